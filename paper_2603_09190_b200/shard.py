"""DB-row sharding across the GPUs of one box (one process per GPU).

Every output row c of DB = db^T (a column of the reference's db) is
independent for b, H and y, and every hint group g (cap consecutive rows) is
independent for t, K and k. Shards are therefore group-aligned:
rank s owns groups [floor(s G / W), floor((s+1) G / W)) = DB rows
[cap g_lo, min(cap g_hi, d1)), holds that slice of DB and H and answers and
compresses it locally; the only collective on the query path is one gather
of the per-shard t (or K) rows -- d1' x 256 B in total at 2048-bit m -- to
the answering rank, done as an all_gather_into_tensor over NCCL/NVLink of
equal-size (zero-padded) slices.
"""

import torch

from .params import Layout


def shard_bounds(d1: int, cap: int, world: int):
    """[(row_lo, row_hi, g_lo, g_hi)] per rank, group aligned."""
    groups = -(-d1 // cap)
    out = []
    for s in range(world):
        g_lo = s * groups // world
        g_hi = (s + 1) * groups // world
        out.append((min(g_lo * cap, d1), min(g_hi * cap, d1), g_lo, g_hi))
    return out


def shard_params(params, rows: int):
    """A params object for one shard: same LWE / Paillier layout, d1 = rows.
    The capacity (hence group boundaries) does not depend on d1."""
    import dataclasses
    return dataclasses.replace(params, d1=rows)


_GATHER_BUFS = {}


def _gather_buffers(t_local, gmax, L, world, group):
    """The zero-padded send slice and the receive buffer of gather_groups,
    kept per (device, stream, shape, group): a rank's slice length never
    changes for fixed bounds, so the padding rows stay zero and a step costs
    one copy + the all_gather (no allocation or memset launches)."""
    dev = t_local.device
    sid = torch.cuda.current_stream(dev).stream_id if dev.type == "cuda" else 0
    key = (str(dev), sid, t_local.dtype, gmax, L, world, id(group), t_local.shape[0])
    bufs = _GATHER_BUFS.get(key)
    if bufs is None:
        bufs = (torch.zeros((gmax, L), dtype=t_local.dtype, device=dev),
                torch.empty((world * gmax, L), dtype=t_local.dtype, device=dev))
        _GATHER_BUFS[key] = bufs
    return bufs


def gather_groups(t_local: torch.Tensor, bounds, rank: int, group=None) -> torch.Tensor:
    """Assemble the full (G, L) answer on every rank from per-rank (g_i, L)
    slices with one all_gather_into_tensor (equal-size padded slices)."""
    import torch.distributed as dist
    world = len(bounds)
    gmax = max(b[3] - b[2] for b in bounds)
    L = t_local.shape[1]
    pad, full = _gather_buffers(t_local, gmax, L, world, group)
    pad[: t_local.shape[0]] = t_local
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(full, pad, group=group)
    else:  # gloo (CPU tests of the multi-rank host logic)
        dist.all_gather(list(full.split(gmax)), pad, group=group)
    parts = [full[s * gmax: s * gmax + (b[3] - b[2])] for s, b in enumerate(bounds)]
    return torch.cat(parts, 0)


class ShardedServer:
    """One rank's share of a DB-row-sharded server (weak or strong scaling).

    db_slice is this rank's (d0, rows) column block of the reference db,
    already cut at shard_bounds()[rank]."""

    def __init__(self, params, db_slice, rank: int, world: int, group=None):
        from .protocol import ServerGlobalState
        lay = Layout(params)
        self.params = params
        self.bounds = shard_bounds(params.d1, lay.cap, world)
        self.rank, self.world, self.group = rank, world, group
        lo, hi, _, _ = self.bounds[rank]
        if db_slice.shape != (params.d0, hi - lo):
            raise ValueError("shard slice shape does not match shard_bounds")
        self.state = ServerGlobalState(shard_params(params, hi - lo), db_slice)

    def answer(self, qu_dev, cko_dev, kctx, t_ld, stream, events=None):
        t_local = self.state.answer_device(qu_dev, cko_dev, kctx, t_ld, stream, events)
        if self.world == 1:
            return t_local
        with torch.cuda.stream(stream):
            return gather_groups(t_local, self.bounds, self.rank, self.group)
