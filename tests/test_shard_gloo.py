"""Multi-rank host logic of the row-sharded server on CPU (gloo, world_size 2).

Each rank computes t for its group-aligned shard (here with the CPU oracle,
standing in for the per-GPU device path) and the shards are assembled with
shard.gather_groups; the result must equal the single-process answer."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_09190_b200.shard import shard_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_bounds_group_aligned():
    for d1, cap, world in [(32768, 63, 2), (92682, 63, 8), (48, 23, 2), (130, 31, 4), (5, 9, 3)]:
        b = shard_bounds(d1, cap, world)
        assert b[0][0] == 0 and b[-1][1] == d1
        groups = -(-d1 // cap)
        assert b[0][2] == 0 and b[-1][3] == groups
        for (lo, hi, glo, ghi), nxt in zip(b, b[1:] + [None]):
            assert lo == min(glo * cap, d1) and hi == min(ghi * cap, d1)
            if nxt:
                assert nxt[0] == hi and nxt[2] == ghi
        sizes = [x[3] - x[2] for x in b]
        assert max(sizes) - min(sizes) <= 1


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import ref
    from paper_2603_09190_b200.shard import gather_groups
    rng = np.random.default_rng(5)
    d0, d1, n, cap, m = 40, 130, 16, 31, (1 << 1023) + 1155
    db = rng.integers(0, 256, (d0, d1), dtype=np.uint8)
    A = rng.integers(0, 1 << 32, (d0, n), dtype=np.uint64)
    qu = rng.integers(0, 1 << 32, d0, dtype=np.uint64)
    ck = [int(x) for x in rng.integers(0, 1 << 62, n, dtype=np.uint64)]
    lo, hi, glo, ghi = shard_bounds(d1, cap, world)[rank]
    part = db[:, lo:hi]
    H = ref.global_hint(part, A, 1 << 32)
    b = ref.db_matvec(part, qu, 1 << 32)
    t = ref.answer_t(H, b, ck, m, cap, 1 << 32, hi - lo)
    limbs = np.array([[(v >> (32 * i)) & 0xFFFFFFFF for i in range(32)] for v in t],
                     dtype=np.uint32).reshape(-1, 32)
    full = gather_groups(torch.from_numpy(limbs.view(np.int32)), shard_bounds(d1, cap, world), rank)
    got = [int.from_bytes(r.numpy().view(np.uint32).astype("<u4").tobytes(), "little") for r in full]
    if rank == 0:
        Hf = ref.global_hint(db, A, 1 << 32)
        want = ref.answer_t(Hf, ref.db_matvec(db, qu, 1 << 32), ck, m, cap, 1 << 32, d1)
        out.put(got == want)
    dist.destroy_process_group()


def test_sharded_answer_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    assert ok
    assert all(p.exitcode == 0 for p in procs)
