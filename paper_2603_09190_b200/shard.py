"""DB-row sharding across the GPUs of one box (one process per GPU).

Every output row c of DB = db^T (a column of the reference's db) is
independent for b, H and y, and every hint group g (cap consecutive rows) is
independent for t, K and k. Shards are therefore group-aligned:
rank s owns groups [floor(s G / W), floor((s+1) G / W)) = DB rows
[cap g_lo, min(cap g_hi, d1)), holds that slice of DB and H and answers and
compresses it locally; the only collective on the query path is one gather
of the per-shard t rows -- d1' x 256 B in total at 2048-bit m -- to the
answering rank, done as an all_gather_into_tensor over NCCL/NVLink of
equal-size (zero-padded) slices.

ShardedPirServer is the reference's PirServer (server.py:29-237) over W
ranks: rank 0 is the front end (registrations, the hint worker, frames,
answers, updates); every rank keeps a rank-local headless PirServer on its
DB slice (its ServerGlobalState, and the slot decompositions of its part of
every client hint for incremental refresh). Two command channels keep the
ranks in lockstep -- each its own process group, so offline hint gathers
never interleave with online answers:

  online  : REGISTER (pk, seed) -> every rank records the client
            ANSWER   broadcast of qu0 + ck_o (4 d0 + n w bytes), per-shard
                     t, one all_gather of the t rows; COMBINED is finished
                     on rank 0 (K = (1 + t m) k mod m^2 over all groups, with
                     the stored hint entries rank 0 keeps for SEPARATE replies)
            UPDATE   each rank's new DB slice sent from rank 0, incremental
                     state on every rank (changed rows found per shard)
  offline : HINTS    a batch of (client, qi) jobs at a db_version: every
                     rank computes (or refreshes) its groups' entries, one
                     all_gather assembles the d1' entries on rank 0, which
                     stores them as the ClientHint SEPARATE returns
                     (protocol.py:352-353)

A rank-local failure never leaves a collective unmatched: every gather
carries a status row, and rank 0 raises (or re-queues a hint job) when any
rank reports one.
"""

import dataclasses
import logging
import threading

import numpy as np
import torch

from .params import Layout
from .server import PirServer

log = logging.getLogger("zippir_b200.shard")


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
    """One rank's share of a DB-row-sharded server state (the bench's
    device-resident timing path; ShardedPirServer is the full server).

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


# -- the sharded PirServer -----------------------------------------------------

class _Channel:
    """Commands and data of one process group, rank 0 -> all and all -> all.
    NCCL groups move device tensors (NVLink); gloo groups host tensors."""

    def __init__(self, group, device):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.nccl = dist.get_backend(group) == "nccl"
        self.device = torch.device(device) if self.nccl else torch.device("cpu")
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.lock = threading.Lock()     # rank 0: one command (and its collectives) at a time

    def command(self, cmd=None):
        box = [cmd]
        self.dist.broadcast_object_list(box, src=0, group=self.group,
                                        device=self.device if self.nccl else None)
        return box[0]

    def bcast_bytes(self, data, nbytes: int) -> torch.Tensor:
        """Rank 0's `data` (bytes-like / ndarray of nbytes) on every rank, as a u8 tensor."""
        t = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        if self.rank == 0:
            src = np.frombuffer(memoryview(data).cast("B"), dtype=np.uint8)
            t.copy_(torch.from_numpy(src.copy()))
        self.dist.broadcast(t, src=0, group=self.group)
        return t

    def gather_rows(self, parts, gmax: int, L: int, status: list) -> torch.Tensor:
        """all_gather of J blocks of (gmax + 1, L) int32 per rank: block j holds
        this rank's rows parts[j] (<= gmax rows, zero padded) and, in its last
        row, status[j] (0 = ok). Returns (world, J, gmax + 1, L)."""
        J = len(parts)
        buf = torch.zeros((J, gmax + 1, L), dtype=torch.int32, device=self.device)
        for j, p in enumerate(parts):
            if p is not None and status[j] == 0:
                buf[j, : p.shape[0], : p.shape[1]] = p.to(self.device)
            buf[j, gmax, 0] = int(status[j])
        full = torch.empty((self.world, J, gmax + 1, L), dtype=torch.int32, device=self.device)
        if self.nccl:
            self.dist.all_gather_into_tensor(full.view(-1), buf.view(-1), group=self.group)
        else:
            self.dist.all_gather(list(full.unbind(0)), buf, group=self.group)
        return full

    def status(self, code: int) -> list:
        """all_gather of one int per rank."""
        t = torch.tensor([int(code)], dtype=torch.int64, device=self.device)
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return [int(x.item()) for x in out]


class DeviceShard:
    """Rank-local part of a sharded server on this rank's GPU: a headless
    PirServer (no workers, no queue) on the DB slice. Its registrations hold
    this rank's part of every client hint, with the slot decomposition for
    incremental refresh."""

    def __init__(self, params, db_slice, basis=None, incremental=True, state=None):
        class _Local(PirServer):
            def _enqueue_missing(self, reg):     # rank 0's front end schedules hints
                pass
        self.srv = _Local(params, db_slice, None, basis, state=state, hint_workers=0,
                          incremental=incremental)

    @property
    def state(self):
        return self.srv.state

    @property
    def version(self) -> int:
        return self.srv.state.db_version

    def new_stream(self):
        return torch.cuda.Stream(self.state.device)

    def register(self, cid: bytes, m: int, seed: bytes):
        from .paillier import PaillierPublicKey
        from .protocol import ClientRegistration
        with self.srv.lock:
            if cid not in self.srv.registrations:
                pk = PaillierPublicKey(m, m.bit_length())
                self.srv.registrations[cid] = ClientRegistration(pk, seed, cid)

    def hints(self, jobs, stream=None) -> list:
        """This shard's part of each (cid, qi) hint at the current version, as
        (g_local, l2) int32 device rows, or None where it could not be made."""
        self.srv._generate_hints(jobs, stream)
        out = []
        for cid, qi in jobs:
            reg = self.srv.registrations.get(cid)
            h = reg.hints.get(qi) if reg is not None else None
            out.append(h.dev if h is not None and h.db_version == self.version else None)
        return out

    def answer_t(self, m: int, ck_bytes: np.ndarray, qu: np.ndarray) -> torch.Tensor:
        from . import protocol
        return protocol.answer_wire(self.srv.state, m, ck_bytes, qu, on_device=True)

    def combine(self, t_rows: torch.Tensor, k_rows, m: int) -> np.ndarray:
        """K = trivial_encrypt(t) k mod m^2 for all groups (protocol.py:354-358)
        on this rank's GPU; t_rows (G, >= lm) int32, k_rows (G, l2) int32."""
        from . import device
        from .bigint import key_ctx
        kctx = key_ctx(m, self.state.device)
        dev = self.state.device
        t = torch.zeros((t_rows.shape[0], kctx.l2), dtype=torch.int32, device=dev)
        t[:, : kctx.lm] = t_rows[:, : kctx.lm].to(dev)
        K = device.combine(t, k_rows.to(dev), kctx)
        return K.cpu().numpy().view(np.uint32)

    def update(self, db_slice):
        self.srv.update_database(db_slice)

    def close(self):
        self.srv.close()


def _limb_rows_to_ints(rows: np.ndarray) -> list:
    from .bigint import limbs_to_ints
    return limbs_to_ints(np.ascontiguousarray(rows, dtype=np.uint32))


class ShardedPirServer(PirServer):
    """PirServer(params, db, store_dir=None, basis=None) over the ranks of
    `group` (default: the world), one per GPU. Every rank constructs it with
    the full db (each keeps its slice) or with db=None and db_slice= its own
    (d0, rows) block. Rank 0 is the server (register / answer / handle_frame
    / update_database / wait_for_hints / close); the other ranks serve its
    commands on background threads until rank 0 closes (join() blocks)."""

    def __init__(self, params, db, store_dir=None, basis=None, *, db_slice=None,
                 group=None, device=None, local_factory=None, local=None, store=None,
                 incremental=True, hint_batch: int = 8, slot_window: int = None):
        import torch.distributed as dist
        self.group = group if group is not None else dist.group.WORLD
        self.rank = dist.get_rank(self.group)
        self.world = dist.get_world_size(self.group)
        lay = Layout(params)
        self.bounds = shard_bounds(params.d1, lay.cap, self.world)
        lo, hi, glo, ghi = self.bounds[self.rank]
        self.gmax = max(b[3] - b[2] for b in self.bounds)
        if local is not None:           # a prebuilt rank-local part (e.g. DeviceShard(state=...))
            self.local = local
        else:
            if db_slice is None:
                db_slice = np.asarray(db)[:, lo:hi]
            if db_slice.shape != (params.d0, hi - lo):
                raise ValueError("shard slice shape does not match shard_bounds")
            factory = local_factory or DeviceShard
            self.local = factory(shard_params(params, hi - lo), db_slice, basis=basis,
                                 incremental=incremental)
        dev = device if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available()
            else torch.device("cpu"))
        # two command channels, each its own process group (created in the
        # same order on every rank)
        ranks = dist.get_process_group_ranks(self.group)
        self.online = _Channel(dist.new_group(ranks), dev)
        self.offline = _Channel(dist.new_group(ranks), dev)
        self._threads = []
        if self.rank == 0:
            PirServer.__init__(self, params, None, store_dir, basis, store=store,
                               state=self.local.state, incremental=incremental,
                               hint_workers=1, hint_batch=hint_batch,
                               slot_window=slot_window)
        else:
            self.params = params
            self._stop = threading.Event()
            self.workers = []
            for loop in (self._online_loop, self._offline_loop):
                th = threading.Thread(target=loop, daemon=True)
                th.start()
                self._threads.append(th)

    # the front end's state is rank 0's local shard state (db_version, device)
    @property
    def state(self):
        return self.local.state

    @state.setter
    def state(self, value):
        pass

    def _worker_stream(self):
        return self.local.new_stream()

    # -- followers ------------------------------------------------------

    def join(self, timeout=None):
        for th in self._threads:
            th.join(timeout)

    def _online_loop(self):
        while True:
            cmd = self.online.command()
            op = cmd[0]
            if op == "STOP":
                return
            try:
                getattr(self, "_do_" + op.lower())(cmd)
            except Exception:
                log.exception("rank %d: online command %s failed", self.rank, op)

    def _offline_loop(self):
        stream = None
        while True:
            cmd = self.offline.command()
            if cmd[0] == "STOP":
                return
            if stream is None:
                stream = self.local.new_stream()
            try:
                with torch.cuda.stream(stream):
                    self._do_hints(cmd, stream)
            except Exception:
                log.exception("rank %d: hint batch failed", self.rank)

    # -- commands (run on every rank, rank 0 included) ------------------

    def _do_register(self, cmd):
        _, cid, m, seed = cmd
        self.local.register(cid, m, seed)

    def _do_answer(self, cmd):
        _, m, w, d0, n = cmd
        raw = self.online.bcast_bytes(None if self.rank else self._payload, 4 * d0 + n * w)
        if self.rank == 0:
            qu, ck = self._payload_arrays
        else:
            host = raw.cpu().numpy()
            qu = host[: 4 * d0].view(np.uint32)
            ck = host[4 * d0:].reshape(n, w)
        status, t = 0, None
        try:
            t = self.local.answer_t(m, ck, qu)
        except Exception as e:
            log.error("rank %d: answer failed: %s", self.rank, e)
            status = 1
        return self.online.gather_rows([t], self.gmax, _width_of(m), [status])

    def _do_update(self, cmd):
        import torch.distributed as dist
        _, d0 = cmd
        lo, hi = self.bounds[self.rank][:2]
        if self.rank == 0:
            db = self._update_db
            for r in range(1, self.world):
                rlo, rhi = self.bounds[r][:2]
                part = torch.from_numpy(np.ascontiguousarray(db[:, rlo:rhi])).to(
                    self.online.device)
                dist.send(part, dst=dist.get_global_rank(self.online.group, r),
                          group=self.online.group)
            mine = np.ascontiguousarray(db[:, lo:hi])
        else:
            part = torch.empty((d0, hi - lo), dtype=torch.uint8, device=self.online.device)
            dist.recv(part, src=dist.get_global_rank(self.online.group, 0),
                      group=self.online.group)
            mine = part.cpu().numpy()
        code = 0
        try:
            self.local.update(mine)
        except Exception as e:
            log.error("rank %d: update failed: %s", self.rank, e)
            code = 1
        return self.online.status(code)

    # hint job status in the gathered block: 0 ok, 1 failed, 2 this rank is at
    # another db_version (rank 0 re-queues the job)
    def _do_hints(self, cmd, stream=None):
        _, jobs, version, l2 = cmd
        if self.local.version != version:
            return self.offline.gather_rows([None] * len(jobs), self.gmax, l2, [2] * len(jobs))
        try:
            got = self.local.hints(jobs, stream)
        except Exception as e:
            log.error("rank %d: hints failed: %s", self.rank, e)
            got = [None] * len(jobs)
        status = [0 if h is not None else 1 for h in got]
        return self.offline.gather_rows(got, self.gmax, l2, status)

    # -- rank 0: the PirServer front end ----------------------------------

    def _restore(self):
        PirServer._restore(self)
        for reg in list(self.registrations.values()):
            self._registered(reg)

    def _registered(self, reg):
        cmd = ("REGISTER", reg.client_id, reg.pk.m, reg.seed)
        with self.online.lock:
            self.online.command(cmd)
            self._do_register(cmd)

    def _generate_hints(self, jobs, stream=None):
        from .paillier import PaillierCiphertext
        from .protocol import ClientHint
        version = self.db_version
        fresh, refresh = self._plan_jobs(jobs, version)
        todo = [(reg, qi) for reg, qi in fresh]
        todo += [(reg, qi) for _, items in refresh.values() for reg, qi, _ in items]
        if not todo:
            return
        l2 = max(_width_of(reg.pk.m2) for reg, _ in todo)
        cmd = ("HINTS", [(reg.client_id, qi) for reg, qi in todo], version, l2)
        with self.offline.lock:
            self.offline.command(cmd)
            full = self._do_hints(cmd, stream)
        done = []
        for j, (reg, qi) in enumerate(todo):
            codes = [int(full[r, j, self.gmax, 0]) for r in range(self.world)]
            if 1 in codes:
                log.error("hint (%s, %d) failed on ranks %s", reg.client_id.hex()[:8], qi,
                          [r for r, c in enumerate(codes) if c == 1])
                continue
            if any(codes):
                self.jobs.put((reg.client_id, qi))      # a rank was at another version
                continue
            rows = self._assemble(full[:, j])
            entries = _limb_rows_to_ints(rows.cpu().numpy().view(np.uint32))
            done.append((reg, qi, ClientHint(qi, version,
                                             [PaillierCiphertext(e) for e in entries],
                                             dev=rows.to(self.local.state.device)
                                             if self.online.nccl else None)))
        self._store_hints(done)

    def _assemble(self, blocks):
        """(world, gmax + 1, L) gathered blocks -> the (G, L) rows in group order."""
        return torch.cat([blocks[r, : b[3] - b[2]] for r, b in enumerate(self.bounds)], 0)

    def _sharded_rows(self, reg, qi, mode, ck_bytes, qu) -> np.ndarray:
        from .protocol import COMBINED
        lay_d0, n = self.params.d0, self.params.lwe.n
        m = reg.pk.m
        qu32 = np.zeros(lay_d0, dtype=np.uint32)
        np.copyto(qu32, np.asarray(qu), casting="unsafe")
        ck = np.ascontiguousarray(ck_bytes, dtype=np.uint8)
        if ck.shape[0] != n:
            raise ValueError("query dimensions do not match the parameters")
        with self.online.lock:
            cmd = ("ANSWER", m, ck.shape[1], lay_d0, n)
            self.online.command(cmd)
            self._payload = qu32.tobytes() + ck.tobytes()
            self._payload_arrays = (qu32, ck)
            full = self._do_answer(cmd)
        if any(int(full[r, 0, self.gmax, 0]) for r in range(self.world)):
            raise RuntimeError("a shard failed to answer")
        t = self._assemble(full[:, 0])
        lm = _width_of(m)
        if mode != COMBINED:
            return t[:, :lm].cpu().numpy().view(np.uint32)
        stored = reg.hints[qi]
        k = stored.dev if stored.dev is not None else torch.from_numpy(
            _ints_rows(stored.entries, _width_of(reg.pk.m2)).view(np.int32))
        return self.local.combine(t, k, m)

    def _respond_rows(self, state, reg, qi, mode, ck_o, qu0):
        rows = self._sharded_rows(reg, qi, mode, ck_o, qu0)
        if mode != "separate":
            from . import counters
            counters.bump("add", self.params.d1_prime)
            counters.bump("group_mult", self.params.d1_prime)
        return rows

    def respond(self, client_id: bytes, qmsg):
        """protocol.respond() over the shards (no hint scheduling): KeyError
        when the client or a fresh hint for the query index is missing."""
        with self.lock:
            reg = self.registrations.get(client_id)
        if reg is None:
            raise KeyError("client not registered")
        stored = reg.hints.get(qmsg.query_index)
        if stored is None or stored.db_version != self.db_version:
            raise KeyError("no hint for this query index and database version")
        return self._respond(None, reg, qmsg)

    def _respond(self, state, reg, qmsg):
        from . import counters
        from .bigint import ints_to_limbs
        from .paillier import PaillierCiphertext
        from .protocol import COMBINED, SEPARATE, ResponseMessage
        if len(qmsg.ck_o) != self.params.lwe.n or len(qmsg.qu0) != self.params.d0:
            raise ValueError("query dimensions do not match the parameters")
        mode = qmsg.mode
        if mode not in (SEPARATE, COMBINED):
            raise ValueError("unknown response mode")
        lm = _width_of(reg.pk.m)
        ck = ints_to_limbs(list(qmsg.ck_o), lm).view(np.uint8).reshape(len(qmsg.ck_o), 4 * lm)
        rows = self._sharded_rows(reg, qmsg.query_index, mode, ck, qmsg.qu0)
        vals = _limb_rows_to_ints(rows)
        stored = reg.hints[qmsg.query_index]
        if mode == SEPARATE:
            return ResponseMessage(SEPARATE, qmsg.query_index, vals, stored.entries)
        counters.bump("add", self.params.d1_prime)
        counters.bump("group_mult", self.params.d1_prime)
        return ResponseMessage(COMBINED, qmsg.query_index, [],
                               [PaillierCiphertext(v) for v in vals])

    def update_database(self, db):
        db = np.asarray(db)
        if db.shape != (self.params.d0, self.params.d1):
            raise ValueError("database shape mismatch")
        with self.online.lock:
            cmd = ("UPDATE", self.params.d0)
            self.online.command(cmd)
            self._update_db = db
            codes = self._do_update(cmd)
            self._update_db = None
        if any(codes):
            raise RuntimeError(f"shard update failed on ranks {[i for i, c in enumerate(codes) if c]}")
        with self.lock:
            regs = list(self.registrations.values())
        for reg in regs:
            if self.store:
                self.store.purge_stale(reg.client_id, self.db_version)
            self._enqueue_missing(reg)

    def close(self):
        if self.rank == 0 and not getattr(self, "_closed", False):
            self._closed = True
            PirServer.close(self)
            with self.offline.lock:
                self.offline.command(("STOP",))
            with self.online.lock:
                self.online.command(("STOP",))
        self.local.close()


def _width_of(x: int) -> int:
    """Warp limb width (32 x limbs-per-lane) of the kernels for an x-sized value."""
    from .bigint import limbs_for_bits
    return limbs_for_bits(int(x).bit_length())


def _ints_rows(entries, L) -> np.ndarray:
    from .bigint import ints_to_limbs
    return ints_to_limbs([c.c if hasattr(c, "c") else int(c) for c in entries], L)
