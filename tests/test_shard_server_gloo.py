"""The row-sharded PirServer (shard.ShardedPirServer) on CPU: gloo,
world_size 2, the full reference API driven on rank 0 -- register, the hint
worker's batches (per-shard parts gathered into d1' entries), answer() and
handle_frame() in both modes, update_database (each rank's slice sent from
rank 0, incremental state per shard), hint regeneration after the update --
every result bit-exact against the single-process oracle of the whole DB and
decoding to the requested record. The rank-local compute is the CPU oracle
(OracleShard below, standing in for shard.DeviceShard's GPU kernels); the
command channels, broadcasts, gathers, status rows and version handling are
the product's."""

import os
import random
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


D0, D1, N, BITS = 24, 40, 16, 256


class OracleShard:
    """DeviceShard's interface on the CPU oracle (test infrastructure)."""

    def __init__(self, params, db_slice, basis=None, incremental=True):
        from types import SimpleNamespace
        from oracle import ref
        self.params = params
        self.db = np.array(db_slice)
        self.A = ref.public_matrix(params.a_seed, params.d0, params.lwe.n, params.lwe.q)
        self.state = SimpleNamespace(db_version=0, device="cpu")
        self.regs = {}
        self._H()

    def _H(self):
        from oracle import ref
        self.H = ref.global_hint(self.db, self.A, self.params.lwe.q)

    @property
    def version(self):
        return self.state.db_version

    def new_stream(self):
        return None

    def register(self, cid, m, seed):
        self.regs.setdefault(cid, (m, seed))

    def hints(self, jobs, stream=None):
        from oracle import c as oc, ref
        from paper_2603_09190_b200.shard import _width_of
        p = self.params
        out = []
        for cid, qi in jobs:
            if cid not in self.regs:
                out.append(None)
                continue
            m, seed = self.regs[cid]
            m2 = m * m
            ck_r = ref.derive_ck_r(m2, seed, qi, p.lwe.n)
            Hs = ref.scale_rows(self.H, p.capacity, p.gamma, self.db.shape[1], p.lwe.n)
            k = oc.multiexp_rows(ck_r, Hs, m2)
            out.append(torch.from_numpy(oc._limbs(k, _width_of(m2)).view(np.int32)))
        return out

    def answer_t(self, m, ck_bytes, qu):
        from oracle import ref
        from paper_2603_09190_b200.shard import _width_of
        p = self.params
        ck = [int.from_bytes(r.tobytes(), "little") for r in np.asarray(ck_bytes, np.uint8)]
        b = ref.db_matvec(self.db, np.asarray(qu, dtype=np.uint64), p.lwe.q)
        t = ref.answer_t(self.H, b, ck, m, p.capacity, p.gamma, self.db.shape[1])
        from oracle import c as oc
        return torch.from_numpy(oc._limbs(t, _width_of(m)).view(np.int32))

    def combine(self, t_rows, k_rows, m):
        from oracle import c as oc, ref
        from paper_2603_09190_b200.shard import _width_of
        t = oc._ints(t_rows.numpy().view(np.uint32))
        k = oc._ints(k_rows.numpy().view(np.uint32))
        return oc._limbs(ref.combined(t, k, m), _width_of(m * m))

    def update(self, db_slice):
        self.db = np.array(db_slice)
        self._H()
        self.state.db_version += 1

    def close(self):
        pass


def _oracle_full(params, db, m, seed, qi, qu, ck):
    from oracle import ref
    A = ref.public_matrix(params.a_seed, params.d0, params.lwe.n, params.lwe.q)
    H = ref.global_hint(db, A, params.lwe.q)
    ck_r = ref.derive_ck_r(m * m, seed, qi, params.lwe.n)
    k = ref.hint_entries(ref.scale_rows(H, params.capacity, params.gamma, params.d1,
                                        params.lwe.n), ck_r, m * m)
    b = ref.db_matvec(db, qu, params.lwe.q)
    t = ref.answer_t(H, b, ck, m, params.capacity, params.gamma, params.d1)
    return k, t, ref.combined(t, k, m)


CPU_CFG = dict(d0=D0, d1=D1, n=N, bits=BITS, sigma=1.0, local="oracle", rows=[3, 17, 33])


def _worker(rank, world, port, out, cfg=CPU_CFG):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _run(rank, out, cfg)
    except Exception as e:                     # report, never hang the other rank
        import traceback
        out.put(("error", rank, traceback.format_exc()))
        raise
    finally:
        dist.destroy_process_group()


def _run(rank, out, cfg):
    import paper_2603_09190_b200 as z
    from oracle import client
    from paper_2603_09190_b200 import wire
    from paper_2603_09190_b200.shard import ShardedPirServer
    D0, D1, N, BITS = cfg["d0"], cfg["d1"], cfg["n"], cfg["bits"]
    params = z.ProtocolParams(z.LweParams(N, 1 << 32, 256, cfg["sigma"]), D0, D1, BITS,
                              hints_per_client=2)
    rng = np.random.default_rng(3)
    db = rng.integers(0, 256, (D0, D1), dtype=np.uint8)
    factory = OracleShard if cfg["local"] == "oracle" else None     # None: DeviceShard (GPU)
    if factory is None:
        torch.cuda.set_device(0)
    srv = ShardedPirServer(params, db, local_factory=factory, hint_batch=4)
    if rank != 0:
        srv.join()
        srv.close()
        return
    checks = {}
    try:
        assert params.d1_prime >= 3 and srv.world == dist.get_world_size()
        r = random.Random(11)
        sk, seed = client.setup(BITS, r)
        pk = z.PaillierPublicKey(sk.m, sk.m.bit_length())
        cid = srv.register(pk, seed)
        srv.wait_for_hints(timeout=120)
        reg = srv.registrations[cid]
        assert sorted(reg.hints) == [0, 1]
        lw = params.lwe
        for version, cur in ((0, db), (1, None)):
            if version == 1:
                db2 = db.copy()
                rows = cfg["rows"]
                db2[:, rows] = rng.integers(0, 256, (D0, len(rows)), dtype=np.uint8)
                srv.update_database(db2)
                assert srv.db_version == 1
                srv.wait_for_hints(timeout=120)
                cur = db2
            for qi, i0 in ((0, 5), (1, 19)):
                h = reg.hints[qi]
                assert h.db_version == version
                qu0, ck_o, _ = client.query(sk, seed, lw.n, lw.q, lw.p, lw.noise_sigma, D0, i0, qi,
                                            r, _A(params))
                k, t, K = _oracle_full(params, cur, sk.m, seed, qi, qu0, ck_o)
                checks[f"v{version}q{qi}_hint"] = [c.c for c in h.entries] == k
                rs = srv.answer(cid, z.QueryMessage(cid, qi, z.SEPARATE, ck_o, qu0))
                checks[f"v{version}q{qi}_t"] = rs.t == t
                rc = srv.answer(cid, z.QueryMessage(cid, qi, z.COMBINED, ck_o, qu0))
                checks[f"v{version}q{qi}_K"] = [c.c for c in rc.k] == K
                got = client.extract(sk, lw.q, lw.p, params.capacity, params.gamma, D1,
                                     combined=[c.c for c in rc.k])
                checks[f"v{version}q{qi}_record"] = got == [int(x) for x in cur[i0]]
                # the wire front end (handle_frame) in both modes
                wl = wire.WireLayout(params)
                for mode_b, want in ((0, (t, k)), (1, (K,))):
                    frame = wire.pack_frame(wire.MSG_QUERY, params.params_hash(),
                                            wire.encode_query(wl, cid, qi, mode_b, ck_o, qu0))
                    rep = wire.unpack_frame(srv.handle_frame(frame[4:])[4:])
                    got = wire.decode_response(wl, rep.body, combined=bool(mode_b))
                    checks[f"v{version}q{qi}_wire{mode_b}"] = got == (qi, *want)
        # errors map as the reference's (ValueError on dimensions)
        with pytest.raises(ValueError):
            srv.answer(cid, z.QueryMessage(cid, 0, z.SEPARATE, [1] * (N - 1), np.zeros(D0)))
        checks["world"] = srv.world == dist.get_world_size() and srv.gmax >= 1
    finally:
        srv.close()
    out.put(("ok", checks))


def _A(params):
    from oracle import ref
    return ref.public_matrix(params.a_seed, params.d0, params.lwe.n, params.lwe.q)


def run_two_ranks(cfg, timeout=300, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, cfg)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=timeout)
    for p in procs:
        p.join(timeout=60)
    assert res[0] == "ok", res
    checks = res[1]
    assert checks and all(checks.values()), {k: v for k, v in checks.items() if not v}
    assert all(p.exitcode == 0 for p in procs)


def test_sharded_pirserver_full_api_gloo():
    run_two_ranks(CPU_CFG)


def test_sharded_pirserver_three_ranks_uneven_groups():
    """Three ranks over 6 groups of 7 rows minus a partial last group (d1 = 40):
    uneven row counts per shard, the same bit-exact API run."""
    run_two_ranks(CPU_CFG, world=3)
