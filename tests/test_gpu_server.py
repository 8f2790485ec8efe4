"""PirServer mirror on the GPU: background hint worker, look-ahead window,
database update with stale-hint regeneration (reference server.py:62-124;
tests test_protocol.py:56-71 update replay, test_acceptance.py:333-360
silent offline)."""

import random

import numpy as np
import pytest

from oracle import client

pytestmark = pytest.mark.gpu


def test_server_update_and_regenerate():
    import paper_2603_09190_b200 as z
    from paper_2603_09190_b200.server import HintPending, PirServer
    rng = random.Random(31)
    params = z.ProtocolParams(z.LweParams(n=64, q=1 << 32, p=256, noise_sigma=6.4), 32, 48, 768,
                              hints_per_client=3)
    db = np.array([[rng.randrange(256) for _ in range(48)] for _ in range(32)])
    srv = PirServer(params, db)
    try:
        sk, seed = client.setup(768, rng)
        pk = z.PaillierPublicKey(sk.m, sk.m.bit_length())
        cid = srv.register(pk, seed)
        srv.wait_for_hints(timeout=120)
        reg = srv.registrations[cid]
        assert sorted(reg.hints) == [0, 1, 2]
        A = srv.state.A

        def ask(qi, i0, mode):
            qu0, ck_o, _ = client.query(sk, seed, 64, 1 << 32, 256, 6.4, 32, i0, qi, rng, A)
            r = srv.answer(cid, z.QueryMessage(cid, qi, mode, ck_o, qu0))
            if mode == z.SEPARATE:
                return client.extract(sk, 1 << 32, 256, params.capacity, 1 << 32, 48,
                                      t=r.t, k=[c.c for c in r.k])
            return client.extract(sk, 1 << 32, 256, params.capacity, 1 << 32, 48,
                                  combined=[c.c for c in r.k])

        assert ask(0, 5, z.SEPARATE) == [int(x) for x in db[5]]
        # database update: hints go stale, the worker regenerates them silently
        db2 = np.array([[rng.randrange(256) for _ in range(48)] for _ in range(32)])
        srv.update_database(db2)
        assert srv.state.db_version == 1
        srv.wait_for_hints(timeout=120)
        # the reference re-enqueues hints_per_client stale indices (server.py:62-70)
        assert all(reg.hints[qi].db_version == 1 for qi in (0, 1, 2))
        assert ask(1, 7, z.COMBINED) == [int(x) for x in db2[7]]
        # a query index outside the window is pending, then served
        with pytest.raises(HintPending):
            ask(9, 0, z.SEPARATE)
        srv.wait_for_hints(timeout=120)
        assert ask(9, 3, z.SEPARATE) == [int(x) for x in db2[3]]
    finally:
        srv.close()


@pytest.mark.parametrize("name", ["ragged", "tiny", "uniform_key", "standard32", "q16"])
def test_incremental_update_bit_exact(golden, name):
    """updated() + refresh_hint() == full rebuild + full hint, bit for bit."""
    import paper_2603_09190_b200 as z
    from conftest import Golden
    g = golden(name)
    params = g.params(z)
    st = z.ServerGlobalState(params, g.db)
    pk = z.PaillierPublicKey(g.m, g.m.bit_length())
    reg = z.ClientRegistration(pk, g.seed, z.client_id_of(pk))
    h_slots = z.hint(st, reg, 0, keep_slots=True)
    assert [c.c for c in h_slots.entries] == g.ints("k")          # slot path == reference
    rng = np.random.default_rng(9)
    db2 = np.array(g.db, dtype=np.uint8, copy=True)
    rows = sorted(set(rng.choice(g.d1, size=max(1, g.d1 // 100), replace=False).tolist())
                  | {0, g.d1 - 1})
    for c in rows:
        db2[:, c] = rng.integers(0, g.lwe["p"], g.d0, dtype=np.uint8)
    st2, changed = st.updated(db2)
    full = z.ServerGlobalState(params, db2, db_version=1)
    assert st2.db_version == 1
    assert np.array_equal(st2.H, full.H)
    assert set(changed.tolist()) <= set(rows)
    h2 = z.refresh_hint(st2, reg, h_slots, changed)
    h_full = z.hint(full, reg, 0)
    assert [c.c for c in h2.entries] == [c.c for c in h_full.entries]
    assert h2.db_version == 1
    # answers against the updated state use the refreshed hint
    reg.hints[0] = h2
    q = z.QueryMessage(reg.client_id, 0, z.SEPARATE, g.ints("ck_o"), g.arr["qu0"])
    assert z.respond(st2, reg, q).t == z.respond(full, reg, q).t


def test_paper_parameters_n1400_3072bit():
    """The paper's setting (cli.py DEFAULT_PARAMS n=1400,
    3072-bit) on the reference's c07 desk shape 256x256 (test_acceptance.py:
    214-217): n % 64 != 0 (CUDA-core hint GEMM), lm = 96 (N = 400 compression
    GEMM), m^2 of 6144 bits (LPL = 6 Montgomery). Bit-exact vs the oracle and
    end-to-end retrieval in both modes."""
    import paper_2603_09190_b200 as z
    from oracle import ref
    rng = random.Random(1400)
    params = z.ProtocolParams(z.LweParams(n=1400, q=1 << 32, p=256, noise_sigma=6.4), 256, 256,
                              3072)
    db = np.array([[rng.randrange(256) for _ in range(256)] for _ in range(256)], dtype=np.uint8)
    st = z.ServerGlobalState(params, db)
    A = ref.public_matrix(b"\x00" * 16, 256, 1400, 1 << 32)
    H = ref.global_hint(db, A, 1 << 32)
    assert np.array_equal(st.H, H)
    sk, seed = client.setup(3072, rng)
    pk = z.PaillierPublicKey(sk.m, sk.m.bit_length())
    reg = z.ClientRegistration(pk, seed, z.client_id_of(pk))
    h = z.hint(st, reg, 0)
    m2 = sk.m * sk.m
    ck_r = ref.derive_ck_r(m2, seed, 0, 1400)
    cap = params.capacity
    Hs = ref.scale_rows(H, cap, 1 << 32, 256, 1400)
    assert [c.c for c in h.entries[:2]] == [ref.multiexp(m2, ck_r, Hs[g]) for g in range(2)]
    reg.hints[0] = h
    i0 = 77
    qu0, ck_o, _ = client.query(sk, seed, 1400, 1 << 32, 256, 6.4, 256, i0, 0, rng, A)
    r = z.respond(st, reg, z.QueryMessage(reg.client_id, 0, z.SEPARATE, ck_o, qu0))
    b = ref.db_matvec(db, qu0, 1 << 32)
    assert r.t == ref.answer_t(H, b, ck_o, sk.m, cap, 1 << 32, 256)
    assert client.extract(sk, 1 << 32, 256, cap, 1 << 32, 256, t=r.t,
                          k=[c.c for c in r.k]) == [int(x) for x in db[i0]]
    rc = z.respond(st, reg, z.QueryMessage(reg.client_id, 0, z.COMBINED, ck_o, qu0))
    assert client.extract(sk, 1 << 32, 256, cap, 1 << 32, 256,
                          combined=[c.c for c in rc.k]) == [int(x) for x in db[i0]]


def test_batched_hints_and_tensor_core_refresh(golden, monkeypatch):
    """hints() for several clients in one tensor-core launch == hint() per
    client; a refresh of two clients through the batched tensor-core path
    (row ids) == full hints on the rebuilt state (BASELINE configs[0] shape,
    2048-bit keys)."""
    import paper_2603_09190_b200 as z
    from paper_2603_09190_b200 import protocol
    g = golden("tiny")
    params = g.params(z)
    st = z.ServerGlobalState(params, g.db)
    regs = []
    for i in range(2):
        sk, seed = client.setup(2048, random.Random(50 + i))
        pk = z.PaillierPublicKey(sk.m, sk.m.bit_length())
        regs.append(z.ClientRegistration(pk, seed, z.client_id_of(pk)))
    hs = z.hints(st, [(regs[0], 0), (regs[1], 3)], keep_slots=True)
    assert [c.c for c in hs[0].entries] == [c.c for c in z.hint(st, regs[0], 0).entries]
    assert [c.c for c in hs[1].entries] == [c.c for c in z.hint(st, regs[1], 3).entries]
    rng = np.random.default_rng(4)
    db2 = np.array(g.db, dtype=np.uint8, copy=True)
    rows = sorted(rng.choice(g.d1, size=40, replace=False).tolist())
    for c in rows:
        db2[:, c] = rng.integers(0, 256, g.d0, dtype=np.uint8)
    st2, changed = st.updated(db2)
    monkeypatch.setattr(protocol, "TC_REFRESH_MIN_ROWS", 1)
    ref_pairs = list(zip(regs, hs))
    out = z.refresh_hints(st2, ref_pairs, changed)
    full = z.ServerGlobalState(params, db2, db_version=1)
    for reg, h, qi in zip(regs, out, (0, 3)):
        assert [c.c for c in h.entries] == [c.c for c in z.hint(full, reg, qi).entries]


def test_tensor_core_hint_failure_falls_back_to_imad(golden, monkeypatch):
    """A tensor-core launch that cannot run (e.g. its workspace does not fit)
    falls back to the IMAD kernels for that batch: same entries."""
    import paper_2603_09190_b200 as z
    from paper_2603_09190_b200 import _lib, device, protocol
    g = golden("tiny")
    st = z.ServerGlobalState(g.params(z), g.db)
    regs = []
    for i in range(2):
        sk, seed = client.setup(2048, random.Random(70 + i))
        pk = z.PaillierPublicKey(sk.m, sk.m.bit_length())
        regs.append(z.ClientRegistration(pk, seed, z.client_id_of(pk)))
    want = [[c.c for c in z.hint(st, r, 0).entries] for r in regs]     # IMAD (< 2048 rows)

    def boom(*a, **k):
        raise _lib.ZpirError("simulated workspace failure")

    monkeypatch.setattr(device, "slot_fixed_tc_many", boom)
    monkeypatch.setattr(protocol, "TC_MIN_ROWS", 1)                       # would take the TC path
    got = [[c.c for c in h.entries] for h in z.hints(st, [(r, 0) for r in regs])]
    assert got == want
