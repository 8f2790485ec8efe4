"""Protocol-level GPU tests mirroring the reference's test_protocol.py
(tests/test_protocol.py:40-113 there): exhaustive toy retrieval in both
modes, zero database, update replay (stale hint refused, regenerated hint
serves), hint determinism per query index -- on the B200 path, with the
oracle's client restatement manufacturing queries and extracting records."""

import random

import numpy as np
import pytest

from oracle import client

pytestmark = pytest.mark.gpu


def _toy(z, d0=4, d1=4, **kw):
    args = dict(lwe=z.LweParams(n=4, q=16, p=4, noise_sigma=0.0, key_dist="binary"),
                d0=d0, d1=d1, paillier_bits=64, scale_regime="standard")
    args.update(kw)
    return z.ProtocolParams(**args)


def _setup(z, rng, params, db=None):
    if db is None:
        db = np.array([[rng.randrange(params.lwe.p) for _ in range(params.d1)]
                       for _ in range(params.d0)])
    state = z.ServerGlobalState(params, db)
    sk, seed = client.setup(params.paillier_bits, rng)
    pk = z.PaillierPublicKey(sk.m, sk.m.bit_length())
    reg = z.ClientRegistration(pk, seed, z.client_id_of(pk))
    return db, state, sk, reg


def _ask(z, params, state, sk, reg, i0, qi, mode, rng, make_hint=True):
    lw = params.lwe
    if make_hint:
        reg.hints[qi] = z.hint(state, reg, qi)
    qu0, ck_o, _ = client.query(sk, reg.seed, lw.n, lw.q, lw.p, lw.noise_sigma, params.d0, i0,
                                qi, rng, state.A)
    r = z.respond(state, reg, z.QueryMessage(reg.client_id, qi, mode, ck_o, qu0))
    kw = dict(t=r.t, k=[c.c for c in r.k]) if mode == z.SEPARATE else \
        dict(combined=[c.c for c in r.k])
    return client.extract(sk, lw.q, lw.p, params.capacity, params.gamma, params.d1, **kw)


@pytest.fixture(scope="module")
def z():
    import paper_2603_09190_b200 as z
    from paper_2603_09190_b200 import _lib, build
    build.build()
    _lib.load()
    return z


def test_end_to_end_exhaustive_toy(z):
    rng = random.Random(0xC0FFEE)
    params = _toy(z)
    db, state, sk, reg = _setup(z, rng, params)
    for i0 in range(4):
        mode = z.SEPARATE if i0 % 2 == 0 else z.COMBINED
        assert _ask(z, params, state, sk, reg, i0, i0, mode, rng) == [int(x) for x in db[i0]]


@pytest.mark.parametrize("shape", [(7, 23), (16, 10), (1, 1)])
def test_end_to_end_toy_shapes(z, shape):
    """Ragged toy shapes incl. a single record of a single symbol."""
    rng = random.Random(sum(shape))
    params = _toy(z, d0=shape[0], d1=shape[1])
    db, state, sk, reg = _setup(z, rng, params)
    for i0 in sorted({0, shape[0] - 1, shape[0] // 2}):
        assert _ask(z, params, state, sk, reg, i0, i0, z.SEPARATE, rng) == \
            [int(x) for x in db[i0]]


def test_zero_database_returns_zero_row(z):
    rng = random.Random(0xC0FFEE)
    params = _toy(z)
    db, state, sk, reg = _setup(z, rng, params, db=np.zeros((4, 4), dtype=np.int64))
    assert _ask(z, params, state, sk, reg, 2, 0, z.SEPARATE, rng) == [0] * 4


def test_database_update_replay(z):
    rng = random.Random(0xC0FFEE)
    params = _toy(z)
    db, state, sk, reg = _setup(z, rng, params)
    assert _ask(z, params, state, sk, reg, 1, 0, z.SEPARATE, rng) == [int(x) for x in db[1]]
    db2 = np.array([[rng.randrange(4) for _ in range(4)] for _ in range(4)])
    state2 = z.ServerGlobalState(params, db2, basis=state.basis, db_version=state.db_version + 1)
    reg.hints[1] = z.hint(state, reg, 1)                     # stale after the swap
    lw = params.lwe
    qu0, ck_o, _ = client.query(sk, reg.seed, lw.n, lw.q, lw.p, 0.0, 4, 3, 1, rng, state2.A)
    q = z.QueryMessage(reg.client_id, 1, z.SEPARATE, ck_o, qu0)
    with pytest.raises(KeyError):
        z.respond(state2, reg, q)
    reg.hints[1] = z.hint(state2, reg, 1)
    r = z.respond(state2, reg, q)
    assert client.extract(sk, lw.q, lw.p, params.capacity, params.gamma, 4, t=r.t,
                          k=[c.c for c in r.k]) == [int(x) for x in db2[3]]
    # the incremental path reaches the same state and hint
    st_inc, changed = state.updated(db2)
    assert np.array_equal(st_inc.H, state2.H)
    assert [c.c for c in z.hint(st_inc, reg, 1).entries] == [c.c for c in reg.hints[1].entries]


def test_hint_is_deterministic_per_index(z):
    rng = random.Random(0xC0FFEE)
    params = _toy(z)
    db, state, sk, reg = _setup(z, rng, params)
    h1 = z.hint(state, reg, 5)
    h2 = z.hint(state, reg, 5)
    assert [c.c for c in h1.entries] == [c.c for c in h2.entries]
    h3 = z.hint(state, reg, 6)
    assert [c.c for c in h1.entries] != [c.c for c in h3.entries]
    assert [client.decrypt(sk, c.c) for c in h1.entries] == \
        [client.decrypt(sk, c.c) for c in h2.entries]


@pytest.mark.parametrize("bits", [1024, 4096])
def test_end_to_end_other_key_sizes(z, bits):
    """Paillier moduli other than the headline's 2048 bits through the whole
    protocol on the device: 1024-bit m (m^2 = 2048 bits, 2 limbs per lane) and
    4096-bit m (m^2 = 8192 bits, 8 limbs per lane; compression on the CUDA-core
    rows kernel): hint, respond in both modes and the client's extraction
    return the requested DB row; t equals the oracle formula."""
    import random
    from oracle import client, ref
    rng = random.Random(bits)
    d0, d1, n = 256, 200, 128
    params = z.ProtocolParams(z.LweParams(n=n, q=1 << 32, p=256, noise_sigma=6.4), d0, d1, bits)
    db = np.array([[rng.randrange(256) for _ in range(d1)] for _ in range(d0)], dtype=np.uint8)
    st = z.ServerGlobalState(params, db)
    sk, seed = client.setup(bits, rng)
    pk = z.PaillierPublicKey(sk.m, sk.m.bit_length())
    reg = z.ClientRegistration(pk, seed, z.client_id_of(pk))
    reg.hints[0] = z.hint(st, reg, 0)
    A = ref.public_matrix(b"\x00" * 16, d0, n, 1 << 32)
    i0 = 101
    qu0, ck_o, _ = client.query(sk, seed, n, 1 << 32, 256, 6.4, d0, i0, 0, rng, A)
    cap = params.capacity
    r = z.respond(st, reg, z.QueryMessage(reg.client_id, 0, z.SEPARATE, ck_o, qu0))
    H = ref.global_hint(db, A, 1 << 32)
    assert r.t == ref.answer_t(H, ref.db_matvec(db, qu0, 1 << 32), ck_o, sk.m, cap, 1 << 32, d1)
    got = client.extract(sk, 1 << 32, 256, cap, 1 << 32, d1, t=r.t, k=[c.c for c in r.k])
    assert got == [int(x) for x in db[i0]]
    rc = z.respond(st, reg, z.QueryMessage(reg.client_id, 0, z.COMBINED, ck_o, qu0))
    got = client.extract(sk, 1 << 32, 256, cap, 1 << 32, d1, combined=[c.c for c in rc.k])
    assert got == [int(x) for x in db[i0]]


@pytest.mark.parametrize("dtype", [np.uint8, np.int64, np.uint16])
def test_symbol_range_check(z, dtype):
    """db.max() >= p raises ValueError (protocol.py:168-169), for u8 databases
    on the device, for wider dtypes on the host -- in the constructor and in
    the incremental update -- and in-range databases of any dtype build the
    same state."""
    import torch
    params = _toy(z, d0=5, d1=7)                        # p = 4
    rng = random.Random(5)
    db = np.array([[rng.randrange(4) for _ in range(7)] for _ in range(5)], dtype=dtype)
    st = z.ServerGlobalState(params, db)
    ref = z.ServerGlobalState(params, db.astype(np.uint8))
    assert torch.equal(st.H_dev, ref.H_dev)
    bad = db.copy()
    bad[4, 6] = 4
    with pytest.raises(ValueError, match="symbol out of range"):
        z.ServerGlobalState(params, bad)
    with pytest.raises(ValueError, match="symbol out of range"):
        st.updated(bad)
    if dtype != np.uint8:
        bad[4, 6] = 260                                 # would wrap to 4 as u8
        with pytest.raises(ValueError, match="symbol out of range"):
            z.ServerGlobalState(params, bad)
    # p = 256: every u8 symbol is in range, no pass over the bytes needed
    p256 = _toy(z, d0=5, d1=7, lwe=z.LweParams(n=4, q=1 << 32, p=256, noise_sigma=0.0,
                                                 key_dist="binary"))
    full = np.full((5, 7), 255, dtype=np.uint8)
    st2, changed = z.ServerGlobalState(p256, full * 0).updated(full)
    assert list(changed) == list(range(7))


def test_combined_op_profile_through_caller_counters(z, monkeypatch):
    """test_protocol.py:147-155 through the drop-in: a caller measuring its own
    `zippir.counters` (here a freshly written minimal module -- the reference
    package does not travel to the GPU box) around respond(COMBINED) sees
    exactly d1' additions and 0 modexp / scalar_mul."""
    import sys
    import types
    from paper_2603_09190_b200 import counters
    tally = {k: 0 for k in counters.NAMES}
    mod = types.ModuleType("zippir.counters")

    def bump(name, amount=1):
        tally[name] += amount
    mod.bump = bump
    monkeypatch.setitem(sys.modules, "zippir.counters", mod)
    rng = random.Random(147)
    params = _toy(z, d0=6, d1=9)
    db, state, sk, reg = _setup(z, rng, params)
    reg.hints[0] = z.hint(state, reg, 0)
    lw = params.lwe
    qu0, ck_o, _ = client.query(sk, reg.seed, lw.n, lw.q, lw.p, lw.noise_sigma, params.d0, 2, 0,
                                rng, state.A)
    before = dict(tally)
    r = z.respond(state, reg, z.QueryMessage(reg.client_id, 0, z.COMBINED, ck_o, qu0))
    delta = {k: tally[k] - before[k] for k in tally}
    assert delta["add"] == params.d1_prime
    assert delta["modexp"] == 0 and delta["scalar_mul"] == 0
    got = client.extract(sk, lw.q, lw.p, params.capacity, params.gamma, params.d1,
                         combined=[c.c for c in r.k])
    assert got == [int(x) for x in db[2]]


def test_pirserver_store_dir_delegation(z, tmp_path, monkeypatch):
    """PirServer(params, db, store_dir) as the reference calls it: the path opens
    zippir.hintstore.HintStore (here a minimal in-memory stand-in registered under
    that name); registrations and generated hints are saved, and a second server
    on the same store_dir restores them."""
    import sys
    import types
    from paper_2603_09190_b200.server import PirServer
    saved = {"regs": {}, "hints": {}}

    class HintStore:
        def __init__(self, root):
            self.root = root

        def save_registration(self, cid, pk, seed):
            saved["regs"][(self.root, cid)] = (pk, seed)

        def load_registrations(self):
            for (root, cid), (pk, seed) in saved["regs"].items():
                if root == self.root:
                    yield cid, pk, seed

        def save_hint(self, cid, qi, version, entries):
            saved["hints"][(self.root, cid, qi, version)] = list(entries)

        def load_hints(self, cid, version):
            return {qi: e for (root, c, qi, v), e in saved["hints"].items()
                    if root == self.root and c == cid and v == version}

        def purge_stale(self, cid, version):
            pass
    mod = types.ModuleType("zippir.hintstore")
    mod.HintStore = HintStore
    monkeypatch.setitem(sys.modules, "zippir.hintstore", mod)
    rng = random.Random(30)
    params = _toy(z, d0=4, d1=8)
    db = np.array([[rng.randrange(params.lwe.p) for _ in range(params.d1)]
                   for _ in range(params.d0)])
    d = str(tmp_path / "store")
    srv = PirServer(params, db, d)
    try:
        sk, seed = client.setup(params.paillier_bits, rng)
        pk = z.PaillierPublicKey(sk.m, sk.m.bit_length())
        cid = srv.register(pk, seed)
        srv.wait_for_hints(timeout=120)
        entries = [c.c for c in srv.registrations[cid].hints[0].entries]
    finally:
        srv.close()
    assert saved["regs"][(d, cid)][1] == seed
    srv2 = PirServer(params, db, d)
    try:
        assert [c.c for c in srv2.registrations[cid].hints[0].entries] == entries
    finally:
        srv2.close()
