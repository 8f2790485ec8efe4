"""GPU parity: the B200 path vs the reference's golden outputs and the oracle.

Bit-exact on every integer output: H, b, hint entries k, t, COMBINED K, and
end-to-end retrieval. Cases (tests/golden): the reference's reduced desk
(test_protocol.py:190-209), ragged shapes, all-zero and all-255 databases,
and BASELINE configs[0] (1024x1024, n=1024, 2048-bit Paillier).
"""

import hashlib
import random

import numpy as np
import pytest

from conftest import GPU_CASES
from oracle import client, ref

pytestmark = pytest.mark.gpu


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def z():
    import paper_2603_09190_b200 as z
    from paper_2603_09190_b200 import _lib, build
    build.build()
    _lib.load()
    return z


_states = {}


def _state(z, g):
    if g.name not in _states:
        _states[g.name] = z.ServerGlobalState(g.params(z), g.db)
    return _states[g.name]


def _reg(z, g):
    pk = z.PaillierPublicKey(g.m, g.m.bit_length())
    return z.ClientRegistration(pk, g.seed, z.client_id_of(pk))


@pytest.mark.parametrize("name", GPU_CASES)
def test_global_hint_bit_exact(z, golden, name):
    g = golden(name)
    st = _state(z, g)
    H = st.H
    assert H.shape == (g.d1, g.lwe["n"])
    assert _sha(H.astype("<u8")) == g.meta["H_sha256"]
    if "H" in g.arr:
        assert np.array_equal(H, g.arr["H"])
    assert np.array_equal(st.A[0], g.arr["A_row0"])


@pytest.mark.parametrize("name", GPU_CASES)
def test_db_matvec_bit_exact(z, golden, name):
    g = golden(name)
    st = _state(z, g)
    assert np.array_equal(st.db_matvec(g.arr["qu0"]), g.arr["b"])


@pytest.mark.parametrize("name", GPU_CASES)
def test_hint_entries_bit_exact(z, golden, name):
    g = golden(name)
    st = _state(z, g)
    reg = _reg(z, g)
    h = z.hint(st, reg, 0)
    assert [c.c for c in h.entries] == g.ints("k")
    assert h.db_version == 0 and h.query_index == 0


@pytest.mark.parametrize("name", GPU_CASES)
def test_respond_separate_and_combined(z, golden, name):
    g = golden(name)
    st = _state(z, g)
    reg = _reg(z, g)
    reg.hints[0] = z.hint(st, reg, 0)
    q = z.QueryMessage(reg.client_id, 0, z.SEPARATE, g.ints("ck_o"), g.arr["qu0"])
    timings = {}
    r = z.respond(st, reg, q, timings=timings)
    assert r.t == g.ints("t")
    assert [c.c for c in r.k] == g.ints("k")
    assert set(timings) == {"db_matvec", "hint_matvec", "total"}
    from paper_2603_09190_b200 import counters
    with counters.measure() as meas:
        rc = z.respond(st, reg, q, mode=z.COMBINED)
    assert [c.c for c in rc.k] == g.ints("K")
    assert meas.delta.modexp == 0 and meas.delta.add == g.groups
    sk = client.SecretKey(g.p, g.q)
    lw = g.lwe
    assert client.extract(sk, lw["q"], lw["p"], g.cap, g.gamma, g.d1, t=r.t,
                          k=[c.c for c in r.k]) == list(g.arr["record"])


@pytest.mark.parametrize("name", ["ragged", "tiny", "uniform_key", "standard32"])
def test_cuda_core_engine_bit_exact(z, golden, name):
    """The CUDA-core engine (IDP4A GEMV, IMAD hint and compression) -- the
    measured alternative to the tcgen05 path -- matches the reference too."""
    g = golden(name)
    st = z.ServerGlobalState(g.params(z), g.db, engine="cuda_core")
    assert np.array_equal(st.H, g.arr["H"]) if "H" in g.arr else True
    assert np.array_equal(st.db_matvec(g.arr["qu0"]), g.arr["b"])
    reg = _reg(z, g)
    reg.hints[0] = z.ClientHint(0, 0, [z.PaillierCiphertext(k) for k in g.ints("k")])
    q = z.QueryMessage(reg.client_id, 0, z.SEPARATE, g.ints("ck_o"), g.arr["qu0"])
    assert z.respond(st, reg, q).t == g.ints("t")
    assert [c.c for c in z.respond(st, reg, q, mode=z.COMBINED).k] == g.ints("K")


def test_respond_repeated_and_threads(z, golden):
    """Graph-replayed answers are stable across calls and threads."""
    import threading
    g = golden("tiny")
    st = _state(z, g)
    reg = _reg(z, g)
    reg.hints[0] = z.ClientHint(0, 0, [z.PaillierCiphertext(k) for k in g.ints("k")])
    q = z.QueryMessage(reg.client_id, 0, z.SEPARATE, g.ints("ck_o"), g.arr["qu0"])
    want = g.ints("t")
    for _ in range(3):
        assert z.respond(st, reg, q).t == want
    errs = []

    def worker():
        try:
            for _ in range(3):
                got = z.respond(st, reg, q).t
                if got != want:
                    errs.append("mismatch")
        except Exception as e:  # noqa: BLE001
            errs.append(repr(e))
    th = [threading.Thread(target=worker) for _ in range(3)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs


def test_respond_errors(z, golden):
    g = golden("desk_reduced")
    st = _state(z, g)
    reg = _reg(z, g)
    q = z.QueryMessage(reg.client_id, 0, z.SEPARATE, g.ints("ck_o"), g.arr["qu0"])
    with pytest.raises(KeyError):
        z.respond(st, reg, q)  # no hint registered
    reg.hints[0] = z.hint(st, reg, 0)
    st2 = z.ServerGlobalState(g.params(z), g.db, db_version=1)
    with pytest.raises(KeyError):
        z.respond(st2, reg, q)  # stale hint
    bad = z.QueryMessage(reg.client_id, 0, z.SEPARATE, g.ints("ck_o")[:-1], g.arr["qu0"])
    with pytest.raises(ValueError):
        z.respond(st, reg, bad)
    with pytest.raises(ValueError):
        z.respond(st, reg, q, mode="bogus")
    with pytest.raises(ValueError):
        z.ServerGlobalState(g.params(z), g.db[:, :-1])
    with pytest.raises(ValueError):
        z.ServerGlobalState(g.params(z), np.full((g.d0, g.d1), 256))


def test_multiexp_kat_gpu(z):
    import json
    import os
    from conftest import GOLDEN
    with open(os.path.join(GOLDEN, "multiexp_kat.json")) as f:
        cases = json.load(f)
    for c in cases:
        m = int(c["m"], 16)
        pk = z.PaillierPublicKey(m, m.bit_length())
        cts = [z.PaillierCiphertext(int(x, 16)) for x in c["bases"]]
        exps = [int(x, 16) for x in c["exps"]]
        assert z.multiexp(pk, cts, exps).c == int(c["result"], 16), (c["bits"], c["tag"])


@pytest.mark.parametrize("bits", [64, 768, 1024, 1536, 2048, 3072])
def test_paillier_matmul_random_vs_oracle(z, bits):
    rng = random.Random(bits)
    sk = client.keygen(bits, rng)
    m2 = sk.m * sk.m
    pk = z.PaillierPublicKey(sk.m, sk.m.bit_length())
    n, rows = 37, 5
    cts = [rng.randrange(m2) for _ in range(n)]
    H = [[rng.randrange(1 << rng.choice([1, 5, 31, 64, 300])) for _ in range(n)] for _ in range(rows)]
    H[2] = [0] * n
    got = z.paillier_matmul(pk, H, [z.PaillierCiphertext(c) for c in cts])
    assert [c.c for c in got] == [ref.multiexp(m2, cts, row) for row in H]
    a = [rng.randrange(m2) for _ in range(9)]
    b = [rng.randrange(m2) for _ in range(9)]
    assert [c.c for c in z.add_batch(pk, a, b)] == [x * y % m2 for x, y in zip(a, b)]


def test_end_to_end_seeded_queries(z):
    """Reference-style statistical correctness at the reduced desk parameters
    (test_protocol.py:190-209): 12 real queries, every row retrieved."""
    rng = random.Random(99)
    params = z.ProtocolParams(z.LweParams(n=64, q=1 << 32, p=256, noise_sigma=6.4), 32, 48, 768)
    db = np.array([[rng.randrange(256) for _ in range(48)] for _ in range(32)])
    st = z.ServerGlobalState(params, db)
    sk, seed = client.setup(768, rng)
    pk = z.PaillierPublicKey(sk.m, sk.m.bit_length())
    reg = z.ClientRegistration(pk, seed, z.client_id_of(pk))
    for qi in range(12):
        i0 = rng.randrange(32)
        reg.hints[qi] = z.hint(st, reg, qi)
        qu0, ck_o, _ = client.query(sk, seed, 64, 1 << 32, 256, 6.4, 32, i0, qi, rng, st.A)
        mode = z.SEPARATE if qi % 2 else z.COMBINED
        r = z.respond(st, reg, z.QueryMessage(reg.client_id, qi, mode, ck_o, qu0))
        if mode == z.SEPARATE:
            rec = client.extract(sk, 1 << 32, 256, params.capacity, 1 << 32, 48, t=r.t,
                                 k=[c.c for c in r.k])
        else:
            rec = client.extract(sk, 1 << 32, 256, params.capacity, 1 << 32, 48,
                                 combined=[c.c for c in r.k])
        assert rec == [int(x) for x in db[i0]]


@pytest.mark.parametrize("nq", [1, 5, 64, 70])
def test_respond_batch_bit_exact(z, golden, nq):
    """Batched answers (one GEMV for all queries, one compression launch) equal
    the per-query reference answers; mixed modes; different clients/moduli."""
    g = golden("tiny")
    st = _state(z, g)
    rng = random.Random(nq)
    A = st.A
    lw = g.lwe
    regs, qs, wants, modes = [], [], [], []
    keys = [client.SecretKey(g.p, g.q)] + [client.keygen(2048, random.Random(1000 + j))
                                            for j in range(2)]
    for i in range(nq):
        sk = keys[i % len(keys)]
        pk = z.PaillierPublicKey(sk.m, sk.m.bit_length())
        seed = bytes([i % 7] * 16)
        reg = z.ClientRegistration(pk, seed, z.client_id_of(pk))
        reg.hints[0] = z.ClientHint(0, 0, [z.PaillierCiphertext(rng.randrange(sk.m * sk.m))
                                           for _ in range(g.groups)])
        qu = np.array([rng.randrange(1 << 32) for _ in range(g.d0)], dtype=np.uint64)
        ck = [rng.randrange(sk.m) for _ in range(lw["n"])]
        mode = z.SEPARATE if i % 3 else z.COMBINED
        regs.append(reg)
        qs.append(z.QueryMessage(reg.client_id, 0, mode, ck, qu))
        modes.append(mode)
    got = z.respond_batch(st, regs, qs)
    for i in sorted({0, min(1, nq - 1), nq // 2, nq - 1}):
        want = z.respond(st, regs[i], qs[i])
        assert got[i].mode == modes[i]
        assert got[i].t == want.t and [c.c for c in got[i].k] == [c.c for c in want.k], i
    # and against the oracle for one query
    b = ref.db_matvec(g.db, qs[-1].qu0, 1 << 32)
    H = st.H
    sk = keys[(nq - 1) % len(keys)]
    t = ref.answer_t(H, b, qs[-1].ck_o, sk.m, g.cap, g.gamma, g.d1)
    if modes[-1] == z.SEPARATE:
        assert got[-1].t == t
    else:
        k = [c.c for c in regs[-1].hints[0].entries]
        assert [c.c for c in got[-1].k] == ref.combined(t, k, sk.m)


@pytest.mark.parametrize("name", ["toy", "uniform_key", "standard32", "q16"])
def test_respond_batch_general_gamma(z, golden, name):
    """Batch scales other than 2^32 through respond_batch (strided positional
    fold for gamma = 2^64, per-row weights otherwise) equal the reference."""
    g = golden(name)
    st = _state(z, g)
    reg = _reg(z, g)
    reg.hints[0] = z.ClientHint(0, 0, [z.PaillierCiphertext(k) for k in g.ints("k")])
    qs = [z.QueryMessage(reg.client_id, 0, md, g.ints("ck_o"), g.arr["qu0"])
          for md in (z.SEPARATE, z.COMBINED, z.SEPARATE)]
    got = z.respond_batch(st, [reg] * 3, qs)
    assert got[0].t == g.ints("t") and got[2].t == g.ints("t")
    assert [c.c for c in got[1].k] == g.ints("K")
