"""GPU parity through the handle-level C ABI (include/zippir_db.h) with host
buffers only (numpy in, numpy out; no torch on this path).

Same golden outputs of the unmodified reference as test_gpu_parity.py:
H, b, t, COMBINED K, hint entries k, the multiexp KATs; plus the row update
against a fresh build and the oracle for batched matvec.
"""

import json
import os
import random

import numpy as np
import pytest

from conftest import GOLDEN, GPU_CASES
from oracle import client, ref

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_2603_09190_b200 import _lib, build, dbapi
    build.build()
    _lib.load()
    return dbapi


def _params(g):
    import paper_2603_09190_b200 as z
    return g.params(z)


@pytest.mark.parametrize("name", GPU_CASES)
def test_handle_api_golden(api, golden, name):
    g = golden(name)
    with api.DeviceDatabase(_params(g), g.db) as d:
        assert d.groups == g.groups
        H = d.global_hint()
        if "H" in g.arr:
            assert np.array_equal(H.astype(np.uint64), g.arr["H"])
        assert np.array_equal(d.db_matvec(g.arr["qu0"]), g.arr["b"])
        assert d.answer(g.arr["qu0"], g.ints("ck_o"), g.m) == g.ints("t")
        assert d.answer_combined(g.arr["qu0"], g.ints("ck_o"), g.m, g.ints("k")) == g.ints("K")
        assert d.client_hint(g.m, g.seed, 0) == g.ints("k")


@pytest.mark.parametrize("name", ["ragged", "standard32", "toy"])
def test_handle_api_cuda_core_and_explicit_A(api, golden, name):
    g = golden(name)
    A = ref.public_matrix(b"\x00" * 16, g.d0, g.lwe["n"], g.lwe["q"])
    with api.DeviceDatabase(_params(g), g.db, A=A, engine="cuda_core") as d:
        assert np.array_equal(d.db_matvec(g.arr["qu0"]), g.arr["b"])
        assert d.answer(g.arr["qu0"], g.ints("ck_o"), g.m) == g.ints("t")
        assert d.client_hint(g.m, g.seed, 0) == g.ints("k")


@pytest.mark.parametrize("name", ["ragged", "uniform_key"])
def test_handle_api_update_rows(api, golden, name):
    g = golden(name)
    params = _params(g)
    rng = np.random.default_rng(5)
    cols = np.array(sorted({0, g.d1 - 1, *rng.choice(g.d1, 7, replace=False).tolist()}))
    vals = rng.integers(0, g.lwe["p"], (cols.size, g.d0), dtype=np.uint8)
    db2 = np.array(g.db, dtype=np.uint8, copy=True)
    db2[:, cols] = vals.T
    with api.DeviceDatabase(params, g.db) as d, api.DeviceDatabase(params, db2) as fresh:
        d.update_rows(cols, vals)
        assert np.array_equal(d.global_hint(), fresh.global_hint())
        qu = g.arr["qu0"]
        assert np.array_equal(d.db_matvec(qu), ref.db_matvec(db2, qu, g.lwe["q"]))
        assert d.answer(qu, g.ints("ck_o"), g.m) == fresh.answer(qu, g.ints("ck_o"), g.m)
        assert d.client_hint(g.m, g.seed, 3) == fresh.client_hint(g.m, g.seed, 3)
        with pytest.raises(ValueError):
            d.update_rows([g.d1], vals[:1])


def test_handle_api_batched_matvec(api, golden):
    g = golden("ragged")
    rng = np.random.default_rng(1)
    Q = rng.integers(0, 1 << 32, (70, g.d0), dtype=np.uint64)   # 64 + 6: two passes
    with api.DeviceDatabase(_params(g), g.db) as d:
        B = d.db_matvec(Q)
    for v in (0, 33, 63, 64, 69):
        assert np.array_equal(B[v], ref.db_matvec(g.db, Q[v], 1 << 32)), v


def test_handle_api_errors(api, golden):
    g = golden("q16")                                  # p = 16: symbols 16..255 are invalid
    bad = np.array(g.db, dtype=np.uint8, copy=True)
    bad[0, 0] = g.lwe["p"]
    with pytest.raises(ValueError, match="symbol out of range"):
        api.DeviceDatabase(_params(g), bad)
    with pytest.raises(ValueError):
        api.DeviceDatabase(_params(g), g.db[:, :-1])
    with api.DeviceDatabase(_params(g), g.db) as d:
        with pytest.raises(ValueError):
            d.answer(g.arr["qu0"][:-1], g.ints("ck_o"), g.m)
        with pytest.raises(ValueError, match="odd"):
            d.answer(g.arr["qu0"], g.ints("ck_o"), g.m + 1)


def test_multiexp_and_montmul_batch_kat(api):
    with open(os.path.join(GOLDEN, "multiexp_kat.json")) as f:
        cases = json.load(f)
    for c in cases:
        m = int(c["m"], 16)
        bases = [int(x, 16) for x in c["bases"]]
        exps = [int(x, 16) for x in c["exps"]]
        got = api.multiexp_batch(bases, [exps, exps[::-1]], m * m)
        assert got[0] == int(c["result"], 16), (c["bits"], c["tag"])
        assert got[1] == ref.multiexp(m * m, bases, exps[::-1]), (c["bits"], c["tag"])
    rng = random.Random(3)
    for bits in (64, 1024, 2048):          # N = m^2: 128 .. 4096 bits
        sk = client.keygen(bits, rng)
        N = sk.m * sk.m
        a = [rng.randrange(N) for _ in range(50)]
        b = [rng.randrange(N) for _ in range(50)]
        assert api.montmul_batch(a, b, N) == [x * y % N for x, y in zip(a, b)]


def test_handle_api_mixed_limb_widths(api, golden):
    """Keys of different widths on one handle, and limb rows wider than the
    modulus (zero top limbs) in and out: results stay exact."""
    g = golden("ragged")
    rng = random.Random(11)
    with api.DeviceDatabase(_params(g), g.db) as d:
        H = d.global_hint().astype(np.uint64)
        qu = g.arr["qu0"]
        b = ref.db_matvec(g.db, qu, 1 << 32)
        for bits in (1024, 1000, 950, 1024):
            m = g.m if bits == 1024 else (rng.getrandbits(bits) | (1 << (bits - 1)) | 1)
            ck = [rng.randrange(m) for _ in range(g.lwe["n"])]
            want = ref.answer_t(H, b, ck, m, g.cap, g.gamma, g.d1)
            assert d.answer(qu, ck, m) == want, bits
        # explicit wider rows through the raw C ABI: L = 33 limbs for a 1024-bit m
        import ctypes
        from paper_2603_09190_b200 import _lib
        from paper_2603_09190_b200.bigint import ints_to_limbs, limbs_to_ints
        L = 33
        ck = g.ints("ck_o")
        q = np.ascontiguousarray(qu.astype(np.uint32))
        c = ints_to_limbs(ck, L)
        mm = ints_to_limbs([g.m], L)
        t = np.empty((g.groups, L), dtype=np.uint32)
        vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        _lib.call("zpir_db_answer", d._h, vp(q), vp(c), vp(mm), L, vp(t))
        assert limbs_to_ints(t) == g.ints("t")
        K = np.empty((g.groups, 2 * L), dtype=np.uint32)
        kin = ints_to_limbs(g.ints("k"), 2 * L)
        _lib.call("zpir_db_answer_combined", d._h, vp(q), vp(c), vp(mm), L, vp(kin), vp(K))
        assert limbs_to_ints(K) == g.ints("K")


def test_handle_api_tensor_core_hint(api, monkeypatch):
    """zpir_db_client_hint on a DB with >= 2048 exponent rows takes the
    tensor-core Pippenger (full Montgomery inverse computed on the host by
    Newton iteration); its entries equal the Python API's IMAD path."""
    import paper_2603_09190_b200 as z
    from paper_2603_09190_b200 import protocol
    rng = random.Random(2048)
    d0, d1, n = 128, 2100, 64
    params = z.ProtocolParams(z.LweParams(n=n, q=1 << 32, p=256, noise_sigma=6.4), d0, d1, 2048)
    db = np.frombuffer(np.random.default_rng(3).bytes(d0 * d1), dtype=np.uint8).reshape(d0, d1)
    sk, seed = client.setup(2048, rng)
    with api.DeviceDatabase(params, db) as d:
        k_tc = d.client_hint(sk.m, seed, 2)
    monkeypatch.setattr(protocol, "TC_MIN_ROWS", 1 << 30)        # IMAD slot_fixed
    st = z.ServerGlobalState(params, db)
    pk = z.PaillierPublicKey(sk.m, sk.m.bit_length())
    reg = z.ClientRegistration(pk, seed, z.client_id_of(pk))
    assert k_tc == [c.c for c in z.hint(st, reg, 2).entries]


def test_handle_api_concurrent_threads(api, golden):
    """The handle ABI from several threads at once (ctypes drops the GIL):
    calls on one handle serialise on its lock and share its pinned staging;
    two handles (and their creation, which shares the process-wide upload
    stages) run side by side. Every answer stays bit-exact."""
    import threading
    import paper_2603_09190_b200 as z
    g = golden("tiny")                                 # BASELINE configs[0]
    qu, ck, m = g.arr["qu0"], g.ints("ck_o"), g.m
    t_want, K_want, k_want = g.ints("t"), g.ints("K"), g.ints("k")
    errors = []
    handles = []
    lock = threading.Lock()
    # a DB above the staged-upload threshold (16 MiB), created from two threads
    big_p = z.ProtocolParams(z.LweParams(1024, 1 << 32, 256, 6.4), 4096, 4160, 2048)
    big = np.frombuffer(np.random.default_rng(3).bytes(4096 * 4160), np.uint8).reshape(4096, 4160)
    big_q = np.random.default_rng(4).integers(0, 1 << 32, 4096, dtype=np.uint64)
    big_b = ref.db_matvec(big, big_q, 1 << 32)

    def create(prm, db, into):
        try:
            d = api.DeviceDatabase(prm, db)
            with lock:
                into.append(d)
        except Exception as e:
            errors.append(e)

    bigs = []
    th = [threading.Thread(target=create, args=a) for a in
          [(big_p, big, bigs), (big_p, big, bigs), (_params(g), g.db, handles),
           (_params(g), g.db, handles)]]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors and len(handles) == 2 and len(bigs) == 2, errors[:1]
    for d in bigs:
        assert np.array_equal(d.db_matvec(big_q), big_b)
        d.close()

    def work(d, i):
        try:
            for _ in range(4):
                if i % 2:
                    assert d.answer_combined(qu, ck, m, k_want) == K_want
                else:
                    assert d.answer(qu, ck, m) == t_want
        except Exception as e:
            errors.append(e)

    th = [threading.Thread(target=work, args=(handles[i % 2], i)) for i in range(6)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for d in handles:
        d.close()
    assert not errors, errors[:1]
