"""Pin the GMP-backed C oracle (oracle/c/zpir_gmp_oracle.c) -- the checker
the BASELINE-size GPU parity tests use -- to the reference's own outputs
(tests/golden, produced by the unmodified reference) on CPU.

* multiexp: all 21 reference multiexp KATs, and every one of the 17 hint
  entries of BASELINE configs[0] (1024 x 1024 DB, n = 1024, 2048-bit key)
  from oracle-computed H and ck_r;
* answer t and COMBINED K: every golden case.
"""

import json
import os

import numpy as np
import pytest

from conftest import ALL_CASES, GOLDEN
from oracle import c as oc
from oracle import ref


def test_gmp_multiexp_kat():
    with open(os.path.join(GOLDEN, "multiexp_kat.json")) as f:
        cases = json.load(f)
    for c in cases:
        m = int(c["m"], 16)
        bases = [int(x, 16) for x in c["bases"]]
        exps = [int(x, 16) for x in c["exps"]]
        got = oc.multiexp_rows(bases, [exps], m * m)
        assert got == [int(c["result"], 16)], (c["bits"], c["tag"])


def test_gmp_multiexp_matches_python_restatement():
    import random
    r = random.Random(5)
    m2 = (r.getrandbits(512) | 1) ** 2
    bases = [r.randrange(m2) for _ in range(40)]
    rows = [[r.getrandbits(r.choice([0, 1, 5, 6, 7, 64, 300])) for _ in range(40)] for _ in range(6)]
    rows.append([0] * 40)
    assert oc.multiexp_rows(bases, rows, m2) == [ref.multiexp(m2, bases, e) for e in rows]


def test_gmp_hint_entries_configs0(golden):
    """All 17 hint entries of BASELINE configs[0] (the reference's golden k)."""
    g = golden("tiny")
    lw = g.lwe
    m2 = g.m * g.m
    ck_r = ref.derive_ck_r(m2, g.seed, 0, lw["n"])
    assert ck_r == g.ints("ck_r")
    A = ref.public_matrix(b"\x00" * 16, g.d0, lw["n"], lw["q"])
    H = oc.hint_rows(g.db, A)
    assert np.array_equal(H.astype(np.uint64), ref.global_hint(g.db, A, lw["q"]))
    E = oc.scaled_exponents(H, g.cap)
    assert oc.multiexp_rows(ck_r, E, m2) == g.ints("k")


@pytest.mark.parametrize("name", ALL_CASES)
def test_gmp_answer_and_combined(golden, name):
    g = golden(name)
    lw = g.lwe
    A = ref.public_matrix(b"\x00" * 16, g.d0, lw["n"], lw["q"])
    H = ref.global_hint(g.db, A, lw["q"])
    t = oc.answer_t(H, g.arr["b"], g.ints("ck_o"), g.m, g.cap, g.gamma, g.d1)
    assert t == g.ints("t")
    assert oc.combined(t, g.ints("k"), g.m) == g.ints("K")


def test_hint_rows_matches_hint_cols():
    rng = np.random.default_rng(3)
    db = rng.integers(0, 256, (300, 200), dtype=np.uint8)
    A = rng.integers(0, 1 << 32, (300, 96), dtype=np.uint64)
    H = oc.hint_rows(db, A, 17, 150)
    assert np.array_equal(H.astype(np.uint64), oc.hint_cols(db, A, list(range(17, 150))))


def test_oracle_compressor_matches_reference_kat():
    """oracle/ref's compressor restatement (the checker of test_gpu_compress)
    against the reference's own outputs (tests/golden/compress_kat.json,
    compress.py:99-258: lwe_compress, fast_lwe_compress, batched and
    fast_batched_lwe_compress)."""
    with open(os.path.join(GOLDEN, "compress_kat.json")) as f:
        cases = json.load(f)
    for c in cases:
        m = int(c["m"], 16)
        ck = [int(x, 16) for x in c["ck"]]
        q = c["q"]
        for ct, want, want_fast in zip(c["cts"], c["lwe_compress"], c["fast_lwe_compress"]):
            got = ref.lwe_compress(m, ck, ct["a"], ct["b"], q)
            assert got == int(want, 16) == int(want_fast, 16), c["bits"]
        cts = [(ct["a"], ct["b"]) for ct in c["cts"][: c["ell"]]]
        got = ref.batched_lwe_compress(m, ck, cts, int(c["gamma"]), q)
        assert got == int(c["batched"], 16) == int(c["fast_batched"], 16), c["bits"]
