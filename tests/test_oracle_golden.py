"""Pin the CPU oracle (oracle/) to the reference's own outputs (tests/golden/).

The golden files were produced by running the unmodified reference package
(tests/golden/make_golden.py); every oracle function used as a checker by the
GPU parity tests is verified here first, on CPU.
"""

import hashlib
import json
import os
import random

import numpy as np
import pytest

from conftest import ALL_CASES, GOLDEN, le_ints
from oracle import client, ref


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", ALL_CASES)
def test_layout_matches_reference(golden, name):
    g = golden(name)
    lw = g.lwe
    gamma, cap, d1p = ref.layout(lw["n"], lw["q"], lw["key_dist"], g.bits,
                                 g.meta["scale_regime"], g.d1)
    assert (gamma, cap, d1p) == (g.gamma, g.cap, g.groups)


@pytest.mark.parametrize("name", ALL_CASES)
def test_public_matrix_and_global_hint(golden, name):
    g = golden(name)
    lw = g.lwe
    A = ref.public_matrix(b"\x00" * 16, g.d0, lw["n"], lw["q"])
    assert _sha(A.astype("<u8")) == g.meta["A_sha256"]
    assert np.array_equal(A[0], g.arr["A_row0"])
    H = ref.global_hint(g.db, A, lw["q"])
    assert _sha(H.astype("<u8")) == g.meta["H_sha256"]
    assert np.array_equal(H[[0, g.d1 // 2, g.d1 - 1]], g.arr["H_rows"])


@pytest.mark.parametrize("name", ALL_CASES)
def test_db_matvec(golden, name):
    g = golden(name)
    b = ref.db_matvec(g.db, g.arr["qu0"], g.lwe["q"])
    assert np.array_equal(b, g.arr["b"])


@pytest.mark.parametrize("name", ALL_CASES)
def test_answer_and_combined(golden, name):
    g = golden(name)
    lw = g.lwe
    A = ref.public_matrix(b"\x00" * 16, g.d0, lw["n"], lw["q"])
    H = ref.global_hint(g.db, A, lw["q"])
    ck_o = g.ints("ck_o")
    t = ref.answer_t(H, g.arr["b"], ck_o, g.m, g.cap, g.gamma, g.d1)
    assert t == g.ints("t")
    assert ref.combined(t, g.ints("k"), g.m) == g.ints("K")


@pytest.mark.parametrize("name", ["toy", "desk_reduced", "zero_db", "ragged", "max_db",
                                  "uniform_key", "standard32", "q16"])
def test_hint_entries(golden, name):
    g = golden(name)
    lw = g.lwe
    m2 = g.m * g.m
    ck_r = ref.derive_ck_r(m2, g.seed, 0, lw["n"])
    assert ck_r == g.ints("ck_r")
    A = ref.public_matrix(b"\x00" * 16, g.d0, lw["n"], lw["q"])
    H = ref.global_hint(g.db, A, lw["q"])
    Hs = ref.scale_rows(H, g.cap, g.gamma, g.d1, lw["n"])
    assert ref.hint_entries(Hs, ck_r, m2) == g.ints("k")


def test_hint_entry_tiny_last_group(golden):
    """BASELINE configs[0]: one (partial, 16-slot) group of the 17."""
    g = golden("tiny")
    lw = g.lwe
    m2 = g.m * g.m
    ck_r = ref.derive_ck_r(m2, g.seed, 0, lw["n"])
    assert ck_r == g.ints("ck_r")
    A = ref.public_matrix(b"\x00" * 16, g.d0, lw["n"], lw["q"])
    db = g.db
    cols = list(range((g.groups - 1) * g.cap, g.d1))
    H = ref.global_hint(db[:, cols], A, lw["q"])
    Hs = ref.scale_rows(H, len(cols), g.gamma, len(cols), lw["n"])
    assert ref.multiexp(m2, ck_r, Hs[0]) == g.ints("k")[-1]


def test_multiexp_kat():
    with open(os.path.join(GOLDEN, "multiexp_kat.json")) as f:
        cases = json.load(f)
    for c in cases:
        m = int(c["m"], 16)
        bases = [int(x, 16) for x in c["bases"]]
        exps = [int(x, 16) for x in c["exps"]]
        assert ref.multiexp(m * m, bases, exps) == int(c["result"], 16), (c["bits"], c["tag"])


def test_prg_kat():
    with open(os.path.join(GOLDEN, "prg_kat.json")) as f:
        k = json.load(f)
    assert ref.Stream(b"\x00" * 16, 3).read(64).hex() == k["stream_seed00_dom3_first64"]
    assert ref.Stream(b"\xab" * 16, 1, (5 << 32) | 7).read(48).hex() == k["stream_seedab_dom1_idx"]
    got = [ref.Stream(bytes(range(16)), 4, i).below((1 << 100) + 12345) for i in range(8)]
    assert [hex(x) for x in got] == k["below"]


@pytest.mark.parametrize("name", ["desk_reduced", "ragged"])
def test_client_restatement_reproduces_reference_query(golden, name):
    """oracle.client consumes random.Random exactly like the reference, so the
    seeded golden query is reproduced bit for bit (pins the input generator)."""
    g = golden(name)
    lw = g.lwe
    rng = random.Random(g.meta["seed"])
    db = np.array([[rng.randrange(lw["p"]) for _ in range(g.d1)] for _ in range(g.d0)])
    assert np.array_equal(db, g.db)
    sk, seed = client.setup(g.bits, rng)
    assert (sk.p, sk.q, seed) == (g.p, g.q, g.seed)
    i0 = rng.randrange(g.d0)
    assert i0 == g.i0
    A = ref.public_matrix(b"\x00" * 16, g.d0, lw["n"], lw["q"])
    qu0, ck_o, _ = client.query(sk, seed, lw["n"], lw["q"], lw["p"], lw["noise_sigma"], g.d0,
                                i0, 0, rng, A)
    assert np.array_equal(qu0, g.arr["qu0"])
    assert ck_o == g.ints("ck_o")
    rec = client.extract(sk, lw["q"], lw["p"], g.cap, g.gamma, g.d1, t=g.ints("t"), k=g.ints("k"))
    assert rec == list(g.arr["record"])
    rec2 = client.extract(sk, lw["q"], lw["p"], g.cap, g.gamma, g.d1, combined=g.ints("K"))
    assert rec2 == list(g.arr["record"])
