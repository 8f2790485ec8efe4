"""The timed CPU baseline (oracle/ref_port.py, the reference's own float64 +
RNS algorithm) reproduces the reference's golden outputs bit for bit."""

import numpy as np
import pytest

from oracle import ref, ref_port


@pytest.mark.parametrize("name", ["desk_reduced", "ragged", "max_db", "tiny"])
def test_port_matches_golden(golden, name):
    g = golden(name)
    lw = g.lwe
    A = ref.public_matrix(b"\x00" * 16, g.d0, lw["n"], lw["q"])
    st = ref_port.PortState(g.db, A, g.cap)
    assert np.array_equal(st.H.astype(np.uint64)[[0, g.d1 // 2, g.d1 - 1]], g.arr["H_rows"])
    assert np.array_equal(st.db_matvec(g.arr["qu0"]), g.arr["b"])
    assert st.respond_t(g.arr["qu0"], g.ints("ck_o"), g.m) == g.ints("t")


def test_basis_matches_reference_constants():
    b = ref_port.Basis(3, 2)
    assert b.primes == [7, 5]
    b = ref_port.Basis()
    assert b.Q > 1 << 6400 and len(set(b.primes)) == 240


def test_chunked_port_matches_oracle():
    """d0 above the float64 exactness bound: the chunked restatement (SURVEY
    8c, BASELINE configs[2]) equals the exact integer oracle."""
    rng = np.random.default_rng(9)
    d0, d1, n = 300, 70, 32
    db = rng.integers(0, 256, (d0, d1), dtype=np.uint8)
    A = rng.integers(0, 1 << 32, (d0, n), dtype=np.uint64)
    qu = rng.integers(0, 1 << 32, d0, dtype=np.uint64)

    class Small(ref_port.PortState):
        CHUNK = 128
    st = Small(db, A, 31, basis=ref_port.Basis(27, 120))
    assert np.array_equal(st.H.astype(np.uint64), ref.global_hint(db, A, 1 << 32))
    b = ref.db_matvec(db, qu, 1 << 32)
    assert np.array_equal(st.db_matvec(qu), b)
    m = (1 << 1023) + 1155
    ck = [int(x) for x in rng.integers(0, 1 << 62, n, dtype=np.uint64)]
    H = ref.global_hint(db, A, 1 << 32)
    assert st.respond_t(qu, ck, m) == ref.answer_t(H, b, ck, m, 31, 1 << 32, d1)
