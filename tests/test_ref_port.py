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
