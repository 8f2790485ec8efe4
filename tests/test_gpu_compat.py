"""The reference's RNS API and operation counters through the drop-in
(rns.py:19-188, paillier.py:134-193 counter bump :192), on the device:

* rns_matmul_mod on matrix_to_rns matrices: the reference's hand case
  (test_rns.py / test_acceptance.py c06) and random instances against Python
  big-integer products, with the reference's ValueErrors;
* ServerGlobalState.basis / .H_rns: rns_matmul_mod(state.basis, state.H_rns,
  ck_o, m) equals the oracle's hv, and the materialised residues equal the
  reference algorithm's H_rns (oracle/ref_port.py, pinned to the goldens);
* hint() bumps group_mult by exactly the reference's count
  (golden hint_group_mults, recorded from the unmodified reference).
"""

import random

import numpy as np
import pytest

from oracle import ref, ref_port

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def z():
    import paper_2603_09190_b200 as z
    from paper_2603_09190_b200 import _lib, build
    build.build()
    _lib.load()
    return z


def test_rns_hand_case_and_random(z):
    from paper_2603_09190_b200 import rns
    basis = rns.build_basis(3, 2)
    assert basis.primes_int == [7, 5] and rns.build_basis(2, 1).primes_int == [3]
    assert rns.rns_matmul_mod(basis, rns.matrix_to_rns(basis, [[2]]), [3], 35, h_bound=2) == [6]
    small = rns.build_basis(7, 4)
    H = np.array([[2]], dtype=object)
    assert rns.rns_matmul_mod(small, rns.matrix_to_rns(small, H), [3], 35, h_bound=2) == [6]
    rng = random.Random(606)
    basis = rns.build_basis(27, 60)
    for bits in (700, 2048, 3072):
        m = rng.getrandbits(bits) | 1 | (1 << (bits - 1))
        for _ in range(4):
            rows, cols = rng.randrange(1, 9), rng.randrange(1, 17)
            Hm = [[rng.randrange(m) for _ in range(cols)] for _ in range(rows)]
            v = [rng.randrange(m) for _ in range(cols)]
            b = basis if bits == 700 else rns.build_basis(27, 480)
            got = rns.rns_matmul_mod(b, rns.matrix_to_rns(b, Hm), v, m)
            assert got == [sum(h * x for h, x in zip(row, v)) % m for row in Hm]
    with pytest.raises(ValueError):
        rns.rns_matmul_mod(basis, rns.matrix_to_rns(basis, [[1, 2]]), [1], 35)
    with pytest.raises(ValueError):       # Q too small for the bound
        tiny = rns.build_basis(3, 2)
        rns.rns_matmul_mod(tiny, rns.matrix_to_rns(tiny, [[5]]), [30], 1001)
    with pytest.raises(ValueError):
        rns.build_basis(28, 2)


@pytest.mark.parametrize("name", ["desk_reduced", "ragged", "uniform_key", "toy"])
def test_state_h_rns(z, golden, name):
    from paper_2603_09190_b200 import rns
    g = golden(name)
    st = z.ServerGlobalState(g.params(z), g.db)
    lw = g.lwe
    A = ref.public_matrix(b"\x00" * 16, g.d0, lw["n"], lw["q"])
    H = ref.global_hint(g.db, A, lw["q"])
    ck = g.ints("ck_o")
    hv = ref.answer_t(H, np.zeros(g.d1, np.uint64), ck, g.m, g.cap, g.gamma, g.d1)
    assert rns.rns_matmul_mod(st.basis, st.H_rns, ck, g.m) == hv
    assert st.H_rns.shape == (240, g.groups, lw["n"])
    if g.gamma == 1 << 32:
        port = ref_port.PortState(g.db, A, g.cap)
        assert np.array_equal(np.asarray(st.H_rns), port.H_rns)
    else:      # residues of the general-gamma scaled rows
        Hs = ref.scale_rows(H, g.cap, g.gamma, g.d1, lw["n"])
        res = np.asarray(st.H_rns)
        primes = st.basis.primes_int
        for i in (0, 7, 239):
            want = np.array([[x % primes[i] for x in row] for row in Hs], dtype=np.float64)
            assert np.array_equal(res[i], want)


@pytest.mark.parametrize("name", ["desk_reduced", "ragged", "zero_db", "max_db", "tiny",
                                  "uniform_key", "q16"])
def test_hint_counts_reference_group_mults(z, golden, name):
    from paper_2603_09190_b200 import counters
    g = golden(name)
    st = z.ServerGlobalState(g.params(z), g.db)
    pk = z.PaillierPublicKey(g.m, g.m.bit_length())
    reg = z.ClientRegistration(pk, g.seed, z.client_id_of(pk))
    with counters.measure() as mm:
        h = z.hint(st, reg, 0)
    assert [c.c for c in h.entries] == g.ints("k")
    assert mm.delta.group_mult == g.meta["hint_group_mults"]
    assert mm.delta.modexp == 0


def test_cko_width_checked(z, golden):
    """ck_o entries at or above 2^(32 lm) raise ValueError on every input path
    (ADVICE r01); entries in [m, 2^(32 lm)) give the exact (H ck_o) mod m."""
    g = golden("desk_reduced")
    st = z.ServerGlobalState(g.params(z), g.db)
    pk = z.PaillierPublicKey(g.m, g.m.bit_length())
    reg = z.ClientRegistration(pk, g.seed, z.client_id_of(pk))
    reg.hints[0] = z.ClientHint(0, 0, [z.PaillierCiphertext(1)] * g.groups)
    ck = g.ints("ck_o")
    lm = -(-g.m.bit_length() // 1024) * 32
    wide = list(ck)
    wide[3] = 1 << (32 * lm)
    with pytest.raises(ValueError):
        z.respond(st, reg, z.QueryMessage(reg.client_id, 0, z.SEPARATE, wide, g.arr["qu0"]))
    big = list(ck)
    big[5] += g.m
    r = z.respond(st, reg, z.QueryMessage(reg.client_id, 0, z.SEPARATE, big, g.arr["qu0"]))
    assert r.t == g.ints("t")


def test_undersized_modulus_exact(z, golden):
    """A modulus narrower than 32 * cap bits (respond() called directly, without
    the server's key-size check): the capacity bound B_g < m no longer holds, the
    answer must still equal the oracle (the captured plan's one-subtraction
    finish is bypassed)."""
    g = golden("desk_reduced")
    st = z.ServerGlobalState(g.params(z), g.db)
    rng = random.Random(5)
    lw = g.lwe
    A = ref.public_matrix(b"\x00" * 16, g.d0, lw["n"], lw["q"])
    H = ref.global_hint(g.db, A, lw["q"])
    for bits in (700, 950):
        m = rng.getrandbits(bits) | (1 << (bits - 1)) | 1
        pk = z.PaillierPublicKey(m, bits)
        reg = z.ClientRegistration(pk, b"\x01" * 16, z.client_id_of(pk))
        reg.hints[0] = z.ClientHint(0, 0, [z.PaillierCiphertext(1)] * g.groups)
        ck = [rng.randrange(m) for _ in range(lw["n"])]
        want = ref.answer_t(H, g.arr["b"], ck, m, g.cap, g.gamma, g.d1)
        r = z.respond(st, reg, z.QueryMessage(reg.client_id, 0, z.SEPARATE, ck, g.arr["qu0"]))
        assert r.t == want, bits
