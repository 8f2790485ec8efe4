"""BASELINE configs[1] at full size on the GPU: a 1 GiB DB (32768 x 32768 u8,
uniform), n = 1024, q = 2^32, 2048-bit Paillier -- the bench's workload --
checked through size-independent properties and sampled oracle values
(the CPU oracle cannot restate the whole answer at this size in seconds):

* retrieval: a real client query (oracle/client.py: binary LWE secret,
  Gaussian error, Paillier-encrypted compression key) answered by respond()
  in both modes decodes to the requested DB row, all 32768 entries;
* b = DB qu mod 2^32 equals the C oracle GEMV, and is linear in qu;
* H = -DB A mod 2^32 equals the C oracle on sampled DB rows;
* t on sampled groups equals the reference formula (oracle/ref.answer_t);
* BASELINE configs[2] (8 GiB, 92682^2) on one GPU: b and sampled t groups.
"""

import random

import numpy as np
import pytest

from oracle import c as oracle_c
from oracle import client, ref

pytestmark = pytest.mark.gpu

D = 32768
N = 1024
Q = 1 << 32


@pytest.fixture(scope="module")
def full():
    import torch
    import paper_2603_09190_b200 as z
    from paper_2603_09190_b200 import _lib, build
    build.build()
    _lib.load()
    db = np.frombuffer(np.random.default_rng(20261020).bytes(D * D), dtype=np.uint8).reshape(D, D)
    params = z.ProtocolParams(z.LweParams(N, Q, 256, 6.4), D, D, 2048)
    st = z.ServerGlobalState(params, db)
    torch.cuda.synchronize()
    return z, params, db, st


def test_fullsize_gemv_oracle_and_linearity(full):
    z, params, db, st = full
    rng = np.random.default_rng(1)
    qa = rng.integers(0, Q, D, dtype=np.uint64)
    qb = rng.integers(0, Q, D, dtype=np.uint64)
    ba, bb = st.db_matvec(qa), st.db_matvec(qb)
    assert np.array_equal(ba, oracle_c.db_matvec(db, qa))
    assert np.array_equal(st.db_matvec((qa + qb) % Q), (ba + bb) % Q)


def test_fullsize_global_hint_sampled_rows(full):
    z, params, db, st = full
    A = ref.public_matrix(b"\x00" * 16, D, N, Q)
    rows = [0, 1, 62, 63, 12345, D - 64, D - 1]
    H = st.H
    assert np.array_equal(H[rows].astype(np.uint64), oracle_c.hint_cols(db, A, rows))


def test_fullsize_retrieval_and_sampled_groups(full):
    """A real client query, hint and answer at the bench's size: the decoded
    row is the DB row (SEPARATE and COMBINED), and t on sampled groups
    equals the reference formula."""
    z, params, db, st = full
    rng = random.Random(33)
    sk, seed = client.setup(2048, rng)
    pk = z.PaillierPublicKey(sk.m, sk.m.bit_length())
    reg = z.ClientRegistration(pk, seed, z.client_id_of(pk))
    reg.hints[0] = z.hint(st, reg, 0)
    A = st.A
    i0 = 4242
    qu0, ck_o, _ = client.query(sk, seed, N, Q, 256, 6.4, D, i0, 0, rng, A)
    r = z.respond(st, reg, z.QueryMessage(reg.client_id, 0, z.SEPARATE, ck_o, qu0))
    cap = params.capacity
    got = client.extract(sk, Q, 256, cap, Q, D, t=r.t, k=[c.c for c in r.k])
    assert got == [int(x) for x in db[i0]]
    # sampled groups against oracle/ref.answer_t (protocol.py:343-351)
    b = st.db_matvec(qu0)
    H = st.H
    for g in (0, 1, 260, params.d1_prime - 1):
        lo, hi = g * cap, min((g + 1) * cap, D)
        want = ref.answer_t(H[lo:hi], b[lo:hi], ck_o, sk.m, cap, Q, hi - lo)
        assert r.t[g] == want[0], g
    rc = z.respond(st, reg, z.QueryMessage(reg.client_id, 0, z.COMBINED, ck_o, qu0))
    got = client.extract(sk, Q, 256, cap, Q, D, combined=[c.c for c in rc.k])
    assert got == [int(x) for x in db[i0]]


def test_fullsize_8gib_gemv_and_sampled_groups():
    """BASELINE configs[2] on one GPU: 92682 x 92682 (8 GiB, d0 > 2^16 so the
    byte-plane sums wrap s32 many times): b equals the C oracle GEMV, t on
    sampled groups (incl. the partial last group) equals the reference formula."""
    import os
    import torch
    import paper_2603_09190_b200 as z
    d = 92682
    try:
        mem = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    except (ValueError, OSError):
        mem = 0
    if mem and mem < 48 * 2**30:
        pytest.skip("needs ~48 GB of host memory")
    db = np.frombuffer(np.random.default_rng(92682).bytes(d * d), dtype=np.uint8).reshape(d, d)
    params = z.ProtocolParams(z.LweParams(N, Q, 256, 6.4), d, d, 2048)
    st = z.ServerGlobalState(params, db)
    qu = np.random.default_rng(2).integers(0, Q, d, dtype=np.uint64)
    b = st.db_matvec(qu)
    assert np.array_equal(b, oracle_c.db_matvec(db, qu))
    sk = client.keygen(2048, random.Random(8))
    pk = z.PaillierPublicKey(sk.m, sk.m.bit_length())
    reg = z.ClientRegistration(pk, b"\x08" * 16, z.client_id_of(pk))
    reg.hints[0] = z.ClientHint(0, 0, [z.PaillierCiphertext(1)] * params.d1_prime)
    r = random.Random(9)
    ck_o = [r.randrange(sk.m) for _ in range(N)]
    t = z.respond(st, reg, z.QueryMessage(reg.client_id, 0, z.SEPARATE, ck_o, qu)).t
    cap = params.capacity
    A = ref.public_matrix(b"\x00" * 16, d, N, Q)
    for g in (0, 777, params.d1_prime - 1):
        lo, hi = g * cap, min((g + 1) * cap, d)
        Hg = oracle_c.hint_cols(db, A, list(range(lo, hi)))
        want = ref.answer_t(Hg, b[lo:hi], ck_o, sk.m, cap, Q, hi - lo)
        assert t[g] == want[0], g
    del st
    torch.cuda.empty_cache()


def test_fullsize_batch_equals_single(full):
    """BASELINE configs[3] shape (queries batched on the N = 256 GEMV and the
    CTA-pair planar compression) at 1 GiB: every query's t equals respond()."""
    z, params, db, st = full
    sk = client.keygen(2048, random.Random(64))
    pk = z.PaillierPublicKey(sk.m, sk.m.bit_length())
    reg = z.ClientRegistration(pk, b"\x40" * 16, z.client_id_of(pk))
    reg.hints[0] = z.ClientHint(0, 0, [z.PaillierCiphertext(1)] * params.d1_prime)
    rng = np.random.default_rng(64)
    r = random.Random(65)
    qms = [z.QueryMessage(reg.client_id, 0, z.SEPARATE, [r.randrange(sk.m) for _ in range(N)],
                          rng.integers(0, Q, D, dtype=np.uint64)) for _ in range(6)]
    outs = z.respond_batch(st, [reg] * len(qms), qms)
    for q, o in zip(qms, outs):
        assert o.t == z.respond(st, reg, q).t
