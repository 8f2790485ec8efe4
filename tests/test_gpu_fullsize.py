"""BASELINE configs[1], [3] and [4] at full size on the GPU: a 1 GiB DB
(32768 x 32768 u8, uniform), n = 1024, q = 2^32, 2048-bit Paillier -- the
bench's workloads -- checked against the CPU oracle computed INDEPENDENTLY of
the device state (H from oracle/c's restatement of db^T A with A from
oracle/ref's ChaCha20, ck_r from oracle/ref, big-integer arithmetic from the
GMP restatement of the reference's multiexp / answer / combine, pinned by
tests/test_oracle_gmp.py) on sampled groups, plus size-independent
properties:

* retrieval: a real client query answered by respond() decodes to the
  requested DB row (SEPARATE and COMBINED);
* b = DB qu mod 2^32 equals the C oracle GEMV, and is linear in qu;
* H = -DB A mod 2^32 equals the C oracle on sampled DB rows;
* t and K on sampled groups equal the oracle;
* the tensor-core hint (the production path at this size) on sampled groups
  incl. the partial last group equals the reference's multiexp over the
  oracle's H_scaled and ck_r (configs[1]/[4]);
* configs[4]: a 1% row update gives the same device H as a full rebuild, and
  refreshed hints (IMAD path, and the tensor-core path for >= 2048 changed
  rows) equal full hints on the rebuilt state and the oracle;
* configs[3]: all 64 batched queries equal respond(), two of them the oracle;
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


@pytest.fixture(scope="module")
def oracle_A():
    return ref.public_matrix(b"\x00" * 16, D, N, Q)


def _groups_H(db, A, cap, groups):
    """Oracle H rows of the given hint groups: {g: (rows, n) u32}."""
    out = {}
    for g in groups:
        lo, hi = g * cap, min((g + 1) * cap, D)
        out[g] = oracle_c.hint_rows(db, A, lo, hi)
    return out


SAMPLE_GROUPS = (0, 1, 260, 520)     # 520 = the partial last group (32768 mod 63 = 8 slots)


@pytest.fixture(scope="module")
def client_a(full, oracle_A):
    """A real client (oracle keygen) with its hint computed by the product
    path -- the tensor-core Pippenger at this size -- and the oracle's H of
    the sampled groups."""
    z, params, db, st = full
    rng = random.Random(33)
    sk, seed = client.setup(2048, rng)
    pk = z.PaillierPublicKey(sk.m, sk.m.bit_length())
    reg = z.ClientRegistration(pk, seed, z.client_id_of(pk))
    nslot = st.layout.groups * st.layout.cap
    assert z.protocol.TC_HINT and nslot >= z.protocol.TC_MIN_ROWS, "tensor-core hint path expected"
    reg.hints[0] = z.hint(st, reg, 0)
    Hg = _groups_H(db, oracle_A, params.capacity, SAMPLE_GROUPS)
    return sk, seed, reg, rng, Hg


def test_fullsize_global_hint_sampled_rows(full, oracle_A):
    z, params, db, st = full
    rows = [0, 1, 62, 63, 12345, D - 64, D - 1]
    H = st.H
    assert np.array_equal(H[rows].astype(np.uint64), oracle_c.hint_cols(db, oracle_A, rows))


def test_fullsize_tc_hint_vs_gmp_oracle(full, client_a):
    """configs[1]/[4]: hint entries from the tensor-core Pippenger equal the
    reference's multiexp k_g = prod_k ck_r[k]^H_scaled[g][k] mod m^2
    (paillier.py:134-193, protocol.py:291-296) over the oracle's H_scaled and
    ck_r, on sampled groups incl. the partial last one."""
    z, params, db, st = full
    sk, seed, reg, _, Hg = client_a
    m2 = sk.m * sk.m
    ck_r = ref.derive_ck_r(m2, seed, 0, N)
    E = np.concatenate([oracle_c.scaled_exponents(Hg[g], params.capacity) for g in SAMPLE_GROUPS])
    want = oracle_c.multiexp_rows(ck_r, E, m2)
    got = [reg.hints[0].entries[g].c for g in SAMPLE_GROUPS]
    assert got == want


def test_fullsize_retrieval_and_sampled_groups(full, client_a, oracle_A):
    """A real client query, hint and answer at the bench's size: the decoded
    row is the DB row (SEPARATE and COMBINED), and t / K on sampled groups
    equal the oracle computed from its own H and b (not the device's)."""
    z, params, db, st = full
    sk, seed, reg, rng, Hg = client_a
    i0 = 4242
    qu0, ck_o, _ = client.query(sk, seed, N, Q, 256, 6.4, D, i0, 0, rng, oracle_A)
    r = z.respond(st, reg, z.QueryMessage(reg.client_id, 0, z.SEPARATE, ck_o, qu0))
    cap = params.capacity
    got = client.extract(sk, Q, 256, cap, Q, D, t=r.t, k=[c.c for c in r.k])
    assert got == [int(x) for x in db[i0]]
    b = oracle_c.db_matvec(db, qu0)
    rc = z.respond(st, reg, z.QueryMessage(reg.client_id, 0, z.COMBINED, ck_o, qu0))
    for g in SAMPLE_GROUPS:
        lo, hi = g * cap, min((g + 1) * cap, D)
        want = oracle_c.answer_t(Hg[g], b[lo:hi], ck_o, sk.m, cap, Q)
        assert r.t[g] == want[0], g
        assert [rc.k[g].c] == oracle_c.combined(want, [reg.hints[0].entries[g].c], sk.m), g
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


def test_fullsize_batch64_vs_single_and_oracle(full, client_a):
    """BASELINE configs[3] at 1 GiB: 64 queries of two clients (different
    moduli, mixed SEPARATE / COMBINED) batched on the N = 256 GEMV and the
    CTA-pair planar compression: every response equals respond(), and two of
    them equal the oracle (C GEMV, oracle H, GMP answer / combine) on sampled
    groups."""
    z, params, db, st = full
    sk_a, _, reg_a, _, Hg = client_a
    sk_b = client.keygen(2048, random.Random(64))
    pk_b = z.PaillierPublicKey(sk_b.m, sk_b.m.bit_length())
    reg_b = z.ClientRegistration(pk_b, b"\x40" * 16, z.client_id_of(pk_b))
    reg_b.hints[0] = z.ClientHint(0, 0, [z.PaillierCiphertext(1)] * params.d1_prime)
    rng = np.random.default_rng(64)
    r = random.Random(65)
    regs, sks, qms = [], [], []
    for i in range(64):
        reg, sk = (reg_a, sk_a) if i % 2 == 0 else (reg_b, sk_b)
        mode = z.COMBINED if i % 8 == 0 else z.SEPARATE
        regs.append(reg)
        sks.append(sk)
        qms.append(z.QueryMessage(reg.client_id, 0, mode, [r.randrange(sk.m) for _ in range(N)],
                                  rng.integers(0, Q, D, dtype=np.uint64)))
    outs = z.respond_batch(st, regs, qms)
    assert len(outs) == 64
    for reg, q, o in zip(regs, qms, outs):
        s1 = z.respond(st, reg, q)
        assert (o.mode, o.t, [c.c for c in o.k]) == (s1.mode, s1.t, [c.c for c in s1.k])
    cap = params.capacity
    for i in (0, 1):      # client a COMBINED, client b SEPARATE
        q, o, sk = qms[i], outs[i], sks[i]
        b = oracle_c.db_matvec(db, q.qu0)
        for g in SAMPLE_GROUPS:
            lo, hi = g * cap, min((g + 1) * cap, D)
            t = oracle_c.answer_t(Hg[g], b[lo:hi], q.ck_o, sk.m, cap, Q)
            if q.mode == z.SEPARATE:
                assert o.t[g] == t[0], (i, g)
            else:
                k = [regs[i].hints[0].entries[g].c]
                assert [o.k[g].c] == oracle_c.combined(t, k, sk.m), (i, g)


def test_fullsize_update_and_refresh(full, client_a, oracle_A):
    """BASELINE configs[4] at 1 GiB: 1% of the DB rows (328 columns of db)
    re-drawn from a seed. ServerGlobalState.updated() gives the same device H
    (and H planes) as a full rebuild; refreshed hints of two clients equal
    full hints on the rebuilt state -- the IMAD row path for 328 rows, then
    the tensor-core row-id path for a second update of 2100 rows -- and the
    GMP oracle on a changed group."""
    import torch
    z, params, db, st = full
    sk_a, seed_a, reg_a, _, _ = client_a
    sk_b = client.keygen(2048, random.Random(77))
    pk_b = z.PaillierPublicKey(sk_b.m, sk_b.m.bit_length())
    reg_b = z.ClientRegistration(pk_b, b"\x4d" * 16, z.client_id_of(pk_b))
    regs = [reg_a, reg_b]
    old = z.hints(st, [(r_, 0) for r_ in regs], keep_slots=True)
    cap = params.capacity
    cur_db, cur_st, cur_h = db, st, old
    for step, (nrows, seed) in enumerate(((D // 100, 91), (2100, 92))):
        rng = np.random.default_rng(seed)
        rows = np.sort(rng.choice(D, size=nrows, replace=False))
        db2 = cur_db.copy()
        db2[:, rows] = rng.integers(0, 256, (D, rows.size), dtype=np.uint8)
        st2, changed = cur_st.updated(db2)
        assert np.array_equal(changed, rows[np.any(db2[:, rows] != cur_db[:, rows], axis=0)])
        rebuilt = z.ServerGlobalState(params, db2, db_version=st2.db_version)
        assert torch.equal(st2.H_dev, rebuilt.H_dev)
        assert torch.equal(st2.H_planes, rebuilt.H_planes)
        use_tc = z.protocol._tc_refresh_pays(st2, len(regs), int(changed.size))
        assert use_tc == (step == 1)     # IMAD row path first, then the tensor-core row-id path
        ref_h = z.hints(rebuilt, [(r_, 0) for r_ in regs])
        new_h = z.refresh_hints(st2, list(zip(regs, cur_h)), changed)
        for a_, b_ in zip(new_h, ref_h):
            assert a_.db_version == b_.db_version == st2.db_version
            assert [c.c for c in a_.entries] == [c.c for c in b_.entries]
        # the oracle on the first changed group (client a)
        g = int(changed[0]) // cap
        lo, hi = g * cap, min((g + 1) * cap, D)
        E = oracle_c.scaled_exponents(oracle_c.hint_rows(db2, oracle_A, lo, hi), cap)
        m2 = sk_a.m * sk_a.m
        want = oracle_c.multiexp_rows(ref.derive_ck_r(m2, seed_a, 0, N), E, m2)
        assert [new_h[0].entries[g].c] == want, (step, g)
        del rebuilt
        cur_db, cur_st, cur_h = db2, st2, new_h
    torch.cuda.empty_cache()
