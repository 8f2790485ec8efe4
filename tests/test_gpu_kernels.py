"""Kernel-level GPU parity through the C ABI: tcgen05 (UMMA) engine vs the
CUDA-core engine vs the oracle, at shapes the golden cases do not reach:
K > 2^15 (s32 wrap of the byte-plane sums), ragged d0/d1, all-255 inputs,
every supported Paillier limb width."""

import random

import numpy as np
import pytest

from oracle import c as oracle_c
from oracle import ref

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    from paper_2603_09190_b200 import _lib, build, device
    build.build()
    _lib.load()
    return torch, device


def _dbt(torch, device, db, rows, ld):
    d0, d1 = db.shape
    dev = torch.device("cuda", 0)
    db_dev = torch.from_numpy(np.ascontiguousarray(db, dtype=np.uint8)).to(dev)
    return device.transpose_db(db_dev, d0, d1, rows, ld)


def _rup(x, m):
    return -(-x // m) * m


@pytest.mark.parametrize("d0,d1,fill", [(1000, 300, None), (70000, 256, None),
                                        (66000, 130, 255), (32768, 1024, None)])
def test_gemv_engines_vs_oracle(env, d0, d1, fill):
    torch, device = env
    rng = np.random.default_rng(d0 + d1)
    db = (np.full((d0, d1), fill, np.uint8) if fill is not None
          else rng.integers(0, 256, (d0, d1), dtype=np.uint8))
    qu = (np.full(d0, 0xFFFFFFFF, np.uint64) if fill is not None
          else rng.integers(0, 1 << 32, d0, dtype=np.uint64))
    want = oracle_c.db_matvec(db, qu)
    rows, ld = _rup(d1, 128), _rup(d0, 64)
    dbt = _dbt(torch, device, db, rows, ld)
    q = np.zeros((1, ld), np.uint32)
    q[0, :d0] = qu
    qd = device.u32_tensor(q, dbt.device)
    b1 = device.to_host_u32(device.gemv(dbt, qd, 0xFFFFFFFF))[0, :d1]
    planes = device.query_planes(qd, 16)
    b2 = device.to_host_u32(device.umma_gemv(dbt, planes, 1))[0, :d1]
    assert np.array_equal(b1.astype(np.uint64), want)
    assert np.array_equal(b2.astype(np.uint64), want)


@pytest.mark.parametrize("nvec", [3, 64])
def test_batched_gemv(env, nvec):
    torch, device = env
    rng = np.random.default_rng(nvec)
    d0, d1 = 4096, 512
    db = rng.integers(0, 256, (d0, d1), dtype=np.uint8)
    Q = rng.integers(0, 1 << 32, (nvec, d0), dtype=np.uint64)
    dbt = _dbt(torch, device, db, d1, d0)
    qd = device.u32_tensor(Q.astype(np.uint32), dbt.device)
    planes = device.query_planes(qd, 16 if nvec <= 4 else 256)
    got = device.to_host_u32(device.umma_gemv(dbt, planes, nvec))
    for v in range(nvec):
        assert np.array_equal(got[v].astype(np.uint64), ref.db_matvec(db, Q[v], 1 << 32)), v


@pytest.mark.parametrize("d0,d1,n", [(777, 130, 256), (4096, 384, 1024), (40000, 128, 64)])
def test_global_hint_engines(env, d0, d1, n):
    torch, device = env
    rng = np.random.default_rng(n)
    db = rng.integers(0, 256, (d0, d1), dtype=np.uint8)
    A = rng.integers(0, 1 << 32, (d0, n), dtype=np.uint64)
    rows, ld, lda = _rup(d1, 128), _rup(d0, 64), _rup(n, 128)
    dbt = _dbt(torch, device, db, rows, ld)
    Ap = np.zeros((ld, lda), np.uint32)
    Ap[:d0, :n] = A
    Ad = device.u32_tensor(Ap, dbt.device)
    H1 = device.to_host_u32(device.global_hint(dbt, Ad, n, 0xFFFFFFFF))[:d1]
    H2 = device.to_host_u32(device.umma_global_hint(dbt, Ad, n, 0xFFFFFFFF))[:d1]
    cols = sorted({0, 1, d1 // 2, d1 - 1} | set(rng.integers(0, d1, 12).tolist()))
    want = oracle_c.hint_cols(db, A, cols)
    assert np.array_equal(H1[cols].astype(np.uint64), want)
    assert np.array_equal(H2, H1)
    # pad rows of H are zero (multiexp reads them as zero exponent limbs)
    assert not device.to_host_u32(device.umma_global_hint(dbt, Ad, n, 0xFFFFFFFF))[d1:].any()


@pytest.mark.parametrize("lm,n", [(32, 64), (64, 1024), (96, 256), (64, 4096)])
def test_answer_rows_engines(env, lm, n):
    torch, device = env
    rng = np.random.default_rng(lm * n)
    rows = 256
    H = rng.integers(0, 1 << 32, (rows, n), dtype=np.uint64).astype(np.uint32)
    H[0] = 0xFFFFFFFF
    b = rng.integers(0, 1 << 32, rows, dtype=np.uint64).astype(np.uint32)
    r = random.Random(lm)
    ck = [r.randrange(1 << (32 * lm)) for _ in range(n)]
    ck[0] = (1 << (32 * lm)) - 1
    from paper_2603_09190_b200.bigint import ints_to_limbs, limbs_to_ints
    dev = torch.device("cuda", 0)
    Hd = device.u32_tensor(H, dev)
    bd = device.u32_tensor(b, dev)
    cd = device.u32_tensor(ints_to_limbs(ck, lm), dev)
    z1 = device.to_host_u32(device.answer_rows(Hd, bd, 0xFFFFFFFF, cd, lm))
    bc = device.build_bc(cd, lm)
    z2 = device.to_host_u32(device.umma_answer_rows(Hd, bc, bd, 0xFFFFFFFF, lm))
    assert np.array_equal(z1, z2)
    zi = limbs_to_ints(z1)
    for row in (0, 1, 77, 255):
        assert zi[row] == sum(int(h) * c for h, c in zip(H[row], ck))


@pytest.mark.parametrize("lm", [32, 64, 96])
@pytest.mark.parametrize("ctas", [1, 3])
def test_umma_few_ctas_multi_tile(env, lm, ctas):
    """Few persistent CTAs -> each walks several tiles, cycling both TMEM
    accumulator buffers (and, for lm = 64, the 32-column overlap hand-off)."""
    torch, device = env
    rng = np.random.default_rng(lm + ctas)
    rows, n = 640, 256
    H = rng.integers(0, 1 << 32, (rows, n), dtype=np.uint64).astype(np.uint32)
    r = random.Random(lm * ctas)
    ck = [r.randrange(1 << (32 * lm)) for _ in range(n)]
    from paper_2603_09190_b200.bigint import ints_to_limbs, limbs_to_ints
    dev = torch.device("cuda", 0)
    Hd = device.u32_tensor(H, dev)
    cd = device.u32_tensor(ints_to_limbs(ck, lm), dev)
    bd = torch.zeros(rows, dtype=torch.int32, device=dev)
    z_ref = device.to_host_u32(device.answer_rows(Hd, bd, 0xFFFFFFFF, cd, lm))
    bc = device.build_bc(cd, lm)
    z = device.to_host_u32(device.umma_answer_rows(Hd, bc, bd, 0xFFFFFFFF, lm, ctas=ctas))
    assert np.array_equal(z, z_ref)
    zi = limbs_to_ints(z)
    for row in (0, 129, 383, 639):
        assert zi[row] == sum(int(h) * c for h, c in zip(H[row], ck))
    # GEMV stream-K on the same few CTAs
    d0 = 5000
    db = rng.integers(0, 256, (d0, rows), dtype=np.uint8)
    qu = rng.integers(0, 1 << 32, d0, dtype=np.uint64)
    ld = _rup(d0, 64)
    dbt = _dbt(torch, device, db, rows, ld)
    q = np.zeros((1, ld), np.uint32)
    q[0, :d0] = qu
    planes = device.query_planes(device.u32_tensor(q, dev), 16)
    b = device.to_host_u32(device.umma_gemv(dbt, planes, 1, ctas=ctas))[0]
    assert np.array_equal(b.astype(np.uint64), oracle_c.db_matvec(db, qu))


@pytest.mark.parametrize("lm,n,rows,nq", [(64, 1024, 384, 1), (32, 64, 256, 1), (64, 100, 128, 3),
                                          (32, 1024, 640, 2), (64, 4096, 128, 1),
                                          (64, 1024, 1152, 8), (64, 1024, 13184, 3)])
@pytest.mark.parametrize("ctas", [0, 2])
def test_planar_compression(env, lm, n, rows, nq, ctas):
    """Planar compression (H byte planes x ck_o byte rows, 4 plane passes per
    tile) == CUDA-core rows, incl. n not a multiple of 128 (zero-padded
    planes), several queries, few persistent CTAs, all-ones extremes, a partial
    pair tile, n = 4096 (ck_o operand too large to stay in shared memory: the
    single-CTA kernel) and 13184 rows (two blocks of row tiles, the last one
    short, in the CTA-pair kernel's unit order)."""
    torch, device = env
    rng = np.random.default_rng(lm * n + nq)
    H = rng.integers(0, 1 << 32, (rows, n), dtype=np.uint64).astype(np.uint32)
    H[0] = 0xFFFFFFFF
    r = random.Random(n + lm)
    from paper_2603_09190_b200.bigint import ints_to_limbs
    dev = torch.device("cuda", 0)
    Hd = device.u32_tensor(H, dev)
    cks = []
    for q in range(nq):
        ck = [r.randrange(1 << (32 * lm)) for _ in range(n)]
        ck[0] = (1 << (32 * lm)) - 1
        cks.append(ck)
    cd = torch.stack([device.u32_tensor(ints_to_limbs(ck, lm), dev) for ck in cks])
    hp = device.h_planes(Hd)
    bp = device.build_bcp(cd, lm)
    z = device.to_host_u32(device.umma_answer_rows_planar(hp, n, bp, lm, ctas=ctas))
    bd = torch.zeros(rows, dtype=torch.int32, device=dev)
    for q in range(nq):
        zr = device.to_host_u32(device.answer_rows(Hd, bd, 0xFFFFFFFF, cd[q].contiguous(), lm))
        assert np.array_equal(z[q], zr), q


@pytest.mark.parametrize("n,rows", [(64, 300), (256, 129), (32, 128), (32, 552)])
def test_slot_fixed_tensor_core(env, n, rows):
    """Tensor-core Pippenger bucket updates (X * y mod N as one int8 GEMM against
    the table of reduced byte shifts of y, buckets left unreduced in 515 bytes)
    == the IMAD warp path, bit for bit (2048-bit m, 4096-bit m^2), incl. zero
    digits, all-255 rows, a partial last tile, and 552 rows = one CTA pair plus
    a 40-row remainder that goes to the IMAD kernel."""
    torch, device = env
    from oracle import client
    from paper_2603_09190_b200.bigint import ints_to_limbs, key_ctx
    dev = torch.device("cuda", 0)
    rng = random.Random(n * 7 + rows)
    sk = client.keygen(2048, random.Random(2048 + n))
    kctx = key_ctx(sk.m, dev)
    m2 = kctx.m2
    bases = device.u32_tensor(ints_to_limbs([rng.randrange(m2) for _ in range(n)], kctx.l2), dev)
    P = device.pow8_table(bases, kctx)
    nrng = np.random.default_rng(n + rows)
    E = nrng.integers(0, 1 << 32, (rows, n), dtype=np.uint64).astype(np.uint32)
    E[0] = 0
    E[1] = 0xFFFFFFFF
    E[2, : n // 2] = 0
    Ed = device.u32_tensor(E, dev)
    W1 = torch.empty((rows, kctx.l2), dtype=torch.int32, device=dev)
    W2 = torch.empty_like(W1)
    device.slot_fixed(P, n, Ed, n, None, rows, kctx, W1)
    device.slot_fixed_tc(P, n, Ed, n, rows, kctx, W2)
    a, b = device.to_host_u32(W1), device.to_host_u32(W2)
    bad = [i for i in range(rows) if not np.array_equal(a[i], b[i])]
    assert not bad, f"{len(bad)} rows differ, first {bad[:5]}"


@pytest.mark.parametrize("m", [(1 << 2048) - 1 - 2 * 12345, (1 << 2047) + 1, None])
def test_slot_fixed_tensor_core_moduli(env, m):
    """The unreduced 515-byte buckets (V < 515 * 255 * N) and the reduce-on-load
    quotient estimate hold for any odd 2048-bit m: m^2 just below 2^4096 (the top
    limb of V is largest), m^2 just above 2^4094 (the estimate's divisor is
    smallest), and a random keygen modulus; bases next to m^2 - 1; every digit
    value appears, buckets are hit back to back (equal digits at consecutive
    positions: the forwarded rows)."""
    torch, device = env
    from oracle import client
    from paper_2603_09190_b200.bigint import ints_to_limbs, key_ctx
    dev = torch.device("cuda", 0)
    if m is None:
        m = client.keygen(2048, random.Random(77)).m
    rng = random.Random(m % 1000)
    n, rows = 32, 260
    kctx = key_ctx(m, dev)
    m2 = kctx.m2
    bases = [m2 - 1 - rng.randrange(1000) for _ in range(n // 2)] + \
        [rng.randrange(m2) for _ in range(n - n // 2)]
    P = device.pow8_table(device.u32_tensor(ints_to_limbs(bases, kctx.l2), dev), kctx)
    nrng = np.random.default_rng(5)
    E = nrng.integers(0, 1 << 32, (rows, n), dtype=np.uint64).astype(np.uint32)
    E[3] = 0x01010101 * 7                       # one bucket, every position
    E[4, :] = np.arange(n, dtype=np.uint32) * 0x01010101 % 256 * 0x01010101
    E[5] = 0xFFFFFFFF
    Ed = device.u32_tensor(E, dev)
    W1 = torch.empty((rows, kctx.l2), dtype=torch.int32, device=dev)
    W2 = torch.empty_like(W1)
    device.slot_fixed(P, n, Ed, n, None, rows, kctx, W1)
    device.slot_fixed_tc(P, n, Ed, n, rows, kctx, W2)
    a, b = device.to_host_u32(W1), device.to_host_u32(W2)
    bad = [i for i in range(rows) if not np.array_equal(a[i], b[i])]
    assert not bad, f"{len(bad)} rows differ, first {bad[:5]}"


@pytest.mark.parametrize("nrow,nsel", [(400, 150), (700, 540)])
def test_slot_fixed_tensor_core_many_clients_row_ids(env, nrow, nsel):
    """One tensor-core launch for three clients (different keys and tables),
    on a row-id subset of the exponent rows (the incremental refresh): every
    client's rows equal its own IMAD slot_fixed; rows outside the subset are
    left untouched. 540 selected rows = one CTA pair plus a 28-row remainder
    on the IMAD kernel, by position in the row-id list."""
    torch, device = env
    from oracle import client
    from paper_2603_09190_b200.bigint import ints_to_limbs, key_ctx
    dev = torch.device("cuda", 0)
    n = 64
    nrng = np.random.default_rng(31)
    E = nrng.integers(0, 1 << 32, (nrow, n), dtype=np.uint64).astype(np.uint32)
    Ed = device.u32_tensor(E, dev)
    rid_h = np.sort(nrng.choice(nrow, size=nsel, replace=False)).astype(np.int32)
    rid = torch.from_numpy(rid_h).to(dev)
    jobs, refs = [], []
    for c in range(3):
        rng = random.Random(900 + c)
        kctx = key_ctx(client.keygen(2048, rng).m, dev)
        bases = device.u32_tensor(ints_to_limbs([rng.randrange(kctx.m2) for _ in range(n)],
                                                kctx.l2), dev)
        P = device.pow8_table(bases, kctx)
        W_ref = torch.zeros((nrow, kctx.l2), dtype=torch.int32, device=dev)
        device.slot_fixed(P, n, Ed, n, rid, len(rid_h), kctx, W_ref)
        W = torch.zeros_like(W_ref)
        jobs.append((P, kctx, W))
        refs.append(W_ref)
    device.slot_fixed_tc_many(jobs, n, Ed, n, len(rid_h), rid=rid)
    for (_, _, W), W_ref in zip(jobs, refs):
        a, b = device.to_host_u32(W_ref), device.to_host_u32(W)
        assert np.array_equal(a, b)
        assert not b[np.setdiff1d(np.arange(nrow), rid_h)].any()


@pytest.mark.parametrize("shape,view", [((4097, 4099), None), (((64 << 20) + 1,), None),
                                        ((11000, 12289), "cols")])
def test_upload_bytes_staged(env, shape, view):
    """device.upload_bytes (pinned stages, threaded host copies) == the plain
    torch copy, at sizes straddling the 16 MiB threshold and the 64 MiB chunk,
    for contiguous and strided (column-sliced) arrays."""
    torch, device = env
    dev = torch.device("cuda", 0)
    a = np.frombuffer(np.random.default_rng(len(shape)).bytes(int(np.prod(shape))),
                      np.uint8).reshape(shape)
    if view == "cols":
        a = a[:, 7:-5]
    stream = torch.cuda.current_stream(dev)
    out = device.upload_bytes(a, dev, stream)
    torch.cuda.synchronize()
    assert out.shape == a.shape
    assert torch.equal(out.cpu(), torch.from_numpy(np.array(a)))   # writable copy
