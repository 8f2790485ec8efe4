"""Device ChaCha20 (csrc/chacha.cu) vs the reference PRG restatement
(oracle/ref.py, pinned to prg.py KATs): public matrix A and the rejection-
sampled ck_r, bit for bit, including non-block-aligned chunk sizes."""

import random

import numpy as np
import pytest

from oracle import client, ref

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    from paper_2603_09190_b200 import _lib, build, device
    build.build()
    _lib.load()
    return torch, device


@pytest.mark.parametrize("d0,n,seed", [(777, 256, b"\x00" * 16), (1024, 1024, b"\x00" * 16),
                                       (33, 5, bytes(range(16)))])
def test_public_matrix(env, d0, n, seed):
    torch, device = env
    lda = -(-n // 128) * 128
    out = torch.zeros((d0 + 3, lda), dtype=torch.int32, device="cuda")
    device.chacha_words32(seed, 3, 0, d0, n, out, lda, 0xFFFFFFFF)
    got = device.to_host_u32(out)
    want = ref.public_matrix(seed, d0, n, 1 << 32) if seed == b"\x00" * 16 else \
        ref.Stream(seed, 3).words_pow2(1 << 32, d0 * n).reshape(d0, n)
    assert np.array_equal(got[:d0, :n].astype(np.uint64), want)
    assert not got[d0:].any() and not got[:, n:].any()


@pytest.mark.parametrize("bits", [64, 768, 2048, 3072])
def test_ck_r_rejection_sampling(env, bits):
    torch, device = env
    from paper_2603_09190_b200.bigint import key_ctx, limbs_to_ints
    rng = random.Random(bits)
    sk = client.keygen(bits, rng)
    kctx = key_ctx(sk.m, torch.device("cuda", 0))
    for seed, qi in [(bytes(16), 0), (bytes([7] * 16), 5), (bytes(range(16)), (1 << 40) + 3)]:
        n = 37
        got = limbs_to_ints(device.to_host_u32(
            device.chacha_below(seed, 1, qi, n, kctx.d_m2, kctx.m2, kctx.l2)))
        assert got == ref.derive_ck_r(kctx.m2, seed, qi, n), (bits, qi)
