"""Standalone LWE->Paillier compressor on the GPU (compress.py:99-258 mirror):
bit-identical ciphertexts vs the oracle restatement of the reference
(including the reference's scalar_mul-based batched path), and decryption to
the LWE phase."""

import random
from types import SimpleNamespace

import numpy as np
import pytest

from oracle import client, ref

pytestmark = pytest.mark.gpu


def _key(z, sk, n, rng, lwe_sk):
    pk = z.PaillierPublicKey(sk.m, sk.m.bit_length())
    ck = [z.PaillierCiphertext(client.encrypt(sk, int(s), rng)) for s in lwe_sk]
    return pk, SimpleNamespace(pk=pk, lwe_params=None, ck=ck, key_scaling=1)


@pytest.mark.parametrize("bits,n,q", [(64, 8, 16), (768, 64, 1 << 32), (2048, 630, 1 << 64)])
def test_lwe_compress_matches_reference(bits, n, q):
    import paper_2603_09190_b200 as z
    from paper_2603_09190_b200 import compress
    rng = random.Random(bits + n)
    sk = client.keygen(bits, rng)
    lwe = SimpleNamespace(n=n, q=q, p=4 if q == 16 else 256, key_dist="binary")
    lwe_sk = [rng.randrange(2) for _ in range(n)]
    pk, ck = _key(z, sk, n, rng, lwe_sk)
    ck.lwe_params = lwe
    cts = []
    for _ in range(5):
        a = [rng.randrange(q) for _ in range(n)]
        b = rng.randrange(q)
        cts.append(SimpleNamespace(a=a, b=b))
    got = compress.lwe_compress_many(ck, cts)
    for ct, cc in zip(cts, got):
        want = ref.lwe_compress(sk.m, [c.c for c in ck.ck], ct.a, ct.b, q)
        assert cc.x.c == want
        # decrypts to the LWE phase b + sum (q - a_i) s_i  (no reduction)
        phase = int(ct.b) + sum((q - int(a)) % q * s for a, s in zip(ct.a, lwe_sk))
        assert client.decrypt(sk, cc.x.c) == phase % sk.m
    assert compress.lwe_compress(ck, cts[0]).x.c == got[0].x.c


def test_batched_compress_matches_reference_scalar_mul_path():
    import paper_2603_09190_b200 as z
    from paper_2603_09190_b200 import compress, counters
    rng = random.Random(7)
    sk = client.keygen(768, rng)
    n, q = 16, 1 << 32
    lwe = SimpleNamespace(n=n, q=q, p=256, key_dist="binary")
    lwe_sk = [rng.randrange(2) for _ in range(n)]
    pk, ck = _key(z, sk, n, rng, lwe_sk)
    ck.lwe_params = lwe
    gamma = q + n * q
    ell = compress.batch_capacity(pk, gamma)
    cts = [SimpleNamespace(a=[rng.randrange(q) for _ in range(n)], b=rng.randrange(q))
           for _ in range(ell)]
    with counters.measure() as meas:
        cc = compress.fast_batched_lwe_compress(ck, cts, gamma)
    assert meas.delta.modexp == 0 and meas.delta.scalar_mul == 0
    want = ref.batched_lwe_compress(sk.m, [c.c for c in ck.ck],
                                    [(ct.a, ct.b) for ct in cts], gamma, q)
    assert cc.x.c == want
    assert compress.batched_lwe_compress(ck, cts, gamma).x.c == want
    with pytest.raises(compress.CapacityExceeded):
        compress.batched_lwe_compress(ck, cts + cts[:1], gamma)


def test_compressor_matches_reference_kat():
    """The GPU compressor against the unmodified reference's outputs
    (tests/golden/compress_kat.json, made by tests/golden/make_golden.py:
    compress.py:99-258 on seeded keys and ciphertexts, binary and uniform
    LWE keys, q = 2^16 / 2^32)."""
    import json
    import os
    import paper_2603_09190_b200 as z
    from paper_2603_09190_b200 import compress
    from conftest import GOLDEN
    with open(os.path.join(GOLDEN, "compress_kat.json")) as f:
        cases = json.load(f)
    for c in cases:
        m = int(c["m"], 16)
        pk = z.PaillierPublicKey(m, m.bit_length())
        lwe = SimpleNamespace(n=c["n"], q=c["q"], p=256, key_dist=c["key_dist"])
        ckl = [z.PaillierCiphertext(int(x, 16)) for x in c["ck"]]
        ck = SimpleNamespace(pk=pk, lwe_params=lwe, ck=ckl, key_scaling=1)
        eck = SimpleNamespace(pk=pk, lwe_params=lwe, eck=[ckl], key_scaling=1)
        cts = [SimpleNamespace(a=ct["a"], b=ct["b"]) for ct in c["cts"]]
        got = compress.lwe_compress_many(ck, cts)
        assert [g.x.c for g in got] == [int(v, 16) for v in c["lwe_compress"]], c["bits"]
        assert [compress.fast_lwe_compress(eck, ct).x.c for ct in cts] == \
            [int(v, 16) for v in c["fast_lwe_compress"]], c["bits"]
        gamma, ell = int(c["gamma"]), c["ell"]
        assert compress.batched_lwe_compress(ck, cts[:ell], gamma).x.c == int(c["batched"], 16)
        assert compress.fast_batched_lwe_compress(ck, cts[:ell], gamma).x.c == \
            int(c["fast_batched"], 16)
