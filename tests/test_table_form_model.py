"""The arithmetic the tensor-core hint kernel relies on (csrc/tc_pippenger.cu,
csrc/bignum.cuh big_reduce_top), checked on Python ints: the table form of a
multiplication by a fixed multiplier keeps unreduced values within 515 bytes,
and the quotient estimates used for reduction never overshoot and leave < 2N."""
import random

import pytest

L = 128                      # limbs of N = m^2 for a 2048-bit m
R = 1 << (32 * L)


def moduli():
    rng = random.Random(11)
    m_hi = (1 << 2048) - 1 - 2 * 12345          # m^2 just below 2^4096
    m_lo = (1 << 2047) + 1                      # m^2 just above 2^4094
    m_rand = rng.getrandbits(2048) | (1 << 2047) | 1
    return [m_hi * m_hi, m_lo * m_lo, m_rand * m_rand]


@pytest.mark.parametrize("N", moduli())
def test_table_product_is_closed_in_515_bytes(N):
    """V = sum_i x_i (y 256^i mod N) == X y (mod N), V < 515 * 255 * N < 2^4120,
    every byte column < 2^25, whatever 515-byte X went in (including the largest)."""
    rng = random.Random(N % 1000003)
    for trial in range(6):
        y = N - 1 - trial if trial < 2 else rng.randrange(N)
        T = [y * pow(256, i, N) % N for i in range(515)]
        X = (1 << (8 * 515)) - 1 if trial % 2 == 0 else rng.getrandbits(8 * 515)
        for _ in range(3):                      # a few positions in a row: the bound is closed
            xb = X.to_bytes(515, "little")
            cols = [0] * 512
            for i, x in enumerate(xb):
                if x:
                    tb = T[i].to_bytes(512, "little")
                    for j in range(512):
                        cols[j] += x * tb[j]
            assert max(cols) < 1 << 25
            V = sum(c << (8 * j) for j, c in enumerate(cols))
            assert V % N == X * y % N
            assert V < 515 * 255 * N and V < 1 << (8 * 515)
            X = V


@pytest.mark.parametrize("N", moduli())
def test_reduce_top_estimates(N):
    """big_reduce_top's callers: q = floor(top bits of V / (top limb of N + 1))
    satisfies q N <= V < (q + 2) N, for the bucket combine (V < 2^4120, 64-bit
    numerator) and for the table walk (V = 256 t, t < N, numerator and divisor
    shifted down by 8 bits)."""
    rng = random.Random(N % 999983)
    s = 32 * (L - 1)
    nt = N >> s
    for trial in range(2000):
        V = rng.choice([rng.getrandbits(4120), 515 * 255 * N - 1 - trial, rng.randrange(N)])
        h, xtop = V >> (32 * L), (V >> s) & 0xFFFFFFFF
        q = ((h << 32) | xtop) // (nt + 1)
        assert q * N <= V < (q + 2) * N
        t = rng.randrange(N) if trial % 3 else N - 1 - trial
        V = 256 * t
        tb, top = t >> (32 * L - 8), (t >> s) & 0xFFFFFFFF
        xt8 = (tb << 24) | (top & 0xFFFFFF)
        q = xt8 // ((nt >> 8) + 1)
        assert q * N <= V < (q + 2) * N
