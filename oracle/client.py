"""Client-side restatement (keygen, query, decrypt, extract) -- TEST INFRASTRUCTURE.

The client is out of scope for the B200 build;
this module only manufactures seeded test inputs (queries, key pairs) and
checks retrieval end to end. It consumes a random.Random exactly as the
reference does, so seeded runs reproduce the reference's golden queries.
"""

import math

import numpy as np

from . import ref

_SMALL_PRIMES = [2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53,
                 59, 61, 67, 71, 73, 79, 83, 89, 97, 101, 103, 107, 109, 113,
                 127, 131, 137, 139, 149]


def is_probable_prime(n: int) -> bool:
    if n < 2:
        return False
    for p in _SMALL_PRIMES[:25]:
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in _SMALL_PRIMES[:25]:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def next_prime(n: int) -> int:
    n += 1
    if n <= 2:
        return 2
    n |= 1
    while not is_probable_prime(n):
        n += 2
    return n


class SecretKey:
    """paillier.py:42-58: CRT decryption constants for g = m + 1."""

    def __init__(self, p: int, q: int):
        self.p, self.q = int(p), int(q)
        self.m = self.p * self.q
        self.bits = self.m.bit_length()
        self.p2, self.q2 = self.p * self.p, self.q * self.q
        g = self.m + 1
        self.hp = pow((pow(g, self.p - 1, self.p2) - 1) // self.p, -1, self.p)
        self.hq = pow((pow(g, self.q - 1, self.q2) - 1) // self.q, -1, self.q)
        self.p_inv_q = pow(self.p, -1, self.q)


def keygen(bits: int, rng) -> SecretKey:
    """paillier.py:69-86 (same rng consumption)."""
    half = bits // 2
    while True:
        p = next_prime(rng.randrange(1 << (half - 1), 1 << half))
        q = next_prime(rng.randrange(1 << (half - 1), 1 << half))
        if p == q or p.bit_length() != half or q.bit_length() != half:
            continue
        m = p * q
        if m.bit_length() != bits or math.gcd(m, (p - 1) * (q - 1)) != 1:
            continue
        return SecretKey(p, q)


def decrypt(sk: SecretKey, c: int) -> int:
    """paillier.py:109-117."""
    c %= sk.m * sk.m
    if math.gcd(c, sk.m) != 1:
        raise ValueError("invalid ciphertext")
    mp = (pow(c, sk.p - 1, sk.p2) - 1) // sk.p * sk.hp % sk.p
    mq = (pow(c, sk.q - 1, sk.q2) - 1) // sk.q * sk.hq % sk.q
    return mp + sk.p * ((mq - mp) * sk.p_inv_q % sk.q)


def setup(bits: int, rng):
    """protocol.py:272-282 -> (secret key, 16-byte seed)."""
    sk = keygen(bits, rng)
    seed = bytes(rng.randrange(256) for _ in range(16))
    return sk, seed


class Gaussian:
    """gaussian.py:14-46 table inverse-CDF sampler."""

    def __init__(self, sigma: float):
        if sigma == 0:
            self.support = np.array([0], dtype=np.int64)
            self.cdf = np.array([2 ** 64 - 1], dtype=np.uint64)
            return
        tail = int(math.ceil(6 * sigma))
        xs = np.arange(-tail, tail + 1, dtype=np.int64)
        w = np.exp(-(xs.astype(np.float64) ** 2) / (2 * sigma * sigma))
        cum = np.cumsum(w / w.sum())
        fixed = np.minimum(np.floor(cum * 2.0 ** 64),
                           np.nextafter(2.0 ** 64, 0)).astype(np.uint64)
        fixed[-1] = np.uint64(2 ** 64 - 1)
        self.support, self.cdf = xs, fixed

    def sample_vector(self, count, rng):
        us = np.array([rng.randrange(1 << 64) for _ in range(count)], dtype=np.uint64)
        idx = np.minimum(np.searchsorted(self.cdf, us, side="right"), len(self.support) - 1)
        return self.support[idx]


def query(sk: SecretKey, seed: bytes, n, q, p, sigma, d0, i0, query_index, rng, A):
    """protocol.py:299-330 -> (qu0 uint64[d0], ck_o list[n], sk_lwe)."""
    m = sk.m
    sk_lwe = np.array([rng.randrange(2) for _ in range(n)], dtype=np.uint64)
    ck_r = ref.derive_ck_r(m * m, seed, query_index, n)
    ck_o = [(int(sk_lwe[i]) - decrypt(sk, c)) % m for i, c in enumerate(ck_r)]
    e = Gaussian(sigma).sample_vector(d0, rng)
    with np.errstate(over="ignore"):
        As = np.asarray(A, dtype=np.uint64) @ sk_lwe
    delta = (2 * q + p) // (2 * p)
    qu0 = np.empty(d0, dtype=np.uint64)
    for i in range(d0):
        qu0[i] = (int(As[i]) + int(e[i]) + (delta if i == i0 else 0)) % q
    return qu0, ck_o, sk_lwe


def extract(sk: SecretKey, q, p, cap, gamma, d1, t=None, k=None, combined=None):
    """protocol.py:368-396 (SEPARATE if t/k given, else COMBINED)."""
    m = sk.m
    if combined is None:
        mu = [(int(tg) + decrypt(sk, int(kg))) % m for tg, kg in zip(t, k)]
    else:
        mu = [decrypt(sk, int(c)) for c in combined]
    delta = (2 * q + p) // (2 * p)
    out = []
    for g, val in enumerate(mu):
        for j in range(min(cap, d1 - g * cap)):
            phase = (val // gamma ** j) % gamma % q
            out.append((2 * phase + delta) // (2 * delta) % p)
    return out


def encrypt(sk: SecretKey, mu: int, rng) -> int:
    """paillier.py:89-101 (same rng consumption)."""
    m, m2 = sk.m, sk.m * sk.m
    while True:
        r = rng.randrange(1, m)
        if math.gcd(r, m) == 1:
            break
    return (1 + mu * m) * pow(r, m, m2) % m2
