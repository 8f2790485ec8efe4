"""Exact CPU restatement of the reference server path -- TEST INFRASTRUCTURE.

Not shipped, never called by the product. Plain numpy (wrapping uint64, which
is exact mod 2^32 after masking) and Python ints. Every function cites the
reference function it restates (paths relative to /root/reference/pkg/src/
zippir/). Pinned against tests/golden/* (reference outputs) by
tests/test_oracle_golden.py.
"""

import hashlib

import numpy as np
from cryptography.hazmat.primitives.ciphers import Cipher, algorithms

DOM_CIPHERTEXT_SAMPLE = 1   # prg.py:15
DOM_PUBLIC_MATRIX = 3       # prg.py:17
MASK32 = (1 << 32) - 1


# -- prg.py:23-57 -----------------------------------------------------------

class Stream:
    """ChaCha20 keystream: key = SHA-256(seed), 16-byte IV = domain byte ||
    15-byte LE index (prg.py:24-27). cryptography's 16-byte ChaCha20 nonce is
    (32-bit LE block counter || 96-bit nonce), i.e. RFC 7539 with counter =
    LE u32 of [domain, i0, i1, i2] and nonce = i[3..14]."""

    def __init__(self, seed: bytes, domain: int, index: int = 0):
        key = hashlib.sha256(seed).digest()
        iv = bytes([domain]) + int(index).to_bytes(15, "little")
        self._enc = Cipher(algorithms.ChaCha20(key, iv), mode=None).encryptor()

    def read(self, nbytes: int) -> bytes:
        return self._enc.update(bytes(nbytes))

    def below(self, bound: int) -> int:
        """Rejection sampling on bitlen(bound-1) bits (prg.py:32-44)."""
        bits = (bound - 1).bit_length()
        if bits == 0:
            return 0
        nbytes = (bits + 7) // 8
        mask = (1 << bits) - 1
        while True:
            x = int.from_bytes(self.read(nbytes), "little") & mask
            if x < bound:
                return x

    def words_pow2(self, bound: int, count: int) -> np.ndarray:
        """integers() for power-of-two bounds: masked LE u64 words (prg.py:50-53)."""
        raw = np.frombuffer(self.read(8 * count), dtype="<u8")
        return raw & np.uint64(bound - 1)


def public_matrix(a_seed: bytes, d0: int, n: int, q: int) -> np.ndarray:
    """protocol.py:91-95 (power-of-two q only, as on the hot path)."""
    assert q & (q - 1) == 0
    return Stream(a_seed, DOM_PUBLIC_MATRIX).words_pow2(q, d0 * n).reshape(d0, n)


def sample_ciphertext(m2: int, seed: bytes, index: int) -> int:
    """paillier.py:206-208."""
    return Stream(seed, DOM_CIPHERTEXT_SAMPLE, index).below(m2)


def derive_ck_r(m2: int, seed: bytes, query_index: int, n: int) -> list:
    """protocol.py:285-288."""
    return [sample_ciphertext(m2, seed, (query_index << 32) | i) for i in range(n)]


# -- protocol.py:62-82 / compress.py:30-43 -----------------------------------

def layout(n, q, key_dist, paillier_bits, scale_regime, d1):
    """(gamma, capacity, d1') exactly as ProtocolParams computes them."""
    binary = key_dist == "binary"
    bound = q + n * q if binary else q + n * q * q          # phase_bound
    if scale_regime == "standard":
        gamma = bound
    else:                                                     # quarter_delta
        gamma = q if binary else q * q
    limit = 1 << (paillier_bits - 1)
    worst = bound - 1
    ell, total, power = 0, 0, 1
    while total + worst * power < limit:
        total += worst * power
        power *= gamma
        ell += 1
    if ell == 0:
        raise ValueError("plaintext modulus cannot hold one slot")
    return gamma, ell, -(-d1 // ell)


# -- protocol.py:195-217, :242-257 -------------------------------------------

def global_hint(db: np.ndarray, A: np.ndarray, q: int, chunk: int = 256) -> np.ndarray:
    """H = (-db^T A) mod q, (d1, n) uint64. Wrapping u64 products are exact
    mod 2^64 hence mod q for q | 2^32 (protocol.py:195-207 / :209-217)."""
    assert q & (q - 1) == 0 and q <= 1 << 32
    dbt = np.ascontiguousarray(np.asarray(db).T).astype(np.uint64)
    A64 = np.asarray(A, dtype=np.uint64)
    out = np.empty((dbt.shape[0], A64.shape[1]), dtype=np.uint64)
    with np.errstate(over="ignore"):
        for s in range(0, dbt.shape[0], chunk):
            g = dbt[s:s + chunk] @ A64
            out[s:s + chunk] = (np.uint64(0) - g) & np.uint64(q - 1)
    return out


def db_matvec(db: np.ndarray, qu: np.ndarray, q: int) -> np.ndarray:
    """b = db^T qu mod q, uint64 (d1) (protocol.py:242-257)."""
    assert q & (q - 1) == 0 and q <= 1 << 32
    with np.errstate(over="ignore"):
        s = np.asarray(db, dtype=np.uint64).T @ np.asarray(qu, dtype=np.uint64)
    return s & np.uint64(q - 1)


def scale_rows(H, cap, gamma, d1, n) -> list:
    """H_scaled[g][k] = sum_j gamma^j H[g*cap+j][k] (protocol.py:219-238)."""
    d1p = -(-d1 // cap)
    rows = []
    for g in range(d1p):
        row = [0] * n
        for j, c in enumerate(range(g * cap, min((g + 1) * cap, d1))):
            gj = gamma ** j
            hc = H[c]
            for k in range(n):
                row[k] += gj * int(hc[k])
        rows.append(row)
    return rows


def scaled_b(b, cap, gamma, d1) -> list:
    """protocol.py:259-269."""
    d1p = -(-d1 // cap)
    return [sum(gamma ** j * int(b[g * cap + j])
                for j in range(min(cap, d1 - g * cap))) for g in range(d1p)]


def answer_t(H, b, ck_o, m, cap, gamma, d1) -> list:
    """t_g = (bs_g + hv_g) mod m (protocol.py:345-350), computed through the
    identity t_g = (sum_j gamma^j (b_c + y_c)) mod m with y_c = sum_k
    H[c,k] ck_o[k] (verified against the reference's RNS
    path by tests/test_oracle_golden.py)."""
    d1p = -(-d1 // cap)
    ck = [int(x) for x in ck_o]
    out = []
    for g in range(d1p):
        acc = 0
        for j, c in enumerate(range(g * cap, min((g + 1) * cap, d1))):
            hc = H[c]
            y = sum(int(hc[k]) * ck[k] for k in range(len(ck)))
            acc += gamma ** j * (int(b[c]) + y)
        out.append(acc % m)
    return out


def combined(t, k, m) -> list:
    """K_g = trivial_encrypt(t_g) * k_g mod m^2 (protocol.py:354-358,
    paillier.py:104-106, :120-123)."""
    m2 = m * m
    return [((1 + (int(tg) % m) * m) % m2) * int(kg) % m2 for tg, kg in zip(t, k)]


# -- paillier.py:134-203 -------------------------------------------------------

def multiexp(m2: int, bases, exps) -> int:
    """prod bases[i]^exps[i] mod m2 by w-bit windows and buckets 1..2^w-1
    with a running-sum combine (paillier.py:134-193). Returns 1 when every
    exponent is zero (paillier.py:145-146)."""
    exps = [int(e) for e in exps]
    if len(exps) != len(bases):
        raise ValueError("dimension mismatch")
    maxbits = max((e.bit_length() for e in exps), default=0)
    if maxbits == 0:
        return 1
    w = min(6, maxbits)
    nwin = -(-maxbits // w)
    mask = (1 << w) - 1
    acc = None
    for win in reversed(range(nwin)):
        if acc is not None:
            for _ in range(w):
                acc = acc * acc % m2
        buckets = {}
        for base, e in zip(bases, exps):
            d = (e >> (win * w)) & mask
            if d:
                buckets[d] = buckets[d] * base % m2 if d in buckets else int(base)
        running = total = None
        for d in range(mask, 0, -1):
            if d in buckets:
                running = buckets[d] if running is None else running * buckets[d] % m2
            if running is not None:
                total = running if total is None else total * running % m2
        if total is not None:
            acc = total if acc is None else acc * total % m2
    return acc % m2


def hint_entries(H_scaled, ck_r, m2) -> list:
    """paillier_matmul (paillier.py:196-203) as used by hint() (protocol.py:291-296)."""
    return [multiexp(m2, ck_r, row) for row in H_scaled]


# -- compress.py:99-258 (server side) -----------------------------------------

def lwe_compress(m: int, ck, a, b, q) -> int:
    """trivial_encrypt(b) * multiexp(ck, (q - a_i) mod q) mod m^2 (compress.py:99-105)."""
    m2 = m * m
    acc = multiexp(m2, [int(c) for c in ck], [(q - int(x)) % q for x in a])
    return (1 + (int(b) % m) * m) % m2 * acc % m2


def batched_lwe_compress(m: int, ck, cts, gamma: int, q) -> int:
    """compress.py:213-221 restated literally: x = Enc~(0); x *= lwe_compress(ct_j)^(gamma^j)."""
    m2 = m * m
    x = 1
    for j, (a, b) in enumerate(cts):
        xj = lwe_compress(m, ck, a, b, q)
        x = x * pow(xj, gamma ** j, m2) % m2
    return x
