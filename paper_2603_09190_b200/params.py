"""Protocol parameters and the batch layout contract.

Same fields, defaults, derived quantities and params_hash bytes as the
reference (lwe.py:25-43, protocol.py:40-95, compress.py:30-43), so objects of
either package can be passed to the other's functions and wire frames keep
the same 32-byte parameter hash.
"""

from dataclasses import dataclass
import hashlib
import math

import numpy as np

from .prg import Stream, DOM_PUBLIC_MATRIX, SEED_BYTES

BINARY = "binary"
UNIFORM = "uniform"
STANDARD = "standard"
QUARTER_DELTA = "quarter_delta"


def round_div(x: int, d: int) -> int:
    """round(x/d), ties away from zero, x >= 0 (lwe.py:20-22)."""
    return (2 * x + d) // (2 * d)


@dataclass(frozen=True)
class LweParams:
    n: int
    q: int
    p: int
    noise_sigma: float = 0.0
    key_dist: str = BINARY

    def __post_init__(self):
        if not (self.n >= 1 and 2 <= self.p < self.q <= 1 << 64):
            raise ValueError("need n >= 1 and p < q <= 2^64")
        if self.delta < 2:
            raise ValueError("scaling factor q/p must be at least 2")
        if self.key_dist not in (BINARY, UNIFORM):
            raise ValueError("unknown key distribution")

    @property
    def delta(self) -> int:
        return round_div(self.q, self.p)


def phase_bound(lwe) -> int:
    """Exclusive bound on b + sum (q - a_i) sk_i (compress.py:30-33)."""
    q, n = lwe.q, lwe.n
    return q + n * q if lwe.key_dist == BINARY else q + n * q * q


def select_scale(lwe, regime: str = STANDARD) -> int:
    """Batch scale gamma (compress.py:36-43)."""
    q = lwe.q
    if regime == STANDARD:
        return phase_bound(lwe)
    if regime == QUARTER_DELTA:
        return q if lwe.key_dist == BINARY else q * q
    raise ValueError("unknown noise regime")


@dataclass(frozen=True)
class ProtocolParams:
    lwe: LweParams
    d0: int
    d1: int
    paillier_bits: int = 3072
    scale_regime: str = QUARTER_DELTA
    a_seed: bytes = b"\x00" * SEED_BYTES
    hints_per_client: int = 4
    delta_fail: float = 2.0 ** -40

    def __post_init__(self):
        if self.lwe.noise_sigma > 0 and not self.correctness_margin() > 1:
            raise ValueError("q/p too small for the target failure probability")

    def correctness_margin(self) -> float:
        lwe = self.lwe
        rhs = 2 * lwe.p * lwe.noise_sigma * math.sqrt(2 * self.d0 * math.log(2 / self.delta_fail))
        return (lwe.q / lwe.p) / rhs if rhs else float("inf")

    @property
    def gamma(self) -> int:
        return select_scale(self.lwe, self.scale_regime)

    @property
    def capacity(self) -> int:
        return capacity_of(self)

    @property
    def d1_prime(self) -> int:
        return -(-self.d1 // self.capacity)

    def params_hash(self) -> bytes:
        return params_hash(self)

    def public_matrix(self):
        return public_matrix(self)


def capacity_of(params) -> int:
    """Largest slot count whose packed worst case stays < 2^(bits-1)
    (protocol.py:66-78)."""
    limit = 1 << (params.paillier_bits - 1)
    worst = phase_bound(params.lwe) - 1
    gamma = select_scale(params.lwe, params.scale_regime)
    ell, total, power = 0, 0, 1
    while total + worst * power < limit:
        total += worst * power
        power *= gamma
        ell += 1
    if ell == 0:
        raise ValueError("plaintext modulus cannot hold one slot")
    return ell


def params_hash(params) -> bytes:
    """SHA-256 over the same repr tuple as protocol.py:84-89."""
    lwe = params.lwe
    blob = repr((lwe.n, lwe.q, lwe.p, lwe.noise_sigma, lwe.key_dist, params.d0, params.d1,
                 params.paillier_bits, params.scale_regime, params.a_seed,
                 params.hints_per_client)).encode()
    return hashlib.sha256(blob).digest()


def public_matrix(params):
    """The (d0, n) uint64 query matrix from the public seed (protocol.py:91-95)."""
    lwe = params.lwe
    return Stream(params.a_seed, DOM_PUBLIC_MATRIX).integers(lwe.q, params.d0 * lwe.n).reshape(
        params.d0, lwe.n)


class Layout:
    """What the device path needs from a params object (ours or the
    reference's): dimensions, q mask, slot capacity, groups."""

    def __init__(self, params):
        lwe = params.lwe
        self.n, self.q, self.p = lwe.n, lwe.q, lwe.p
        self.d0, self.d1 = params.d0, params.d1
        self.bits = params.paillier_bits
        self.gamma = select_scale(lwe, params.scale_regime)
        self.cap = capacity_of(params)
        self.groups = -(-self.d1 // self.cap)
        if self.q & (self.q - 1) or self.q > 1 << 32:
            raise NotImplementedError(
                f"the B200 path needs q a power of two <= 2^32 (got q={self.q}); there is no "
                "CPU fallback")
        if self.p > 256:
            raise NotImplementedError("the device layout stores one byte per DB symbol (p <= 256)")
        self.qmask = (self.q - 1) & 0xFFFFFFFF
        # slot stride of the positional group fold: gamma = 2^(32 s) (binary key,
        # quarter-delta: s = 1; uniform key: s = 2); 0 = general gamma
        self.stride = {1 << 32: 1, 1 << 64: 2}.get(self.gamma, 0)
        self.gamma_words = np.frombuffer(self.gamma.to_bytes(32, "little"), dtype="<u4").copy() \
            if self.gamma.bit_length() <= 256 else None
        if self.gamma_words is None:
            raise NotImplementedError("batch scale gamma wider than 256 bits")
        # device padding: DB rows (d1) to 128 and to whole groups; K (d0) to 64
        self.rows = _round_up(max(self.d1, self.groups * self.cap), 128)
        self.ld = _round_up(self.d0, 64)
        self.lda = _round_up(self.n, 128)


def _round_up(x, m):
    return -(-x // m) * m
