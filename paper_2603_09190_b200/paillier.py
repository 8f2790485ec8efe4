"""Paillier server-side operations on the B200 path.

Types mirror paillier.py:24-66 of the reference (PaillierPublicKey,
PaillierCiphertext); the group arithmetic the server performs --
multi-exponentiation (paillier.py:134-193), homomorphic matrix-vector
products (:196-203) and batched additions (:120-123) -- runs in the warp
Montgomery kernels (csrc/multiexp.cu, csrc/answer.cu). Seeded ciphertext
sampling (:206-208) stays on the host PRG. Keygen, encryption and
decryption are client operations and are not part of this package.
"""

from dataclasses import dataclass
import struct

import numpy as np
import torch

from . import counters, device
from .bigint import ints_to_limbs, key_ctx, limbs_to_ints
from .prg import Stream, DOM_CIPHERTEXT_SAMPLE


class InvalidCiphertext(Exception):
    """Ciphertext not invertible modulo m^2 (paillier.py:20-21)."""


@dataclass(frozen=True)
class PaillierPublicKey:
    m: int
    bit_length: int

    @property
    def m2(self):
        return self.m * self.m

    def serialize(self) -> bytes:
        nbytes = (self.m.bit_length() + 7) // 8
        return struct.pack("<I", nbytes) + self.m.to_bytes(nbytes, "little")


@dataclass
class PaillierCiphertext:
    c: int

    def serialize(self) -> bytes:
        nbytes = (self.c.bit_length() + 7) // 8
        return struct.pack("<I", nbytes) + self.c.to_bytes(nbytes, "little")


def trivial_encrypt(pk, v: int) -> PaillierCiphertext:
    """(m+1)^v = 1 + v m mod m^2 (paillier.py:104-106); a closed form, no
    group arithmetic. On the response path it is fused into zpir_combine."""
    return PaillierCiphertext((1 + (v % pk.m) * pk.m) % pk.m2)


def sample_ciphertext(pk, seed: bytes, index: int) -> PaillierCiphertext:
    """Uniform element of [0, m^2) from (seed, index) (paillier.py:206-208)."""
    return PaillierCiphertext(Stream(seed, DOM_CIPHERTEXT_SAMPLE, index).below(pk.m2))


def _cvals(cts, m2):
    return [(c.c if hasattr(c, "c") else int(c)) % m2 for c in cts]


def paillier_matmul(pk, H, v, stream=None):
    """Homomorphic H . v: entry g = prod_k v[k]^H[g][k] mod m^2
    (paillier.py:196-203), all rows in one device multi-exponentiation."""
    rows = [[int(e) for e in row] for row in H]
    for row in rows:
        if len(row) != len(v):
            raise ValueError("dimension mismatch")
        if any(e < 0 for e in row):
            raise ValueError("exponents must be nonnegative")
    if not rows:
        return []
    n = len(v)
    if n == 0:
        return [PaillierCiphertext(1) for _ in rows]
    dev = device.require_cuda()
    kctx = key_ctx(pk.m, dev)
    maxbits = max(e.bit_length() for row in rows for e in row)
    elimbs = max(1, -(-maxbits // 32))
    bases = device.u32_tensor(ints_to_limbs(_cvals(v, kctx.m2), kctx.l2), dev)
    flat = [e for row in rows for e in row]
    E = device.u32_tensor(ints_to_limbs(flat, elimbs), dev)
    out = device.multiexp(bases, E, len(rows), n * elimbs, elimbs, 1, elimbs, kctx, stream)
    res = limbs_to_ints(device.to_host_u32(out))
    counters.bump("group_mult", len(rows) * n)
    return [PaillierCiphertext(r) for r in res]


def multiexp(pk, cts, exps) -> PaillierCiphertext:
    """prod cts[i]^exps[i] mod m^2 (paillier.py:134-193); group
    multiplications only (no general powmod)."""
    exps = [int(e) for e in exps]
    if len(exps) != len(cts):
        raise ValueError("dimension mismatch")
    return paillier_matmul(pk, [exps], cts)[0]


def add_batch(pk, a, b, stream=None) -> list:
    """[a_i * b_i mod m^2]: batched homomorphic addition (paillier.py:120-123)."""
    if len(a) != len(b):
        raise ValueError("dimension mismatch")
    if not a:
        return []
    dev = device.require_cuda()
    kctx = key_ctx(pk.m, dev)
    da = device.u32_tensor(ints_to_limbs(_cvals(a, kctx.m2), kctx.l2), dev)
    db = device.u32_tensor(ints_to_limbs(_cvals(b, kctx.m2), kctx.l2), dev)
    out = device.mulmod(da, db, kctx.l2, kctx.d_m2, kctx.c2.np, kctx.d_r2sq, stream)
    counters.bump("add", len(a))
    counters.bump("group_mult", len(a))
    return [PaillierCiphertext(r) for r in limbs_to_ints(device.to_host_u32(out))]


def add(pk, a, b) -> PaillierCiphertext:
    return add_batch(pk, [a], [b])[0]
