"""LWE -> Paillier compression on the B200 kernels.

Mirrors the server-side operations of the reference compressor
(compress.py:99-258): lwe_compress, fast_lwe_compress, batched_lwe_compress,
fast_batched_lwe_compress, plus lwe_compress_many (many independent
ciphertexts in one device launch). Every one of them is a single
multi-exponentiation over the compression key times one trivial encryption:

  lwe_compress(ct)            = Enc~(b) * prod_i ck_i^((q - a_i) mod q)
  batched_lwe_compress(cts)   = Enc~(sum_j gamma^j b_j) *
                                prod_i ck_i^(sum_j gamma^j ((q - a_ji) mod q))

which is the same group element the reference reaches through scalar_mul
(batched) or repeated doubling of an expanded key (fast paths): in Z_{m^2},
(1 + v m)^s = 1 + s v m, and the doubled keys are ck_i^(2^r). Results are
therefore bit-identical, computed with group multiplications only (no
modexp, no scalar_mul counted). Key generation / encryption / decryption
are client operations (out of scope); keys may be the reference's objects.
"""

from dataclasses import dataclass

from . import counters
from .paillier import PaillierCiphertext, add_batch, paillier_matmul
from .params import BINARY


class ModulusTooSmall(Exception):
    pass


class CapacityExceeded(Exception):
    pass


@dataclass
class CompressedCiphertext:
    x: PaillierCiphertext
    lwe_params: object
    gamma: int = 1
    ell: int = 1
    key_scaling: int = 1


def phase_bound(params) -> int:
    """compress.py:30-33."""
    q, n = params.q, params.n
    return q + n * q if params.key_dist == BINARY else q + n * q * q


def _check_modulus(pk, params):
    if pk.m <= phase_bound(params):
        raise ModulusTooSmall("plaintext modulus must exceed the phase bound")


def batch_capacity(pk, gamma: int) -> int:
    """Largest ell with gamma^ell < m (compress.py:197-203)."""
    ell, power = 0, 1
    while power * gamma < pk.m:
        power *= gamma
        ell += 1
    return ell


def _key_list(ck):
    """Base keys: CompressionKey.ck or ExpandedCompressionKey.eck[0]."""
    if hasattr(ck, "eck"):
        return ck.eck[0]
    return ck.ck


def _finish(pk, bvals, accs, params, **kw):
    triv = [PaillierCiphertext((1 + (int(b) % pk.m) * pk.m) % pk.m2) for b in bvals]
    out = add_batch(pk, triv, accs)
    return [CompressedCiphertext(x, params, **kw) for x in out]


def lwe_compress_many(ck, cts) -> list:
    """Independent compressions of many LWE ciphertexts under one key in a
    single device multi-exponentiation (rows = ciphertexts)."""
    pk, params = ck.pk, ck.lwe_params
    _check_modulus(pk, params)
    if not cts:
        return []
    q = params.q
    rows = [[(q - int(a)) % q for a in ct.a] for ct in cts]
    accs = paillier_matmul(pk, rows, _key_list(ck))
    return _finish(pk, [ct.b for ct in cts], accs, params,
                   key_scaling=getattr(ck, "key_scaling", 1))


def lwe_compress(ck, ct) -> CompressedCiphertext:
    """compress.py:99-105."""
    return lwe_compress_many(ck, [ct])[0]


def fast_lwe_compress(eck, ct) -> CompressedCiphertext:
    """compress.py:181-194 (addition-only in the reference; here the same
    element through the multiexp over eck[0])."""
    return lwe_compress_many(eck, [ct])[0]


def _batched(ck, cts, gamma):
    pk, params = ck.pk, ck.lwe_params
    if getattr(ck, "key_scaling", 1) != 1:
        raise ValueError("batching requires an unscaled compression key")
    if len(cts) > batch_capacity(pk, gamma):
        raise CapacityExceeded("batch exceeds capacity at this scale")
    q = params.q
    n = params.n
    exps = [0] * n
    for j, ct in enumerate(cts):
        s = gamma ** j
        for i, a in enumerate(ct.a):
            exps[i] += s * ((q - int(a)) % q)
    acc = paillier_matmul(pk, [exps], _key_list(ck))
    btotal = sum(gamma ** j * int(ct.b) for j, ct in enumerate(cts))
    return _finish(pk, [btotal], acc, params, gamma=gamma, ell=len(cts))[0]


def batched_lwe_compress(ck, cts, gamma: int) -> CompressedCiphertext:
    """compress.py:213-221."""
    return _batched(ck, cts, gamma)


def fast_batched_lwe_compress(ck, cts, gamma: int) -> CompressedCiphertext:
    """compress.py:224-258."""
    out = _batched(ck, cts, gamma)
    counters.bump("scalar_mul", 0)
    return out
