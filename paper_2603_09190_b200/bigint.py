"""Python int <-> little-endian u32 limb arrays, and Montgomery contexts.

Host-side layout plumbing only (no arithmetic on the data path): the device
kernels take limbs; the reference's API takes and returns Python ints
(PaillierCiphertext.c, QueryMessage.ck_o, ResponseMessage.t).
"""

import threading

import numpy as np

# limbs-per-lane widths the warp kernels are instantiated for (csrc/*.cu)
SUPPORTED_LPL = (1, 2, 3, 4, 6, 8)


def limbs_for_bits(bits: int) -> int:
    """Smallest supported warp width (32 * LPL limbs) holding `bits` bits."""
    need = -(-bits // 32)
    for lpl in SUPPORTED_LPL:
        if 32 * lpl >= need:
            return 32 * lpl
    raise NotImplementedError(f"{bits}-bit moduli exceed the widest kernel (8192 bits)")


def _conv():
    global _CONV
    if _CONV is None:
        from . import build
        build.build_conv()
        from . import _zpir_conv
        _CONV = _zpir_conv
    return _CONV


_CONV = None


def ints_to_limbs(values, nlimbs: int, out=None) -> np.ndarray:
    """(len(values), nlimbs) uint32, little-endian limbs (C loop over
    _PyLong_AsByteArray). ValueError on negative or too-wide values."""
    if not isinstance(values, (list, tuple)):
        values = list(values)
    if out is None:
        out = np.empty((len(values), nlimbs), dtype=np.uint32)
    _conv().ints_into(values, out, nlimbs)
    return out


def limbs_to_ints(arr) -> list:
    a = np.ascontiguousarray(arr, dtype="<u4")
    rows, nl = a.shape
    return _conv().ints_from(a, rows, nl)


class ModCtx:
    """Montgomery context of an odd modulus N at a warp width of L limbs:
    N limbs, n' = -N^-1 mod 2^32, R = 2^(32 L), extra tables on demand."""

    def __init__(self, N: int, limbs: int):
        if N % 2 == 0 or N <= 1:
            raise ValueError("Montgomery modulus must be odd and > 1")
        self.N = N
        self.limbs = limbs
        self.R = 1 << (32 * limbs)
        if N >= self.R:
            raise ValueError("modulus wider than the limb width")
        self.np = (-pow(N, -1, 1 << 32)) % (1 << 32)
        self.n_limbs = ints_to_limbs([N], limbs)[0]
        self.r2 = ints_to_limbs([self.R * self.R % N], limbs)[0]

    def rpow(self, count: int) -> np.ndarray:
        """R^(s+1) mod N for s < count, (count, limbs)."""
        return ints_to_limbs([pow(self.R, s + 1, self.N) for s in range(count)], self.limbs)


class KeyCtx:
    """Per-Paillier-key device constants (cached per modulus m)."""

    def __init__(self, m: int, device):
        import torch
        self.m = m
        self.m2 = m * m
        bits = m.bit_length()
        self.lm = limbs_for_bits(bits)
        self.l2 = limbs_for_bits(2 * bits)
        self.cm = ModCtx(m, self.lm)
        self.c2 = ModCtx(self.m2, self.l2)
        self.mr = ints_to_limbs([m * self.c2.R % self.m2], self.l2)[0]
        dev = lambda a: torch.from_numpy(np.array(a, dtype=np.uint32).view(np.int32)).to(device)
        self.d_m = dev(self.cm.n_limbs)
        self.d_m2 = dev(self.c2.n_limbs)
        self.d_r2sq = dev(self.c2.r2)
        self.d_mr = dev(self.mr)
        self.d_one2 = dev(ints_to_limbs([self.c2.R % self.m2], self.l2)[0])  # Montgomery 1
        self._rpow = {}
        self._dev = dev
        self._lock = threading.Lock()

    def d_gamma_table(self, gamma: int, cap: int):
        """{gamma^j R mod m, gamma^j R^2 mod m} for j < cap (general-gamma answers)."""
        key = ("g", gamma, cap)
        with self._lock:
            t = self._rpow.get(key)
            if t is None:
                m, R = self.m, self.cm.R
                vals = []
                g = 1
                for _ in range(cap):
                    vals += [g * R % m, g * R * R % m]
                    g = g * gamma % m
                t = self._rpow[key] = self._dev(ints_to_limbs(vals, self.lm))
            return t

    def d_rpow(self, nchunks: int):
        with self._lock:
            t = self._rpow.get(nchunks)
            if t is None:
                t = self._rpow[nchunks] = self._dev(self.cm.rpow(nchunks))
            return t


_key_cache = {}
_key_lock = threading.Lock()


def key_ctx(m: int, device) -> KeyCtx:
    k = (m, str(device))
    with _key_lock:
        ctx = _key_cache.get(k)
        if ctx is None:
            if len(_key_cache) > 4096:
                _key_cache.clear()
            ctx = _key_cache[k] = KeyCtx(m, device)
        return ctx
