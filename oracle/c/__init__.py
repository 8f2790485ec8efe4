"""ctypes wrappers of the plain-C oracle -- TEST INFRASTRUCTURE ONLY.

zpir_oracle.c      integer GEMV / global-hint restatements (OpenMP)
zpir_gmp_oracle.c  big-integer restatements over libgmp.so.10: the reference's
                   windowed multiexp (paillier.py:134-193), the answer t
                   (protocol.py:343-350) and COMBINED (:354-358)
"""

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "zpir_oracle.c")
GMP_SRC = os.path.join(HERE, "zpir_gmp_oracle.c")
LIB = os.path.join(HERE, "..", "_build", "liboracle.so")
GMP_LIB = os.path.join(HERE, "..", "_build", "liboracle_gmp.so")
_lib = None
_gmp = None


def _stale(out, src):
    return not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(src)


def build(force=False):
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    if force or _stale(LIB, SRC):
        subprocess.check_call(["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-shared", "-fPIC",
                               SRC, "-o", LIB])
    if force or _stale(GMP_LIB, GMP_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", GMP_SRC, "-o",
                               GMP_LIB, "-l:libgmp.so.10"])
    return LIB


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(LIB)
    return _lib


def _load_gmp():
    global _gmp
    if _gmp is None:
        build()
        _gmp = ctypes.CDLL(GMP_LIB)
    return _gmp


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _i(x):
    return ctypes.c_int64(int(x))


def db_matvec(db, qu):
    db = np.ascontiguousarray(db, dtype=np.uint8)
    d0, d1 = db.shape
    q = np.ascontiguousarray(np.asarray(qu, dtype=np.uint64).astype(np.uint32))
    out = np.empty(d1, dtype=np.uint32)
    _load().oracle_db_matvec(_p(db), _i(d0), _i(d1), _p(q), _p(out))
    return out.astype(np.uint64)


def hint_cols(db, A, cols):
    db = np.ascontiguousarray(db, dtype=np.uint8)
    d0, d1 = db.shape
    A32 = np.ascontiguousarray(np.asarray(A).astype(np.uint32))
    n = A32.shape[1]
    c = np.ascontiguousarray(np.asarray(cols, dtype=np.int64))
    out = np.empty((len(c), n), dtype=np.uint32)
    _load().oracle_hint_cols(_p(db), _i(d0), _i(d1), _p(A32), _i(n), _p(c), _i(len(c)), _p(out))
    return out.astype(np.uint64)


def hint_rows(db, A, lo=0, hi=None):
    """H rows [lo, hi) = -(db^T A)[lo:hi] mod 2^32 as uint32 (cache-blocked)."""
    db = np.ascontiguousarray(db, dtype=np.uint8)
    d0, d1 = db.shape
    hi = d1 if hi is None else hi
    A32 = np.ascontiguousarray(np.asarray(A).astype(np.uint32))
    n = A32.shape[1]
    out = np.empty((hi - lo, n), dtype=np.uint32)
    _load().oracle_hint_rows(_p(db), _i(d0), _i(d1), _p(A32), _i(n), _i(lo), _i(hi), _p(out))
    return out


# -- big integers as little-endian u32 limb rows -------------------------------

def _limbs(vals, L):
    out = np.zeros((len(vals), L), dtype="<u4")
    for i, v in enumerate(vals):
        v = int(v)
        if v < 0 or v.bit_length() > 32 * L:
            raise ValueError("value does not fit the limb width")
        out[i] = np.frombuffer(v.to_bytes(4 * L, "little"), dtype="<u4")
    return out


def _ints(arr):
    a = np.ascontiguousarray(arr, dtype="<u4")
    return [int.from_bytes(a[i].tobytes(), "little") for i in range(a.shape[0])]


def _nl(x):
    return max(1, -(-int(x).bit_length() // 32))


def multiexp_rows(bases, exps, mod):
    """[prod_k bases[k]^exps[r][k] mod `mod` for each row r] by the reference's
    windowed multiexp (paillier.py:134-193). `exps` is either a list of rows
    of Python ints or a (rows, n, Le) u32 limb array (little-endian words)."""
    n = len(bases)
    Lm = _nl(mod)
    B = _limbs(bases, max(Lm, max((_nl(b) for b in bases), default=1)))
    if isinstance(exps, np.ndarray):
        E = np.ascontiguousarray(exps, dtype="<u4")
        if E.ndim != 3 or E.shape[1] != n:
            raise ValueError("exps must be (rows, n, Le)")
    else:
        Le = max((_nl(e) for row in exps for e in row), default=1)
        E = np.stack([_limbs(row, Le) for row in exps]) if exps else \
            np.zeros((0, n, 1), dtype="<u4")
        if E.shape[1] != n:
            raise ValueError("dimension mismatch")
    rows, _, Le = E.shape
    M = _limbs([mod], Lm)
    out = np.zeros((rows, Lm), dtype="<u4")
    rc = _load_gmp().oracle_gmp_multiexp(_p(B), _i(n), _i(B.shape[1]), _p(E), _i(rows), _i(Le),
                                         _p(M), _i(Lm), _p(out), _i(Lm))
    if rc:
        raise RuntimeError("oracle_gmp_multiexp: result wider than the modulus")
    return _ints(out)


def answer_t(H, b, ck_o, m, cap, gamma, d1=None):
    """t_g = (sum_j gamma^j (b_c + y_c)) mod m for all groups (protocol.py:343-350)."""
    H = np.ascontiguousarray(np.asarray(H).astype(np.uint32))
    d1 = H.shape[0] if d1 is None else d1
    n = H.shape[1]
    b32 = np.ascontiguousarray(np.asarray(b, dtype=np.uint64)[:d1].astype(np.uint32))
    Lm = _nl(m)
    C = _limbs(ck_o, Lm)
    if C.shape[0] != n:
        raise ValueError("dimension mismatch")
    M = _limbs([m], Lm)
    G = _limbs([gamma], _nl(gamma))
    groups = -(-d1 // cap)
    out = np.zeros((groups, Lm), dtype="<u4")
    rc = _load_gmp().oracle_gmp_answer_t(_p(H), _p(b32), _i(d1), _i(n), _p(C), _i(Lm), _p(M),
                                         _i(Lm), _p(G), _i(G.shape[1]), _i(cap), _p(out), _i(Lm))
    if rc:
        raise RuntimeError("oracle_gmp_answer_t failed")
    return _ints(out)


def combined(t, k, m):
    """K_g = trivial_encrypt(t_g) k_g mod m^2 (protocol.py:354-358)."""
    Lm = _nl(m)
    L2 = _nl(m * m)
    T = _limbs(t, Lm)
    Kk = _limbs(k, L2)
    out = np.zeros((len(t), L2), dtype="<u4")
    rc = _load_gmp().oracle_gmp_combine(_p(T), _i(Lm), _p(Kk), _i(L2), _i(len(t)),
                                        _p(_limbs([m], Lm)), _i(Lm), _p(out), _i(L2))
    if rc:
        raise RuntimeError("oracle_gmp_combine failed")
    return _ints(out)


def scaled_exponents(H, cap, groups=None):
    """The hint's exponent rows H_scaled[g][k] = sum_j 2^(32 j) H[g cap + j][k]
    (protocol.py:219-238, gamma = 2^32 layout) as a (G, n, cap) u32 limb
    array: limb j of exponent (g, k) is H[g cap + j][k]."""
    H = np.asarray(H).astype(np.uint32)
    d1, n = H.shape
    G = -(-d1 // cap)
    sel = range(G) if groups is None else groups
    out = np.zeros((len(sel), n, cap), dtype="<u4")
    for i, g in enumerate(sel):
        blk = H[g * cap:min((g + 1) * cap, d1)]
        out[i, :, : blk.shape[0]] = blk.T
    return out
