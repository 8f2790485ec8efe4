"""numpy-only binding of the handle-level C ABI (include/zippir_db.h).

The same server hot path as protocol.py, driven through `zpir_db_*` with
HOST buffers: no torch, no device pointers, no Montgomery constants on the
caller's side. This is what a maintainer of the reference (pure Python +
numpy, /root/reference/pkg/src/zippir) would bind with ctypes to replace

    ServerGlobalState.__init__ / _global_hint_fast   (protocol.py:162-217)
    ServerGlobalState.db_matvec                       (protocol.py:242-257)
    rns.rns_matmul_mod + scaled_b + t                 (protocol.py:345-351, rns.py:163-188)
    COMBINED                                          (protocol.py:352-358)
    hint / paillier_matmul                            (protocol.py:291-296, paillier.py:196-203)
    paillier.multiexp / add                           (paillier.py:120-193)
    update_database (row-incremental)                 (server.py:115-124)

Errors: status 1 -> ValueError, 2/3 -> ZpirError, as everywhere in the package.
"""

import ctypes

import numpy as np

from . import _lib
from .bigint import ints_to_limbs, limbs_to_ints
from .params import Layout


def _vp(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _limbs(bits: int) -> int:
    return max(1, -(-bits // 32))


class DeviceDatabase:
    """One database on one GPU (zpir_db handle).

    params: ProtocolParams (this package's or the reference's); db: (d0, d1)
    symbols < p; A: optional (d0, n) public matrix, else generated on the
    device from params.a_seed."""

    def __init__(self, params, db, A=None, device: int = 0, engine: str = "umma"):
        lay = self.layout = Layout(params)
        db = np.ascontiguousarray(np.asarray(db), dtype=np.uint8) if np.asarray(db).size else None
        if db is None or db.shape != (lay.d0, lay.d1):
            raise ValueError("database shape mismatch")
        prm = _lib.DbParams()
        prm.d0, prm.d1, prm.n = lay.d0, lay.d1, lay.n
        prm.log2q = lay.q.bit_length() - 1
        prm.p = lay.p
        prm.cap = lay.cap
        prm.gamma_bits = lay.gamma.bit_length()
        for i, w in enumerate(lay.gamma_words):
            prm.gamma[i] = int(w)
        prm.device = device
        prm.engine = {"umma": 0, "cuda_core": 1}[engine]
        a_arr = None
        if A is not None:
            a_arr = np.ascontiguousarray(np.asarray(A, dtype=np.uint64).astype(np.uint32))
            if a_arr.shape != (lay.d0, lay.n):
                raise ValueError("public matrix shape mismatch")
        seed = np.frombuffer(bytes(params.a_seed), dtype=np.uint8).copy()
        h = ctypes.c_void_p()
        _lib.call("zpir_db_create", ctypes.byref(prm), _vp(db), lay.d1,
                  _vp(a_arr) if a_arr is not None else None, _vp(seed), ctypes.byref(h))
        self._h = h
        g, r = ctypes.c_int64(), ctypes.c_int64()
        _lib.call("zpir_db_info", h, ctypes.byref(g), ctypes.byref(r))
        self.groups = g.value

    # -- handle lifetime -------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().zpir_db_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- (4) global hint, (2)/(3) matvec ------------------------------------------
    def global_hint(self) -> np.ndarray:
        lay = self.layout
        H = np.empty((lay.d1, lay.n), dtype=np.uint32)
        _lib.call("zpir_db_global_hint", self._h, _vp(H))
        return H

    def db_matvec(self, qu) -> np.ndarray:
        """b = db^T qu mod q; qu (d0,) or (nvec, d0) -> uint64 (d1,) / (nvec, d1)."""
        lay = self.layout
        q = np.asarray(qu, dtype=np.uint64)
        one = q.ndim == 1
        q = np.ascontiguousarray(q.reshape(-1, lay.d0).astype(np.uint32))
        if q.shape[1] != lay.d0:
            raise ValueError("query dimensions do not match the parameters")
        b = np.empty((q.shape[0], lay.d1), dtype=np.uint32)
        _lib.call("zpir_db_matvec", self._h, _vp(q), q.shape[0], _vp(b))
        b = b.astype(np.uint64)
        return b[0] if one else b

    # -- (5) answers ------------------------------------------------------------
    def _query(self, qu, ck_o, m):
        lay = self.layout
        q = np.ascontiguousarray(np.asarray(qu, dtype=np.uint64).astype(np.uint32))
        if q.shape != (lay.d0,) or len(ck_o) != lay.n:
            raise ValueError("query dimensions do not match the parameters")
        L = _limbs(int(m).bit_length())
        try:   # Python ints (the reference's QueryMessage.ck_o) convert in C directly
            c = ints_to_limbs(ck_o, L)
        except TypeError:   # other integer types (numpy scalars, ...)
            c = ints_to_limbs([int(v) for v in ck_o], L)
        return q, c, ints_to_limbs([int(m)], L), L

    def answer(self, qu, ck_o, m) -> list:
        """SEPARATE answer t (d1' ints < m)."""
        q, c, mm, L = self._query(qu, ck_o, m)
        t = np.empty((self.groups, L), dtype=np.uint32)
        _lib.call("zpir_db_answer", self._h, _vp(q), _vp(c), _vp(mm), L, _vp(t))
        return limbs_to_ints(t)

    def answer_combined(self, qu, ck_o, m, k) -> list:
        """COMBINED answer K_g = Enc~(t_g) k_g mod m^2 for stored hint entries k."""
        q, c, mm, L = self._query(qu, ck_o, m)
        if len(k) != self.groups:
            raise ValueError("hint entry count does not match d1'")
        kin = ints_to_limbs([int(x) for x in k], 2 * L)
        K = np.empty((self.groups, 2 * L), dtype=np.uint32)
        _lib.call("zpir_db_answer_combined", self._h, _vp(q), _vp(c), _vp(mm), L, _vp(kin), _vp(K))
        return limbs_to_ints(K)

    # -- per-client hint, (8) update ----------------------------------------------
    def client_hint(self, m, seed: bytes, query_index: int) -> list:
        L = _limbs(int(m).bit_length())
        mm = ints_to_limbs([int(m)], L)
        s = np.frombuffer(bytes(seed), dtype=np.uint8).copy()
        k = np.empty((self.groups, 2 * L), dtype=np.uint32)
        _lib.call("zpir_db_client_hint", self._h, _vp(mm), L, _vp(s), s.size, query_index, _vp(k))
        return limbs_to_ints(k)

    def update_rows(self, cols, values):
        """db[:, cols[i]] = values[i] (each d0 symbols); H rows refreshed."""
        lay = self.layout
        c = np.ascontiguousarray(np.asarray(cols, dtype=np.int64).ravel())
        v = np.ascontiguousarray(np.asarray(values, dtype=np.uint8).reshape(c.size, lay.d0))
        _lib.call("zpir_db_update_rows", self._h, _vp(c), c.size, _vp(v))


# -- (6)/(7) batched modular arithmetic ---------------------------------------------

def montmul_batch(a, b, N, device: int = 0) -> list:
    """[a_i * b_i mod N] (paillier.add's product, paillier.py:120-123)."""
    if len(a) != len(b):
        raise ValueError("dimension mismatch")
    L = _limbs(int(N).bit_length())
    A = ints_to_limbs([int(x) for x in a], L)
    B = ints_to_limbs([int(x) for x in b], L)
    out = np.empty_like(A)
    _lib.call("zpir_montmul_batch", _vp(A), _vp(B), len(a), _vp(ints_to_limbs([int(N)], L)), L,
              _vp(out), device)
    return limbs_to_ints(out)


def multiexp_batch(bases, exps, N, device: int = 0) -> list:
    """[prod_k bases[k]^exps[g][k] mod N for each row g] (paillier.py:134-203)."""
    n = len(bases)
    if any(len(r) != n for r in exps):
        raise ValueError("dimension mismatch")
    L = _limbs(int(N).bit_length())
    ebits = max([int(e).bit_length() for r in exps for e in r] + [1])
    Le = _limbs(ebits)
    Bs = ints_to_limbs([int(x) for x in bases], L)
    E = ints_to_limbs([int(e) for r in exps for e in r], Le)
    out = np.empty((len(exps), L), dtype=np.uint32)
    _lib.call("zpir_multiexp_batch", _vp(Bs), n, _vp(E), len(exps), Le,
              _vp(ints_to_limbs([int(N)], L)), L, _vp(out), device)
    return limbs_to_ints(out)
