"""ctypes wrapper of oracle/c/zpir_oracle.c -- TEST INFRASTRUCTURE ONLY."""

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "zpir_oracle.c")
LIB = os.path.join(HERE, "..", "_build", "liboracle.so")
_lib = None


def build(force=False):
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-shared", "-fPIC",
                               SRC, "-o", LIB])
    return LIB


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(LIB)
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def db_matvec(db, qu):
    db = np.ascontiguousarray(db, dtype=np.uint8)
    d0, d1 = db.shape
    q = np.ascontiguousarray(np.asarray(qu, dtype=np.uint64).astype(np.uint32))
    out = np.empty(d1, dtype=np.uint32)
    _load().oracle_db_matvec(_p(db), ctypes.c_int64(d0), ctypes.c_int64(d1), _p(q), _p(out))
    return out.astype(np.uint64)


def hint_cols(db, A, cols):
    db = np.ascontiguousarray(db, dtype=np.uint8)
    d0, d1 = db.shape
    A32 = np.ascontiguousarray(np.asarray(A).astype(np.uint32))
    n = A32.shape[1]
    c = np.ascontiguousarray(np.asarray(cols, dtype=np.int64))
    out = np.empty((len(c), n), dtype=np.uint32)
    _load().oracle_hint_cols(_p(db), ctypes.c_int64(d0), ctypes.c_int64(d1), _p(A32),
                             ctypes.c_int64(n), _p(c), ctypes.c_int64(len(c)), _p(out))
    return out.astype(np.uint64)
