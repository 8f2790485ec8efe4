"""ctypes binding of libzpir_b200.so (the C ABI in include/zippir_b200.h).

This is the Python-side FFI the reference would bind. It
fails loudly: if the shared library is missing or no CUDA device is present,
every entry raises -- there is no CPU fallback anywhere in the product.
ctypes releases the GIL for the duration of each foreign call, so the
connection threads and the hint worker can overlap GPU submissions.
"""

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libzpir_b200.so")

_c_i64 = ctypes.c_int64
_c_int = ctypes.c_int
_c_u32 = ctypes.c_uint32
_p = ctypes.c_void_p

class DbParams(ctypes.Structure):
    """zpir_db_params (include/zippir_db.h)."""
    _fields_ = [("d0", ctypes.c_int64), ("d1", ctypes.c_int64), ("n", ctypes.c_int64),
                ("log2q", ctypes.c_int32), ("p", ctypes.c_int32), ("cap", ctypes.c_int32),
                ("gamma_bits", ctypes.c_int32), ("gamma", ctypes.c_uint32 * 8),
                ("device", ctypes.c_int32), ("engine", ctypes.c_int32)]


_SIGS = {
    "zpir_abi_version": ([], _c_int),
    "zpir_event_record": ([_p, _p], _c_int),
    "zpir_stream_wait_event": ([_p, _p], _c_int),
    "zpir_graph_launch": ([_p, _p], _c_int),
    # handle-level ABI (include/zippir_db.h), host buffers
    "zpir_db_create": ([ctypes.POINTER(DbParams), _p, _c_i64, _p, _p, ctypes.POINTER(_p)], _c_int),
    "zpir_db_destroy": ([_p], _c_int),
    "zpir_db_info": ([_p, ctypes.POINTER(_c_i64), ctypes.POINTER(_c_i64)], _c_int),
    "zpir_db_global_hint": ([_p, _p], _c_int),
    "zpir_db_matvec": ([_p, _p, _c_i64, _p], _c_int),
    "zpir_db_answer": ([_p, _p, _p, _p, _c_int, _p], _c_int),
    "zpir_db_answer_combined": ([_p, _p, _p, _p, _c_int, _p, _p], _c_int),
    "zpir_db_client_hint": ([_p, _p, _c_int, _p, _c_i64, ctypes.c_uint64, _p], _c_int),
    "zpir_db_update_rows": ([_p, _p, _c_i64, _p], _c_int),
    "zpir_montmul_batch": ([_p, _p, _c_i64, _p, _c_int, _p, _c_int], _c_int),
    "zpir_multiexp_batch": ([_p, _c_i64, _p, _c_i64, _c_int, _p, _c_int, _p, _c_int], _c_int),
    "zpir_last_error": ([], ctypes.c_char_p),
    "zpir_host_device_pointer": ([_p, ctypes.POINTER(_p)], _c_int),
    "zpir_rns_residues": ([_p, _c_i64, _c_i64, _c_int, _c_int, _p, _p, _c_int, _c_i64, _p, _p],
                          _c_int),
    "zpir_multiexp_opcount": ([_p, _c_i64, _c_i64, _c_int, _c_int, _c_i64, _p, _p], _c_int),
    "zpir_transpose_db": ([_p, _c_i64, _c_i64, _c_i64, _p, _c_i64, _c_i64, _p], _c_int),
    "zpir_global_hint": ([_p, _c_i64, _c_i64, _p, _c_i64, _c_i64, _p, _c_u32, _p], _c_int),
    "zpir_gemv_workspace_bytes": ([_c_i64, _c_i64], _c_i64),
    "zpir_gemv": ([_p, _c_i64, _c_i64, _p, _c_i64, _p, _c_u32, _p, _p], _c_int),
    "zpir_answer_rows": ([_p, _c_i64, _c_i64, _p, _c_u32, _p, _c_int, _p, _p], _c_int),
    "zpir_answer_groups": ([_p, _p, _c_u32, _c_i64, _c_int, _c_i64, _c_int, _p, _c_u32, _p,
                            _c_int, _c_int, _p, _c_i64, _p], _c_int),
    "zpir_combine": ([_p, _p, _c_i64, _c_int, _p, _c_u32, _p, _p, _p, _p], _c_int),
    "zpir_mulmod": ([_p, _p, _c_i64, _c_int, _p, _c_u32, _p, _p, _p], _c_int),
    "zpir_multiexp_workspace_bytes": ([_c_i64, _c_i64, _c_int, _c_int], _c_i64),
    "zpir_multiexp": ([_p, _c_i64, _p, _c_i64, _c_i64, _c_i64, _c_i64, _c_int, _c_int, _p,
                       _c_u32, _p, _p, _p, _c_i64, _p], _c_int),
    "zpir_query_planes": ([_p, _c_i64, _c_i64, _p, _c_i64, _p], _c_int),
    "zpir_umma_gemv": ([_p, _c_i64, _c_i64, _p, _c_i64, _p, _c_int, _p], _c_int),
    "zpir_build_aplanes": ([_p, _c_i64, _c_i64, _c_i64, _p, _p], _c_int),
    "zpir_umma_global_hint": ([_p, _c_i64, _c_i64, _p, _c_i64, _p, _c_u32, _p], _c_int),
    "zpir_build_bc": ([_p, _c_i64, _c_int, _c_int, _p, _p], _c_int),
    "zpir_umma_answer_rows": ([_p, _c_i64, _c_i64, _p, _c_int, _p, _c_u32, _c_int, _p, _c_int,
                               _p], _c_int),
    "zpir_build_bc_batch": ([_p, _c_i64, _c_int, _c_int, _c_int, _p, _p], _c_int),
    "zpir_umma_answer_rows_batch": ([_p, _c_i64, _c_i64, _p, _c_int, _c_int, _c_int, _p, _p],
                                    _c_int),
    "zpir_answer_groups_batch": ([_p, _c_i64, _p, _c_i64, _c_u32, _c_i64, _c_int, _c_i64, _c_int,
                                  _p, _p, _p, _c_int, _p, _p, _c_i64, _c_int, _c_int, _p], _c_int),
    "zpir_multiexp_rows": ([_p, _c_i64, _p, _p, _c_i64, _c_i64, _c_i64, _c_i64, _c_int, _c_int,
                            _p, _c_u32, _p, _p, _c_int, _p, _p, _c_i64, _p], _c_int),
    "zpir_slot_combine": ([_p, _c_int, _p, _c_i64, _c_int, _p, _c_u32, _p, _c_int, _p, _p], _c_int),
    "zpir_slot_combine_many": ([_c_int, _p, _p, _p, _p, _c_int, _p, _c_i64, _c_int, _p, _c_int, _p],
                               _c_int),
    "zpir_answer_general": ([_p, _p, _c_u32, _c_i64, _c_int, _c_i64, _c_int, _p, _c_u32, _p, _p, _p,
                             _c_i64, _p], _c_int),
    "zpir_pow8_table": ([_p, _c_i64, _c_int, _p, _c_u32, _p, _p, _p], _c_int),
    "zpir_slot_fixed": ([_p, _c_i64, _p, _c_i64, _p, _c_i64, _c_int, _p, _c_u32, _p, _p, _p],
                        _c_int),
    "zpir_groups_z": ([_p, _c_i64, _c_i64, _c_int, _c_i64, _c_int, _p, _p, _p, _c_int, _p, _p,
                       _c_i64, _c_int, _c_int, _p], _c_int),
    "zpir_groups_finish": ([_p, _p, _c_i64, _c_u32, _c_i64, _c_int, _c_i64, _c_int, _p, _p, _c_i64,
                            _c_int, _c_int, _p], _c_int),
    "zpir_chacha_words32": ([ctypes.c_char_p, ctypes.c_char_p, _c_i64, _c_i64, _p, _c_i64, _c_u32,
                             _p], _c_int),
    "zpir_chacha_below": ([ctypes.c_char_p, _c_u32, ctypes.c_uint64, _c_i64, _p, _c_int, _c_int, _p,
                           _p], _c_int),
    "zpir_digits_to_limbs": ([_p, _c_i64, _c_int, _p, _c_int, _p], _c_int),
    "zpir_limbs_to_digits": ([_p, _c_i64, _c_int, _c_i64, _p, _c_int, _p], _c_int),
    "zpir_rows_differ": ([_p, _p, _c_i64, _c_i64, _p, _p], _c_int),
    "zpir_move_rows": ([_p, _p, _c_i64, _p, _c_i64, _c_int, _p], _c_int),
    "zpir_memcpy_async": ([_p, _p, _c_i64, _c_int, _p], _c_int),
    "zpir_probe_imad": ([_c_int, _c_int, ctypes.POINTER(ctypes.c_float)], _c_int),
    "zpir_h_planes": ([_p, _c_i64, _c_i64, _p, _p], _c_int),
    "zpir_slot_fixed_tc": ([_p, _c_i64, _p, _c_i64, _c_i64, _c_int, _p, _c_u32, _p, _p, _p],
                           _c_int),
    "zpir_slot_fixed_tc_many": ([_c_int, _p, _p, _p, _p, _p, _c_i64, _p, _c_i64, _p, _c_i64, _p],
                                _c_int),
    "zpir_slot_fixed_tc_workspace": ([_c_i64, _c_i64, _c_int], _c_i64),
    "zpir_build_bcp": ([_p, _c_i64, _c_int, _c_int, _p, _p], _c_int),
    "zpir_umma_answer_rows_planar": ([_p, _c_i64, _c_i64, _p, _c_int, _c_int, _c_int, _p, _c_int,
                                      _p], _c_int),
    "zpir_probe_umma_i8": ([_c_int, _c_int, _c_int, ctypes.POINTER(ctypes.c_float)], _c_int),
}

EXPORTED = tuple(_SIGS)

_lock = threading.Lock()
_lib = None


class ZpirError(RuntimeError):
    """CUDA-side failure reported by the C ABI (status 2/3)."""


def load(path=LIB_PATH):
    """Load and type the shared library (no GPU needed just to load)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ImportError(
                f"{path} is missing: build it with `python -m paper_2603_09190_b200.build` "
                "(the B200 path has no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
        return lib


def lib():
    return _lib if _lib is not None else load()


def call(name, *args):
    """Invoke an entry point; map status codes to exceptions."""
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        msg = (lib().zpir_last_error() or b"").decode(errors="replace")
        if rc == 1:
            raise ValueError(f"{name}: {msg}")
        raise ZpirError(f"{name} failed ({rc}): {msg}")
    return rc


def ptr(t):
    """Device pointer of a torch tensor as a c_void_p-compatible int."""
    return ctypes.c_void_p(t.data_ptr())


def stream_handle(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)
