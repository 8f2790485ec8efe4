"""The C-ABI library loads on CPU and exports every symbol include/*.h declares."""

import glob
import os
import re

from conftest import ROOT


def _declared():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(zpir_\w+)\s*\(", src))
    return names


def test_header_declares_entry_points():
    d = _declared()
    assert {"zpir_gemv", "zpir_global_hint", "zpir_multiexp", "zpir_answer_rows",
            "zpir_answer_groups", "zpir_combine"} <= d


def test_library_loads_and_exports_all():
    from paper_2603_09190_b200 import _lib, build
    build.build()
    lib = _lib.load()
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_lib.EXPORTED) == _declared()
    assert lib.zpir_abi_version() == 1


def test_status_codes_without_gpu():
    """Input validation happens before any CUDA call: status 1 -> ValueError."""
    import pytest
    from paper_2603_09190_b200 import _lib
    _lib.load()
    with pytest.raises(ValueError):
        # rows not a multiple of 128
        _lib.call("zpir_gemv", None, 100, 64, None, 1, None, 0xFFFFFFFF, None, None)
    assert b"multiple of 128" in _lib.lib().zpir_last_error()


def test_handle_api_validates_before_cuda():
    """zpir_db_create rejects bad parameters / symbols with status 1 on CPU."""
    import ctypes
    import numpy as np
    import pytest
    from paper_2603_09190_b200 import _lib
    _lib.load()
    prm = _lib.DbParams()
    prm.d0, prm.d1, prm.n, prm.log2q, prm.p, prm.cap, prm.gamma_bits = 4, 4, 4, 32, 4, 9, 33
    prm.gamma[1] = 1
    db = np.full((4, 4), 7, dtype=np.uint8)        # 7 >= p = 4
    h = ctypes.c_void_p()
    seed = np.zeros(16, dtype=np.uint8)
    args = (ctypes.byref(prm), db.ctypes.data_as(ctypes.c_void_p), 4, None,
            seed.ctypes.data_as(ctypes.c_void_p), ctypes.byref(h))
    with pytest.raises(ValueError, match="symbol out of range"):
        _lib.call("zpir_db_create", *args)
    db[:] = 1
    prm.gamma_bits = 40                            # inconsistent with gamma
    with pytest.raises(ValueError, match="gamma_bits"):
        _lib.call("zpir_db_create", *args)
    prm.gamma_bits, prm.log2q = 33, 40
    with pytest.raises(ValueError, match="bad parameters"):
        _lib.call("zpir_db_create", *args)
    assert _lib.lib().zpir_db_destroy(None) == 0
