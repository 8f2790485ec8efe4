"""Database files written by the reference (dbfile.py) load into the device
layout unchanged (tests/golden/*.zpirdb from make_golden.py)."""

import os
import struct

import numpy as np
import pytest

from conftest import GOLDEN


def test_load_reference_file(golden):
    from paper_2603_09190_b200 import dbfile
    g = golden("desk_reduced")
    f = dbfile.load(os.path.join(GOLDEN, "desk_reduced.zpirdb"))
    assert (f.d0, f.d1, f.p, f.record_bytes) == (32, 48, 256, 48)
    assert f.symbols.dtype == np.uint8 and np.array_equal(f.symbols, g.db)


def test_load_ingested_p16():
    from paper_2603_09190_b200 import dbfile
    f = dbfile.load(os.path.join(GOLDEN, "ingest_p16.zpirdb"))
    raw = np.arange(80, dtype=np.int64)
    want = np.stack([raw & 15, raw >> 4], axis=1).reshape(8, 20)   # dbfile.py:77-85
    assert (f.p, f.record_bytes) == (16, 10) and np.array_equal(f.symbols, want)


def test_load_errors(tmp_path):
    from paper_2603_09190_b200 import dbfile
    src = open(os.path.join(GOLDEN, "ingest_p16.zpirdb"), "rb").read()
    cases = {
        "short": (src[:10], "shorter than header"),
        "magic": (b"X" + src[1:], "bad magic"),
        "version": (src[:8] + struct.pack("<I", 2) + src[12:], "unsupported database version"),
        "size": (src[:-1], "does not match header shape"),
        "range": (src[:-1] + b"\x10", "symbol out of range"),
    }
    for name, (data, msg) in cases.items():
        p = tmp_path / f"{name}.zpirdb"
        p.write_bytes(data)
        with pytest.raises(dbfile.DatabaseError, match=msg):
            dbfile.load(str(p))
    assert issubclass(dbfile.DatabaseError, ValueError)


@pytest.mark.gpu
def test_load_state_bit_exact(golden):
    import paper_2603_09190_b200 as z
    from paper_2603_09190_b200 import dbfile
    g = golden("desk_reduced")
    st = dbfile.load_state(g.params(z), os.path.join(GOLDEN, "desk_reduced.zpirdb"))
    assert np.array_equal(st.H, g.arr["H"])
    assert np.array_equal(st.db_matvec(g.arr["qu0"]), g.arr["b"])
    with pytest.raises(dbfile.DatabaseError):
        dbfile.load_state(g.params(z), os.path.join(GOLDEN, "ingest_p16.zpirdb"))
