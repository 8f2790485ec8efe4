"""Database file -> device layout loader.

Reads the reference's on-disk format (dbfile.py:1-57: header
struct "<8sIQQIQ" = magic "ZPIRDB1\\0", version 1, d0, d1, p, record_bytes;
then d0*d1 row-major symbols, one byte each for p <= 256, else u64 LE) with
the same DatabaseError cases, but memory-maps the body and hands it to the
device as the u8 array it already is: the reference materialises an int64
copy (8 bytes per symbol, 8 GiB for the 1 GiB config) before its own
float64 copy. Files with p > 256 are rejected (the device layout stores one
byte per symbol).
"""

import os
import struct
from dataclasses import dataclass

import numpy as np

MAGIC = b"ZPIRDB1\x00"
DB_VERSION = 1
HEADER = struct.Struct("<8sIQQIQ")


class DatabaseError(ValueError):
    pass


@dataclass
class DatabaseFile:
    d0: int
    d1: int
    p: int
    record_bytes: int
    symbols: np.ndarray   # (d0, d1) uint8, memory-mapped read-only


def load(path: str, check_range: bool = True) -> DatabaseFile:
    size = os.path.getsize(path)
    if size < HEADER.size:
        raise DatabaseError("file shorter than header")
    with open(path, "rb") as fh:
        magic, version, d0, d1, p, record_bytes = HEADER.unpack(fh.read(HEADER.size))
    if magic != MAGIC:
        raise DatabaseError("bad magic")
    if version != DB_VERSION:
        raise DatabaseError(f"unsupported database version {version}")
    width = 1 if p <= 256 else 8
    if size - HEADER.size != d0 * d1 * width:
        raise DatabaseError("symbol count does not match header shape")
    if width != 1:
        raise NotImplementedError("the device layout stores one byte per symbol (p <= 256)")
    if d0 * d1:
        symbols = np.memmap(path, dtype=np.uint8, mode="r", offset=HEADER.size, shape=(d0, d1))
    else:
        symbols = np.zeros((d0, d1), dtype=np.uint8)
    if check_range and symbols.size and int(symbols.max()) >= p:
        raise DatabaseError("symbol out of range")
    return DatabaseFile(d0, d1, p, record_bytes, symbols)


def load_state(params, path: str, **kw):
    """ServerGlobalState for the database stored at `path` (cli.py:53-56 +
    protocol.py:162); shape and p must match the parameters."""
    from .protocol import ServerGlobalState
    f = load(path, check_range=False)   # the state checks the range against lwe.p
    if (f.d0, f.d1) != (params.d0, params.d1):
        raise DatabaseError("database shape does not match the parameters")
    if f.p != params.lwe.p:
        raise DatabaseError("database alphabet does not match the parameters")
    return ServerGlobalState(params, f.symbols, **kw)
