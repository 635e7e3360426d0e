"""NSTW1 record container (reference container.py:1-64): the on-disk format of network
weights and cached layer statistics, kept byte-compatible so weight/stat files written by
either implementation load in the other.

Layout: magic b"NSTW1", then per record: u32 name length, UTF-8 name, u8 dtype tag
(0 = f32, 1 = f64), u32 rank, u32 dims[rank], little-endian values.
"""

from __future__ import annotations

import struct

import numpy as np

from .errors import FormatError

MAGIC = b"NSTW1"
_DTYPES = (np.dtype("<f4"), np.dtype("<f8"))


def write_records(path, records: dict) -> None:
    out = bytearray(MAGIC)
    for name, arr in records.items():
        a = np.asarray(arr)
        tag = 0 if a.dtype == np.float32 else 1
        a = np.ascontiguousarray(a, dtype=_DTYPES[tag])
        key = name.encode("utf-8")
        out += struct.pack("<I", len(key)) + key
        out += struct.pack("<BI", tag, a.ndim) + struct.pack(f"<{a.ndim}I", *a.shape)
        out += a.tobytes()
    with open(path, "wb") as f:
        f.write(bytes(out))


def read_records(path) -> dict:
    with open(path, "rb") as f:
        buf = f.read()
    if buf[:5] != MAGIC:
        raise FormatError(f"{path}: bad magic {buf[:5]!r}, expected {MAGIC!r}")
    pos = 5
    recs = {}

    def need(n, what):
        if pos + n > len(buf):
            raise FormatError(f"{path}: truncated while reading {what}")

    while pos < len(buf):
        need(4, "record name length")
        (ln,) = struct.unpack_from("<I", buf, pos)
        pos += 4
        need(ln, "record name")
        name = buf[pos:pos + ln].decode("utf-8")
        pos += ln
        need(5, f"{name} header")
        tag, rank = struct.unpack_from("<BI", buf, pos)
        pos += 5
        if tag > 1:
            raise FormatError(f"{path}: record {name} has unknown dtype tag {tag}")
        need(4 * rank, f"{name} dims")
        dims = struct.unpack_from(f"<{rank}I", buf, pos)
        pos += 4 * rank
        dt = _DTYPES[tag]
        nbytes = int(np.prod(dims, dtype=np.int64)) * dt.itemsize
        need(nbytes, f"{name} data")
        recs[name] = np.frombuffer(buf, dtype=dt, count=nbytes // dt.itemsize, offset=pos).reshape(dims).copy()
        pos += nbytes
    return recs
