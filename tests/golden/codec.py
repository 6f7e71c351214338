"""Compact on-disk form of packed trace records for the golden fixtures:
column-major arrays of the 48-byte csg_packed_record, LZMA-compressed."""
from __future__ import annotations

import lzma
import struct

import numpy as np

from paper_2509_03018_b200._abi import RECORD_DTYPE

# byte columns of the record: (offset, width)
_COLS = [(0, 8), (8, 8), (16, 4), (20, 4), (24, 4), (28, 1), (29, 1), (32, 8), (40, 8)]


def dump(records: np.ndarray) -> bytes:
    raw = np.ascontiguousarray(records, dtype=RECORD_DTYPE).view(np.uint8).reshape(-1, 48)
    parts = [struct.pack("<Q", len(records))]
    for off, w in _COLS:
        parts.append(np.ascontiguousarray(raw[:, off:off + w]).tobytes())
    return lzma.compress(b"".join(parts), preset=9)


def load(blob: bytes) -> np.ndarray:
    data = lzma.decompress(blob)
    n = struct.unpack_from("<Q", data, 0)[0]
    raw = np.zeros((n, 48), dtype=np.uint8)
    pos = 8
    for off, w in _COLS:
        raw[:, off:off + w] = np.frombuffer(data, dtype=np.uint8, count=n * w,
                                            offset=pos).reshape(n, w)
        pos += n * w
    return raw.reshape(-1).view(RECORD_DTYPE).copy()


def save_file(path: str, records: np.ndarray):
    with open(path, "wb") as f:
        f.write(dump(records))


def load_file(path: str) -> np.ndarray:
    with open(path, "rb") as f:
        return load(f.read())
