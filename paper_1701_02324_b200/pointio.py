"""PTS1 / CSV point and vector files (data.py:125-217 of the reference).

PTS1 layout: the 4 bytes ``PTS1``, n and d as little-endian u64, then n * d
little-endian float64 values, row-major.  Vectors (weights, right-hand
sides, labels, solutions) are PTS1 files with d = 1.  Malformed files raise
``PointFormatError`` (a ValueError) naming the file and the offending byte
or line, as the reference does.
"""

from __future__ import annotations

import struct

import numpy as np

from .data import PointSet

PTS1_MAGIC = b"PTS1"
_HDR = struct.Struct("<4sQQ")


class PointFormatError(ValueError):
    """Malformed points file (bad magic, truncation, bad CSV cell)."""


def save_points(ps, path, format="binary"):
    coords = ps.coords if isinstance(ps, PointSet) else np.atleast_2d(np.asarray(ps, dtype=np.float64))
    if format == "binary":
        with open(path, "wb") as fh:
            fh.write(_HDR.pack(PTS1_MAGIC, coords.shape[0], coords.shape[1]))
            fh.write(np.ascontiguousarray(coords, dtype="<f8").tobytes())
    elif format == "csv":
        with open(path, "w") as fh:
            fh.writelines(",".join(f"{v:.17g}" for v in row) + "\n" for row in coords)
    else:
        raise ValueError(f"unknown format {format!r}")


def load_points(path, format="binary"):
    if format == "csv":
        return _read_csv(path)
    if format != "binary":
        raise ValueError(f"unknown format {format!r}")
    with open(path, "rb") as fh:
        head = fh.read(_HDR.size)
        if len(head) < _HDR.size:
            raise PointFormatError(f"{path}: truncated header ({len(head)} of {_HDR.size} bytes)")
        magic, n, d = _HDR.unpack(head)
        if magic != PTS1_MAGIC:
            raise PointFormatError(f"{path}: bad magic {magic!r} at byte 0")
        want = 8 * n * d
        body = fh.read(want)
    if len(body) < want:
        raise PointFormatError(f"{path}: truncated payload at byte {_HDR.size + len(body)} "
                               f"(expected {want} payload bytes)")
    return PointSet(np.frombuffer(body, dtype="<f8").reshape(n, d).astype(np.float64))


def _read_csv(path):
    rows, width = [], None
    with open(path) as fh:
        for lineno, raw in enumerate(fh, start=1):
            line = raw.strip()
            if not line:
                continue
            cells = line.split(",")
            width = len(cells) if width is None else width
            if len(cells) != width:
                raise PointFormatError(f"{path}: line {lineno}: expected {width} columns, got {len(cells)}")
            vals = []
            for c in cells:
                try:
                    vals.append(float(c))
                except ValueError:
                    raise PointFormatError(f"{path}: line {lineno}: non-numeric cell {c.strip()!r}") from None
            rows.append(vals)
    if not rows:
        raise PointFormatError(f"{path}: no data rows")
    return PointSet(np.asarray(rows, dtype=np.float64))


def save_vector(values, path):
    save_points(PointSet(np.asarray(values, dtype=np.float64).reshape(-1, 1)), path)


def load_vector(path):
    ps = load_points(path)
    if ps.d != 1:
        raise PointFormatError(f"{path}: expected a d=1 vector file, got d={ps.d}")
    return np.array(ps.coords[:, 0])


def normalize_unit_box(ps):
    """Affine map of every coordinate onto [0, 1] (constant ones stay 0)."""
    lo = ps.coords.min(axis=0)
    span = ps.coords.max(axis=0) - lo
    span[span == 0.0] = 1.0
    return PointSet((ps.coords - lo) / span)
