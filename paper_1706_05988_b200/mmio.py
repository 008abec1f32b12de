"""Matrix Market coordinate I/O, byte-compatible with `kpl.mmio`.

Reader: `%%MatrixMarket matrix coordinate real|integer symmetric|general`,
one-based indices, the stored triangle of symmetric files mirrored, gzip
detected from the magic bytes, duplicates summed through
`SparseMatrix.from_coo` (which also validates symmetry).  Writer: the lower
triangle in row order, `%.17g` values, so write -> read round-trips bitwise
and files match the reference's `write_matrix_market` byte for byte.
"""

from __future__ import annotations

import gzip
import io
import os

import numpy as np

from .sparse import SparseMatrix


class MatrixMarketError(ValueError):
    """Malformed or unsupported Matrix Market content."""


def _text(source) -> list:
    if isinstance(source, (str, os.PathLike)):
        with open(source, "rb") as fh:
            data = fh.read()
    elif isinstance(source, (bytes, bytearray)):
        data = bytes(source)
    else:
        data = source.read()
    if data[:2] == b"\x1f\x8b":
        data = gzip.decompress(data)
    return data.decode("ascii", errors="replace").splitlines()


def read_matrix_market(source) -> SparseMatrix:
    lines = _text(source)
    if not lines:
        raise MatrixMarketError("empty input")
    head = lines[0].split()
    if len(head) != 5 or head[0] != "%%MatrixMarket":
        raise MatrixMarketError(f"malformed header: {lines[0].strip()!r}")
    obj, fmt, fld, sym = (h.lower() for h in head[1:])
    if obj != "matrix" or fmt != "coordinate":
        raise MatrixMarketError(f"unsupported object/format: {obj} {fmt}")
    if fld not in ("real", "integer"):
        raise MatrixMarketError(f"unsupported field (need real values): {fld}")
    if sym not in ("symmetric", "general"):
        raise MatrixMarketError(f"unsupported symmetry: {sym}")
    body = (ln for ln in lines[1:] if ln.strip() and not ln.startswith("%"))
    size_line = next(body, None)
    if size_line is None or len(size_line.split()) != 3:
        raise MatrixMarketError(f"malformed size line: {size_line!r}")
    nr, nc, nnz = (int(t) for t in size_line.split())
    if nr != nc:
        raise MatrixMarketError(f"matrix is not square: {nr} x {nc}")
    entries = [ln.split() for ln in body]
    if len(entries) != nnz:
        raise MatrixMarketError(f"expected {nnz} entries, found {len(entries)}")
    if any(len(e) != 3 for e in entries):
        raise MatrixMarketError("malformed entry line")
    rows = np.array([int(e[0]) - 1 for e in entries], dtype=np.int64)
    cols = np.array([int(e[1]) - 1 for e in entries], dtype=np.int64)
    vals = np.array([float(e[2]) for e in entries], dtype=np.float64)
    if nnz and (rows.min() < 0 or cols.min() < 0 or rows.max() >= nr or cols.max() >= nc):
        raise MatrixMarketError("index out of range")
    if sym == "symmetric":
        off = rows != cols
        rows, cols, vals = (np.concatenate([rows, cols[off]]), np.concatenate([cols, rows[off]]),
                            np.concatenate([vals, vals[off]]))
    try:
        return SparseMatrix.from_coo(nr, rows, cols, vals)
    except ValueError as exc:
        raise MatrixMarketError(str(exc)) from exc


def write_matrix_market(A, sink) -> None:
    """Lower triangle, coordinate real symmetric, `%.17g` values."""
    rows = np.repeat(np.arange(A.n), np.diff(A.row_ptr))
    low = A.col_idx <= rows
    r, c, v = rows[low] + 1, np.asarray(A.col_idx)[low] + 1, np.asarray(A.values)[low]
    out = io.StringIO()
    out.write("%%MatrixMarket matrix coordinate real symmetric\n")
    out.write(f"{A.n} {A.n} {len(v)}\n")
    for i, j, x in zip(r.tolist(), c.tolist(), v.tolist()):
        out.write("%d %d %.17g\n" % (i, j, x))
    data = out.getvalue().encode("ascii")
    if isinstance(sink, (str, os.PathLike)):
        with open(sink, "wb") as fh:
            fh.write(data)
    else:
        sink.write(data)
