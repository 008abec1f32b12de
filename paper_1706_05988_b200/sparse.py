"""Host-side sparse types and generators of the drop-in API.

Mirrors the reference's `kpl.sparse` surface (`pkg/src/kpl/sparse.py`) so a
caller can switch imports: `SparseMatrix` (CSR with sorted columns, validated
symmetric on construction, `mu`, `norm_inf`, `diagonal`, `from_coo`,
`from_dense`, `to_dense`), `laplacian_2d`, `random_spd`.  Host arrays stay
numpy (int64 indices, as the reference stores them); the device copy is the
int32 CSR built lazily by `paper_1706_05988_b200.device` on first use.

Matrix-free operators (`Stencil2D`, `Stencil3D`) describe the same unscaled
Dirichlet Laplacians without storing them; the solver runs them through the
fused stencil kernel.  Their action equals `csr_matvec` on the assembled
matrix bit for bit ("Stencil operator").

No arithmetic of the solve happens here: `spmv`, `dot`, `axpy` of the
reference's level-1/2 API are provided by `paper_1706_05988_b200.ops` on the
device.
"""

from __future__ import annotations

import numpy as np

SYMMETRY_RTOL = 1e-14                      # sparse.py:22


class SparseMatrix:
    """Symmetric CSR matrix; same constructor contract as sparse.py:25-88."""

    __slots__ = ("n", "row_ptr", "col_idx", "values", "mu", "_device")

    def __init__(self, n, row_ptr, col_idx, values, *, check_symmetry=True):
        n = int(n)
        row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
        col_idx = np.ascontiguousarray(col_idx, dtype=np.int64)
        values = np.ascontiguousarray(values, dtype=np.float64)
        if n < 1:
            raise ValueError("matrix dimension must be >= 1")
        if row_ptr.shape != (n + 1,):
            raise ValueError("row_ptr must have n + 1 entries")
        if row_ptr[0] != 0 or row_ptr[-1] != len(values) or len(col_idx) != len(values):
            raise ValueError("row_ptr endpoints inconsistent with value count")
        counts = np.diff(row_ptr)
        if np.any(counts < 0):
            raise ValueError("row_ptr must be non-decreasing")
        if len(col_idx) and (col_idx.min() < 0 or col_idx.max() >= n):
            raise ValueError("column index out of range")
        rows = np.repeat(np.arange(n, dtype=np.int64), counts)
        if len(col_idx) > 1:
            same_row = rows[1:] == rows[:-1]
            if np.any(same_row & (col_idx[1:] <= col_idx[:-1])):
                raise ValueError("column indices must be strictly increasing within rows")
        self.n = n
        self.row_ptr = row_ptr
        self.col_idx = col_idx
        self.values = values
        self.mu = int(counts.max()) if n else 0
        self._device = None
        if check_symmetry:
            self._check_symmetry(rows)

    def _check_symmetry(self, rows):
        """sparse.py:74-87."""
        order = np.lexsort((rows, self.col_idx))
        if not (np.array_equal(self.col_idx[order], rows)
                and np.array_equal(rows[order], self.col_idx)):
            raise ValueError("sparsity pattern is not symmetric")
        mirrored = self.values[order]
        tol = SYMMETRY_RTOL * np.maximum(np.abs(self.values), 1.0)
        bad = np.abs(self.values - mirrored) > tol
        if np.any(bad):
            k = int(np.nonzero(bad)[0][0])
            raise ValueError(
                f"matrix is not numerically symmetric at entry ({rows[k]}, {self.col_idx[k]})")

    @classmethod
    def from_coo(cls, n, rows, cols, vals):
        """sparse.py:89-110: duplicates summed after a stable (row, col) sort."""
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        vals = np.asarray(vals, dtype=np.float64)
        if len(rows) and (rows.min() < 0 or rows.max() >= n or cols.min() < 0 or cols.max() >= n):
            raise ValueError("coordinate index out of range")
        order = np.lexsort((cols, rows))
        rows, cols, vals = rows[order], cols[order], vals[order]
        if len(rows):
            keep = np.empty(len(rows), dtype=bool)
            keep[0] = True
            keep[1:] = (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])
            group = np.cumsum(keep) - 1
            summed = np.zeros(int(group[-1]) + 1)
            np.add.at(summed, group, vals)
            rows, cols, vals = rows[keep], cols[keep], summed
        row_ptr = np.zeros(n + 1, dtype=np.int64)
        np.add.at(row_ptr, rows + 1, 1)
        np.cumsum(row_ptr, out=row_ptr)
        return cls(n, row_ptr, cols, vals)

    @classmethod
    def from_dense(cls, a, drop_tol=0.0):
        """sparse.py:112-120."""
        a = np.asarray(a, dtype=np.float64)
        n = a.shape[0]
        if a.shape != (n, n):
            raise ValueError("dense input must be square")
        rows, cols = np.nonzero(np.abs(a) > drop_tol)
        return cls.from_coo(n, rows, cols, a[rows, cols])

    def to_dense(self):
        out = np.zeros((self.n, self.n))
        rows = np.repeat(np.arange(self.n), np.diff(self.row_ptr))
        out[rows, self.col_idx] = self.values
        return out

    def diagonal(self):
        """sparse.py:129-136 (vectorised; columns are sorted and unique)."""
        rows = np.repeat(np.arange(self.n), np.diff(self.row_ptr))
        d = np.zeros(self.n)
        on = self.col_idx == rows
        d[rows[on]] = self.values[on]
        return d

    def norm_inf(self):
        """sparse.py:138-143 (max absolute row sum).  np.bincount adds the
        weights in input order per bin, i.e. the same sequence of additions as
        the reference's np.add.at, so the value is bitwise identical."""
        counts = np.diff(self.row_ptr)
        sums = np.bincount(np.repeat(np.arange(self.n), counts), weights=np.abs(self.values),
                           minlength=self.n)
        return float(sums.max())

    @property
    def nnz(self):
        return len(self.values)

    def __repr__(self):
        return f"SparseMatrix(n={self.n}, nnz={self.nnz}, mu={self.mu})"


def laplacian_2d(nx: int, ny: int) -> SparseMatrix:
    """sparse.py:188-214: unscaled 5-point Dirichlet Laplacian, id = ix + nx*iy."""
    if nx < 1 or ny < 1:
        raise ValueError("grid dimensions must be >= 1")
    return _assemble_laplacian(nx, 1, ny, 4.0)


def random_spd(n: int, cond: float = 100.0, seed: int = 0) -> SparseMatrix:
    """sparse.py:217-228: dense QR construction, log-spaced spectrum, stored as CSR."""
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.normal(size=(n, n)))
    lam = np.logspace(0.0, np.log10(cond), n) if n > 1 else np.ones(1)
    a = (q * lam) @ q.T
    a = (a + a.T) / 2.0
    return SparseMatrix.from_dense(a)


def _assemble_laplacian(NX, NY, NZ, diag, check_symmetry=True):
    """CSR of the unscaled Dirichlet Laplacian on (NX, NY, NZ), rows in id order,
    columns ascending (z-1, y-1, x-1, id, x+1, y+1, z+1).  Built directly in
    sorted order (no COO sort), so 256^3-class grids assemble in seconds; the
    result equals `SparseMatrix.from_coo` of the same triplets (tested)."""
    return _assemble_7pt(NX, NY, NZ, None, diag, check_symmetry)


def _assemble_7pt(NX, NY, NZ, face, diag_const, check_symmetry=True):
    """Shared 7-point CSR assembly.  `face` is None (constant -1 couplings and
    diagonal `diag_const`) or a tuple (kx, ky, kz) of face-coefficient arrays
    with shapes (NZ, NY, NX+1), (NZ, NY+1, NX), (NZ+1, NY, NX)."""
    n = NX * NY * NZ
    z, y, x = np.meshgrid(np.arange(NZ), np.arange(NY), np.arange(NX), indexing="ij")
    x = x.ravel()
    y = y.ravel()
    z = z.ravel()
    ids = np.arange(n, dtype=np.int64)
    sxy = NX * NY
    # (present mask, column offset, value) in ascending column order
    if face is None:
        ones = None
        offs = [(z > 0, -sxy), (y > 0, -NX), (x > 0, -1), (None, 0),
                (x < NX - 1, 1), (y < NY - 1, NX), (z < NZ - 1, sxy)]
        vals_of = lambda k, m: np.full(int(m.sum()) if m is not None else n, -1.0)
        dvals = np.full(n, float(diag_const))
    else:
        kx, ky, kz = face
        kxf = kx.reshape(NZ, NY, NX + 1)
        kyf = ky.reshape(NZ, NY + 1, NX)
        kzf = kz.reshape(NZ + 1, NY, NX)
        left = kxf[:, :, :-1].ravel()
        right = kxf[:, :, 1:].ravel()
        down = kyf[:, :-1, :].ravel()
        up = kyf[:, 1:, :].ravel()
        back = kzf[:-1].ravel()
        front = kzf[1:].ravel()
        # diag_i = kx[..,ix] + kx[..,ix+1] + ky[.,iy,.] + ky[.,iy+1,.] + kz[iz] + kz[iz+1]
        dvals = left + right + down + up + back + front
        coup = {-sxy: back, -NX: down, -1: left, 1: right, NX: up, sxy: front}
        offs = [(z > 0, -sxy), (y > 0, -NX), (x > 0, -1), (None, 0),
                (x < NX - 1, 1), (y < NY - 1, NX), (z < NZ - 1, sxy)]
        vals_of = lambda k, m: -coup[k][m]
    counts = np.ones(n, dtype=np.int64)
    for m, k in offs:
        if m is not None:
            counts += m
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    nnz = int(row_ptr[-1])
    col_idx = np.empty(nnz, dtype=np.int64)
    values = np.empty(nnz, dtype=np.float64)
    pos = row_ptr[:-1].copy()
    for m, k in offs:
        if m is None:
            col_idx[pos] = ids
            values[pos] = dvals
            pos += 1
        else:
            sel = pos[m]
            col_idx[sel] = ids[m] + k
            values[sel] = vals_of(k, m)
            pos += m
    return SparseMatrix(n, row_ptr, col_idx, values, check_symmetry=check_symmetry)
