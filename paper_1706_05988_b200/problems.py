"""Problem generators and matrix-free operators for the BASELINE.json configs.

The reference ships only `laplacian_2d` and `random_spd`
(`pkg/src/kpl/sparse.py:188-228`); the 3D, variable-coefficient and random
banded generators below follow SURVEY.md Appendix C, with the reference's
conventions (unscaled, Dirichlet truncation, id = x + NX*(y + NY*z), columns
ascending).  Right-hand sides follow `harness.build_rhs`
(`pkg/src/kpl/harness.py:84-88`).
"""

from __future__ import annotations

import numpy as np

from .sparse import SparseMatrix, _assemble_7pt


class _Stencil:
    """Matrix-free unscaled Dirichlet Laplacian on an (NX, NY, NZ) grid.

    Exposes the parts of `SparseMatrix` the solvers read (`n`, `mu`,
    `norm_inf`, `diagonal`) so it can be passed wherever a matrix is
    accepted.  Its action is the reference's `csr_matvec` on the assembled
    Laplacian, term order included.
    """

    diag_value = 0.0

    def __init__(self, NX, NY, NZ):
        if min(NX, NY, NZ) < 1:
            raise ValueError("grid dimensions must be >= 1")
        self.NX, self.NY, self.NZ = int(NX), int(NY), int(NZ)
        self.n = self.NX * self.NY * self.NZ
        self._device = None

    def stencil_spec(self):
        """Device geometry (NX, NY, NZ, diag); id = x + NX*(y + NY*z)."""
        return (self.NX, self.NY, self.NZ, float(self.diag_value))

    def slab_spec(self):
        """Geometry whose last axis is split into z-slabs by the multi-GPU
        solver: 3D grids as they are; a 2D grid as (nx, 1, ny), so its rows
        become the slab axis.  Same element order as stencil_spec."""
        return self.stencil_spec()

    @property
    def mu(self):
        k = 1
        for d in (self.NX, self.NY, self.NZ):
            k += 2 if d >= 3 else (1 if d == 2 else 0)
        return k

    def norm_inf(self):
        nb = 0
        for d in (self.NX, self.NY, self.NZ):
            nb += 2 if d >= 3 else (1 if d == 2 else 0)
        return float(self.diag_value + nb)

    def diagonal(self):
        return np.full(self.n, float(self.diag_value))

    def to_csr(self) -> SparseMatrix:
        return _assemble_7pt(self.NX, self.NY, self.NZ, None, self.diag_value)

    @property
    def nnz(self):
        n, (NX, NY, NZ) = self.n, (self.NX, self.NY, self.NZ)
        return n + 2 * ((NX - 1) * NY * NZ + NX * (NY - 1) * NZ + NX * NY * (NZ - 1))


class Stencil2D(_Stencil):
    """5-point Laplacian on nx-by-ny (the operator of `laplacian_2d(nx, ny)`).

    Runs on the device as the grid (nx, 1, ny): the sweep marches over the
    rows (the z axis of the 3D machinery) with 512-wide row tiles."""

    diag_value = 4.0

    def __init__(self, nx, ny):
        super().__init__(nx, 1, ny)
        self.nx, self.ny = int(nx), int(ny)

    def __repr__(self):
        return f"Stencil2D({self.nx}x{self.ny})"


class Stencil3D(_Stencil):
    """7-point Laplacian on nx-by-ny-by-nz (diag 6, -1 couplings)."""

    diag_value = 6.0

    def __repr__(self):
        return f"Stencil3D({self.NX}x{self.NY}x{self.NZ})"


def laplacian_3d(nx, ny, nz) -> SparseMatrix:
    """Assembled 7-point Laplacian (first bullet)."""
    return _assemble_7pt(nx, ny, nz, None, 6.0)


def varcoef_faces(N, seed=0, sigma_log=2.0):
    """Face coefficients k_f = exp(N(0, sigma_log^2)) drawn in the Appendix C
    order: kx (N, N, N+1) [iz, iy, x-face], then ky (N, N+1, N), then kz (N+1, N, N)."""
    rng = np.random.default_rng(seed)
    kx = np.exp(rng.normal(0.0, sigma_log, (N, N, N + 1)))
    ky = np.exp(rng.normal(0.0, sigma_log, (N, N + 1, N)))
    kz = np.exp(rng.normal(0.0, sigma_log, (N + 1, N, N)))
    return kx, ky, kz


def varcoef_3d(N, seed=0, sigma_log=2.0, check_symmetry=True) -> SparseMatrix:
    """Config 4: variable-coefficient 7-point diffusion on N^3 (Appendix C)."""
    return _assemble_7pt(N, N, N, varcoef_faces(N, seed, sigma_log), 0.0,
                         check_symmetry=check_symmetry)


def varcoef_3d_coo(N, seed=0, sigma_log=2.0):
    """COO triplets of `varcoef_3d` (used to check assembly against from_coo)."""
    A = varcoef_3d(N, seed, sigma_log, check_symmetry=False)
    rows = np.repeat(np.arange(A.n), np.diff(A.row_ptr))
    return A.n, rows, A.col_idx.copy(), A.values.copy()


def banded_spd_coo(n, seed=0, per_row=11, band=50_000):
    """Config 5 triplets (Appendix C): per row `per_row` off-diagonal columns at
    offsets uniform in [1, band] with a random sign, dropped outside [0, n),
    values uniform in [-1, 0), plus the mirrored entries.  The diagonal is
    added by `banded_spd` after duplicates are summed."""
    rng = np.random.default_rng(seed)
    rows = np.repeat(np.arange(n, dtype=np.int64), per_row)
    off = rng.integers(1, band + 1, size=rows.size) * rng.choice(np.array([-1, 1]), size=rows.size)
    vals = rng.uniform(-1.0, 0.0, size=rows.size)
    cols = rows + off
    keep = (cols >= 0) & (cols < n)
    rows, cols, vals = rows[keep], cols[keep], vals[keep]
    return (np.concatenate([rows, cols]), np.concatenate([cols, rows]),
            np.concatenate([vals, vals]))


def banded_spd(n, seed=0, per_row=11, band=50_000) -> SparseMatrix:
    """Config 5: random banded, structurally symmetric, strictly diagonally
    dominant SPD matrix; diag = sum |off-diagonal| + 1e-3 per row."""
    r, c, v = banded_spd_coo(n, seed, per_row, band)
    off = SparseMatrix.from_coo(n, r, c, v)
    rows = np.repeat(np.arange(n), np.diff(off.row_ptr))
    absum = np.zeros(n)
    np.add.at(absum, rows, np.abs(off.values))
    d = absum + 1e-3
    # insert the diagonal into each (sorted) row
    counts = np.diff(off.row_ptr) + 1
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    nnz = int(row_ptr[-1])
    col_idx = np.empty(nnz, dtype=np.int64)
    values = np.empty(nnz)
    below = np.zeros(n, dtype=np.int64)
    np.add.at(below, rows[off.col_idx < rows], 1)
    # position of the diagonal inside each new row
    dpos = row_ptr[:-1] + below
    is_diag = np.zeros(nnz, dtype=bool)
    is_diag[dpos] = True
    col_idx[dpos] = np.arange(n)
    values[dpos] = d
    col_idx[~is_diag] = off.col_idx
    values[~is_diag] = off.values
    return SparseMatrix(n, row_ptr, col_idx, values)


def build_rhs(A, rhs_mode="ones_solution"):
    """harness.py:84-88: `ones_rhs` -> b_j = 1/sqrt(n); `ones_solution` -> b = A xhat
    with xhat_j = 1/sqrt(n).  The product runs on the device (same term order
    as the reference's csr_matvec)."""
    entries = np.full(A.n, 1.0 / np.sqrt(A.n))
    if rhs_mode == "ones_rhs":
        return entries
    if rhs_mode != "ones_solution":
        raise ValueError(f"unknown rhs_mode {rhs_mode!r}")
    from .ops import spmv
    return spmv(A, entries)
