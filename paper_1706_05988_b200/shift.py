"""Shift selection for p-CG-sh: the reference's a-posteriori rule.

Host-side analysis of a solver's (alpha, beta) history -- O(i) 4x4 products
per grid point, exactly as the reference does it -- plus the workflow of
`pkg/scripts/shift_study.py:18-64` with the solves on the device:

  1. baseline p-CG solve (device) -> coefficient history
  2. `default_sigma_grid(A, M)`                    stability.py:207-232
  3. psi_i(sigma) on the grid (`select_shift`)     stability.py:157-204
  4. margin rule: smallest sigma with psi <= 4 * min psi   shift_study.py:46-51

Every function restates the reference's arithmetic with the same numpy
calls (4x4 `@`, cyclic Jacobi rotations), so psi values are bit-identical
to the reference's on the same history (tests/test_shift.py pins this
against fixtures produced by the unmodified reference).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class CoefficientHistory:
    """alpha_k, beta_k for k = 1 .. len (stability.py:26-55)."""

    alphas: np.ndarray
    betas: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "alphas", np.asarray(self.alphas, dtype=np.float64))
        object.__setattr__(self, "betas", np.asarray(self.betas, dtype=np.float64))
        if self.alphas.shape != self.betas.shape or self.alphas.ndim != 1:
            raise ValueError("alphas and betas must be 1-D and equally long")
        if not (np.all(np.isfinite(self.alphas)) and np.all(np.isfinite(self.betas))):
            raise ValueError("coefficients must be finite")

    def __len__(self):
        return len(self.alphas)

    @classmethod
    def from_result(cls, result):
        recs = [rec for rec in result.history if rec.iter >= 1]
        return cls(np.array([rec.alpha for rec in recs]), np.array([rec.beta for rec in recs]))


def propagation_matrix(alpha: float, beta: float, sigma: float) -> np.ndarray:
    """stability.py:58-71: one-iteration propagation of the gap stack (f, g, h, j)."""
    ab = alpha * beta
    return np.array([
        [1.0, -ab, -alpha, 0.0],
        [0.0, beta, 1.0, 0.0],
        [0.0, -ab * sigma, 1.0 - alpha * sigma, -ab],
        [0.0, 0.0, 0.0, beta],
    ])


def _jacobi_max_eigenvalue(S: np.ndarray, tol: float) -> float:
    """stability.py:104-137: largest eigenvalue of a symmetric 4x4, cyclic Jacobi."""
    a = S.copy()
    n = a.shape[0]
    for _ in range(60):
        off = 0.0
        total = 0.0
        for p in range(n):
            for q in range(n):
                total += a[p, q] * a[p, q]
                if p != q:
                    off += a[p, q] * a[p, q]
        if off <= tol * tol * total or total == 0.0:
            break
        for p in range(n - 1):
            for q in range(p + 1, n):
                apq = a[p, q]
                if apq == 0.0:
                    continue
                tau = (a[q, q] - a[p, p]) / (2.0 * apq)
                if abs(tau) > 1e150:
                    t = 1.0 / (2.0 * tau)
                else:
                    t = np.sign(tau) / (abs(tau) + np.hypot(1.0, tau))
                    if tau == 0.0:
                        t = 1.0
                c = 1.0 / np.hypot(1.0, t)
                s = t * c
                rot = np.eye(n)
                rot[p, p] = rot[q, q] = c
                rot[p, q] = s
                rot[q, p] = -s
                a = rot.T @ a @ rot
    return float(np.max(np.diag(a)))


def matrix_2norm(P: np.ndarray, tol: float = 1e-14) -> float:
    """stability.py:140-154: largest singular value; +inf once entries overflow."""
    P = np.asarray(P, dtype=np.float64)
    if not np.all(np.isfinite(P)):
        return float("inf")
    with np.errstate(over="ignore"):
        S = P.T @ P
    if not np.all(np.isfinite(S)):
        return float("inf")
    lam = _jacobi_max_eigenvalue(S, tol)
    return float(np.sqrt(lam)) if lam > 0.0 else 0.0


def amplification_factor(hist: CoefficientHistory, i: int, shift: float) -> float:
    """stability.py:157-176: worst 2-norm over all window products ending at i."""
    if not 1 <= i <= len(hist):
        raise IndexError(f"iteration index i={i} outside history of length {len(hist)}")
    prod = None
    best = 0.0
    with np.errstate(over="ignore", invalid="ignore"):
        for j in range(i, 0, -1):
            pj = propagation_matrix(hist.alphas[j - 1], hist.betas[j - 1], shift)
            prod = pj if prod is None else prod @ pj
            nrm = matrix_2norm(prod)
            if nrm > best:
                best = nrm
            if np.isinf(best):
                break
    return best


@dataclass(frozen=True)
class ShiftSweep:
    grid: np.ndarray
    psi_values: np.ndarray
    argmin: float
    iter: int


def select_shift(hist: CoefficientHistory, i: int, grid) -> ShiftSweep:
    """stability.py:189-204: psi on the grid, ties toward the smaller shift."""
    grid = np.asarray(grid, dtype=np.float64)
    if grid.size == 0:
        raise ValueError("shift grid must be nonempty")
    values = np.array([amplification_factor(hist, i, s) for s in grid])
    best = 0
    for k in range(1, len(grid)):
        if values[k] < values[best] or (values[k] == values[best] and grid[k] < grid[best]):
            best = k
    return ShiftSweep(grid, values, float(grid[best]), i)


def default_sigma_grid(A, M=None, npoints: int = 81) -> np.ndarray:
    """stability.py:207-232: 0, log-spaced 1e-2..1, linear 1..2*Gershgorin bound
    (Jacobi-scaled when M is Jacobi)."""
    if hasattr(A, "stencil_spec"):
        sums = None
        rowmax = float(A.norm_inf())
        if M is not None and getattr(M, "kind", None) == "jacobi":
            inv = getattr(M, "inv_const", None)
            inv = float(inv) if inv is not None else float(np.asarray(M.inv_diag)[0])
            hi = 2.0 * (rowmax * inv)
        else:
            hi = 2.0 * rowmax
    else:
        counts = np.diff(A.row_ptr)
        rows = np.repeat(np.arange(A.n), counts)
        sums = np.zeros(A.n)
        np.add.at(sums, rows, np.abs(A.values))
        if M is not None and getattr(M, "kind", None) == "jacobi":
            hi = 2.0 * float((sums * M.inv_diag).max())
        else:
            hi = 2.0 * float(sums.max())
    if hi <= 1.0:
        body = np.geomspace(hi / 1000.0, hi, npoints - 1)
    else:
        n_log = (npoints - 1) // 3
        n_lin = npoints - 1 - n_log
        body = np.concatenate([np.geomspace(1e-2, 1.0, n_log, endpoint=False),
                               np.linspace(1.0, hi, n_lin)])
    return np.concatenate([[0.0], body])


def margin_rule(sweep: ShiftSweep, factor: float = 4.0) -> float:
    """shift_study.py:46-51: smallest grid shift with psi <= factor * min psi."""
    floor = factor * sweep.psi_values.min()
    return float(sweep.grid[np.argmax(sweep.psi_values <= floor)])


def choose_shift(A, M, b, *, max_iters, rtol=0.0, i=None, grid=None, solve=None):
    """The reference's selection workflow (shift_study.py:18-64) with the
    baseline p-CG solve on the device.  Returns (sigma, sweep, baseline)."""
    if solve is None:
        from .solvers import SolverConfig, solve as dev_solve
        base = dev_solve(A, M, b, None, SolverConfig(method="pcg", max_iters=max_iters, rtol=rtol))
    else:
        base = solve(A, M, b)
    hist = CoefficientHistory.from_result(base)
    it = i if i is not None else base.iterations
    g = default_sigma_grid(A, M) if grid is None else np.asarray(grid, dtype=np.float64)
    sw = select_shift(hist, it, g)
    return margin_rule(sw), sw, base
