"""Preconditioners of the drop-in API (mirror of pkg/src/kpl/precond.py).

Only identity and Jacobi run on the device (the `north_star` path).  The
reference's IC(0) (`make_ic0`, precond.py:134-154) is out of scope this
round; passing an IC(0) preconditioner to a solver raises
NotImplementedError rather than running anything on the CPU.

`apply` is the device operation m = M^-1 v used inside the fused sweeps; the
host-side `apply` here exists for API parity and computes on the device too.
"""

from __future__ import annotations

import numpy as np


class PreconditionerBreakdown(ArithmeticError):
    """precond.py:20-25 (raised by IC(0) in the reference)."""

    def __init__(self, row):
        self.row = row
        super().__init__(f"nonpositive pivot in IC(0) factorization at row {row}")


class Preconditioner:
    """`kind` in {"identity", "jacobi"}; Jacobi keeps `inv_diag = 1 / diag(A)`.

    For matrix-free stencils the diagonal is constant, so `inv_const` holds
    the single value fl(1/diag) and `inv_diag` is materialised only on access.
    """

    __slots__ = ("kind", "_inv_diag", "inv_const", "n_rows", "mu_tilde", "_device")

    def __init__(self, kind, inv_diag=None, inv_const=None, n=None):
        self.kind = kind
        self._inv_diag = None if inv_diag is None else np.ascontiguousarray(inv_diag, dtype=np.float64)
        self.inv_const = inv_const
        self.n_rows = n if n is not None else (None if inv_diag is None else len(inv_diag))
        self.mu_tilde = 1
        self._device = None

    @property
    def inv_diag(self):
        if self._inv_diag is None and self.inv_const is not None:
            self._inv_diag = np.full(self.n_rows, self.inv_const)
        return self._inv_diag

    @property
    def n(self):
        return self.n_rows

    def apply(self, v):
        """M^-1 v.  Identity returns v itself (precond.py:84-85)."""
        if self.kind == "identity":
            return v
        from .ops import _jacobi_apply
        return _jacobi_apply(self, v)

    def norm_estimate(self):
        if self.kind == "identity":
            return 1.0
        if self.inv_const is not None:
            return float(self.inv_const)
        return float(self.inv_diag.max())

    def __repr__(self):
        return f"Preconditioner(kind={self.kind!r}, n={self.n})"


def identity() -> Preconditioner:
    return Preconditioner("identity")


def make_jacobi(A) -> Preconditioner:
    """precond.py:124-131: inverse diagonal; requires a strictly positive diagonal."""
    if hasattr(A, "stencil_spec"):
        d = float(A.stencil_spec()[3])
        if d <= 0.0:
            raise ValueError("nonpositive diagonal entry at row 0")
        return Preconditioner("jacobi", inv_const=1.0 / d, n=A.n)
    d = A.diagonal()
    bad = np.nonzero(d <= 0.0)[0]
    if len(bad):
        raise ValueError(f"nonpositive diagonal entry at row {bad[0]}")
    return Preconditioner("jacobi", inv_diag=1.0 / d)


def make_ic0(A, eta: float = 0.0):
    raise NotImplementedError(
        "IC(0) is outside this build's device scope (SURVEY.md 8f-4); "
        "use identity() or make_jacobi()")
