"""Preconditioners of the drop-in API (mirror of pkg/src/kpl/precond.py).

identity, Jacobi and IC(0) all run on the device:

* Jacobi: m = v * inv_diag inside the fused sweeps (a constant for stencils);
* IC(0) (`make_ic0`, precond.py:134-154): the factor is computed on the device
  by a sync-free row sweep (kpl_ic0_factor, _kernels.py:77-115), and every
  apply is the forward + backward substitution pair (kpl_ic0 sweeps,
  _kernels.py:55-74) -- bit-identical to the reference.  Host work is index
  bookkeeping only: the lower pattern, its transpose permutation, mu_tilde.

`apply` is the device operation m = M^-1 v (kpl_precond_apply); inside the
solvers the same kernels run between the fused sweeps.
"""

from __future__ import annotations

import os

import numpy as np


class PreconditionerBreakdown(ArithmeticError):
    """precond.py:20-25 (raised by IC(0) in the reference)."""

    def __init__(self, row):
        self.row = row
        super().__init__(f"nonpositive pivot in IC(0) factorization at row {row}")


class Preconditioner:
    """`kind` in {"identity", "jacobi", "ic0"}; Jacobi keeps `inv_diag = 1 / diag(A)`.

    For matrix-free stencils the diagonal is constant, so `inv_const` holds
    the single value fl(1/diag) and `inv_diag` is materialised only on access.
    IC(0) keeps its factor on the device (`ic`, an `Ic0Factor`).
    """

    __slots__ = ("kind", "_inv_diag", "inv_const", "n_rows", "mu_tilde", "_device", "ic",
                 "_norm_estimate", "__weakref__")

    def __init__(self, kind, inv_diag=None, inv_const=None, n=None, ic=None, mu_tilde=1):
        self.kind = kind
        self._inv_diag = None if inv_diag is None else np.ascontiguousarray(inv_diag, dtype=np.float64)
        self.inv_const = inv_const
        self.n_rows = n if n is not None else (None if inv_diag is None else len(inv_diag))
        self.mu_tilde = mu_tilde
        self._device = None
        self.ic = ic
        self._norm_estimate = None

    @property
    def inv_diag(self):
        if self._inv_diag is None and self.inv_const is not None:
            self._inv_diag = np.full(self.n_rows, self.inv_const)
        return self._inv_diag

    @property
    def n(self):
        return self.n_rows

    @property
    def _l(self):
        """Host (row_ptr, col_idx, l_values) of the IC(0) factor (the
        reference's `Preconditioner._l`)."""
        return None if self.ic is None else self.ic.host_lower()

    def host_lower(self):
        return self._l

    def apply(self, v):
        """M^-1 v on the device.  Identity returns v itself (precond.py:84-85)."""
        if self.kind == "identity":
            return v
        from .ops import precond_apply
        return precond_apply(self, v)

    def norm_estimate(self):
        """precond.py:96-118: 1 (identity), max(inv_diag) (Jacobi), or 20
        power-iteration steps on the applied operator (IC(0), device ops)."""
        if self.kind == "identity":
            return 1.0
        if self.kind == "jacobi":
            if self.inv_const is not None:
                return float(self.inv_const)
            return float(self.inv_diag.max())
        if self._norm_estimate is None:
            from .ops import dot, norm2
            v = np.full(self.n, 1.0 / np.sqrt(self.n))
            lam = 1.0
            for _ in range(20):
                w = self.apply(v)
                lam = dot(v, w)
                nw = norm2(w)
                if nw == 0.0:
                    break
                v = w / nw
            self._norm_estimate = abs(float(lam))
        return self._norm_estimate

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


class Ic0Factor:
    """Device-resident IC(0) factor: L (lower CSR, diagonal last) and
    U = L^T (diagonal first), int32 indices, fp64 values."""

    def __init__(self, n, l_ptr, l_col, l_val, u_ptr, u_col, u_val, host_ptr, host_col,
                 l_order=None, u_order=None):
        self.n = n
        self.l_ptr, self.l_col, self.l_val = l_ptr, l_col, l_val
        self.u_ptr, self.u_col, self.u_val = u_ptr, u_col, u_val
        self.l_order, self.u_order = l_order, u_order
        self._host = (host_ptr, host_col)

    def host_lower(self):
        ptr, col = self._host
        return ptr, col, self.l_val.cpu().numpy()


def ic0_from_host(lower, upper, device):
    """Upload a host IC(0) factor as the reference stores it (precond.py:64-70):
    `lower` = (row_ptr, col_idx, values) of L, diagonal last per row; `upper` =
    its transpose from _transpose_csr (precond.py:46-53), diagonal first.  No
    arithmetic: the factor values are the reference's own."""
    from . import device as D
    t = D.torch()
    ptr, cols, lval = (np.asarray(a) for a in lower)
    tptr, tcols, uval = (np.asarray(a) for a in upper)
    n = len(ptr) - 1
    if len(cols) >= 2**31:
        raise ValueError("factor too large for int32 indices")
    i32 = lambda a: t.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(device)
    f64 = lambda a: t.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(device)
    return Ic0Factor(n, i32(ptr), i32(cols), f64(lval), i32(tptr), i32(tcols), f64(uval),
                     np.asarray(ptr, dtype=np.int64), np.asarray(cols, dtype=np.int64))


def _lower_pattern(A):
    """precond.py:28-43 index part: the lower triangle's row pointer, columns
    and the positions of its entries in A.values (diagonal last per row)."""
    n = A.n
    row_ptr = np.asarray(A.row_ptr, dtype=np.int64)
    col_idx = np.asarray(A.col_idx, dtype=np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(row_ptr))
    keep = np.flatnonzero(col_idx <= rows)
    ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows[keep], minlength=n), out=ptr[1:])
    cols = col_idx[keep]
    last = ptr[1:] - 1
    if np.any(ptr[1:] == ptr[:-1]) or np.any(cols[last] != np.arange(n)):
        raise ValueError("matrix has a structurally missing diagonal entry")
    return ptr, cols, keep


def _transpose_perm(n, ptr, cols):
    """precond.py:46-53 index part: CSR pattern of the transpose and the
    permutation taking the factor's values to it (rows of a column ascending)."""
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(ptr))
    perm = np.lexsort((rows, cols))
    tptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(cols, minlength=n), out=tptr[1:])
    return tptr, rows[perm], perm


def make_ic0(A, eta: float = 0.0) -> Preconditioner:
    """precond.py:134-154: IC(0) of A + eta*diag(diag(A)) on the pattern of
    lower(A), factored on the device.  Raises PreconditionerBreakdown(row)
    for the first non-positive pivot."""
    if eta < 0.0:
        raise ValueError("compensation shift eta must be >= 0")
    from . import _lib
    from . import device as D
    if hasattr(A, "stencil_spec"):
        A = A.to_csr()
    ptr, cols, keep = _lower_pattern(A)
    n, nnz = A.n, len(cols)
    if nnz >= 2**31:
        raise ValueError("factor too large for int32 indices")
    dev = D.require_cuda()
    t = D.torch()
    i32 = lambda a: t.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(dev)
    l_ptr, l_col = i32(ptr), i32(cols)
    a_val = t.from_numpy(np.ascontiguousarray(np.asarray(A.values)[keep], dtype=np.float64)).to(dev)
    l_val = t.empty(nnz, dtype=t.float64, device=dev)
    lib = _lib.load()
    scratch = t.empty(int(lib.kpl_ic0_scratch_bytes(n)), dtype=t.uint8, device=dev)
    level = t.empty(n, dtype=t.int32, device=dev)

    # natural row order by default: its i-1 neighbours sit in the same warp and
    # the rows of a CTA are contiguous (measured faster than level order on
    # 2D/3D Laplacians); KPL_IC0_ORDER=level sorts rows by dependency level
    natural = os.environ.get("KPL_IC0_ORDER", "natural") != "level"

    def order_of(rp, ci, upper):
        # rows sorted by dependency level: the sweeps' topological processing order
        if natural:
            return None
        _lib.check(lib.kpl_ic0_levels(n, D.ptr(rp), D.ptr(ci), upper, D.ptr(level), D.ptr(scratch),
                                      D.stream_handle()), "IC(0) levels")
        return i32(np.argsort(level.cpu().numpy(), kind="stable"))

    l_order = order_of(l_ptr, l_col, 0)
    bad = _lib._i64(-1)
    import ctypes
    _lib.check(lib.kpl_ic0_factor(n, D.ptr(l_ptr), D.ptr(l_col), D.ptr(l_order), D.ptr(a_val), 1.0 + eta,
                                  D.ptr(l_val), D.ptr(scratch), ctypes.byref(bad), D.stream_handle()),
               "IC(0) factor")
    if bad.value >= 0:
        raise PreconditionerBreakdown(int(bad.value))
    tptr, trows, perm = _transpose_perm(n, ptr, cols)
    u_val = t.empty(nnz, dtype=t.float64, device=dev)
    perm_d = i32(perm)
    _lib.check(lib.kpl_gather(nnz, D.ptr(perm_d), D.ptr(l_val), D.ptr(u_val), D.stream_handle()),
               "IC(0) transpose")
    u_ptr, u_col = i32(tptr), i32(trows)
    u_order = order_of(u_ptr, u_col, 1)
    counts = np.diff(ptr)
    mu_tilde = int((counts + np.bincount(cols, minlength=n) - 1).max())
    ic = Ic0Factor(n, l_ptr, l_col, l_val, u_ptr, u_col, u_val, ptr, cols, l_order, u_order)
    return Preconditioner("ic0", n=n, ic=ic, mu_tilde=mu_tilde)
