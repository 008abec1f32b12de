"""CPU oracle: a numpy/C restatement of the reference `kpl` solvers.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package
(`paper_1706_05988_b200`) imports this module; only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s CPU legs (`cpu_baseline`,
`--impl reference`) use it, and only as the checker / the timed CPU baseline.

What it restates (file:line into the read-only reference `pkg/src/kpl/`):

* `blocked_dot`      -> `_kernels.py:15-41`   (C, oracle/csrc/oracle_kernels.c)
* `csr_matvec`       -> `_kernels.py:44-52`   (C)
* `axpy`             -> `sparse.py:172-180`   (alpha == 0 -> exact copy)
* `norm2`            -> `sparse.py:183-185`
* `_sub2`            -> `solvers.py:170-178`
* `_pipelined_scalars` -> `solvers.py:194-230`
* `_rnorm_true_wanted` -> `solvers.py:233-234`
* `gap_vectors` / `measure_gaps` -> `solvers.py:142-167`
* `solve_cg`         -> `solvers.py:237-294`
* `solve_pcg`        -> `solvers.py:297-357`
* `solve_pcg_shifted` -> `solvers.py:360-422`
* `solve_pcg_var_shifted` -> `solvers.py:425-498`
* `_ReplacementTrigger` / `solve_pcg_rr` -> `solvers.py:501-608`
* Jacobi apply       -> `precond.py:82-94` (`v * inv_diag`; identity returns v)
* IC(0)              -> `precond.py:28-53, :134-154`, `_kernels.py:55-115` (C: lower/upper
                        solves and the factor)
* `laplacian_2d`     -> `sparse.py:188-214`; `random_spd` -> `sparse.py:217-228`
* `from_coo`         -> `sparse.py:89-110`

Pinning: tests/test_oracle_golden.py checks every function here bit for bit
against fixtures produced by running the unmodified reference in the build
container (tests/golden/make_golden.py, committed with its outputs).

Two hooks make the oracle a checker for the GPU path:

* `dot=` replaces the reduction order (default: the reference's 8-lane
  blocked order).  `oracle.gpu_order` supplies the GPU's deterministic tree
  order so GPU histories can be compared bit for bit.
* operators may be CSR triplets or a `StencilSpec` (matrix-free Laplacian in
  the reference's CSR summation order, bitwise equal to `csr_matvec`).
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field

import numpy as np

UNIT_ROUNDOFF = float(np.finfo(np.float64).eps) / 2.0          # solvers.py:42
DEFAULT_RR_THRESHOLD = math.sqrt(UNIT_ROUNDOFF)                 # solvers.py:46

# history columns: iter, alpha, beta, gamma, delta, rnorm_recursive,
# rnorm_true, gap_f, gap_g, gap_h, gap_j  (None -> NaN)
NCOL = 11

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")
_lib = None


def _clib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            from . import build as _b
            _b.build()
        lib = ctypes.CDLL(_LIB_PATH)
        d = ctypes.c_double
        i64 = ctypes.c_int64
        p = ctypes.c_void_p
        lib.orc_blocked_dot.restype = d
        lib.orc_blocked_dot.argtypes = [i64, p, p]
        lib.orc_csr_matvec.restype = None
        lib.orc_csr_matvec.argtypes = [i64, p, p, p, p, p]
        lib.orc_stencil_matvec.restype = None
        lib.orc_stencil_matvec.argtypes = [i64, i64, i64, d, p, p]
        for name in ("orc_lower_solve", "orc_upper_solve"):
            getattr(lib, name).restype = None
            getattr(lib, name).argtypes = [i64, p, p, p, p, p]
        lib.orc_ic0_factor.restype = i64
        lib.orc_ic0_factor.argtypes = [i64, p, p, p, p]
        _lib = lib
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


class BreakdownError(ArithmeticError):
    """solvers.py:51-57."""

    def __init__(self, iteration, what):
        self.iteration = iteration
        self.what = what
        super().__init__(f"breakdown at iteration {iteration}: {what}")


# --------------------------------------------------------------------------
# operators
# --------------------------------------------------------------------------

@dataclass
class CSR:
    """Plain CSR triplet (int64 indices like sparse.py:48-50)."""
    n: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        self.row_ptr = np.ascontiguousarray(self.row_ptr, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(self.col_idx, dtype=np.int64)
        self.values = np.ascontiguousarray(self.values, dtype=np.float64)

    @property
    def mu(self):
        return int(np.diff(self.row_ptr).max())

    def norm_inf(self):
        """sparse.py:138-143."""
        counts = np.diff(self.row_ptr)
        sums = np.zeros(self.n)
        np.add.at(sums, np.repeat(np.arange(self.n), counts), np.abs(self.values))
        return float(sums.max())

    def diagonal(self):
        rows = np.repeat(np.arange(self.n), np.diff(self.row_ptr))
        d = np.zeros(self.n)
        on = self.col_idx == rows
        d[rows[on]] = self.values[on]
        return d


@dataclass
class StencilSpec:
    """Matrix-free unscaled Dirichlet Laplacian on (NX, NY, NZ).

    2D nx-by-ny grids are (nx, 1, ny) with diag 4; 3D grids use diag 6.
    """
    NX: int
    NY: int
    NZ: int
    diag: float

    @property
    def n(self):
        return self.NX * self.NY * self.NZ

    @property
    def mu(self):
        # stored entries per row of the equivalent CSR (interior row)
        k = 1
        for d in (self.NX, self.NY, self.NZ):
            k += 2 if d >= 3 else (1 if d == 2 else 0)
        return k

    def norm_inf(self):
        # max |row sum|: diag + number of neighbours of the best-connected row
        nb = 0
        for d in (self.NX, self.NY, self.NZ):
            nb += 2 if d >= 3 else (1 if d == 2 else 0)
        return float(self.diag + nb)

    def diagonal(self):
        return np.full(self.n, self.diag)


def as_oracle_operator(A):
    """Accept reference SparseMatrix, package SparseMatrix/Stencil, or oracle types."""
    if isinstance(A, (CSR, StencilSpec)):
        return A
    if hasattr(A, "stencil_spec"):
        NX, NY, NZ, diag = A.stencil_spec()
        return StencilSpec(NX, NY, NZ, diag)
    return CSR(A.n, A.row_ptr, A.col_idx, A.values)


def spmv(A, v):
    """sparse.py:153-160 -> _kernels.csr_matvec (or its matrix-free twin)."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    out = np.empty(A.n)
    lib = _clib()
    if isinstance(A, StencilSpec):
        lib.orc_stencil_matvec(A.NX, A.NY, A.NZ, float(A.diag), _ptr(v), _ptr(out))
    else:
        lib.orc_csr_matvec(A.n, _ptr(A.row_ptr), _ptr(A.col_idx), _ptr(A.values),
                           _ptr(v), _ptr(out))
    return out


def blocked_dot(u, v):
    """_kernels.py:15-41 via the C restatement."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    if u.shape != v.shape or u.ndim != 1:
        raise ValueError("dimension mismatch in dot")
    return float(_clib().orc_blocked_dot(len(u), _ptr(u), _ptr(v)))


def blocked_dot_numpy(u, v):
    """Same order as blocked_dot in pure numpy (add.accumulate is sequential)."""
    n = len(u)
    lim = n - n % 8
    prod = (u[:lim] * v[:lim]).reshape(-1, 8)
    if lim:
        lanes = np.add.accumulate(prod, axis=0)[-1]
    else:
        lanes = np.zeros(8)
    tail = 0.0
    for j in range(lim, n):
        tail += float(u[j] * v[j])
    a = lanes
    return float((((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]))) + tail)


def axpy(alpha, x, y):
    """sparse.py:172-180."""
    if x.shape != y.shape:
        raise ValueError("dimension mismatch in axpy")
    if alpha == 0.0:
        return y.copy()
    return alpha * x + y


class Precond:
    """precond.py:56-131: identity, Jacobi, IC(0) (`lower` = (row_ptr,
    col_idx, l_values) of L, `upper` = the same for L^T)."""

    def __init__(self, kind="identity", inv_diag=None, lower=None, upper=None):
        self.kind = kind
        self.inv_diag = inv_diag
        self.lower = lower
        self.upper = upper

    def apply(self, v):
        if self.kind == "identity":
            return v                                     # precond.py:84-85
        if self.kind == "jacobi":
            return v * self.inv_diag                     # precond.py:88-89
        v = np.ascontiguousarray(v, dtype=np.float64)   # precond.py:90-94
        n = len(v)
        y, out = np.empty(n), np.empty(n)
        lib = _clib()
        lib.orc_lower_solve(n, *(_ptr(a) for a in self.lower), _ptr(v), _ptr(y))
        lib.orc_upper_solve(n, *(_ptr(a) for a in self.upper), _ptr(y), _ptr(out))
        return out


class PreconditionerBreakdown(ArithmeticError):
    """precond.py:20-25."""

    def __init__(self, row):
        self.row = row
        super().__init__(f"nonpositive pivot in IC(0) factorization at row {row}")


def lower_pattern(A, eta=0.0):
    """precond.py:28-43: lower triangle of A (diagonal last per row), the
    diagonal scaled by (1 + eta) when eta != 0."""
    n = A.n
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(A.row_ptr))
    keep = A.col_idx <= rows
    cols = np.ascontiguousarray(A.col_idx[keep], dtype=np.int64)
    vals = np.array(A.values[keep], dtype=np.float64)
    ptr = np.zeros(n + 1, dtype=np.int64)
    ptr[1:] = np.cumsum(np.bincount(rows[keep], minlength=n))
    dpos = ptr[1:] - 1
    if np.any(ptr[1:] == ptr[:-1]) or np.any(cols[dpos] != np.arange(n)):
        raise ValueError("matrix has a structurally missing diagonal entry")
    if eta:
        vals[dpos] *= 1.0 + eta
    return ptr, cols, vals


def transpose_pattern(n, ptr, cols, vals):
    """precond.py:46-53: CSR of the transpose, rows of each column in order."""
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(ptr))
    perm = np.lexsort((rows, cols))
    tptr = np.zeros(n + 1, dtype=np.int64)
    tptr[1:] = np.cumsum(np.bincount(cols, minlength=n))
    return tptr, np.ascontiguousarray(rows[perm]), np.ascontiguousarray(vals[perm])


def make_ic0(A, eta=0.0):
    """precond.py:134-154 with the factor of _kernels.py:77-115 (C)."""
    if eta < 0.0:
        raise ValueError("compensation shift eta must be >= 0")
    ptr, cols, avals = lower_pattern(A, eta)
    lvals = np.zeros_like(avals)
    bad = int(_clib().orc_ic0_factor(A.n, _ptr(ptr), _ptr(cols), _ptr(avals), _ptr(lvals)))
    if bad >= 0:
        raise PreconditionerBreakdown(bad)
    lower = (ptr, cols, lvals)
    return Precond("ic0", lower=lower, upper=transpose_pattern(A.n, *lower))


def identity():
    return Precond("identity")


def make_jacobi(A):
    """precond.py:124-131."""
    d = A.diagonal()
    if np.any(d <= 0.0):
        raise ValueError(f"nonpositive diagonal entry at row {int(np.nonzero(d <= 0.0)[0][0])}")
    return Precond("jacobi", 1.0 / d)


def as_oracle_precond(M):
    if M is None:
        return identity()
    if isinstance(M, Precond):
        return M
    kind = getattr(M, "kind", "identity")
    if kind == "identity":
        return identity()
    if kind == "jacobi":
        inv = M.inv_diag
        if hasattr(inv, "cpu"):
            inv = inv.cpu().numpy()
        return Precond("jacobi", np.asarray(inv, dtype=np.float64))
    if kind == "ic0":
        lower = tuple(np.ascontiguousarray(a, dtype=t) for a, t in
                      zip(M.host_lower(), (np.int64, np.int64, np.float64)))
        return Precond("ic0", lower=lower, upper=transpose_pattern(len(lower[0]) - 1, *lower))
    raise ValueError(f"oracle supports identity/jacobi/ic0, not {kind!r}")


# --------------------------------------------------------------------------
# solver pieces
# --------------------------------------------------------------------------

@dataclass
class Config:
    """Mirror of SolverConfig (solvers.py:60-86)."""
    method: str = "cg"
    shift: float = 0.0
    shift_schedule: tuple | None = None
    max_iters: int = 100
    rtol: float = 0.0
    track_gaps: bool = False
    rr_threshold: float = DEFAULT_RR_THRESHOLD


@dataclass
class Result:
    x: np.ndarray
    converged: bool
    iterations: int
    history: np.ndarray                       # [iterations+1, NCOL]
    replacements: list = field(default_factory=list)


def _cfg(cfg):
    if isinstance(cfg, Config):
        return cfg
    return Config(**{k: getattr(cfg, k) for k in Config.__dataclass_fields__})


def _sub2(base, a, xv, c, yv):
    """solvers.py:170-178."""
    if c == 0.0:
        return base - a * xv
    return base - (a * xv + c * yv)


def pipelined_scalars(i, gamma, delta, gamma_prev, alpha_prev, last):
    """solvers.py:194-230, verbatim logic."""
    if i == 0:
        beta = 0.0
        if delta > 0.0:
            alpha = gamma / delta
        elif last:
            alpha = 0.0
        elif gamma <= 0.0:
            raise BreakdownError(i, "nonpositive (r, u)")
        else:
            raise BreakdownError(i, "nonpositive curvature (w, u)")
        return beta, alpha
    beta = gamma / gamma_prev if gamma_prev != 0.0 else 0.0
    if last:
        if gamma == 0.0 or delta == 0.0:
            return beta, 0.0
        denom = delta / gamma - beta / alpha_prev
        alpha = 1.0 / denom if denom != 0.0 else 0.0
        return beta, (alpha if math.isfinite(alpha) else 0.0)
    if gamma == 0.0:
        raise BreakdownError(i, "vanishing (r, u)")
    denom = delta / gamma - beta / alpha_prev
    if denom == 0.0:
        raise BreakdownError(i, "vanishing alpha denominator")
    alpha = 1.0 / denom
    if not (math.isfinite(alpha) and math.isfinite(beta)):
        raise BreakdownError(i, "non-finite coefficients")
    return beta, alpha


def _rnorm_true_wanted(cfg, i, last):
    return cfg.track_gaps or last or (i % 10 == 0)


def _row(i, alpha, beta, gamma, delta, rnorm, true=None, gaps=(None,) * 4):
    vals = [i, alpha, beta, gamma, delta, rnorm, true, *gaps]
    return [np.nan if v is None else float(v) for v in vals]


def _check(A, b, x0):
    b = np.asarray(b, dtype=np.float64)
    if b.shape != (A.n,):
        raise ValueError("right-hand side dimension mismatch")
    x0 = np.zeros(A.n) if x0 is None else np.asarray(x0, dtype=np.float64)
    if x0.shape != (A.n,):
        raise ValueError("initial guess dimension mismatch")
    return b, x0


def _gaps(A, b, x, r, u, w, s, t, p, q, z, sigma_prev, dot):
    """solvers.py:142-167 (pipelined states)."""
    norm = lambda v: float(np.sqrt(dot(v, v)))
    true_r = b - spmv(A, x)
    f = true_r - r
    if w is None:
        return norm(true_r), (norm(f), None, None, None)
    h = axpy(-sigma_prev, r, spmv(A, u)) - w
    g = axpy(-sigma_prev, t, spmv(A, p)) - s
    j = spmv(A, q) - z
    return norm(true_r), (norm(f), norm(g), norm(h), norm(j))


def _record(A, b, cfg, i, last, alpha, beta, gamma, delta, rnorm, dot, vecs):
    x = vecs[0]
    if cfg.track_gaps:
        true, gaps = _gaps(A, b, *vecs, dot=dot)
        return _row(i, alpha, beta, gamma, delta, rnorm, true, gaps)
    true = None
    if _rnorm_true_wanted(cfg, i, last):
        tr = b - spmv(A, x)
        true = float(np.sqrt(dot(tr, tr)))
    return _row(i, alpha, beta, gamma, delta, rnorm, true)


def solve_cg(A, M, b, x0, cfg, dot=blocked_dot, callback=None):
    """solvers.py:237-294."""
    A = as_oracle_operator(A)
    M = as_oracle_precond(M)
    cfg = _cfg(cfg)
    b, x0 = _check(A, b, x0)
    norm = lambda v: float(np.sqrt(dot(v, v)))
    bnorm = norm(b)
    x = x0.copy()
    r = b - spmv(A, x)
    u = M.apply(r)
    p = np.zeros(A.n)
    gamma_prev = 0.0
    hist = []
    converged = False
    i = 0
    for i in range(cfg.max_iters + 1):
        gamma = dot(r, u)
        rnorm = norm(r)
        converged = rnorm == 0.0 or (cfg.rtol > 0.0 and rnorm <= cfg.rtol * bnorm)
        last = converged or i == cfg.max_iters
        if i == 0:
            beta = 0.0
        else:
            beta = gamma / gamma_prev if gamma_prev > 0.0 else 0.0
        if not last and gamma <= 0.0:
            raise BreakdownError(i, "nonpositive (r, u)")
        p = axpy(beta, p, u)
        s = spmv(A, p)
        delta = dot(s, p)
        if last:
            alpha = gamma / delta if delta > 0.0 else 0.0
        elif delta <= 0.0:
            raise BreakdownError(i, "nonpositive curvature (s, p)")
        else:
            alpha = gamma / delta
        if cfg.track_gaps:
            true_r = b - spmv(A, x)
            row = _row(i, alpha, beta, gamma, delta, rnorm, norm(true_r),
                       (norm(true_r - r), None, None, None))
        else:
            row = _record(A, b, cfg, i, last, alpha, beta, gamma, delta, rnorm, dot, (x,))
        hist.append(row)
        if callback is not None:
            callback(dict(iter=i, x=x, r=r, u=u, p_prev=p, s_prev=s))
        if last:
            break
        x = axpy(alpha, p, x)
        r = r - alpha * s
        u = M.apply(r)
        gamma_prev = gamma
    return Result(x, converged, i, np.array(hist))


def solve_pcg_shifted(A, M, b, x0, cfg, dot=blocked_dot, callback=None):
    """solvers.py:360-422 (also solve_pcg, :297-357, as the shift=0 case:
    axpy(0, r, w) is an exact copy and _sub2 with c=0 is the two-term update,
    so the shifted recurrences with sigma=0 are the plain p-CG ones)."""
    A = as_oracle_operator(A)
    M = as_oracle_precond(M)
    cfg = _cfg(cfg)
    sigma = float(cfg.shift) if cfg.method == "pcg_sh" else 0.0
    b, x0 = _check(A, b, x0)
    norm = lambda v: float(np.sqrt(dot(v, v)))
    bnorm = norm(b)
    x = x0.copy()
    r = b - spmv(A, x)
    u = M.apply(r)
    w = axpy(-sigma, r, spmv(A, u))
    z = np.zeros(A.n)
    q = np.zeros(A.n)
    s = np.zeros(A.n)
    t = np.zeros(A.n)
    p = np.zeros(A.n)
    gamma_prev = 0.0
    alpha_prev = 1.0
    hist = []
    converged = False
    i = 0
    for i in range(cfg.max_iters + 1):
        gamma = dot(r, u)
        delta = dot(axpy(sigma, r, w), u)
        rnorm = norm(r)
        converged = rnorm == 0.0 or (cfg.rtol > 0.0 and rnorm <= cfg.rtol * bnorm)
        last = converged or i == cfg.max_iters
        beta, alpha = pipelined_scalars(i, gamma, delta, gamma_prev, alpha_prev, last)
        hist.append(_record(A, b, cfg, i, last, alpha, beta, gamma, delta, rnorm, dot,
                            (x, r, u, w, s, t, p, q, z, sigma)))
        if callback is not None:
            callback(dict(iter=i, x=x, r=r, u=u, w=w, s_prev=s, t_prev=t,
                          p_prev=p, q_prev=q, z_prev=z))
        if last:
            break
        m = M.apply(w)
        n = spmv(A, m)
        z = axpy(beta, z, n)
        q = axpy(beta, q, m)
        s = axpy(beta, s, w)
        t = axpy(beta, t, r)
        p = axpy(beta, p, u)
        x = axpy(alpha, p, x)
        asig = alpha * sigma
        r = _sub2(r, alpha, s, asig, t)
        u = _sub2(u, alpha, q, asig, p)
        w = w - alpha * z
        gamma_prev = gamma
        alpha_prev = alpha
    return Result(x, converged, i, np.array(hist))


def solve_pcg(A, M, b, x0, cfg, dot=blocked_dot, callback=None):
    """solvers.py:297-357: identical operation sequence to the shifted solver
    at sigma = 0 (reference test_solvers.py:73-90 pins that bitwise)."""
    cfg = _cfg(cfg)
    c0 = Config(**{**cfg.__dict__, "method": "pcg", "shift": 0.0})
    return solve_pcg_shifted(A, M, b, x0, c0, dot=dot, callback=callback)


def solve_pcg_var_shifted(A, M, b, x0, cfg, dot=blocked_dot, callback=None):
    """solvers.py:425-498."""
    A = as_oracle_operator(A)
    M = as_oracle_precond(M)
    cfg = _cfg(cfg)
    b, x0 = _check(A, b, x0)
    sched = np.asarray(cfg.shift_schedule, dtype=np.float64)
    if sched.ndim != 1 or len(sched) < cfg.max_iters + 1:
        raise ValueError("shift schedule must provide max_iters + 1 values")
    norm = lambda v: float(np.sqrt(dot(v, v)))
    bnorm = norm(b)
    x = x0.copy()
    r = b - spmv(A, x)
    u = M.apply(r)
    w = axpy(-sched[0], r, spmv(A, u))
    z = np.zeros(A.n)
    q = np.zeros(A.n)
    s = np.zeros(A.n)
    t = np.zeros(A.n)
    p = np.zeros(A.n)
    gamma_prev = 0.0
    alpha_prev = 1.0
    hist = []
    converged = False
    i = 0
    for i in range(cfg.max_iters + 1):
        sigma_prev = float(sched[i])
        sigma_cur = float(sched[i + 1]) if i + 1 < len(sched) else None
        gamma = dot(r, u)
        delta = dot(axpy(sigma_prev, r, w), u)
        rnorm = norm(r)
        converged = rnorm == 0.0 or (cfg.rtol > 0.0 and rnorm <= cfg.rtol * bnorm)
        last = converged or i == cfg.max_iters
        beta, alpha = pipelined_scalars(i, gamma, delta, gamma_prev, alpha_prev, last)
        hist.append(_record(A, b, cfg, i, last, alpha, beta, gamma, delta, rnorm, dot,
                            (x, r, u, w, s, t, p, q, z, sigma_prev)))
        if last:
            break
        m = M.apply(w)
        n = spmv(A, m)
        dsig = sigma_cur - sigma_prev
        t = axpy(beta, t, r)
        p = axpy(beta, p, u)
        s = axpy(-dsig, t, axpy(beta, s, w))
        q = axpy(-dsig, p, axpy(beta, q, m))
        zbase = axpy(beta, z, n)
        if dsig == 0.0:
            z = zbase
        else:
            z = axpy(-dsig, axpy(sigma_cur, t, s), zbase)
        x = axpy(alpha, p, x)
        w = _sub2(w, alpha, z, dsig, r)
        asig = alpha * sigma_cur
        r = _sub2(r, alpha, s, asig, t)
        u = _sub2(u, alpha, q, asig, p)
        gamma_prev = gamma
        alpha_prev = alpha
    return Result(x, converged, i, np.array(hist))


class ReplacementTrigger:
    """solvers.py:501-532."""

    def __init__(self, mu, n, norm_inf, bnorm, tau):
        self.tau = tau
        self.eps = UNIT_ROUNDOFF
        self.coef = (mu * math.sqrt(n) + 1.0) * norm_inf
        self.e = 0.0
        self.held = False
        self.bnorm = bnorm

    def start(self, xnorm, rnorm):
        self.e = self.eps * (self.coef * xnorm + self.bnorm)
        self.held = self.e <= self.tau * rnorm

    def update(self, xnorm, rnorm):
        self.e += self.eps * (self.coef * xnorm + rnorm)
        ok = self.e <= self.tau * rnorm
        fire = self.held and not ok and self.tau > 0.0
        self.held = ok
        return fire

    def reset(self, xnorm, rnorm):
        self.e = self.eps * (self.coef * xnorm + rnorm)
        self.held = self.e <= self.tau * rnorm


def solve_pcg_rr(A, M, b, x0, cfg, dot=blocked_dot, callback=None):
    """solvers.py:535-608."""
    A = as_oracle_operator(A)
    M = as_oracle_precond(M)
    cfg = _cfg(cfg)
    b, x0 = _check(A, b, x0)
    norm = lambda v: float(np.sqrt(dot(v, v)))
    bnorm = norm(b)
    trig = ReplacementTrigger(A.mu, A.n, A.norm_inf(), bnorm, cfg.rr_threshold)
    x = x0.copy()
    r = b - spmv(A, x)
    u = M.apply(r)
    w = spmv(A, u)
    z = np.zeros(A.n)
    q = np.zeros(A.n)
    s = np.zeros(A.n)
    t = np.zeros(A.n)
    p = np.zeros(A.n)
    trig.start(norm(x), norm(r))
    gamma_prev = 0.0
    alpha_prev = 1.0
    hist = []
    reps = []
    converged = False
    i = 0
    for i in range(cfg.max_iters + 1):
        gamma = dot(r, u)
        delta = dot(w, u)
        rnorm = norm(r)
        converged = rnorm == 0.0 or (cfg.rtol > 0.0 and rnorm <= cfg.rtol * bnorm)
        last = converged or i == cfg.max_iters
        beta, alpha = pipelined_scalars(i, gamma, delta, gamma_prev, alpha_prev, last)
        hist.append(_record(A, b, cfg, i, last, alpha, beta, gamma, delta, rnorm, dot,
                            (x, r, u, w, s, t, p, q, z, 0.0)))
        if last:
            break
        m = M.apply(w)
        n = spmv(A, m)
        z = axpy(beta, z, n)
        q = axpy(beta, q, m)
        s = axpy(beta, s, w)
        t = axpy(beta, t, r)
        p = axpy(beta, p, u)
        x = axpy(alpha, p, x)
        r = r - alpha * s
        u = u - alpha * q
        w = w - alpha * z
        gamma_prev = gamma
        alpha_prev = alpha
        if trig.update(norm(x), norm(r)):
            r = b - spmv(A, x)
            u = M.apply(r)
            w = spmv(A, u)
            s = spmv(A, p)
            q = M.apply(s)
            z = spmv(A, q)
            reps.append(i + 1)
            trig.reset(norm(x), norm(r))
    return Result(x, converged, i, np.array(hist), reps)


SOLVERS = {
    "cg": solve_cg,
    "pcg": solve_pcg,
    "pcg_sh": solve_pcg_shifted,
    "pcg_var_sh": solve_pcg_var_shifted,
    "pcg_rr": solve_pcg_rr,
}


def solve(A, M, b, x0, cfg, dot=blocked_dot, callback=None):
    """solvers.py:620-623."""
    cfg = _cfg(cfg)
    return SOLVERS[cfg.method](A, M, b, x0, cfg, dot=dot, callback=callback)


# --------------------------------------------------------------------------
# generators restated from the reference (sparse.py)
# --------------------------------------------------------------------------

def from_coo(n, rows, cols, vals):
    """sparse.py:89-110 (duplicates summed with np.add.at in sorted order)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
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
    return CSR(n, row_ptr, cols, vals)


def laplacian_2d(nx, ny):
    """sparse.py:188-214."""
    n = nx * ny
    ids = np.arange(n, dtype=np.int64)
    ix = ids % nx
    iy = ids // nx
    rows = [ids]
    cols = [ids]
    vals = [np.full(n, 4.0)]
    for mask, shift in ((iy > 0, -nx), (ix > 0, -1), (ix < nx - 1, 1), (iy < ny - 1, nx)):
        rows.append(ids[mask])
        cols.append(ids[mask] + shift)
        vals.append(np.full(int(mask.sum()), -1.0))
    return from_coo(n, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals))


def random_spd(n, cond=100.0, seed=0):
    """sparse.py:217-228 (dense QR construction, stored as CSR)."""
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.normal(size=(n, n)))
    lam = np.logspace(0.0, np.log10(cond), n) if n > 1 else np.ones(1)
    a = (q * lam) @ q.T
    a = (a + a.T) / 2.0
    rows, cols = np.nonzero(np.abs(a) > 0.0)
    return from_coo(n, rows, cols, a[rows, cols])
