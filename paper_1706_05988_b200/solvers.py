"""Drop-in solver entry points (mirror of pkg/src/kpl/solvers.py) on the B200.

Same signatures, dataclasses and error conventions as the reference:

    solve(A, M, b, x0, cfg, callback=None) -> SolveResult      solvers.py:620-623
    solve_cg / solve_pcg / solve_pcg_shifted / solve_pcg_rr     :237 / :297 / :360 / :535
    SolverConfig, IterationRecord, SolveResult, SolverState, BreakdownError

Every vector operation runs in libkpl_b200.so; the host loop only enqueues
chunks of iterations and polls a 128-byte device status word (no per-
iteration synchronisation).  History rows live in a device table copied back
once at the end.  `A` may be a reference or package `SparseMatrix` (uploaded
as int32 CSR) or a `Stencil2D`/`Stencil3D` (matrix-free); `b`/`x0` may be
numpy arrays (the result `x` is numpy) or CUDA tensors (the result stays on
the device).

Numerics: elementwise work is bitwise identical to the reference; dot
products use the deterministic GPU tree order, so histories match
the reference's within rounding and match the oracle run with the same order
bit for bit.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib, device as D

# unit roundoff of binary64 round-to-nearest (solvers.py:42)
UNIT_ROUNDOFF = float(np.finfo(np.float64).eps) / 2.0
DEFAULT_RR_THRESHOLD = math.sqrt(UNIT_ROUNDOFF)          # solvers.py:46
_METHODS = ("cg", "pcg", "pcg_sh", "pcg_var_sh", "pcg_rr")
_CODE = {"cg": _lib.KPL_M_CG, "pcg": _lib.KPL_M_PCG, "pcg_sh": _lib.KPL_M_PCG_SH,
         "pcg_var_sh": _lib.KPL_M_PCG_VAR_SH, "pcg_rr": _lib.KPL_M_PCG_RR}
HC = _lib.KPL_HIST_COLS


def records_from(h, rows):
    """Device history table [rows, 10] -> IterationRecord list (NaN -> None)."""
    opt = lambda v: None if np.isnan(v) else float(v)
    return [IterationRecord(i, *(float(c) for c in h[i, :5]), rnorm_true=opt(h[i, 5]),
                            gap_f=opt(h[i, 6]), gap_g=opt(h[i, 7]), gap_h=opt(h[i, 8]),
                            gap_j=opt(h[i, 9]))
            for i in range(rows)]


def make_kcfg(cfg, A, dm, device):
    """kpl_cfg for `cfg`; returns (kcfg, keep-alive tensors)."""
    c = _lib.KplCfg()
    c.method = _CODE[cfg.method]
    c.track_gaps = 1 if cfg.track_gaps else 0
    c.shift = float(cfg.shift)
    c.max_iters = int(cfg.max_iters)
    c.rtol = float(cfg.rtol)
    c.rr_threshold = float(cfg.rr_threshold)
    keep = []
    if cfg.method == "pcg_rr":
        # _ReplacementTrigger.coef = (mu*sqrt(n) + 1) * ||A||_inf (solvers.py:514)
        if getattr(dm, "rr_coef", None) is None:
            dm.rr_coef = (A.mu * math.sqrt(A.n) + 1.0) * A.norm_inf()
        c.rr_coef = dm.rr_coef
    if cfg.method == "pcg_var_sh":
        sched = np.asarray(cfg.shift_schedule, dtype=np.float64)
        if sched.ndim != 1 or len(sched) < cfg.max_iters + 1:
            raise ValueError("shift schedule must provide max_iters + 1 values")   # solvers.py:439-440
        t = D.torch()
        dsched = t.from_numpy(np.ascontiguousarray(sched[:cfg.max_iters + 1])).to(device)
        keep.append(dsched)
        c.shift_schedule = dsched.data_ptr()
        c.shift = float(sched[0])
    return c, keep


class BreakdownError(ArithmeticError):
    """A denominator that must be positive for SPD inputs was not (solvers.py:51-57)."""

    def __init__(self, iteration, what):
        self.iteration = iteration
        self.what = what
        super().__init__(f"breakdown at iteration {iteration}: {what}")


@dataclass(frozen=True)
class SolverConfig:
    """solvers.py:60-86 (same fields, defaults and validation)."""
    method: str = "cg"
    shift: float = 0.0
    shift_schedule: tuple | None = None
    max_iters: int = 100
    rtol: float = 0.0
    track_gaps: bool = False
    rr_threshold: float = DEFAULT_RR_THRESHOLD

    def __post_init__(self):
        if self.method not in _METHODS:
            raise ValueError(f"unknown method {self.method!r}")
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")
        if self.rtol < 0.0:
            raise ValueError("rtol must be >= 0")
        if not math.isfinite(self.shift):
            raise ValueError("shift must be finite")
        if self.method == "pcg_var_sh":
            if self.shift_schedule is None:
                raise ValueError("pcg_var_sh requires a shift schedule")
            if len(self.shift_schedule) < self.max_iters + 1:
                raise ValueError(
                    "shift schedule must provide max_iters + 1 values "
                    "(the entry before iteration 0, then one per iteration)")


@dataclass(slots=True)
class IterationRecord:
    iter: int
    alpha: float
    beta: float
    gamma: float
    delta: float
    rnorm_recursive: float
    rnorm_true: float | None = None
    gap_f: float | None = None
    gap_g: float | None = None
    gap_h: float | None = None
    gap_j: float | None = None


@dataclass(slots=True)
class SolveResult:
    x: object
    converged: bool
    iterations: int
    history: list
    replacements: list = field(default_factory=list)


@dataclass(slots=True)
class SolverState:
    """Callback payload (solvers.py:113-139).  Vectors are host copies taken
    at the record point (the device vectors keep evolving)."""
    iter: int
    x: np.ndarray
    r: np.ndarray
    u: np.ndarray
    alpha: float
    beta: float
    gamma: float
    delta: float
    w: np.ndarray | None = None
    s_prev: np.ndarray | None = None
    t_prev: np.ndarray | None = None
    p_prev: np.ndarray | None = None
    q_prev: np.ndarray | None = None
    z_prev: np.ndarray | None = None
    sigma_prev: float = 0.0
    sigma: float | None = None


# ------------------------------------------------------------------ engine

def _assembled(A):
    """CSR form of a matrix-free stencil, built once per stencil object."""
    csr = getattr(A, "_csr", None)
    if csr is None:
        csr = A.to_csr()
        A._csr = csr
    return csr


class _Solve:
    """One solve: device vectors, workspace, and the host enqueue loop."""

    # stencil problems up to this size run as persistent cooperative launches
    # (one launch per chunk of iterations, grid barriers instead of kernel
    # boundaries): there the per-iteration launch latency, not HBM, dominates.
    # Measured crossover (tools/small_time.py, us/iteration persistent vs
    # launches): 2D 200^2 13.3/17.5, 300^2 18.1/26.3, 400^2 21.3/28.1, 600^2
    # 38.7/24.0; 3D 64x24x32 11.1/12.6, 48^3 15.6/14.6, 64^3 23.2/19.7 -- the
    # redundant per-CTA fold grows with the item count.
    PERSISTENT_MAX_N = 1 << 16
    PERSISTENT_MAX_N_2D = 1 << 18

    def __init__(self, A, M, b, x0, cfg: SolverConfig, *, zc=0, vx=0, chunk_blocks=0, slab_view=False,
                 persistent=None, alloc=None):
        self.device = dev = D.require_cuda()
        t = D.torch()
        self.cfg = cfg
        self.A = A
        if getattr(M, "kind", None) == "ic0" and hasattr(A, "stencil_spec"):
            A = _assembled(A)            # IC(0) runs with the CSR form (bitwise the same operator)
        self.dm = D.device_matrix(A, dev)
        self.dp = D.device_precond(M, self.dm, dev)
        n = self.n = self.dm.n
        self.b, self.host_io = D.to_device_f64(b, n, dev, "right-hand side")
        self.x0 = None
        if x0 is not None:
            self.x0, _ = D.to_device_f64(x0, n, dev, "initial guess")
        geom = A.slab_spec()[:3] if (slab_view and hasattr(A, "slab_spec")) else None
        self.op = D.make_op(self.dm, self.dp, zc=zc, vx=vx, chunk_blocks=chunk_blocks, geometry=geom)
        self.kcfg, self._keep = make_kcfg(cfg, A, self.dm, dev)
        ident = self.dp.identity
        f64 = dict(dtype=t.float64, device=dev)
        # `alloc(count, dtype)`: where the solver's vectors and workspace live (default: the
        # torch caching allocator; the guard-band tests pass views into poisoned arenas)
        alloc = alloc or (lambda cnt, dt: t.empty(cnt, dtype=dt, device=dev))
        emp = lambda: alloc(n, t.float64)
        self.x = emp()
        self.r = emp()
        self.u = self.r if ident else emp()
        if cfg.method == "cg":
            self.p = emp()
            self.p1 = emp()
            self.s = emp()
            self.w0 = self.w1 = self.z = self.q = self.t = None
        else:
            self.w0, self.w1 = emp(), emp()
            self.z, self.s, self.t = emp(), emp(), emp()
            self.q = self.s if ident else emp()
            self.p = self.t if ident else emp()
            self.p1 = None
        v = _lib.KplVecs()
        for name in ("x", "r", "u", "w0", "w1", "z", "q", "s", "t", "p", "p1", "b"):
            setattr(v, name, D.ptr(getattr(self, name)))
        self.vecs = v
        lib = _lib.load()
        nbytes = lib.kpl_workspace_bytes(self.op, cfg.max_iters)
        _lib.check(nbytes if nbytes < 0 else 0, "workspace size")
        self.ws = alloc(int(nbytes), t.uint8)
        self.hist_off = lib.kpl_history_offset(self.op)
        self.reps_off = lib.kpl_replacements_offset(self.op, cfg.max_iters)
        self.status = _lib.KplStatus()
        if persistent is None and os.environ.get("KPL_NO_PERSISTENT") == "1":
            persistent = False
        if persistent is None:
            lim = self.PERSISTENT_MAX_N_2D if self.op.ny == 1 else self.PERSISTENT_MAX_N
            persistent = (self.dm.kind == _lib.KPL_OP_STENCIL and n <= lim
                          and cfg.method in ("pcg", "pcg_sh", "pcg_var_sh") and not cfg.track_gaps
                          and self.op.order == _lib.KPL_ORDER_TREE)
        self.persistent = bool(persistent)
        # p-CG-rr: replacement sweeps only when the device trigger fired (host-issued
        # at the next status poll) instead of four predicated launches per iteration;
        # KPL_RR_EAGER=1 keeps the per-iteration launches
        self.lazy_rr = (cfg.method == "pcg_rr" and not self.persistent
                        and os.environ.get("KPL_RR_EAGER") != "1")
        # classic CG records row i in the first half of pass i, so the final
        # row max_iters needs one more pass than the pipelined solvers
        self.limit = cfg.max_iters + (1 if cfg.method == "cg" else 0)

    # -- device calls ---------------------------------------------------
    def init(self):
        lib = _lib.load()
        _lib.check(lib.kpl_solver_init(self.op, self.kcfg, self.vecs, D.ptr(self.x0),
                                       D.ptr(self.ws), D.stream_handle()), "solver init")
        self.issued = 0

    def iterate(self, count):
        lib = _lib.load()
        count = min(count, self.limit - self.issued)
        if count <= 0:
            return
        if self.persistent:
            _lib.check(lib.kpl_solver_iterate_persistent(self.op, self.kcfg, self.vecs, self.issued, count,
                                                         D.ptr(self.ws), D.stream_handle()), "solver iterate")
        else:
            flags = _lib.KPL_ITER_LAZY_REPLACE if self.lazy_rr else 0
            _lib.check(lib.kpl_solver_iterate2(self.op, self.kcfg, self.vecs, self.issued, count, flags,
                                               D.ptr(self.ws), D.stream_handle()), "solver iterate")
        self.issued += count

    def replace_if_fired(self, st):
        """Lazy p-CG-rr: the trigger fired at record row st.iter + 1 and the
        iterations issued after it were predicated off -- run the replacement
        (which records that row) and continue from there."""
        if not (self.lazy_rr and st.state == _lib.KPL_ST_RUNNING and st.fire):
            return False
        _lib.check(_lib.load().kpl_solver_replace(self.op, self.kcfg, self.vecs, D.ptr(self.ws),
                                                  D.stream_handle()), "replacement")
        self.issued = int(st.iter) + 1
        return True

    def read_status(self):
        _lib.check(_lib.load().kpl_read_status(D.ptr(self.ws), self.status, D.stream_handle()),
                   "status")
        return self.status

    def finish(self):
        _lib.check(_lib.load().kpl_solver_finish(self.op, self.kcfg, self.vecs, D.ptr(self.ws),
                                                 D.stream_handle()), "solver finish")

    def cg_pass(self, j, which):
        _lib.check(_lib.load().kpl_solver_cg_pass(self.op, self.kcfg, self.vecs, j, which,
                                                  D.ptr(self.ws), D.stream_handle()), "cg pass")

    def _run_cg_callback(self, callback):
        j = 0
        while self.read_status().state == _lib.KPL_ST_RUNNING:
            self.cg_pass(j, 1)                 # record point of row j (solvers.py:269-287)
            st = self.read_status()
            if st.state == _lib.KPL_ST_BREAKDOWN:
                break
            self._callback(callback)
            if st.state != _lib.KPL_ST_RUNNING:
                break
            self.cg_pass(j, 2)                 # x, r, u updates + head of row j+1
            j += 1
        return self.result()

    def run(self, callback=None):
        self.init()
        if callback is not None and self.cfg.method == "cg":
            return self._run_cg_callback(callback)
        # persistent launches stop on the device at convergence, so they can
        # start with longer chunks (fewer status round trips)
        chunk = 1 if callback is not None else (64 if self.persistent else 8)
        st = self.read_status()
        if callback is not None:
            self._callback(callback)
        while st.state == _lib.KPL_ST_RUNNING and (self.issued < self.limit or st.fire):
            if self.replace_if_fired(st):
                st = self.read_status()
                if callback is not None and st.state != _lib.KPL_ST_BREAKDOWN:
                    self._callback(callback)
                continue
            self.iterate(chunk)
            st = self.read_status()
            if callback is not None:
                if st.state != _lib.KPL_ST_BREAKDOWN and not st.fire:
                    self._callback(callback)
            else:
                # lazy p-CG-rr: a fired trigger idles the rest of the chunk, so keep chunks short
                chunk = min(chunk * 2, 32 if self.lazy_rr else 256)
        return self.result()

    # -- results ---------------------------------------------------------
    def _raise_breakdown(self, st):
        msg = _lib.load().kpl_breakdown_message(st.bd_code).decode()
        if st.bd_code >= 7:                      # device-side failure, not arithmetic breakdown
            raise _lib.KplError(f"device solve failed: {msg}")
        raise BreakdownError(int(st.bd_iter), msg)

    def history_array(self, rows):
        t = D.torch()
        raw = self.ws[self.hist_off:self.hist_off + 8 * HC * rows]
        return raw.view(t.float64).reshape(rows, HC).cpu().numpy()

    def result(self):
        st = self.read_status()
        if st.state == _lib.KPL_ST_BREAKDOWN:
            self._raise_breakdown(st)
        if st.state != _lib.KPL_ST_DONE:
            raise _lib.KplError(f"device solve ended in state {st.state} at row {st.iter}")
        self.finish()
        st = self.read_status()
        iters = int(st.iter)
        history = records_from(self.history_array(iters + 1), iters + 1)
        reps = []
        if st.n_replacements:
            t = D.torch()
            raw = self.ws[self.reps_off:self.reps_off + 8 * int(st.n_replacements)]
            reps = [int(v) for v in raw.view(t.int64).cpu().numpy()]
        if self.host_io == "numpy":
            x = D.to_numpy_f64(self.x)
        elif self.host_io == "host":
            t = D.torch()
            x = t.empty(self.n, dtype=t.float64, pin_memory=True)
            x.copy_(self.x, non_blocking=True)
            t.cuda.current_stream().synchronize()
        else:
            x = self.x
        return SolveResult(x, bool(st.converged), iters, history, reps)

    def _callback(self, callback):
        """Slow path: one synchronisation and host copies per record point."""
        st = self.status
        i = int(st.iter)
        if i < 0:
            return
        h = self.history_array(i + 1)[i]
        host = lambda v: None if v is None else v.cpu().numpy().copy()
        sig = sig_cur = float(self.cfg.shift) if self.cfg.method == "pcg_sh" else 0.0
        if self.cfg.method == "pcg_var_sh":
            sched = self.cfg.shift_schedule
            sig = float(sched[i])
            sig_cur = float(sched[i + 1]) if i + 1 < len(sched) else None
        if self.cfg.method == "cg":
            par = (i + 1) & 1      # p written by pass 1 of row i
            state = SolverState(i, host(self.x), host(self.r), host(self.u), *map(float, h[:4]),
                                p_prev=host(self.p1 if par else self.p), s_prev=host(self.s))
        else:
            w = self.w1 if (i & 1) else self.w0
            state = SolverState(i, host(self.x), host(self.r), host(self.u), *map(float, h[:4]),
                                w=host(w), s_prev=host(self.s), t_prev=host(self.t),
                                p_prev=host(self.p), q_prev=host(self.q), z_prev=host(self.z),
                                sigma_prev=sig, sigma=sig_cur)
        callback(state)


def _solve(A, M, b, x0, cfg, callback):
    return _Solve(A, M, b, x0, cfg).run(callback)


def solve_cg(A, M, b, x0, cfg: SolverConfig, callback=None) -> SolveResult:
    """Classic preconditioned CG (solvers.py:237-294) on the device."""
    return _solve(A, M, b, x0, _as(cfg, "cg"), callback)


def solve_pcg(A, M, b, x0, cfg: SolverConfig, callback=None) -> SolveResult:
    """Pipelined CG (solvers.py:297-357) on the device."""
    return _solve(A, M, b, x0, _as(cfg, "pcg"), callback)


def solve_pcg_shifted(A, M, b, x0, cfg: SolverConfig, callback=None) -> SolveResult:
    """Shifted pipelined CG, Alg. 3 (solvers.py:360-422) on the device."""
    return _solve(A, M, b, x0, _as(cfg, "pcg_sh"), callback)


def solve_pcg_rr(A, M, b, x0, cfg: SolverConfig, callback=None) -> SolveResult:
    """Pipelined CG with automated residual replacement (solvers.py:535-608)."""
    return _solve(A, M, b, x0, _as(cfg, "pcg_rr"), callback)


def solve_pcg_var_shifted(A, M, b, x0, cfg: SolverConfig, callback=None) -> SolveResult:
    """Variable-shift p-CG, Alg. 4 (solvers.py:425-498) on the device."""
    return _solve(A, M, b, x0, _as(cfg, "pcg_var_sh"), callback)


def _as(cfg, method):
    """The reference's solve_* functions ignore cfg.method; mirror that."""
    if cfg.method == method:
        return cfg
    from dataclasses import replace
    return replace(cfg, method=method)


_SOLVERS = {
    "cg": solve_cg,
    "pcg": solve_pcg,
    "pcg_sh": solve_pcg_shifted,
    "pcg_var_sh": solve_pcg_var_shifted,
    "pcg_rr": solve_pcg_rr,
}


def solve(A, M, b, x0, cfg: SolverConfig, callback=None) -> SolveResult:
    """Dispatch on cfg.method (solvers.py:620-623)."""
    return _SOLVERS[cfg.method](A, M, b, x0, cfg, callback=callback)
