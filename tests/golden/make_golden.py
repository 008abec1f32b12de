#!/usr/bin/env python3
"""Generate golden fixtures by running the UNMODIFIED reference `kpl`.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Outputs tests/golden/*.npz.  These pin the CPU oracle (oracle/kpl_oracle.py)
bit for bit; the GPU parity tests then compare the device path with the
oracle.  Nothing at test time reads /root/reference.
"""

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import kpl  # noqa: E402  (the reference package)
from kpl import (BreakdownError, SolverConfig, SparseMatrix, laplacian_2d,  # noqa: E402
                 make_jacobi, random_spd, solve, spmv)
from kpl import _kernels  # noqa: E402

from paper_1706_05988_b200 import problems  # noqa: E402  (generators only: no device use)

COLS = ("iter", "alpha", "beta", "gamma", "delta", "rnorm_recursive", "rnorm_true",
        "gap_f", "gap_g", "gap_h", "gap_j")


def hist_array(res):
    return np.array([[np.nan if getattr(r, c) is None else float(getattr(r, c)) for c in COLS]
                     for r in res.history])


def digest(x):
    return hashlib.sha256(np.ascontiguousarray(x, dtype=np.float64).tobytes()).hexdigest()


def csr_arrays(A, prefix):
    return {f"{prefix}_n": np.int64(A.n), f"{prefix}_row_ptr": A.row_ptr,
            f"{prefix}_col_idx": A.col_idx, f"{prefix}_values": A.values}


def run_case(out, tag, A, M, b, cfg, keep_x=False):
    res = solve(A, M, b, None, cfg)
    out[f"{tag}_hist"] = hist_array(res)
    out[f"{tag}_iters"] = np.int64(res.iterations)
    out[f"{tag}_converged"] = np.bool_(res.converged)
    out[f"{tag}_xsha"] = np.array(digest(res.x))
    out[f"{tag}_xsub"] = res.x[::97].copy()
    out[f"{tag}_reps"] = np.array(res.replacements, dtype=np.int64)
    if keep_x:
        out[f"{tag}_x"] = res.x.copy()
    print(f"  {tag}: iters={res.iterations} conv={res.converged} "
          f"final_true={res.history[-1].rnorm_true}")
    return res


def kernels():
    out = {}
    rng = np.random.default_rng(2024)
    for n in (0, 1, 7, 8, 9, 15, 16, 17, 100, 1001, 4099):
        u = rng.normal(size=n) * 10.0 ** rng.integers(-8, 8, size=n)
        v = rng.normal(size=n)
        out[f"dot_{n}_u"] = u
        out[f"dot_{n}_v"] = v
        out[f"dot_{n}_r"] = np.float64(_kernels.blocked_dot(u, v))
    for tag, A in (("lap37x23", laplacian_2d(37, 23)),
                   ("rspd12", random_spd(12, cond=50.0, seed=3))):
        v = rng.normal(size=A.n)
        v[::5] = 0.0
        v[1::7] = -0.0
        out.update(csr_arrays(A, tag))
        out[f"{tag}_v"] = v
        out[f"{tag}_Av"] = spmv(A, v)
    # 3D 7-point and variable-coefficient assemblies through the reference's from_coo
    n, r, c, v = problems.varcoef_3d_coo(6, seed=0)
    Avc = SparseMatrix.from_coo(n, r, c, v)
    out.update(csr_arrays(Avc, "varcoef6"))
    A3 = problems.laplacian_3d(5, 4, 3)
    rows = np.repeat(np.arange(A3.n), np.diff(A3.row_ptr))
    A3r = SparseMatrix.from_coo(A3.n, rows[::-1], A3.col_idx[::-1], A3.values[::-1])
    out.update(csr_arrays(A3r, "lap3d_543"))
    rb, cb, vb = problems.banded_spd_coo(3000, seed=0, band=100)
    Ab = SparseMatrix.from_coo(3000, rb, cb, vb)
    out.update(csr_arrays(Ab, "bandoff3000"))
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **out)


def solvers_small():
    """Reference unit-test problems (test_solvers.py / test_acceptance.py)."""
    out = {}
    methods = (("cg", {}), ("pcg", {}), ("pcg_sh", {"shift": 0.9}),
               ("pcg_var_sh", {"shift_schedule": tuple(0.1 * k for k in range(62))}),
               ("pcg_rr", {}), ("pcg_rr0", {"rr_threshold": 0.0}))
    probs = {
        "rspd48": (random_spd(48, cond=1e3, seed=21), 1 / np.sqrt(48.0)),
        "rspd64s3": (random_spd(64, cond=1e4, seed=3), 1 / 8.0),
    }
    for pname, (A, xval) in probs.items():
        b = spmv(A, np.full(A.n, xval))
        out.update(csr_arrays(A, pname))
        out[f"{pname}_b"] = b
        for gaps in (False, True):
            for mname, extra in methods:
                meth = "pcg_rr" if mname == "pcg_rr0" else mname
                cfg = SolverConfig(method=meth, max_iters=60, rtol=0.0, track_gaps=gaps, **extra)
                run_case(out, f"{pname}_{mname}_{'g' if gaps else 'n'}", A, None, b, cfg, keep_x=True)
    # laplacian_2d(5,4) p-CG-sh sigma=1 with gaps (test_solvers.py:148-159)
    A = laplacian_2d(5, 4)
    b = np.full(A.n, 1 / np.sqrt(A.n))
    out["lap5x4_b"] = b
    run_case(out, "lap5x4_pcgsh", A, None, b,
             SolverConfig(method="pcg_sh", shift=1.0, max_iters=3, track_gaps=True), keep_x=True)
    # identity matrix (test_solvers.py:70-90)
    A = SparseMatrix.from_dense(np.eye(5))
    b = np.random.default_rng(1234).normal(size=5)
    out["eye5_b"] = b
    for m in ("cg", "pcg"):
        run_case(out, f"eye5_{m}", A, None, b, SolverConfig(method=m, max_iters=10, rtol=1e-12),
                 keep_x=True)
    # breakdown (test_solvers.py:198-206)
    A = SparseMatrix.from_dense(np.array([[1.0, 0.0], [0.0, -1.0]]))
    for m in ("cg", "pcg", "pcg_sh"):
        try:
            solve(A, None, np.array([0.5, 1.0]), None, SolverConfig(method=m, max_iters=5))
            out[f"indef_{m}"] = np.array("no breakdown")
        except BreakdownError as e:
            out[f"indef_{m}"] = np.array(f"{e.iteration}|{e.what}")
    np.savez_compressed(os.path.join(HERE, "solvers_small.npz"), **out)


def config1():
    """BASELINE.json config 1 and the Table-1 lapl200 runs."""
    out = {}
    A = laplacian_2d(200, 200)
    b = spmv(A, np.full(A.n, 1.0 / np.sqrt(A.n)))
    out["b_sha"] = np.array(digest(b))
    sig = 2.1320754716981134
    for m, extra in (("cg", {}), ("pcg", {}), ("pcg_sh", {"shift": sig}), ("pcg_rr", {})):
        run_case(out, f"cfg1_{m}", A, None, b,
                 SolverConfig(method=m, max_iters=2000, rtol=1e-12, **extra))
    bt = np.full(A.n, 1.0 / np.sqrt(A.n))
    for m, extra in (("cg", {}), ("pcg", {}), ("pcg_sh", {"shift": 4.0}), ("pcg_rr", {})):
        run_case(out, f"tab1_{m}", A, None, bt,
                 SolverConfig(method=m, max_iters=500, rtol=0.0, **extra))
    np.savez_compressed(os.path.join(HERE, "config1.npz"), **out)


def jacobi_and_3d():
    out = {}
    # config-2 recipe at reduced size: 2D, Jacobi, xhat ~ U[0,1) seed 0
    A = laplacian_2d(64, 48)
    M = make_jacobi(A)
    xh = np.random.default_rng(0).random(A.n)
    b = spmv(A, xh)
    out["j2d_b_sha"] = np.array(digest(b))
    sig = 0.49238826317067413
    for m, extra in (("cg", {}), ("pcg", {}), ("pcg_sh", {"shift": sig}), ("pcg_rr", {})):
        run_case(out, f"j2d_{m}", A, M, b,
                 SolverConfig(method=m, max_iters=1000, rtol=1e-10, **extra))
    # config-3 recipe at reduced size: 3D 7-point M=I, b = A 1/sqrt(n), fixed iterations
    A3 = problems.laplacian_3d(12, 10, 8)
    rows = np.repeat(np.arange(A3.n), np.diff(A3.row_ptr))
    A3r = SparseMatrix.from_coo(A3.n, rows, A3.col_idx, A3.values)
    b3 = spmv(A3r, np.full(A3.n, 1 / np.sqrt(A3.n)))
    out["l3d_b_sha"] = np.array(digest(b3))
    for m, extra in (("pcg", {}), ("pcg_sh", {"shift": 2.30188679245283}), ("cg", {})):
        run_case(out, f"l3d_{m}", A3r, None, b3,
                 SolverConfig(method=m, max_iters=120, rtol=0.0, **extra))
    # config-4 recipe at 8^3: variable coefficients, Jacobi, b ~ N(0,1) seed 1
    n, r, c, v = problems.varcoef_3d_coo(8, seed=0)
    Av = SparseMatrix.from_coo(n, r, c, v)
    Mv = make_jacobi(Av)
    bv = np.random.default_rng(1).standard_normal(n)
    out.update(csr_arrays(Av, "vc8"))
    out["vc8_b"] = bv
    for m, extra in (("cg", {}), ("pcg_sh", {"shift": 0.49238826317067413}), ("pcg", {})):
        run_case(out, f"vc8_{m}", Av, Mv, bv,
                 SolverConfig(method=m, max_iters=400, rtol=1e-12, **extra), keep_x=True)
    # config-5 recipe at n=20000, band 2000
    Ab = problems.banded_spd(20000, seed=0, band=2000)
    Abr = SparseMatrix(Ab.n, Ab.row_ptr, Ab.col_idx, Ab.values)
    Mb = make_jacobi(Abr)
    xb = np.random.default_rng(1).standard_normal(Ab.n)
    bb = spmv(Abr, xb)
    for k in ("row_ptr", "col_idx", "values"):
        out[f"band20k_{k}_sha"] = np.array(digest(getattr(Abr, k).astype(np.float64)))
    out["band20k_b_sha"] = np.array(digest(bb))
    for m, extra in (("cg", {}), ("pcg_sh", {"shift": 0.4124626382901352}), ("pcg_rr", {})):
        run_case(out, f"band20k_{m}", Abr, Mb, bb,
                 SolverConfig(method=m, max_iters=300, rtol=1e-10, **extra))
    np.savez_compressed(os.path.join(HERE, "jacobi_3d.npz"), **out)


def shift_selection():
    """stability.py sweep + shift_study.py:46-51 margin rule on reference histories."""
    from kpl import CoefficientHistory, default_sigma_grid, select_shift
    out = {}
    cases = []
    A = laplacian_2d(200, 200)
    b = spmv(A, np.full(A.n, 1.0 / np.sqrt(A.n)))
    cases.append(("cfg1", A, None, b, 2000, 1e-12))
    Aj = laplacian_2d(64, 48)
    Mj = make_jacobi(Aj)
    bj = spmv(Aj, np.random.default_rng(0).random(Aj.n))
    cases.append(("j2d", Aj, Mj, bj, 1000, 1e-10))
    for tag, A_, M_, b_, maxit, rtol in cases:
        base = solve(A_, M_, b_, None, SolverConfig(method="pcg", max_iters=maxit, rtol=rtol))
        hist = CoefficientHistory.from_result(base)
        grid = default_sigma_grid(A_, M_)
        sw = select_shift(hist, base.iterations, grid)
        floor = 4.0 * sw.psi_values.min()
        chosen = float(sw.grid[np.argmax(sw.psi_values <= floor)])
        out[f"{tag}_alphas"] = hist.alphas
        out[f"{tag}_betas"] = hist.betas
        out[f"{tag}_i"] = np.int64(base.iterations)
        out[f"{tag}_grid"] = grid
        out[f"{tag}_psi"] = sw.psi_values
        out[f"{tag}_argmin"] = np.float64(sw.argmin)
        out[f"{tag}_chosen"] = np.float64(chosen)
        print(f"  {tag}: i={base.iterations} argmin={sw.argmin} chosen={chosen!r}")
    np.savez_compressed(os.path.join(HERE, "shift.npz"), **out)


def formats():
    """Reference history CSV/JSON and Matrix Market bytes (harness.py:99-130, mmio.py:103-122)."""
    import io
    from kpl import emit_history, write_matrix_market
    out = {}
    A = laplacian_2d(5, 4)
    b = np.full(A.n, 1 / np.sqrt(A.n))
    for tag, cfg in (("gaps", SolverConfig(method="pcg_sh", shift=1.0, max_iters=12, track_gaps=True)),
                     ("plain", SolverConfig(method="pcg_rr", max_iters=25))):
        res = solve(A, None, b, None, cfg)
        out[f"{tag}_hist"] = hist_array(res)
        for fmt in ("csv", "json"):
            sink = io.StringIO()
            emit_history(res.history, fmt, sink)
            out[f"{tag}_{fmt}"] = np.frombuffer(sink.getvalue().encode("ascii"), dtype=np.uint8)
    for tag, M in (("lap5x4", laplacian_2d(5, 4)), ("rspd6", random_spd(6, cond=30.0, seed=2))):
        sink = io.BytesIO()
        write_matrix_market(M, sink)
        out[f"mm_{tag}"] = np.frombuffer(sink.getvalue(), dtype=np.uint8)
        out.update(csr_arrays(M, f"mmA_{tag}"))
    np.savez_compressed(os.path.join(HERE, "formats.npz"), **out)


def ic0():
    """IC(0) factor, apply and solves (precond.py:134-154, _kernels.py:55-115)."""
    from kpl import PreconditionerBreakdown, make_ic0
    out = {}
    rng = np.random.default_rng(77)
    cases = (("lap12x9", laplacian_2d(12, 9), 0.0),
             ("rspd40", random_spd(40, cond=1e3, seed=5), 0.0),
             ("rspd40e", random_spd(40, cond=1e3, seed=5), 0.25),
             ("vc5", SparseMatrix(*_csr_args(problems.varcoef_3d(5, seed=2))), 0.0),
             ("band3k", SparseMatrix(*_csr_args(problems.banded_spd(3000, seed=4, band=100))), 0.1))
    for tag, A, eta in cases:
        M = make_ic0(A, eta=eta)
        out.update(csr_arrays(A, tag))
        out[f"{tag}_eta"] = np.float64(eta)
        out[f"{tag}_L_row_ptr"], out[f"{tag}_L_col_idx"], out[f"{tag}_L_values"] = M._l
        out[f"{tag}_mu_tilde"] = np.int64(M.mu_tilde)
        v = rng.normal(size=A.n)
        v[::11] = -0.0
        out[f"{tag}_v"] = v
        out[f"{tag}_Mv"] = M.apply(v)
    try:
        make_ic0(SparseMatrix.from_dense(np.array([[1.0, 2.0], [2.0, 1.0]])), eta=0.0)
    except PreconditionerBreakdown as exc:
        out["indef_row"] = np.int64(exc.row)
    # solves: 2D Laplacian 30x20 and var-coef 6^3, IC(0) eta 0
    A = laplacian_2d(30, 20)
    M = make_ic0(A, eta=0.0)
    b = spmv(A, np.full(A.n, 1.0 / np.sqrt(A.n)))
    out["l2_b"] = b
    sched = tuple(0.05 * (k % 7) for k in range(82))
    for m, extra in (("cg", {}), ("pcg", {}), ("pcg_sh", {"shift": 0.5}),
                     ("pcg_var_sh", {"shift_schedule": sched}), ("pcg_rr", {}),
                     ("pcg_rrx", {"rtol": 0.0})):
        for gaps in (False, True):
            meth = "pcg_rr" if m == "pcg_rrx" else m      # rrx: past convergence, replacements fire
            kw = {"rtol": 1e-10, **extra}
            run_case(out, f"l2_{m}_{'g' if gaps else 'n'}", A, M, b,
                     SolverConfig(method=meth, max_iters=80, track_gaps=gaps, **kw), keep_x=True)
    A = SparseMatrix(*_csr_args(problems.varcoef_3d(6, seed=0)))
    M = make_ic0(A, eta=0.0)
    b = spmv(A, np.random.default_rng(3).standard_normal(A.n))
    out["v6_b"] = b
    for m, extra in (("cg", {}), ("pcg_sh", {"shift": 0.3}), ("pcg_rr", {})):
        run_case(out, f"v6_{m}", A, M, b, SolverConfig(method=m, max_iters=300, rtol=1e-12, **extra),
                 keep_x=True)
    np.savez_compressed(os.path.join(HERE, "ic0.npz"), **out)


def _csr_args(A):
    return A.n, A.row_ptr, A.col_idx, A.values


if __name__ == "__main__":
    print("reference kpl", kpl.__version__, "from", kpl.__file__)
    only = sys.argv[1:]
    for name, fn in (("kernels", kernels), ("solvers_small", solvers_small), ("config1", config1),
                     ("jacobi_3d", jacobi_and_3d), ("shift", shift_selection), ("formats", formats),
                     ("ic0", ic0)):
        if not only or name in only:
            fn()
