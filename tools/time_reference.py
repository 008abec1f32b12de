#!/usr/bin/env python3
"""Time the UNMODIFIED reference solver (`kpl.solve`, pkg/src/kpl/solvers.py:611-623)
on the GPU box's host, one core.

The reference package is installed (not copied into the repo) with

    python -m pip install --no-index --no-build-isolation --no-deps --target baseline/_ref <copy of pkg/>

(baseline/_ref is git-ignored and travels to the GPU box).  Run there as

    taskset -c 0 env OMP_NUM_THREADS=1 NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tools/time_reference.py [--configs 1,5,2,4] [--full2]

Per BASELINE.md 3: one JIT warm-up solve (max_iters=1), then time.perf_counter
around `solve` only (matrix and rhs construction excluded); configs 1 and 5 run
to tolerance; config 2 runs to tolerance with --full2 (~25 min per method),
else 200 iterations for the rate; config 4 (256^3 CSR) 50 iterations for the
rate.  The matrices are the same arrays the device runs on (this package's
host generators for configs 4 and 5).
"""

import argparse
import json
import math
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.path.insert(1, ROOT)

import numpy as np  # noqa: E402

import kpl  # noqa: E402  (the reference package)


def host():
    model = None
    with open("/proc/cpuinfo") as f:
        for line in f:
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    aff = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else None
    return {"cpu_model": model, "host_cores": os.cpu_count(), "cores_used": 1, "affinity_cpus": aff,
            "python": platform.python_version(), "numpy": np.__version__}


def run(tag, A, M, b, method, shift, max_iters, rtol):
    kpl.solve(A, M, b, None, kpl.SolverConfig(method=method, shift=shift, max_iters=1, rtol=0.0))  # JIT
    bn = float(kpl.norm2(b))
    t0 = time.perf_counter()
    res = kpl.solve(A, M, b, None, kpl.SolverConfig(method=method, shift=shift, max_iters=max_iters, rtol=rtol))
    dt = time.perf_counter() - t0
    out = {"config": tag, "method": method, "shift": shift, "n": A.n, "iterations": res.iterations,
           "converged": res.converged, "final_true_rel": res.history[-1].rnorm_true / bn,
           "seconds": dt, "s_per_iteration": dt / max(res.iterations, 1),
           "iterations_per_s": max(res.iterations, 1) / dt, "impl": "reference kpl.solve", **host()}
    print(json.dumps(out), flush=True)


def config1():
    A = kpl.laplacian_2d(200, 200)
    b = kpl.spmv(A, np.full(A.n, 1.0 / math.sqrt(A.n)))
    for m, sh in (("cg", 0.0), ("pcg", 0.0), ("pcg_sh", 2.1320754716981134), ("pcg_rr", 0.0)):
        run("1", A, None, b, m, sh, 2000, 1e-12)


def as_ref(A):
    return kpl.SparseMatrix(A.n, np.asarray(A.row_ptr, dtype=np.int64), np.asarray(A.col_idx, dtype=np.int64),
                            np.asarray(A.values, dtype=np.float64))


def config2(full):
    A = kpl.laplacian_2d(2048, 2048)
    M = kpl.make_jacobi(A)
    b = kpl.spmv(A, np.random.default_rng(0).random(A.n))
    it = 20000 if full else 200
    run("2" if full else "2 (200-iteration rate)", A, M, b, "pcg_sh", 0.49238826317067413, it,
        1e-10 if full else 0.0)
    if full:
        run("2", A, M, b, "cg", 0.0, it, 1e-10)


def config4():
    from paper_1706_05988_b200 import problems
    A = as_ref(problems.varcoef_3d(256, seed=0, check_symmetry=False))
    M = kpl.make_jacobi(A)
    b = np.random.default_rng(1).standard_normal(A.n)
    run("4 (50-iteration rate)", A, M, b, "pcg_sh", 0.49238826317067413, 50, 0.0)


def config5():
    from paper_1706_05988_b200 import problems
    A = as_ref(problems.banded_spd(2_000_000, seed=0))
    M = kpl.make_jacobi(A)
    b = kpl.spmv(A, np.random.default_rng(1).standard_normal(A.n))
    for m, sh in (("cg", 0.0), ("pcg", 0.0), ("pcg_sh", 0.4124626382901352), ("pcg_rr", 0.0)):
        run("5", A, M, b, m, sh, 2000, 1e-10)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,5,2,4")
    ap.add_argument("--full2", action="store_true")
    a = ap.parse_args()
    for c in a.configs.split(","):
        {"1": config1, "2": lambda: config2(a.full2), "4": config4, "5": config5}[c]()
