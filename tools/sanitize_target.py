#!/usr/bin/env python3
"""Small runs of every kernel family, for compute-sanitizer.

    compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck \\
        python tools/sanitize_target.py [family ...]

Families: tma (TMA-fed 3D sweep), reg (register stencil sweep), persist
(persistent small-problem solver), csr (split CSR SpMV + chunk sweep, pipelined
SpMV), sorted (column-sorted SpMV), band (window SpMV), ic0 (IC(0) factor +
substitution sweeps), peer (virtual-rank peer exchange: fused sweep with the
deferred fold, post kernels, finalize), order (reference reduction order).
Each runs a few iterations and checks the result against a second run of the
same solve (bitwise), so a sanitizer-visible fault also shows as a mismatch.
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1706_05988_b200 as K  # noqa: E402
from paper_1706_05988_b200 import problems  # noqa: E402


def same(a, b):
    return all((x.alpha, x.beta, x.gamma, x.delta, x.rnorm_recursive) ==
               (y.alpha, y.beta, y.gamma, y.delta, y.rnorm_recursive) for x, y in zip(a.history, b.history))


def solve_twice(A, M, b, **kw):
    cfg = K.SolverConfig(**kw)
    r1 = K.solve(A, M, b, None, cfg)
    r2 = K.solve(A, M, b, None, cfg)
    assert same(r1, r2), "repeat mismatch"
    return r1


def tma():
    os.environ["KPL_NO_PERSISTENT"] = "1"        # small grids: force the per-sweep TMA launches
    A = K.Stencil3D(64, 16, 12)
    b = K.spmv(A, np.random.default_rng(0).standard_normal(A.n))
    solve_twice(A, None, b, method="pcg_sh", shift=1.0, max_iters=12, rtol=0.0)
    A2 = K.Stencil2D(1024, 40)
    solve_twice(A2, K.make_jacobi(A2), np.ones(A2.n), method="pcg_sh", shift=0.4, max_iters=12, rtol=0.0)
    del os.environ["KPL_NO_PERSISTENT"]


def reg():
    A = K.Stencil3D(33, 9, 20)          # odd nx: register sweep (rr / gaps: never persistent)
    solve_twice(A, None, np.ones(A.n), method="pcg_rr", max_iters=12, rtol=0.0)
    solve_twice(A, None, np.ones(A.n), method="cg", max_iters=12, rtol=0.0, track_gaps=True)


def persist():
    A = K.Stencil2D(60, 50)
    solve_twice(A, None, np.ones(A.n), method="pcg_sh", shift=2.0, max_iters=40, rtol=1e-12)


def csr():
    A = problems.varcoef_3d(10, seed=1)
    solve_twice(A, K.make_jacobi(A), np.ones(A.n), method="pcg_sh", shift=0.5, max_iters=15, rtol=0.0)
    B = problems.banded_spd(6000, seed=2, band=900)
    solve_twice(B, K.make_jacobi(B), np.ones(B.n), method="pcg_rr", max_iters=15, rtol=0.0)


def sorted_():
    os.environ["KPL_CSR_GATHER"] = "sorted"
    B = problems.banded_spd(9000, seed=3, band=3000)
    solve_twice(B, K.make_jacobi(B), np.ones(B.n), method="pcg_sh", shift=0.4, max_iters=10, rtol=0.0)
    os.environ["KPL_CSR_GATHER"] = "csr"


def ic0():
    A = K.laplacian_2d(30, 20)
    M = K.make_ic0(A)
    solve_twice(A, M, np.ones(A.n), method="pcg_sh", shift=0.3, max_iters=10, rtol=0.0)


def peer():
    from paper_1706_05988_b200.distributed import LocalPeerComm, SlabPlan, solve_distributed
    A = K.Stencil3D(64, 16, 16)
    b = K.spmv(A, np.random.default_rng(1).standard_normal(A.n))
    plan = SlabPlan(64, 16, 16, 2, 4)
    for fused, fold in ((True, True), (True, False), (False, False)):
        cfg = K.SolverConfig(method="pcg_sh", shift=1.0, max_iters=14, rtol=0.0)
        solve_distributed(A, None, [b[plan.local_slice(r)] for r in range(2)], None, cfg,
                          comm=LocalPeerComm(2, fused=fused, fold=fold), zc=4)
    torch.cuda.synchronize()


def order():
    A = K.laplacian_2d(40, 30)
    with K.reduction_order("reference"):
        solve_twice(A, None, np.ones(A.n), method="pcg_sh", shift=1.0, max_iters=10, rtol=0.0)


FAMILIES = {"tma": tma, "reg": reg, "persist": persist, "csr": csr, "sorted": sorted_, "ic0": ic0,
            "peer": peer, "order": order}

if __name__ == "__main__":
    for f in (sys.argv[1:] or list(FAMILIES)):
        FAMILIES[f]()
        torch.cuda.synchronize()
        print("ok", f, flush=True)
