"""Device time of 9 fused iteration sweeps of a stencil problem (A/B timing helper).

    python tools/stencil_iter_time.py [--grid 3d512|2d2048] [--jacobi] [--zc 0,8,14,28]

zc = planes (3D) / rows (2D) per reduction chunk; 0 = the library's default.
"""
import argparse
import ctypes
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1706_05988_b200 as K  # noqa: E402
from paper_1706_05988_b200 import _lib, device as D  # noqa: E402
from paper_1706_05988_b200.solvers import _Solve  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--grid", default="3d512")
ap.add_argument("--jacobi", action="store_true")
ap.add_argument("--zc", default="0")
a = ap.parse_args()
if a.grid.startswith("3d"):
    N = int(a.grid[2:])
    A = K.Stencil3D(N, N, N)
else:
    N = int(a.grid[2:])
    A = K.Stencil2D(N, N)
M = K.make_jacobi(A) if a.jacobi else None
per_dof = 144 if a.jacobi else 96
b = K.spmv(A, torch.full((A.n,), 1 / math.sqrt(A.n), dtype=torch.float64, device="cuda"))
for zc in [int(v) for v in a.zc.split(",")]:
    best = 1e9
    for rep in range(3):
        S = _Solve(A, M, b, None, K.SolverConfig(method="pcg_sh", shift=0.5, max_iters=100), zc=zc,
                   persistent=False)
        lib = _lib.load()
        it = lambda j, k: _lib.check(lib.kpl_solver_iterate(S.op, S.kcfg, S.vecs, j, k, D.ptr(S.ws),
                                                            D.stream_handle()), "iterate")
        S.init(); it(0, 1); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); it(1, 9); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 9)

    out = (ctypes.c_int64 * 8)()
    _lib.load().kpl_reduction_layout(S.op, out)
    print(os.path.basename(os.environ.get("KPL_LIB", "libkpl_b200.so")), a.grid, "jacobi" if a.jacobi else "identity", f"zc={zc} (layout zc={out[3]}, items={out[6] * out[7]})",
          f"{best * 1000:.1f} us/sweep", f"{per_dof * A.n / best / 1e6:.0f} GB/s", flush=True)
