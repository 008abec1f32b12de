"""Per-sweep time of the fused iteration vs the chunk length zc (2D / 3D)."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1706_05988_b200 as K
from paper_1706_05988_b200.solvers import _Solve
cases = [("2D2048-jacobi", K.Stencil2D(2048, 2048), True), ("3D512", K.Stencil3D(512, 512, 512), False)]
if os.environ.get("ZC_2D_ONLY"):
    cases = cases[:1]
for name, A, jac in cases:
    M = K.make_jacobi(A) if jac else None
    b = K.spmv(A, torch.as_tensor(np.random.default_rng(0).random(A.n), device="cuda"))
    per = (144 if jac else 96) * A.n
    zcs = [int(z) for z in os.environ.get("ZCS", "1,2,4,8,16,32").split(",")]
    for zc in zcs:
        S = _Solve(A, M, b, None, K.SolverConfig(method="pcg_sh", shift=0.5, max_iters=100), zc=zc)
        S.init(); S.iterate(1); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); S.iterate(9); e1.record(); torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 9
        print(name, "zc", zc, f"{t*1e3:.1f} us/sweep", f"{per / t / 1e6:.0f} GB/s", flush=True)
