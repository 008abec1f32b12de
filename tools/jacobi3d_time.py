"""Per-sweep time of the fused iteration with a constant-diagonal Jacobi
(8 TMA streams, 144 B/DOF) on 3D grids vs the 2D 2048^2 case."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1706_05988_b200 as K
from paper_1706_05988_b200.solvers import _Solve
for name, A in [("3D512-jacobi", K.Stencil3D(512, 512, 512)), ("3D384-jacobi", K.Stencil3D(384, 384, 384)),
                ("2D2048-jacobi", K.Stencil2D(2048, 2048)), ("2D4096-jacobi", K.Stencil2D(4096, 4096))]:
    M = K.make_jacobi(A)
    b = K.spmv(A, torch.full((A.n,), 1 / math.sqrt(A.n), dtype=torch.float64, device="cuda"))
    S = _Solve(A, M, b, None, K.SolverConfig(method="pcg_sh", shift=0.5, max_iters=100))
    S.init(); S.iterate(1); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); S.iterate(9); e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 9
    print(name, f"{t*1e3:.1f} us/sweep", f"{144 * A.n / t / 1e6:.0f} GB/s", flush=True)
    del S, b
    torch.cuda.empty_cache()
