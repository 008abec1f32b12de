"""Device time of N fused 3D iteration sweeps at 512^3 (A/B timing helper)."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1706_05988_b200 as K
from paper_1706_05988_b200.solvers import _Solve
N = int(os.environ.get("N3", "512"))
A = K.Stencil3D(N, N, N)
b = K.spmv(A, torch.full((A.n,), 1 / math.sqrt(A.n), dtype=torch.float64, device="cuda"))
for rep in range(2):
    S = _Solve(A, None, b, None, K.SolverConfig(method="pcg_sh", shift=2.3, max_iters=100))
    S.init(); S.iterate(1); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); S.iterate(9); e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 9
    print(os.path.basename(os.environ.get("KPL_LIB", "default")), f"{t:.4f} ms/sweep",
          f"{96 * A.n / t / 1e6:.0f} GB/s")
