"""Config 1 (200^2, M=I) p-CG-sh solve timing (launch-list target)."""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1706_05988_b200 as K
A = K.Stencil2D(200, 200)
b = K.spmv(A, torch.full((A.n,), 1 / math.sqrt(A.n), dtype=torch.float64, device="cuda"))
cfg = K.SolverConfig(method="pcg_sh", shift=2.1320754716981134, max_iters=2000, rtol=1e-12)
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    r = K.solve(A, None, b, None, cfg)
    torch.cuda.synchronize()
    print(f"solve {1e3*(time.perf_counter()-t):.2f} ms, {r.iterations} it, {1e6*(time.perf_counter()-t)/r.iterations:.1f} us/it")
