"""Time `count` persistent iterations of config 1 (kernel components A/B)."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1706_05988_b200 as K
from paper_1706_05988_b200.solvers import _Solve
A = K.Stencil2D(200, 200)
b = K.spmv(A, torch.full((A.n,), 1 / math.sqrt(A.n), dtype=torch.float64, device="cuda"))
cfg = K.SolverConfig(method="pcg_sh", shift=2.1320754716981134, max_iters=2000, rtol=0.0)
for rep in range(3):
    S = _Solve(A, None, b, None, cfg, persistent=True)
    S.init()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); S.iterate(400); e1.record(); torch.cuda.synchronize()
    print(f"{os.environ.get('KPL_LIB','default')}: 400 it {e0.elapsed_time(e1):.3f} ms = {e0.elapsed_time(e1)/400*1e3:.2f} us/it")
