"""Where a config-3 solve's time goes: device time of init, of the iteration
chunks (incl. cadence) and of the whole K.solve call, CUDA events."""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1706_05988_b200 as K
from paper_1706_05988_b200.solvers import _Solve
A = K.Stencil3D(512, 512, 512)
b = K.spmv(A, torch.full((A.n,), 1 / math.sqrt(A.n), dtype=torch.float64, device="cuda"))
cfg = K.SolverConfig(method="pcg_sh", shift=2.30188679245283, max_iters=500, rtol=0.0)
for rep in range(3):
    K.solve(A, None, b, None, cfg)
E = lambda: torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0, e1 = E(), E()
e0.record(); K.solve(A, None, b, None, cfg); e1.record(); torch.cuda.synchronize()
print(f"K.solve total {e0.elapsed_time(e1):.2f} ms")
t0 = time.perf_counter()
S = _Solve(A, None, b, None, cfg)
torch.cuda.synchronize(); t1 = time.perf_counter()
a0, a1 = E(), E()
a0.record(); S.init(); a1.record(); torch.cuda.synchronize()
print(f"_Solve() host {1e3*(t1-t0):.2f} ms; init {a0.elapsed_time(a1):.2f} ms")
tot = 0.0
chunk = 8
while S.issued < S.limit:
    c0, c1 = E(), E()
    c0.record(); S.iterate(chunk); c1.record(); torch.cuda.synchronize()
    tot += c0.elapsed_time(c1)
    chunk = min(chunk * 2, 256)
print(f"iterate chunks {tot:.2f} ms = {tot / 500:.4f} ms/iteration")
r0, r1 = E(), E()
r0.record(); res = S.result(); r1.record(); torch.cuda.synchronize()
print(f"result {r0.elapsed_time(r1):.2f} ms")
S = _Solve(A, None, b, None, cfg)
S.init(); S.iterate(1); torch.cuda.synchronize()
c0, c1, c2 = E(), E(), E()
c0.record(); S.iterate(9); c1.record(); S.iterate(10); c2.record(); torch.cuda.synchronize()
t9, t10 = c0.elapsed_time(c1), c1.elapsed_time(c2)
print(f"9 ITER {t9:.3f} ms ({t9/9:.4f}/it); TRUE + 10 ITER {t10:.3f} ms -> TRUE ~ {t10 - 10 * t9 / 9:.3f} ms")
