"""Where does the e2e time go?  (pinned alloc, H2D, D2H, solve)"""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1706_05988_b200 as K

n = 512 ** 3
dev = torch.device("cuda", 0)
ev = lambda: torch.cuda.Event(enable_timing=True)
for rep in range(3):
    t0 = time.perf_counter()
    h = torch.empty(n, dtype=torch.float64, pin_memory=True)
    t1 = time.perf_counter()
    print(f"pinned alloc 1 GiB: {1e3*(t1-t0):.1f} ms")
    del h
d = torch.ones(n, dtype=torch.float64, device=dev)
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
for rep in range(3):
    a, b = ev(), ev()
    a.record(); d2 = h.to(dev, non_blocking=True); b.record(); torch.cuda.synchronize()
    print(f"H2D 1 GiB: {a.elapsed_time(b):.1f} ms  ({8*n/a.elapsed_time(b)/1e6:.1f} GB/s)")
    a, b = ev(), ev()
    a.record(); h.copy_(d, non_blocking=True); b.record(); torch.cuda.synchronize()
    print(f"D2H 1 GiB: {a.elapsed_time(b):.1f} ms  ({8*n/a.elapsed_time(b)/1e6:.1f} GB/s)")
A = K.Stencil3D(512, 512, 512)
b = K.spmv(A, torch.full((n,), 1 / math.sqrt(n), dtype=torch.float64, device=dev))
cfg = K.SolverConfig(method="pcg_sh", shift=2.30188679245283, max_iters=500)
bh = torch.empty(n, dtype=torch.float64, pin_memory=True); bh.copy_(b)
for kind, arg in (("device", b), ("host", bh), ("device", b), ("host", bh)):
    torch.cuda.synchronize()
    a, c = ev(), ev()
    t0 = time.perf_counter()
    a.record(); r = K.solve(A, None, arg, None, cfg); c.record(); torch.cuda.synchronize()
    print(f"solve {kind}: {a.elapsed_time(c):.1f} ms (wall {1e3*(time.perf_counter()-t0):.1f})")
