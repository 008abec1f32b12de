"""Config-1 style small solves: per-iteration device time of the persistent
path and of per-iteration launches (A/B helper; set KPL_PERSIST_CLUSTER=0 for
the grid-barrier layout)."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1706_05988_b200 as K
from paper_1706_05988_b200.solvers import _Solve
tag = os.environ.get("KPL_PERSIST_CLUSTER", "1")
sizes = [("2D200", K.Stencil2D(200, 200)), ("2D300", K.Stencil2D(300, 300)), ("2D400", K.Stencil2D(400, 400)),
         ("2D600", K.Stencil2D(600, 600)), ("3D48", K.Stencil3D(48, 48, 48)), ("3D64", K.Stencil3D(64, 64, 64)),
         ("3D80", K.Stencil3D(80, 80, 80)), ("3D96", K.Stencil3D(96, 96, 96))]
for name, A in sizes:
    b = K.spmv(A, torch.full((A.n,), 1 / math.sqrt(A.n), dtype=torch.float64, device="cuda"))
    for method, pers in [("pcg_sh", True), ("pcg_sh", False)]:
        cfg = K.SolverConfig(method=method, shift=2.13 if method == "pcg_sh" else 0.0, max_iters=2000, rtol=0.0)
        ts = []
        for rep in range(3):
            S = _Solve(A, None, b, None, cfg, persistent=pers)
            S.init()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); S.iterate(200); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 200 * 1e3)
        print(f"cluster={tag} {name} {method} persistent={pers}: {min(ts):.2f} us/it", flush=True)
