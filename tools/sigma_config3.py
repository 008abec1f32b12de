"""Config 3's shift from the reference's selection rule, recomputed at full size
('recompute it there from the p-CG history at i=500'): device
p-CG, 500 iterations, then the host-side psi sweep + margin rule (shift.py)."""
import json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1706_05988_b200 as K
from paper_1706_05988_b200 import shift

order = os.environ.get("SIGMA_ORDER", "tree")
K.set_reduction_order(order)
for N in [int(v) for v in os.environ.get("SIGMA_N", "128,256,512").split(",")]:
    A = K.Stencil3D(N, N, N)
    b = K.spmv(A, torch.full((A.n,), 1 / math.sqrt(A.n), dtype=torch.float64, device="cuda"))
    t0 = time.perf_counter()
    sigma, sw, base = shift.choose_shift(A, None, b, max_iters=500, rtol=0.0)
    t1 = time.perf_counter()
    bn = float(torch.linalg.norm(b))
    k = int(sw.psi_values.argmin())
    sh = K.solve(A, None, b, None, K.SolverConfig(method="pcg_sh", shift=sigma, max_iters=500, rtol=0.0))
    print(json.dumps({"N": N, "order": order, "sigma": sigma, "psi_at_sigma": float(sw.psi_values[list(sw.grid).index(sigma)]),
                      "argmin": float(sw.grid[k]), "psi_min": float(sw.psi_values[k]),
                      "psi_at_0": float(sw.psi_values[0]),
                      "pcg_true_rel_500": base.history[-1].rnorm_true / bn,
                      "pcg_sh_true_rel_500": sh.history[-1].rnorm_true / bn,
                      "seconds_pcg_plus_sweep": t1 - t0}), flush=True)
    del b, base, sh
    torch.cuda.empty_cache()
