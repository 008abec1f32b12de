"""ms/iteration of the CSR configs (2-CSR, 4, 5) for A/B builds."""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1706_05988_b200 as K
from paper_1706_05988_b200 import problems
dev = "cuda"
probs = {}
probs["c2c"] = (K.laplacian_2d(2048, 2048), np.random.default_rng(0).random(2048 * 2048), 0.49238826317067413)
probs["c4"] = (problems.varcoef_3d(256, seed=0, check_symmetry=False), np.random.default_rng(1).standard_normal(256 ** 3), 0.49238826317067413)
probs["c5"] = (problems.banded_spd(2_000_000, seed=0), np.random.default_rng(1).standard_normal(2_000_000), 0.4124626382901352)
for name, (A, v, sig) in probs.items():
    M = K.make_jacobi(A)
    b = torch.as_tensor(v, device=dev)
    cfg = K.SolverConfig(method="pcg_sh", shift=sig, max_iters=60)
    K.solve(A, M, b, None, cfg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); r = K.solve(A, M, b, None, cfg); e1.record(); torch.cuda.synchronize()
    print(name, os.environ.get("KPL_LIB", "default"), f"{e0.elapsed_time(e1)/60:.4f} ms/iter", r.history[-1].rnorm_recursive)
