"""Device time of N iteration sweeps (no result check) -- A/B timing helper."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1706_05988_b200 as K
from paper_1706_05988_b200 import problems
from paper_1706_05988_b200.solvers import _Solve
probs = {
    "c2c": (K.laplacian_2d(2048, 2048), np.random.default_rng(0).random(2048 * 2048)),
    "c4": (problems.varcoef_3d(256, seed=0, check_symmetry=False), np.random.default_rng(1).standard_normal(256 ** 3)),
    "c5": (problems.banded_spd(2_000_000, seed=0), np.random.default_rng(1).standard_normal(2_000_000)),
}
for name, (A, v) in probs.items():
    M = K.make_jacobi(A)
    b = torch.as_tensor(v, device="cuda")
    S = _Solve(A, M, b, None, K.SolverConfig(method="pcg_sh", shift=0.4, max_iters=100))
    S.init(); S.iterate(1); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); S.iterate(9); e1.record(); torch.cuda.synchronize()
    print(name, os.path.basename(os.environ.get("KPL_LIB", "default")), f"{e0.elapsed_time(e1)/9:.4f} ms/sweep")
