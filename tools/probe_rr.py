"""Small pcg_rr run on a banded CSR matrix (for launch-list profiling)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1706_05988_b200 as K  # noqa: E402
from paper_1706_05988_b200 import problems  # noqa: E402

A = problems.banded_spd(400_000, seed=0, band=10_000)
M = K.make_jacobi(A)
b = torch.as_tensor(np.random.default_rng(1).standard_normal(A.n), device="cuda")
for m in ("pcg_sh", "pcg_rr"):
    K.solve(A, M, b, None, K.SolverConfig(method=m, max_iters=5))
    torch.cuda.synchronize()
    t = time.time()
    r = K.solve(A, M, b, None, K.SolverConfig(method=m, max_iters=30))
    torch.cuda.synchronize()
    print(m, r.iterations, (time.time() - t) / 30 * 1e3, "ms/iter", r.replacements)
