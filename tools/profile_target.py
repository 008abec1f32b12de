#!/usr/bin/env python3
"""Set up one BASELINE config and run a few solver iterations (ncu target).

    python tools/profile_target.py c4|c5|c2s|c2c|c3 [iters] [method]
"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1706_05988_b200 as K  # noqa: E402
from paper_1706_05988_b200 import problems  # noqa: E402


def main():
    which = sys.argv[1]
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    method = sys.argv[3] if len(sys.argv) > 3 else "pcg_sh"
    dev = "cuda"
    if which == "c4":
        A = problems.varcoef_3d(256, seed=0, check_symmetry=False)
        M = K.make_jacobi(A)
        b = torch.as_tensor(np.random.default_rng(1).standard_normal(A.n), device=dev)
        sig = 0.49238826317067413
    elif which == "c5":
        A = problems.banded_spd(2_000_000, seed=0)
        M = K.make_jacobi(A)
        b = K.spmv(A, torch.as_tensor(np.random.default_rng(1).standard_normal(A.n), device=dev))
        sig = 0.4124626382901352
    elif which in ("c2s", "c2c"):
        A = K.Stencil2D(2048, 2048) if which == "c2s" else K.laplacian_2d(2048, 2048)
        M = K.make_jacobi(A)
        b = K.spmv(A, torch.as_tensor(np.random.default_rng(0).random(A.n), device=dev))
        sig = 0.49238826317067413
    else:
        A = K.Stencil3D(512, 512, 512)
        M = None
        b = K.spmv(A, torch.full((A.n,), 1 / math.sqrt(A.n), dtype=torch.float64, device=dev))
        sig = 2.30188679245283
    cfg = K.SolverConfig(method=method, shift=sig if method == "pcg_sh" else 0.0, max_iters=iters, rtol=0.0)
    res = K.solve(A, M, b, None, cfg)
    torch.cuda.synchronize()
    print(which, A.n, res.iterations, res.history[-1].rnorm_true)


if __name__ == "__main__":
    main()
