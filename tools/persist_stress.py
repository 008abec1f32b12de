"""Stress the persistent small-problem solver: repeat one solve and compare
its history and x with the per-iteration-launch path (bitwise)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_05988_b200 as K  # noqa: E402
from paper_1706_05988_b200.solvers import _Solve  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
A = K.Stencil3D(64, 24, 32)
b = K.spmv(A, np.random.default_rng(2).normal(size=A.n))
cfg = K.SolverConfig(method="pcg_sh", shift=2.30188679245283, max_iters=80, rtol=1e-10)
ref = _Solve(A, None, b, None, cfg, zc=4, slab_view=True, persistent=False).run()
print("reference done", flush=True)
bad = 0
for i in range(reps):
    res = _Solve(A, None, b, None, cfg, zc=4, slab_view=True, persistent=True).run()
    h1 = [(r.alpha, r.rnorm_true) for r in res.history]
    h0 = [(r.alpha, r.rnorm_true) for r in ref.history]
    print(f"rep {i} done", flush=True) if i < 3 else None
    ok = h1 == h0 and np.asarray(res.x).tobytes() == np.asarray(ref.x).tobytes()
    if not ok:
        bad += 1
        d = [k for k, (a, c) in enumerate(zip(h1, h0)) if a != c]
        print(f"rep {i}: mismatch rows {d[:10]}", flush=True)
print(f"persistent stress: {bad}/{reps} mismatching", flush=True)
