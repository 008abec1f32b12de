"""Stress the persistent solver on a 2D grid (config-1-like); optional
KPL_TRACE=1 prints every C-ABI call (use with CUDA_LAUNCH_BLOCKING=1 to find
a kernel that does not finish)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_05988_b200 as K  # noqa: E402
from paper_1706_05988_b200 import _lib  # noqa: E402
from paper_1706_05988_b200.solvers import _Solve  # noqa: E402

if os.environ.get("KPL_TRACE") == "1":
    lib = _lib.load()

    class Tr:
        def __getattr__(self, name):
            fn = getattr(lib, name)

            def w(*a):
                print("call", name, flush=True)
                return fn(*a)
            return w
    _lib._lib = Tr()

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
nx = int(sys.argv[2]) if len(sys.argv) > 2 else 200
A = K.Stencil2D(nx, nx)
b = np.full(A.n, 1.0 / np.sqrt(A.n))
cfg = K.SolverConfig(method="pcg_sh", shift=4.0, max_iters=500, rtol=0.0)
ref = _Solve(A, None, b, None, cfg, persistent=False).run()
print("reference done", flush=True)
bad = 0
for i in range(reps):
    res = _Solve(A, None, b, None, cfg, persistent=True).run()
    ok = [(r.alpha, r.rnorm_true) for r in res.history] == [(r.alpha, r.rnorm_true) for r in ref.history]
    bad += not ok
    if i < 3 or not ok:
        print(f"rep {i} ok={ok}", flush=True)
print(f"persistent stress 2d: {bad}/{reps} mismatching", flush=True)
