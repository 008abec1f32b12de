"""Repeat whole solves while another stream keeps the GPU busy; every repeat must reproduce the first run's
history and x bit for bit (races in the producer/consumer kernels show up as rare differences).

    python tools/stress_solve.py [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1706_05988_b200 as K  # noqa: E402
from paper_1706_05988_b200 import problems  # noqa: E402

REPS = int(sys.argv[1]) if len(sys.argv) > 1 else 20


def hist(res):
    f = lambda v: np.nan if v is None else v
    return np.array([[f(r.alpha), f(r.beta), f(r.gamma), f(r.delta), f(r.rnorm_recursive), f(r.rnorm_true)]
                     for r in res.history], dtype=np.float64)


CASES = [
    ("tma3d 128^3 pcg_sh", lambda: (K.Stencil3D(128, 128, 128), None), dict(method="pcg_sh", shift=2.3, max_iters=120, rtol=0.0), "tree"),
    ("tma2d 1024x512 jacobi pcg_sh", lambda: (K.Stencil2D(1024, 512), "jacobi"), dict(method="pcg_sh", shift=0.49, max_iters=150, rtol=0.0), "tree"),
    ("register 3d 65x40x33 pcg_rr", lambda: (K.Stencil3D(65, 40, 33), None), dict(method="pcg_rr", max_iters=150, rtol=1e-12), "tree"),
    ("persistent 200^2 pcg_sh", lambda: (K.Stencil2D(200, 200), None), dict(method="pcg_sh", shift=2.13, max_iters=450, rtol=1e-12), "tree"),
    ("csr band 400k pcg_sh", lambda: (problems.banded_spd(400_000, seed=2), "jacobi"), dict(method="pcg_sh", shift=0.41, max_iters=60, rtol=1e-10), "tree"),
    ("csr band 400k cg", lambda: (problems.banded_spd(400_000, seed=2), "jacobi"), dict(method="cg", max_iters=60, rtol=1e-10), "tree"),
    ("csr band 400k pcg_rr", lambda: (problems.banded_spd(400_000, seed=2), "jacobi"), dict(method="pcg_rr", max_iters=60, rtol=1e-10), "tree"),
    ("csr varcoef 48^3 pcg_sh", lambda: (problems.varcoef_3d(48, seed=1), "jacobi"), dict(method="pcg_sh", shift=0.49, max_iters=200, rtol=1e-10), "tree"),
    ("reference order 512x256 pcg_sh", lambda: (K.Stencil2D(512, 256), None), dict(method="pcg_sh", shift=1.5, max_iters=30, rtol=0.0), "reference"),
    ("ic0 lap 60x50 pcg_sh", lambda: (K.laplacian_2d(60, 50), "ic0"), dict(method="pcg_sh", shift=0.3, max_iters=80, rtol=1e-10), "tree"),
]

side = torch.cuda.Stream()
junk = torch.empty(48 << 20, dtype=torch.float64, device="cuda")
total_bad = 0
for name, make, kw, order in CASES:
    A, mk = make()
    M = {"jacobi": K.make_jacobi, "ic0": K.make_ic0}.get(mk, lambda a: None)(A)
    b = torch.as_tensor(np.random.default_rng(3).standard_normal(A.n), device="cuda")
    first = None
    bad = 0
    with K.reduction_order(order):
        for rep in range(REPS):
            with torch.cuda.stream(side):
                junk.normal_()
                junk.mul_(1.0001)
            res = K.solve(A, M, b, None, K.SolverConfig(**kw))
            cur = (hist(res).tobytes(), res.x.cpu().numpy().tobytes(), res.iterations)
            if first is None:
                first = cur
            elif cur != first:
                bad += 1
    total_bad += bad
    print(f"{name}: {bad}/{REPS - 1} repeats differ", flush=True)
torch.cuda.synchronize()
print("stress_solve:", "FAILED" if total_bad else "ok", flush=True)
