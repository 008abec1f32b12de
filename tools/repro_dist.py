"""Repro of a distributed fuzz mismatch: compare the 1-GPU solve (persistent
and launches) with P virtual ranks through every exchange path."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_1706_05988_b200 as K
from paper_1706_05988_b200.distributed import LocalComm, LocalPeerComm, SlabPlan, solve_distributed
from paper_1706_05988_b200.solvers import _Solve

dims = tuple(int(v) for v in os.environ.get("DIMS", "40,6,33").split(","))
P, zc = int(os.environ.get("P", "3")), int(os.environ.get("ZC", "1"))
method = os.environ.get("METHOD", "pcg")
A = K.Stencil3D(*dims)
b = np.random.default_rng(0).standard_normal(A.n)
cfg = K.SolverConfig(method=method, max_iters=110, rtol=1e-12)
plan = SlabPlan(*dims, P, zc)
h = lambda r: [(x.alpha, x.beta, x.rnorm_true) for x in r.history]
ref_l = _Solve(A, None, b, None, cfg, zc=zc, slab_view=True, persistent=False).run()
ref_p = _Solve(A, None, b, None, cfg, zc=zc, slab_view=True, persistent=True).run()
print("persistent == launches:", h(ref_p) == h(ref_l), ref_p.iterations, ref_l.iterations)
for name, comm in [("LocalComm", LocalComm(P)), ("peer fused", LocalPeerComm(P)), ("peer post", LocalPeerComm(P, fused=False))]:
    res = solve_distributed(A, None, [b[plan.local_slice(r)] for r in range(P)], None, cfg, comm=comm, zc=zc)
    hh = h(res)
    d = next((i for i, (u, v) in enumerate(zip(hh, h(ref_l))) if u != v), None)
    print(f"{name}: iterations {res.iterations} vs {ref_l.iterations}; first differing row {d}", hh[d] if d is not None else "", h(ref_l)[d] if d is not None else "")
