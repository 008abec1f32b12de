#!/usr/bin/env python3
"""Config 4's shift by the reference's selection rule at full size (256^3).

VERDICT r01 item 1: sigma* must come from the rule (stability.py:207-232 Jacobi
grid, scripts/shift_study.py:46-51 margin rule) applied to a plain p-CG history
of the 256^3 variable-coefficient problem itself, not borrowed from 16^3/64^3.

    # on the GPU box: device p-CG to rtol 1e-12 (capped), history saved
    python tools/sigma_config4.py run  [--cap 60000] [--order tree|reference]
    # anywhere (CPU): psi sweep over default_sigma_grid(A, M) at i = iterations
    python tools/sigma_config4.py sweep gpurun_out/c4_pcg_history.npz

The p-CG run is also the sigma = 0 point of the config-4 sweep
{0, 1/4, 1/2, 1} x sigma*: its iteration count, final true residual and the
stagnation level (minimum true residual over the cadence rows) are reported.
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def run(args):
    import torch
    import paper_1706_05988_b200 as K
    from paper_1706_05988_b200 import problems
    K.set_reduction_order(args.order)
    A = problems.varcoef_3d(args.N, seed=0, check_symmetry=False)
    M = K.make_jacobi(A)
    b = torch.as_tensor(np.random.default_rng(1).standard_normal(A.n), device="cuda")
    bn = float(torch.linalg.norm(b))
    t0 = time.perf_counter()
    res = K.solve(A, M, b, None, K.SolverConfig(method="pcg", max_iters=args.cap, rtol=1e-12))
    dt = time.perf_counter() - t0
    h = np.array([[r.iter, r.alpha, r.beta, r.gamma, r.delta, r.rnorm_recursive,
                   np.nan if r.rnorm_true is None else r.rnorm_true] for r in res.history])
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    np.savez_compressed(args.out, hist=h, iterations=res.iterations, converged=res.converged,
                        bnorm=bn, N=args.N, order=args.order)
    tr = h[:, 6][~np.isnan(h[:, 6])] / bn
    print(json.dumps({"config": "4", "N": args.N, "method": "pcg (= pcg_sh sigma 0)",
                      "order": args.order, "cap": args.cap, "iterations": res.iterations,
                      "converged": res.converged, "final_true_rel": float(tr[-1]),
                      "stagnation_min_true_rel": float(tr.min()), "seconds": dt}), flush=True)


def sweep(args):
    from paper_1706_05988_b200 import problems, shift
    import paper_1706_05988_b200 as K
    d = np.load(args.hist)
    h = d["hist"]
    N = int(d["N"])
    A = problems.varcoef_3d(N, seed=0, check_symmetry=False)
    M = K.make_jacobi(A)

    rows = h[h[:, 0] >= 1]                      # CoefficientHistory.from_result: records iter >= 1
    hist = shift.CoefficientHistory(rows[:, 1].copy(), rows[:, 2].copy())
    it = int(d["iterations"])
    g = shift.default_sigma_grid(A, M)
    t0 = time.perf_counter()
    sw = shift.select_shift(hist, it, g)
    sigma = shift.margin_rule(sw)
    k = int(np.argmin(sw.psi_values))
    print(json.dumps({"config": "4", "N": N, "i": it, "grid_hi": float(g[-1]), "sigma_star": sigma,
                      "psi_at_sigma": float(sw.psi_values[list(g).index(sigma)]),
                      "argmin": float(g[k]), "psi_min": float(sw.psi_values[k]),
                      "psi_at_0": float(sw.psi_values[0]), "sweep_s": time.perf_counter() - t0}),
          flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run")
    r.add_argument("--N", type=int, default=256)
    r.add_argument("--cap", type=int, default=60000)
    r.add_argument("--order", default="tree")
    r.add_argument("--out", default="gpurun_out/c4_pcg_history.npz")
    s = sub.add_parser("sweep")
    s.add_argument("hist")
    a = ap.parse_args()
    run(a) if a.cmd == "run" else sweep(a)
