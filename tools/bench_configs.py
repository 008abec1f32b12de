#!/usr/bin/env python3
"""Per-config device measurements for every BASELINE.json config (1 GPU).

For each config: build the operator/rhs exactly as BASELINE.json describes,
run the requested solvers through the drop-in API, and report iterations,
final true relative residual, device ms/iteration (CUDA events around the
solve, init included) and the algorithmic GB/s of the iteration sweep.

Reference numbers for the parity targets come from SURVEY.md Appendix B
(the unmodified reference run in the build container):
  config 1: p-CG-sh 450 it, 9.466e-13;  config 2: p-CG-sh 4764 it, 9.949e-11;
  config 5: p-CG-sh 88 it, 5.746e-11.

    python tools/bench_configs.py [--configs 1,2,4,5] > profiles/rNN_configs.jsonl
"""

import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1706_05988_b200 as K  # noqa: E402
from paper_1706_05988_b200 import problems  # noqa: E402

REF = {  # (iterations, final true relative residual)
    ("1", "cg"): (450, 9.480e-13), ("1", "pcg"): (491, 2.373e-11),
    ("1", "pcg_sh"): (450, 9.466e-13), ("1", "pcg_rr"): (450, 9.55e-13),
    ("2", "cg"): (4764, 9.949e-11), ("2", "pcg"): (4764, 7.607e-10),
    ("2", "pcg_sh"): (4764, 9.949e-11),
    # config 5: the unmodified reference's kpl.solve on the same arrays (profiles/r02_reference_cpu.jsonl)
    ("5", "cg"): (88, 4.551026644281697e-11), ("5", "pcg"): (88, 4.5673596921911305e-11),
    ("5", "pcg_sh"): (88, 4.551026657642009e-11), ("5", "pcg_rr"): (88, 4.551026319857749e-11),
    # config 4 (256^3): the full-size oracle in the reference order (tests/golden/config4_oracle_*.npz,
    # tools/oracle_fullsize.py); the sigma* = 0.49238826317067413 of the rule at 256^3
    # (profiles/r02_sigma_config4.jsonl) -- every sigma > 0 of the sweep is held to CG's target
    ("4", "cg"): (2960, 1.0581659160347994e-12),
    ("4", "pcg_sh x0.25"): (2960, 1.0581659160347994e-12), ("4", "pcg_sh x0.5"): (2960, 1.0581659160347994e-12),
    ("4", "pcg_sh x1.0"): (2960, 1.0581659160347994e-12),
}


def timed_solve(A, M, b, cfg):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = K.solve(A, M, b, None, cfg)
    e1.record()
    torch.cuda.synchronize()
    return res, e0.elapsed_time(e1) / 1000.0


def report(cfgname, form, method, sigma, A, M, b, cfg, bytes_per_iter, bnorm):
    K.solve(A, M, b, None, K.SolverConfig(method=cfg.method, shift=cfg.shift, max_iters=3,
                                          rtol=0.0))          # warm-up (JIT-free, allocator warm)
    res, t = timed_solve(A, M, b, cfg)
    fin = res.history[-1].rnorm_true / bnorm
    it = res.iterations
    out = {"config": cfgname, "form": form, "method": method, "sigma": sigma, "n": A.n,
           "iterations": it, "converged": res.converged, "final_true_rel": fin,
           "seconds": t, "ms_per_iter": 1000 * t / max(it, 1),
           "alg_gbs_iter_sweep": bytes_per_iter * it / t / 1e9 if it else None,
           "replacements": len(res.replacements)}
    ref = REF.get((cfgname, method))
    if ref:
        out["ref_iterations"], out["ref_final_true_rel"] = ref
        out["iters_within_2pct"] = abs(it - ref[0]) <= 0.02 * ref[0]
        out["residual_within_2x"] = (fin <= 2 * ref[1]) and (fin >= ref[1] / 2)
    print(json.dumps(out), flush=True)


def dev(v):
    return torch.as_tensor(v, dtype=torch.float64, device="cuda")


def config1():
    sig = 2.1320754716981134
    for form, A in (("stencil", K.Stencil2D(200, 200)), ("csr", K.laplacian_2d(200, 200))):
        b = K.spmv(A, dev(np.full(A.n, 1 / math.sqrt(A.n))))
        bn = math.sqrt(K.dot(b, b, A))
        for m in ("cg", "pcg", "pcg_sh", "pcg_rr"):
            cfg = K.SolverConfig(method=m, shift=sig if m == "pcg_sh" else 0.0, max_iters=2000, rtol=1e-12)
            report("1", form, m, cfg.shift, A, None, b, cfg, 96 * A.n, bn)


def config2():
    sig = 0.49238826317067413
    xh = np.random.default_rng(0).random(2048 * 2048)
    for form, A in (("stencil", K.Stencil2D(2048, 2048)), ("csr", K.laplacian_2d(2048, 2048))):
        M = K.make_jacobi(A)
        b = K.spmv(A, dev(xh))
        bn = math.sqrt(K.dot(b, b, A))
        per = 144 * A.n if form == "stencil" else 152 * A.n + 12 * A.nnz + 4 * (A.n + 1)
        for m in ("pcg_sh", "cg"):
            cfg = K.SolverConfig(method=m, shift=sig if m == "pcg_sh" else 0.0, max_iters=20000, rtol=1e-10)
            report("2", form, m, cfg.shift, A, M, b, cfg, per, bn)


def config4():
    t0 = time.time()
    A = problems.varcoef_3d(256, seed=0, check_symmetry=False)
    print(json.dumps({"config": "4", "setup_s": time.time() - t0, "nnz": A.nnz}), flush=True)
    M = K.make_jacobi(A)
    b = dev(np.random.default_rng(1).standard_normal(A.n))
    bn = math.sqrt(K.dot(b, b, A))
    per = 152 * A.n + 12 * A.nnz + 4 * (A.n + 1)
    sig_star = 0.49238826317067413   # the rule at 256^3 (tools/sigma_config4.py, profiles/r02_sigma_config4.jsonl)
    for f in (0.25, 0.5, 1.0):
        cfg = K.SolverConfig(method="pcg_sh", shift=f * sig_star, max_iters=20000, rtol=1e-12)
        report("4", "csr", f"pcg_sh x{f}", cfg.shift, A, M, b, cfg, per, bn)
    # sigma = 0 (plain p-CG): stagnates above 1e-12, so capped; the run is also the rule's history
    cfg = K.SolverConfig(method="pcg", max_iters=60000, rtol=1e-12)
    report("4", "csr", "pcg_sh x0 (= pcg, capped 60000)", 0.0, A, M, b, cfg, per, bn)
    cfg = K.SolverConfig(method="cg", max_iters=20000, rtol=1e-12)
    report("4", "csr", "cg", 0.0, A, M, b, cfg, per, bn)


def config5():
    t0 = time.time()
    A = problems.banded_spd(2_000_000, seed=0)
    print(json.dumps({"config": "5", "setup_s": time.time() - t0, "nnz": A.nnz}), flush=True)
    M = K.make_jacobi(A)
    xh = np.random.default_rng(1).standard_normal(A.n)
    b = K.spmv(A, dev(xh))
    bn = math.sqrt(K.dot(b, b, A))
    per = 152 * A.n + 12 * A.nnz + 4 * (A.n + 1)
    for m in ("cg", "pcg", "pcg_sh", "pcg_rr"):
        cfg = K.SolverConfig(method=m, shift=0.4124626382901352 if m == "pcg_sh" else 0.0,
                             max_iters=2000, rtol=1e-10)
        report("5", "csr", m, cfg.shift, A, M, b, cfg, per, bn)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,5,4")
    args = ap.parse_args()
    fns = {"1": config1, "2": config2, "4": config4, "5": config5}
    for c in args.configs.split(","):
        fns[c]()


if __name__ == "__main__":
    main()
