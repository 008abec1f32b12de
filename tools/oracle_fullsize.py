#!/usr/bin/env python3
"""Full-size oracle runs for BASELINE configs 3 and 4 (TEST INFRASTRUCTURE).

VERDICT r01 'Next round' item 1: pin the 512^3 and 256^3 configs against the
reference algorithm at full size.  The oracle (`oracle/kpl_oracle.py`, pinned
bit for bit to the unmodified reference by tests/test_oracle_golden.py) runs in
the reference's own reduction order (blocked_dot, `_kernels.py:15-41`), one
core, and its outputs are committed under tests/golden/ so the `-m gpu` suite
can compare the device run in the reference order bit for bit.

    python tools/oracle_fullsize.py config3            # 512^3, 500 it, ~45 min
    python tools/oracle_fullsize.py config4 cg         # 256^3 var-coef CG to 1e-12
    python tools/oracle_fullsize.py config4 pcg_sh SIG # p-CG-sh at shift SIG

Config 3 (BASELINE.json configs[2]): 3D 7-point 512^3, matrix-free, M = I,
b = A * 1/sqrt(n), x0 = 0, 500 fixed p-CG-sh iterations (rtol 0),
sigma = 2.30188679245283 (profiles/r01_sigma_config3.jsonl).
Config 4 (configs[3]): varcoef_3d(256, seed 0), Jacobi, b ~ N(0,1) from
default_rng(1), x0 = 0, rtol 1e-12.
"""

import hashlib
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import kpl_oracle as O  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
SIGMA3 = 2.30188679245283


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def config3(N=512, iters=500):
    A = O.StencilSpec(N, N, N, 6.0)
    b = O.spmv(A, np.full(A.n, 1.0 / math.sqrt(A.n)))
    t0 = time.time()
    res = O.solve_pcg_shifted(A, None, b, None,
                              O.Config(method="pcg_sh", shift=SIGMA3, max_iters=iters, rtol=0.0))
    dt = time.time() - t0
    bn = math.sqrt(O.blocked_dot(b, b))
    tag = f"c3_{N}"
    out = {f"{tag}_hist": res.history, f"{tag}_iters": res.iterations,
           f"{tag}_xsha": sha(res.x), f"{tag}_bsha": sha(b), f"{tag}_bnorm": bn,
           f"{tag}_x_sum": float(np.sum(res.x)), f"{tag}_seconds": dt}
    np.savez_compressed(os.path.join(GOLD, f"config3_oracle_{N}.npz"), **out)
    print(json.dumps({"config": "3", "N": N, "iterations": res.iterations,
                      "final_true_rel": res.history[-1, 6] / bn, "xsha": sha(res.x),
                      "seconds": dt, "s_per_iter": dt / max(res.iterations, 1)}), flush=True)


def config4(method, sigma=0.0, N=256, max_iters=20000):
    from paper_1706_05988_b200 import problems   # host-side generator (pinned at 8^3 by golden)
    t0 = time.time()
    A = problems.varcoef_3d(N, seed=0, check_symmetry=False)
    Ao = O.CSR(A.n, A.row_ptr, A.col_idx, A.values)
    M = O.make_jacobi(Ao)
    b = np.random.default_rng(1).standard_normal(A.n)
    setup = time.time() - t0
    t0 = time.time()
    res = O.solve(Ao, M, b, None, O.Config(method=method, shift=sigma, max_iters=max_iters,
                                           rtol=1e-12))
    dt = time.time() - t0
    bn = math.sqrt(O.blocked_dot(b, b))
    tag = f"c4_{N}_{method}" + (f"_{sigma!r}" if method == "pcg_sh" else "")
    safe = tag.replace(".", "p")
    out = {"hist": res.history, "iters": res.iterations, "converged": res.converged,
           "xsha": sha(res.x), "bsha": sha(b), "bnorm": bn, "sigma": sigma,
           "a_sha": sha(A.values), "cols_sha": hashlib.sha256(
               np.ascontiguousarray(A.col_idx, dtype=np.int64).tobytes()).hexdigest(),
           "seconds": dt}
    np.savez_compressed(os.path.join(GOLD, f"config4_oracle_{safe}.npz"), **out)
    print(json.dumps({"config": "4", "N": N, "method": method, "sigma": sigma,
                      "iterations": res.iterations, "converged": res.converged,
                      "final_true_rel": res.history[-1, 6] / bn, "setup_s": setup,
                      "seconds": dt, "s_per_iter": dt / max(res.iterations, 1)}), flush=True)


if __name__ == "__main__":
    what = sys.argv[1]
    if what == "config3":
        config3(int(sys.argv[2]) if len(sys.argv) > 2 else 512)
    elif what == "config4":
        m = sys.argv[2]
        s = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
        N = int(sys.argv[4]) if len(sys.argv) > 4 else 256
        config4(m, s, N)
    else:
        raise SystemExit(__doc__)
