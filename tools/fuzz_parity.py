"""Randomised device-vs-oracle parity sweep (tree order, the device's own
layout), bitwise: random stencil shapes / CSR matrices, methods, shifts,
preconditioners, x0, gaps; breakdowns must match too.

    python tools/fuzz_parity.py [cases] [seed]
"""
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import paper_1706_05988_b200 as K  # noqa: E402
from paper_1706_05988_b200 import problems  # noqa: E402
from oracle import kpl_oracle as O  # noqa: E402
from gpu_helpers import gpu_dot, hist6, oracle_hist6, same_bits  # noqa: E402


def random_case(rng):
    kind = str(rng.choice(["s2", "s3", "csr_lap", "csr_rspd", "csr_band"]))
    if kind == "s2":
        A = K.Stencil2D(int(rng.integers(1, 300)), int(rng.integers(1, 120)))
    elif kind == "s3":
        A = K.Stencil3D(int(rng.integers(1, 90)), int(rng.integers(1, 30)), int(rng.integers(1, 40)))
    elif kind == "csr_lap":
        A = K.laplacian_2d(int(rng.integers(1, 90)), int(rng.integers(1, 90)))
    elif kind == "csr_rspd":
        A = K.random_spd(int(rng.integers(2, 120)), cond=float(rng.uniform(2, 1e4)), seed=int(rng.integers(1000)))
    else:
        A = problems.banded_spd(int(rng.integers(300, 30000)), seed=int(rng.integers(1000)),
                                band=int(rng.integers(2, 400)))
    method = str(rng.choice(["cg", "pcg", "pcg_sh", "pcg_rr", "pcg_var_sh"]))
    jac = bool(rng.integers(2))
    gaps = bool(rng.integers(4) == 0)
    maxit = int(rng.integers(1, 120))
    kw = dict(method=method, max_iters=maxit, rtol=float(rng.choice([0.0, 1e-8, 1e-12])), track_gaps=gaps)
    if method == "pcg_sh":
        kw["shift"] = float(rng.uniform(0, 3))
    if method == "pcg_var_sh":
        kw["shift_schedule"] = tuple(float(v) for v in rng.uniform(0, 2, maxit + 1))
    if method == "pcg_rr":
        kw["rr_threshold"] = float(rng.choice([1e-8, 1e-4, 0.0]))
    b = rng.standard_normal(A.n)
    x0 = rng.standard_normal(A.n) if rng.integers(3) == 0 else None
    desc = f"{kind} n={A.n} {method} jac={jac} gaps={gaps} maxit={maxit} x0={x0 is not None}"
    return A, jac, kw, b, x0, desc


def check_case(A, jac, kw, b, x0):
    """True when the device and the oracle (device dot order) agree bit for bit."""
    M = K.make_jacobi(A) if jac else None
    Mo = O.make_jacobi(O.as_oracle_operator(A)) if jac else None
    res = err = ores = oerr = None
    try:
        res = K.solve(A, M, b, x0, K.SolverConfig(**kw))
    except Exception as e:
        err = e
    try:
        ores = O.solve(A, Mo, b, x0, O.Config(**kw), dot=gpu_dot(A))
    except Exception as e:
        oerr = e
    if err is not None or oerr is not None:
        return type(err).__name__ == type(oerr).__name__ and str(err) == str(oerr)
    ok = (res.iterations == ores.iterations and same_bits(hist6(res), oracle_hist6(ores))
          and same_bits(np.asarray(res.x), ores.x) and res.replacements == list(ores.replacements))
    if ok and kw["track_gaps"]:
        gd = np.array([[r.gap_f, r.gap_g, r.gap_h, r.gap_j] for r in res.history], dtype=float)
        ok = same_bits(np.nan_to_num(gd, nan=-1.0), np.nan_to_num(ores.history[:, 7:11], nan=-1.0))
    return ok


def run(cases, seed, log=print):
    """Descriptions of the failing cases."""
    rng = np.random.default_rng(seed)
    failures = []
    for c in range(cases):
        A, jac, kw, b, x0, desc = random_case(rng)
        try:
            ok = check_case(A, jac, kw, b, x0)
        except Exception:
            ok = False
            log(traceback.format_exc())
        if not ok:
            failures.append(f"case {c}: {desc}")
            log("MISMATCH", failures[-1])
    return failures


if __name__ == "__main__":
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    fails = run(cases, int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    print(f"fuzz parity: {len(fails)}/{cases} failing", flush=True)
