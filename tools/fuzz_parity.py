"""Randomised device-vs-oracle parity sweep (tree order, the device's own
layout), bitwise: random stencil shapes / CSR matrices, methods, shifts,
preconditioners, x0, gaps; breakdowns must match too.

    python tools/fuzz_parity.py [cases] [seed] [tree|reference|dist]
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
    jac = str(rng.choice(["none", "jacobi", "ic0"], p=[0.4, 0.4, 0.2]))
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


def precs(A, pc):
    """(device, oracle) preconditioners; IC(0) breakdowns propagate."""
    if pc == "jacobi":
        return K.make_jacobi(A), O.make_jacobi(O.as_oracle_operator(A))
    if pc == "ic0":
        Ac = A.to_csr() if hasattr(A, "to_csr") else A
        return K.make_ic0(A), O.make_ic0(O.as_oracle_operator(Ac))
    return None, None


def check_case(A, jac, kw, b, x0):
    """True when the device and the oracle (device dot order) agree bit for bit."""
    try:
        M, Mo = precs(A, jac)
    except Exception:
        return None                            # IC(0) breakdown of this matrix: nothing to solve
    res = err = ores = oerr = None
    try:
        res = K.solve(A, M, b, x0, K.SolverConfig(**kw))
    except Exception as e:
        err = e
    try:
        Ao = A.to_csr() if (jac == "ic0" and hasattr(A, "to_csr")) else A   # IC(0) runs the CSR form
        ores = O.solve(Ao, Mo, b, x0, O.Config(**kw), dot=gpu_dot(Ao))
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


def check_case_reference_order(A, jac, kw, b, x0):
    """Reference reduction order (single GPU) vs the oracle with the
    reference's own blocked_dot: bit for bit."""
    try:
        M, Mo = precs(A, jac)
    except Exception:
        return None
    res = err = ores = oerr = None
    try:
        with K.reduction_order("reference"):
            res = K.solve(A, M, b, x0, K.SolverConfig(**kw))
    except Exception as e:
        err = e
    try:
        ores = O.solve(O.as_oracle_operator(A), Mo, b, x0, O.Config(**kw))
    except Exception as e:
        oerr = e
    if err is not None or oerr is not None:
        return type(err).__name__ == type(oerr).__name__ and str(err) == str(oerr)
    return (res.iterations == ores.iterations and same_bits(hist6(res), oracle_hist6(ores))
            and same_bits(np.asarray(res.x), ores.x) and res.replacements == list(ores.replacements))


INFO = [""]


def check_case_distributed(A, jac, kw, b, x0, rng):
    """P virtual ranks (host NCCL-style exchange, fused or post-kernel peer
    exchange) vs one GPU, bit for bit."""
    from paper_1706_05988_b200.distributed import LocalComm, LocalPeerComm, RowPlan, SlabPlan, solve_distributed
    from paper_1706_05988_b200.solvers import _Solve
    if jac == "ic0":
        return None                              # IC(0) is single-GPU
    M = K.make_jacobi(A) if jac == "jacobi" else None
    cfg = K.SolverConfig(**kw)
    kinds = [lambda P: LocalComm(P), lambda P: LocalPeerComm(P), lambda P: LocalPeerComm(P, fused=False)]
    make_comm = kinds[int(rng.integers(3))]
    comm_name = lambda c: type(c).__name__ + ("" if not hasattr(c, "fused") else f"(fused={c.fused})")
    split = lambda v, plan, P: None if v is None else [v[plan.local_slice(r)] for r in range(P)]
    if hasattr(A, "stencil_spec"):
        NX, NY, NZ, _ = A.slab_spec() if hasattr(A, "slab_spec") else A.stencil_spec()
        Ps = [p for p in (2, 3, 4, 8) if NZ % p == 0]
        if not Ps:
            return None                      # not partitionable: skipped
        P = int(rng.choice(Ps))
        nzl = NZ // P
        zc = max(z for z in (1, 2, 4, 8) if nzl % z == 0)
        plan = SlabPlan(NX, NY, NZ, P, zc)
        comm = make_comm(P)
        INFO[0] = f"dims={(NX, NY, NZ)} P={P} zc={zc} comm={comm_name(comm)} kw={kw}"
        try:
            ref = _Solve(A, M, b, x0, cfg, zc=zc, slab_view=True).run()
            res = solve_distributed(A, M, [b[plan.local_slice(r)] for r in range(P)], split(x0, plan, P), cfg,
                                    comm=comm, zc=zc)
        except Exception as e:
            return "Breakdown" in type(e).__name__
    else:
        if A.n < 2 * 256:
            return None
        P = int(rng.integers(2, min(8, A.n // 256) + 1))
        try:
            plan = RowPlan(A, P, chunk_blocks=1)
        except ValueError:
            return None
        comm = make_comm(P)
        INFO[0] = f"P={P} comm={comm_name(comm)} kw={kw}"
        try:
            ref = _Solve(A, M, b, x0, cfg, chunk_blocks=1).run()
            res = solve_distributed(A, M, [b[plan.local_slice(r)] for r in range(P)], split(x0, plan, P), cfg,
                                    comm=comm, chunk_blocks=1)
        except Exception as e:
            return "Breakdown" in type(e).__name__
    x = np.concatenate([xi.cpu().numpy() for xi in res.x])
    return (res.iterations == ref.iterations and same_bits(hist6(res), hist6(ref))
            and same_bits(x, np.asarray(ref.x)) and res.replacements == ref.replacements)


def run(cases, seed, log=print, mode="tree"):
    """Descriptions of the failing cases (mode: tree | reference | dist)."""
    rng = np.random.default_rng(seed)
    failures = []
    skipped = 0
    for c in range(cases):
        A, jac, kw, b, x0, desc = random_case(rng)
        try:
            if mode == "reference":
                ok = check_case_reference_order(A, jac, kw, b, x0)
            elif mode == "dist":
                ok = check_case_distributed(A, jac, kw, b, x0, rng)
            else:
                ok = check_case(A, jac, kw, b, x0)
        except Exception:
            ok = False
            log(traceback.format_exc())
        if ok is None:
            skipped += 1
        elif not ok:
            failures.append(f"case {c}: {desc} {INFO[0] if mode == 'dist' else ''}")
            log("MISMATCH", failures[-1])
    if skipped:
        log(f"({skipped} of {cases} cases not applicable in mode {mode})")
    return failures


if __name__ == "__main__":
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    mode = sys.argv[3] if len(sys.argv) > 3 else "tree"
    fails = run(cases, int(sys.argv[2]) if len(sys.argv) > 2 else 0, mode=mode)
    print(f"fuzz parity ({mode}): {len(fails)}/{cases} failing", flush=True)
