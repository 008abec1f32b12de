"""Command line front end, mirroring `kpl`'s (pkg/src/kpl/cli.py) on the B200.

    python -m paper_1706_05988_b200.cli solve --matrix stencil3:128x128x128 --method pcg-sh \
        --shift 2.3 --maxit 500 --history h.csv
    python -m paper_1706_05988_b200.cli analyze-shift --history h.csv --iter 500 --matrix lapl:200x200
    python -m paper_1706_05988_b200.cli gen --matrix lapl:200x200 --out lap.mtx

Same flags, printed lines and exit codes (0 ok, 1 error, 2 usage) as the
reference for `solve`, `analyze-shift` and `gen`; `fetch`/`bench` (network)
are not part of this build.
"""

from __future__ import annotations

import argparse
import sys

import numpy as np

from .device import reduction_order
from .harness import RunConfig, load_matrix, parse_sigma_grid, run_analyze_shift, run_solve
from .mmio import write_matrix_market
from .shift import default_sigma_grid
from .solvers import DEFAULT_RR_THRESHOLD, SolverConfig

METHODS = {"cg": "cg", "pcg": "pcg", "pcg-sh": "pcg_sh", "pcg-var-sh": "pcg_var_sh", "pcg-rr": "pcg_rr"}


def _schedule(path):
    with open(path, encoding="ascii") as fh:
        return tuple(float(ln) for ln in fh if ln.strip())


def cmd_solve(a) -> int:
    solver = SolverConfig(method=METHODS[a.method], shift=a.shift,
                          shift_schedule=_schedule(a.shift_schedule) if a.shift_schedule else None,
                          max_iters=a.maxit, rtol=a.rtol, track_gaps=a.track_gaps,
                          rr_threshold=a.rr_threshold)
    cfg = RunConfig(matrix_source=a.matrix, rhs_mode=a.rhs.replace("-", "_"), precond=a.precond,
                    ic_eta=a.ic_shift, solver=solver, output_format=a.format,
                    output_path=a.history, seed=a.seed)
    with reduction_order(a.reduction_order):
        res, _, _, _ = run_solve(cfg)
    last = res.history[-1]
    print(f"method={a.method} n-iterations={res.iterations} converged={res.converged}")
    print(f"recursive residual norm: {last.rnorm_recursive:.6e}")
    if last.rnorm_true is not None:
        print(f"true residual norm:      {last.rnorm_true:.6e}")
    if res.replacements:
        print(f"replacements at iterations: {res.replacements}")
    if a.history:
        print(f"history written to {a.history}")
    return 0


def cmd_analyze_shift(a) -> int:
    if a.sigma_grid:
        grid = parse_sigma_grid(a.sigma_grid)
    elif a.matrix:
        grid = default_sigma_grid(load_matrix(a.matrix))
    else:
        print("error: provide --sigma-grid or --matrix for a default grid", file=sys.stderr)
        return 2
    sw = run_analyze_shift(a.history, a.iter, grid, output=a.output)
    k0 = int(np.argmin(np.abs(sw.grid)))
    print(f"iteration used: {sw.iter}")
    print(f"psi at sigma={sw.grid[k0]:g}: {sw.psi_values[k0]:.6e}")
    print(f"argmin sigma*: {sw.argmin:g} (psi {sw.psi_values.min():.6e})")
    if a.output:
        print(f"sweep written to {a.output}")
    return 0


def cmd_gen(a) -> int:
    A = load_matrix(a.matrix, seed=a.seed)
    if hasattr(A, "to_csr"):
        A = A.to_csr()
    write_matrix_market(A, a.out)
    print(f"wrote {a.out} (n={A.n}, nnz={A.nnz})")
    return 0


def main(argv=None) -> int:
    p = argparse.ArgumentParser(prog="kpl-b200", description="Shifted pipelined CG on the B200.")
    sub = p.add_subparsers(dest="command", required=True)
    s = sub.add_parser("solve", help="run one solver and emit its history")
    s.add_argument("--matrix", required=True,
                   help="Matrix Market path, lapl:NXxNY, stencil:NXxNY, stencil3:NXxNYxNZ, rand:N[:COND]")
    s.add_argument("--rhs", choices=["ones-solution", "ones-rhs"], default="ones-solution")
    s.add_argument("--precond", choices=["none", "jacobi", "ic0"], default="none")
    s.add_argument("--ic-shift", type=float, default=0.0, metavar="ETA")
    s.add_argument("--method", choices=sorted(METHODS), default="cg")
    s.add_argument("--shift", type=float, default=0.0, metavar="SIGMA")
    s.add_argument("--shift-schedule", metavar="FILE")
    s.add_argument("--maxit", type=int, default=100)
    s.add_argument("--rtol", type=float, default=0.0)
    s.add_argument("--track-gaps", action="store_true")
    s.add_argument("--rr-threshold", type=float, default=DEFAULT_RR_THRESHOLD)
    s.add_argument("--history", metavar="PATH")
    s.add_argument("--format", choices=["csv", "json"], default="csv")
    s.add_argument("--seed", type=int, default=0)
    s.add_argument("--reduction-order", choices=["tree", "reference"], default="tree",
                   help="dot-product order: the device tree (default) or the reference's "
                        "blocked order (bit-identical to the reference's output)")
    s.set_defaults(func=cmd_solve)
    an = sub.add_parser("analyze-shift", help="sweep the amplification factor over shifts")
    an.add_argument("--history", required=True, metavar="PATH")
    an.add_argument("--iter", type=int, required=True)
    an.add_argument("--sigma-grid", metavar="LO:STEP:HI")
    an.add_argument("--matrix")
    an.add_argument("--output", metavar="PATH")
    an.set_defaults(func=cmd_analyze_shift)
    g = sub.add_parser("gen", help="generate a matrix and write Matrix Market")
    g.add_argument("--matrix", required=True)
    g.add_argument("--out", required=True)
    g.add_argument("--seed", type=int, default=0)
    g.set_defaults(func=cmd_gen)
    a = p.parse_args(argv)
    try:
        return a.func(a)
    except Exception as exc:          # cli.py:169-173: any error -> exit 1
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
