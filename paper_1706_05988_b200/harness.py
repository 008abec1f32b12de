"""Run orchestration and on-disk formats, device-backed.

The reference's harness (`pkg/src/kpl/harness.py`) wraps solves in a
`RunConfig`, resolves matrix sources, builds right-hand sides and
preconditioners, and writes iteration histories as CSV or JSON.  The same
surface here runs the solve on the B200 and keeps every file format
byte-compatible, so histories written by either side load in the other and
`kpl analyze-shift` style analyses run unchanged:

* history CSV: fixed column set `HISTORY_COLUMNS`, reals with 17 significant
  digits (`%.17g`), integers plain, None as an empty cell (harness.py:99-130);
* history JSON: a list of objects, one per record, `indent=1`, trailing
  newline;
* sigma/psi sweep CSV: header `sigma,psi`, `%.17g,%.17g` rows (:214-218).

Matrix sources: a Matrix Market path, `lapl:<nx>x<ny>` (assembled 5-point
Laplacian), `rand:<n>[:<cond>]` (dense random SPD), and -- B200 additions --
`stencil:<nx>x<ny>` / `stencil3:<nx>x<ny>x<nz>` for the matrix-free operators.
Network fetching of the Table-1 matrices is out of scope.
"""

from __future__ import annotations

import json
import os
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .mmio import read_matrix_market
from .precond import identity, make_ic0, make_jacobi
from .problems import Stencil2D, Stencil3D, build_rhs
from .shift import CoefficientHistory, ShiftSweep, select_shift
from .solvers import IterationRecord, SolverConfig, solve
from .sparse import laplacian_2d, random_spd

HISTORY_COLUMNS = ("iter", "alpha", "beta", "gamma", "delta", "rnorm_recursive", "rnorm_true",
                   "gap_f", "gap_g", "gap_h", "gap_j")


@dataclass(frozen=True)
class RunConfig:
    """One solve: matrix source, rhs convention, preconditioner, solver (harness.py:38-66)."""

    matrix_source: str
    rhs_mode: str = "ones_solution"
    precond: str = "none"
    ic_eta: float = 0.0
    solver: SolverConfig = field(default_factory=SolverConfig)
    output_format: str = "csv"
    output_path: str | None = None
    seed: int = 0

    def __post_init__(self):
        if self.rhs_mode not in ("ones_solution", "ones_rhs"):
            raise ValueError(f"unknown rhs_mode {self.rhs_mode!r}")
        if self.precond not in ("none", "jacobi", "ic0"):
            raise ValueError(f"unknown preconditioner {self.precond!r}")
        if self.ic_eta < 0.0:
            raise ValueError("ic_eta must be >= 0")
        if self.output_format not in ("csv", "json"):
            raise ValueError(f"unknown output format {self.output_format!r}")


def _dims(spec, count, what):
    parts = spec.split("x")
    if len(parts) != count:
        raise ValueError(f"bad {what} spec, expected {'x'.join(['<n>'] * count)}")
    return [int(p) for p in parts]


def load_matrix(source: str, seed: int = 0):
    """Resolve a matrix source string (generator spec or Matrix Market path)."""
    if source.startswith("lapl:"):
        nx, ny = _dims(source[5:], 2, f"Laplacian {source!r}")
        return laplacian_2d(nx, ny)
    if source.startswith("stencil:"):
        nx, ny = _dims(source[8:], 2, f"stencil {source!r}")
        return Stencil2D(nx, ny)
    if source.startswith("stencil3:"):
        nx, ny, nz = _dims(source[9:], 3, f"stencil {source!r}")
        return Stencil3D(nx, ny, nz)
    if source.startswith("rand:"):
        parts = source[5:].split(":")
        cond = float(parts[1]) if len(parts) > 1 else 100.0
        return random_spd(int(parts[0]), cond=cond, seed=seed)
    return read_matrix_market(source)


def build_preconditioner(A, kind: str, eta: float = 0.0):
    """harness.py:91-96."""
    if kind == "none":
        return identity()
    if kind == "jacobi":
        return make_jacobi(A)
    return make_ic0(A, eta)


def _cell(value) -> str:
    """One CSV cell: empty for None/NaN, plain integers, 17 significant digits."""
    if value is None or (isinstance(value, float) and value != value):
        return ""
    if isinstance(value, (int, np.integer)) and not isinstance(value, bool):
        return str(int(value))
    return "%.17g" % value


def emit_history(records, fmt: str, sink) -> None:
    """Write records as CSV or JSON; reals round-trip bitwise."""
    if not records:
        raise ValueError("no records to emit")
    if fmt == "csv":
        lines = [",".join(HISTORY_COLUMNS)]
        lines += [",".join(_cell(getattr(r, c)) for c in HISTORY_COLUMNS) for r in records]
        text = "\n".join(lines) + "\n"
    elif fmt == "json":
        text = json.dumps([{c: getattr(r, c) for c in HISTORY_COLUMNS} for r in records], indent=1) + "\n"
    else:
        raise ValueError(f"unknown history format {fmt!r}")
    if isinstance(sink, (str, os.PathLike)):
        with open(sink, "w", encoding="ascii", newline="") as fh:
            fh.write(text)
    else:
        sink.write(text)


def load_history(source) -> list:
    """Parse a CSV or JSON history (either side's) into IterationRecords."""
    text = Path(source).read_text(encoding="ascii") if isinstance(source, (str, os.PathLike)) \
        else source.read()
    text = text.lstrip()
    if text.startswith("["):
        return [IterationRecord(**{c: row.get(c) for c in HISTORY_COLUMNS}) for row in json.loads(text)]
    lines = text.splitlines()
    if tuple(lines[0].split(",")) != HISTORY_COLUMNS:
        raise ValueError(f"unexpected history header: {lines[0]!r}")
    out = []
    for line in lines[1:]:
        if not line.strip():
            continue
        row = {}
        for c, cell in zip(HISTORY_COLUMNS, line.split(",")):
            row[c] = None if cell == "" else (int(cell) if c == "iter" else float(cell))
        out.append(IterationRecord(**row))
    return out


def run_solve(cfg: RunConfig, callback=None):
    """Resolve, solve on the device, emit the history; returns (result, A, M, b)."""
    A = load_matrix(cfg.matrix_source, seed=cfg.seed)
    b = build_rhs(A, cfg.rhs_mode)
    M = build_preconditioner(A, cfg.precond, cfg.ic_eta)
    result = solve(A, M, b, None, cfg.solver, callback=callback)
    if cfg.output_path is not None:
        emit_history(result.history, cfg.output_format, cfg.output_path)
    return result, A, M, b


def parse_sigma_grid(spec: str) -> np.ndarray:
    """Inclusive `lo:step:hi` grid (harness.py:180-189)."""
    parts = spec.split(":")
    if len(parts) != 3:
        raise ValueError(f"bad grid spec {spec!r}, expected lo:step:hi")
    lo, step, hi = (float(p) for p in parts)
    if step <= 0 or hi < lo:
        raise ValueError(f"bad grid spec {spec!r}")
    return lo + step * np.arange(int(round((hi - lo) / step)) + 1)


def run_analyze_shift(history_source, iteration: int, grid, output=None) -> ShiftSweep:
    """Amplification-factor sweep from a stored history (harness.py:192-220);
    truncates to the records available and writes a `sigma,psi` CSV."""
    recs = load_history(history_source)
    hist = CoefficientHistory(np.array([r.alpha for r in recs if r.iter >= 1]),
                              np.array([r.beta for r in recs if r.iter >= 1]))
    if len(hist) == 0:
        raise ValueError("history too short: no usable coefficient records")
    if isinstance(grid, str):
        grid = parse_sigma_grid(grid)
    sweep = select_shift(hist, min(iteration, len(hist)), grid)
    if output is not None:
        text = "sigma,psi\n" + "".join("%.17g,%.17g\n" % (s, v)
                                       for s, v in zip(sweep.grid, sweep.psi_values))
        if isinstance(output, (str, os.PathLike)):
            with open(output, "w", encoding="ascii", newline="") as fh:
                fh.write(text)
        else:
            output.write(text)
    return sweep
