"""B200-native shifted pipelined CG (arXiv 1706.05988), drop-in for `kpl`'s solver path.

The public names mirror the reference package (`pkg/src/kpl/__init__.py`):
solver entry points, configuration/record types, sparse matrix type and
generators, preconditioners, and level-1/2 operations.  All arithmetic runs in
hand-written sm_100a CUDA kernels (libkpl_b200.so) -- there is no CPU path.
"""

from .sparse import SparseMatrix, laplacian_2d, random_spd
from .problems import (Stencil2D, Stencil3D, banded_spd, build_rhs, laplacian_3d,
                       varcoef_3d)
from .precond import (Preconditioner, PreconditionerBreakdown, identity, make_ic0,
                      make_jacobi)
from .solvers import (BreakdownError, DEFAULT_RR_THRESHOLD, IterationRecord, SolveResult,
                      SolverConfig, SolverState, UNIT_ROUNDOFF, solve, solve_cg, solve_pcg,
                      solve_pcg_rr, solve_pcg_shifted, solve_pcg_var_shifted)
from .ops import axpy, dot, norm2, spmv
from .device import get_reduction_order, reduction_order, set_reduction_order
from .mmio import MatrixMarketError, read_matrix_market, write_matrix_market
from .shift import (CoefficientHistory, ShiftSweep, amplification_factor, choose_shift,
                    default_sigma_grid, margin_rule, matrix_2norm, propagation_matrix, select_shift)
from .harness import (HISTORY_COLUMNS, RunConfig, build_preconditioner, emit_history, load_history,
                      load_matrix, parse_sigma_grid, run_analyze_shift, run_solve)

__version__ = "0.1.0"
