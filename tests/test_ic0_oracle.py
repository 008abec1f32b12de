"""Pin the oracle's IC(0) restatement (oracle/csrc/oracle_kernels.c:
orc_ic0_factor / orc_lower_solve / orc_upper_solve, oracle/kpl_oracle.py:
lower_pattern / transpose_pattern / make_ic0) bit for bit against fixtures
produced by the unmodified reference (tests/golden/ic0.npz)."""

import hashlib

import numpy as np
import pytest

from conftest import hist_equal
from oracle import kpl_oracle as O

CASES = ("lap12x9", "rspd40", "rspd40e", "vc5", "band3k")


def sha(x):
    return hashlib.sha256(np.ascontiguousarray(x, dtype=np.float64).tobytes()).hexdigest()


def csr(g, tag):
    return O.CSR(int(g[f"{tag}_n"]), g[f"{tag}_row_ptr"], g[f"{tag}_col_idx"], g[f"{tag}_values"])


@pytest.mark.parametrize("tag", CASES)
def test_ic0_factor_and_apply_golden(gold_ic0, tag):
    g = gold_ic0
    A = csr(g, tag)
    M = O.make_ic0(A, eta=float(g[f"{tag}_eta"]))
    ptr, cols, vals = M.lower
    assert np.array_equal(ptr, g[f"{tag}_L_row_ptr"])
    assert np.array_equal(cols, g[f"{tag}_L_col_idx"])
    assert vals.tobytes() == g[f"{tag}_L_values"].tobytes()
    assert M.apply(g[f"{tag}_v"]).tobytes() == g[f"{tag}_Mv"].tobytes()


def test_ic0_breakdown_row_golden(gold_ic0):
    A = O.CSR(2, np.array([0, 2, 4]), np.array([0, 1, 0, 1]), np.array([1.0, 2.0, 2.0, 1.0]))
    with pytest.raises(O.PreconditionerBreakdown) as exc:
        O.make_ic0(A)
    assert exc.value.row == int(gold_ic0["indef_row"])


def test_ic0_rejects_negative_eta_and_missing_diagonal():
    A = O.CSR(2, np.array([0, 1, 2]), np.array([0, 1]), np.array([1.0, 1.0]))
    with pytest.raises(ValueError):
        O.make_ic0(A, eta=-0.1)
    B = O.CSR(2, np.array([0, 1, 2]), np.array([1, 0]), np.array([1.0, 1.0]))
    with pytest.raises(ValueError, match="diagonal"):
        O.make_ic0(B)


L2 = (("cg", {}), ("pcg", {}), ("pcg_sh", {"shift": 0.5}),
      ("pcg_var_sh", {"shift_schedule": tuple(0.05 * (k % 7) for k in range(82))}),
      ("pcg_rr", {}), ("pcg_rrx", {"rtol": 0.0}))


def check(g, tag, res):
    assert res.iterations == int(g[f"{tag}_iters"]), tag
    assert bool(res.converged) == bool(g[f"{tag}_converged"]), tag
    assert hist_equal(res.history, g[f"{tag}_hist"]), tag
    assert list(res.replacements) == list(g[f"{tag}_reps"]), tag
    assert res.x.tobytes() == g[f"{tag}_x"].tobytes(), tag


@pytest.mark.parametrize("gaps", [False, True])
@pytest.mark.parametrize("m,extra", L2)
def test_ic0_solves_golden(gold_ic0, m, extra, gaps):
    g = gold_ic0
    A = O.laplacian_2d(30, 20)
    M = O.make_ic0(A)
    meth = "pcg_rr" if m == "pcg_rrx" else m
    kw = {"rtol": 1e-10, **extra}
    res = O.solve(A, M, g["l2_b"], None, O.Config(method=meth, max_iters=80, track_gaps=gaps, **kw))
    check(g, f"l2_{m}_{'g' if gaps else 'n'}", res)


@pytest.mark.parametrize("m,extra", [("cg", {}), ("pcg_sh", {"shift": 0.3}), ("pcg_rr", {})])
def test_ic0_varcoef_solves_golden(gold_ic0, m, extra):
    from paper_1706_05988_b200 import problems
    g = gold_ic0
    Ap = problems.varcoef_3d(6, seed=0)
    A = O.CSR(Ap.n, Ap.row_ptr, Ap.col_idx, Ap.values)
    res = O.solve(A, O.make_ic0(A), g["v6_b"], None, O.Config(method=m, max_iters=300, rtol=1e-12, **extra))
    check(g, f"v6_{m}", res)
