"""IC(0) on the device: factor, apply and every solver with
an IC(0) preconditioner, checked bit for bit against the unmodified
reference's fixtures (tests/golden/ic0.npz) and against the oracle.

Mirrors the reference's own IC(0) tests (pkg/tests/test_precond.py:41-150)
where they state properties rather than values."""

import hashlib

import numpy as np
import pytest

from conftest import hist_equal
from gpu_helpers import first_diff, gpu_dot, hist11
from oracle import kpl_oracle as O
import paper_1706_05988_b200 as K
from paper_1706_05988_b200 import problems

pytestmark = pytest.mark.gpu

CASES = ("lap12x9", "rspd40", "rspd40e", "vc5", "band3k")


def sha(x):
    return hashlib.sha256(np.ascontiguousarray(x, dtype=np.float64).tobytes()).hexdigest()


def csr(g, tag):
    return K.SparseMatrix(int(g[f"{tag}_n"]), g[f"{tag}_row_ptr"], g[f"{tag}_col_idx"],
                          g[f"{tag}_values"])


@pytest.mark.parametrize("tag", CASES)
def test_factor_and_apply_equal_reference(gold_ic0, tag):
    g = gold_ic0
    M = K.make_ic0(csr(g, tag), eta=float(g[f"{tag}_eta"]))
    ptr, cols, vals = M._l
    assert np.array_equal(ptr, g[f"{tag}_L_row_ptr"])
    assert np.array_equal(cols, g[f"{tag}_L_col_idx"])
    assert vals.tobytes() == g[f"{tag}_L_values"].tobytes(), first_diff(vals, g[f"{tag}_L_values"])
    assert M.mu_tilde == int(g[f"{tag}_mu_tilde"])
    out = M.apply(g[f"{tag}_v"])
    assert out.tobytes() == g[f"{tag}_Mv"].tobytes(), first_diff(out, g[f"{tag}_Mv"])


def test_apply_is_repeatable():
    """The substitution sweeps re-arm their own flags: many applies in a row
    (and interleaved with another factor's) give identical bits."""
    A = K.laplacian_2d(40, 33)
    M1, M2 = K.make_ic0(A), K.make_ic0(A, eta=0.5)
    v = np.random.default_rng(0).normal(size=A.n)
    r1, r2 = M1.apply(v), M2.apply(v)
    for _ in range(5):
        assert M1.apply(v).tobytes() == r1.tobytes()
        assert M2.apply(v).tobytes() == r2.tobytes()


def test_breakdown_row_equals_reference(gold_ic0):
    A = K.SparseMatrix.from_dense(np.array([[1.0, 2.0], [2.0, 1.0]]))
    with pytest.raises(K.PreconditionerBreakdown) as exc:
        K.make_ic0(A, eta=0.0)
    assert exc.value.row == int(gold_ic0["indef_row"])


def test_diagonal_and_compensation_shift():
    """test_precond.py:41-51."""
    d = np.array([4.0, 9.0, 16.0])
    M = K.make_ic0(K.SparseMatrix.from_dense(np.diag(d)), eta=0.0)
    v = np.ones(3)
    assert np.allclose(M.apply(v), v / d, rtol=1e-15)
    M = K.make_ic0(K.SparseMatrix.from_dense(np.eye(3)), eta=0.5)
    v = np.array([3.0, 6.0, 9.0])
    assert np.allclose(M.apply(v), v / 1.5, rtol=1e-15)


def test_full_pattern_is_complete_cholesky():
    """test_precond.py:70-76."""
    rng = np.random.default_rng(3)
    q, _ = np.linalg.qr(rng.normal(size=(8, 8)))
    a = q @ np.diag(np.linspace(1.0, 10.0, 8)) @ q.T
    a = (a + a.T) / 2
    M = K.make_ic0(K.SparseMatrix.from_dense(a), eta=0.0)
    v = rng.normal(size=8)
    expected = np.linalg.solve(a, v)
    assert np.linalg.norm(M.apply(v) - expected) <= 1e-10 * np.linalg.norm(expected)
    exact = np.linalg.norm(np.linalg.inv(a), 2)
    assert M.norm_estimate() == pytest.approx(exact, rel=0.1)


def test_defining_equations_on_laplacian():
    """test_precond.py:54-67: L L^T reproduces lower(A) on its pattern."""
    A = K.laplacian_2d(4, 4)
    ptr, cols, vals = K.make_ic0(A)._l
    L = np.zeros((A.n, A.n))
    for i in range(A.n):
        L[i, cols[ptr[i]:ptr[i + 1]]] = vals[ptr[i]:ptr[i + 1]]
    dense = A.to_dense()
    err = np.abs(L @ L.T - dense)[np.tril(dense) != 0]
    assert err.max() <= 1e-12


def test_negative_eta_rejected():
    with pytest.raises(ValueError):
        K.make_ic0(K.laplacian_2d(2, 2), eta=-0.1)


L2 = (("cg", {}), ("pcg", {}), ("pcg_sh", {"shift": 0.5}),
      ("pcg_var_sh", {"shift_schedule": tuple(0.05 * (k % 7) for k in range(82))}),
      ("pcg_rr", {}), ("pcg_rrx", {"rtol": 0.0}))


def check(g, tag, res):
    h = hist11(res)
    want = g[f"{tag}_hist"]
    assert h.tobytes() == np.ascontiguousarray(want).tobytes(), f"{tag}: {first_diff(h, want)}"
    assert res.iterations == int(g[f"{tag}_iters"]), tag
    assert bool(res.converged) == bool(g[f"{tag}_converged"]), tag
    assert list(res.replacements) == list(g[f"{tag}_reps"]), tag
    assert res.x.tobytes() == g[f"{tag}_x"].tobytes(), tag


@pytest.mark.parametrize("gaps", [False, True])
@pytest.mark.parametrize("m,extra", L2)
def test_ic0_solves_equal_reference(gold_ic0, m, extra, gaps):
    """Reference reduction order: every solver with IC(0) reproduces the
    reference's history, replacements and x bit for bit."""
    g = gold_ic0
    A = K.laplacian_2d(30, 20)
    M = K.make_ic0(A)
    meth = "pcg_rr" if m == "pcg_rrx" else m
    kw = {"rtol": 1e-10, **extra}
    with K.reduction_order("reference"):
        res = K.solve(A, M, g["l2_b"], None, K.SolverConfig(method=meth, max_iters=80, track_gaps=gaps, **kw))
    check(g, f"l2_{m}_{'g' if gaps else 'n'}", res)


@pytest.mark.parametrize("m,extra", [("cg", {}), ("pcg_sh", {"shift": 0.3}), ("pcg_rr", {})])
def test_ic0_varcoef_solves_equal_reference(gold_ic0, m, extra):
    g = gold_ic0
    A = problems.varcoef_3d(6, seed=0)
    with K.reduction_order("reference"):
        res = K.solve(A, K.make_ic0(A), g["v6_b"], None,
                      K.SolverConfig(method=m, max_iters=300, rtol=1e-12, **extra))
    check(g, f"v6_{m}", res)


@pytest.mark.parametrize("m,extra", [("cg", {}), ("pcg_sh", {"shift": 0.5}), ("pcg_rr", {"rtol": 0.0})])
def test_ic0_tree_order_bitwise_vs_oracle(m, extra):
    """Default (tree) order: device == oracle run with the device's reduction order."""
    A = K.laplacian_2d(30, 20)
    M = K.make_ic0(A)
    b = K.build_rhs(A)
    kw = {"rtol": 1e-10, **extra}
    res = K.solve(A, M, b, None, K.SolverConfig(method=m, max_iters=80, **kw))
    oA = O.as_oracle_operator(A)
    ores = O.solve(oA, O.as_oracle_precond(M), b, None, O.Config(method=m, max_iters=80, **kw),
                   dot=gpu_dot(A))
    assert hist_equal(hist11(res), ores.history), first_diff(hist11(res), ores.history)
    assert res.x.tobytes() == ores.x.tobytes()
    assert list(res.replacements) == list(ores.replacements)


def test_ic0_with_stencil_operator_equals_csr():
    """A matrix-free Stencil2D with IC(0) runs on its CSR form: same bits."""
    S, A = K.Stencil2D(30, 20), K.laplacian_2d(30, 20)
    b = K.build_rhs(A)
    cfg = K.SolverConfig(method="pcg_sh", shift=0.5, max_iters=60, rtol=1e-10)
    r1 = K.solve(S, K.make_ic0(S), b, None, cfg)
    r2 = K.solve(A, K.make_ic0(A), b, None, cfg)
    assert hist11(r1).tobytes() == hist11(r2).tobytes()
    assert r1.x.tobytes() == r2.x.tobytes()


def test_ic0_larger_problem_converges():
    """2D 256x256 Laplacian (65k rows, 511 wavefronts): the sync-free
    substitution handles long dependency chains; IC(0) needs far fewer
    iterations than no preconditioner."""
    A = K.laplacian_2d(256, 256)
    b = K.build_rhs(A)
    cfg = K.SolverConfig(method="pcg_sh", shift=0.3, max_iters=1000, rtol=1e-10)
    r_ic = K.solve(A, K.make_ic0(A), b, None, cfg)
    r_id = K.solve(A, None, b, None, K.SolverConfig(method="pcg_sh", shift=2.0, max_iters=1000, rtol=1e-10))
    assert r_ic.converged
    assert r_ic.iterations < 0.6 * r_id.iterations
    true = np.linalg.norm(b - K.spmv(A, r_ic.x)) / np.linalg.norm(b)
    assert true < 1e-9
