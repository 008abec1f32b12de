"""The reference's acceptance criteria (pkg/tests/test_acceptance.py) re-run on
the device path.  Criteria 2-4 and 8 are host analyses of histories/vectors
(stability module) and are covered by the oracle/shift tests; 9 needs network.
"""

import math

import numpy as np
import pytest

import paper_1706_05988_b200 as K

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ITERS = 500
SIGMA_STAR = 4.0


@pytest.fixture(scope="module")
def lapl200():
    A = K.Stencil2D(200, 200)
    return A, np.full(A.n, 1.0 / np.sqrt(A.n))


@pytest.fixture(scope="module")
def finals(lapl200):
    A, b = lapl200
    out = {}
    for key, method, shift in (("cg", "cg", 0.0), ("pcg", "pcg", 0.0), ("pcg_sh", "pcg_sh", SIGMA_STAR)):
        res = K.solve(A, None, b, None, K.SolverConfig(method=method, shift=shift, max_iters=ITERS))
        out[key] = res.history[-1].rnorm_true
    return out


def test_criterion_01_reference_accuracy_levels(finals):
    """test_acceptance.py:96-104 (the pipelined stagnation level is reduction-order
    dependent: 3.3e-7 with the reference order, ~1e-7 with trees)."""
    assert finals["cg"] <= 6.8e-11
    assert 1e-9 <= finals["pcg"] <= 3.1e-6
    assert finals["pcg_sh"] <= 6.8e-11


def test_criterion_05_bitwise_reductions(lapl200):
    """test_acceptance.py:167-197 on the device: degenerate variants reproduce
    their parents bit for bit, gaps included."""
    A, b = lapl200
    kw = dict(max_iters=120, track_gaps=True)
    rec = lambda r: [(h.iter, h.alpha, h.beta, h.gamma, h.delta, h.rnorm_recursive, h.rnorm_true,
                      h.gap_f, h.gap_g, h.gap_h, h.gap_j) for h in r.history]
    base = K.solve(A, None, b, None, K.SolverConfig(method="pcg", **kw))
    assert rec(K.solve(A, None, b, None, K.SolverConfig(method="pcg_sh", shift=0.0, **kw))) == rec(base)
    rr0 = K.solve(A, None, b, None, K.SolverConfig(method="pcg_rr", rr_threshold=0.0, **kw))
    assert rec(rr0) == rec(base) and rr0.replacements == []
    sh = K.solve(A, None, b, None, K.SolverConfig(method="pcg_sh", shift=SIGMA_STAR, **kw))
    var = K.solve(A, None, b, None, K.SolverConfig(method="pcg_var_sh",
                                                   shift_schedule=(SIGMA_STAR,) * 121, **kw))
    assert rec(var) == rec(sh)
    for seed in range(4):
        An = K.random_spd(64, cond=1e4, seed=seed)
        bn = K.spmv(An, np.full(64, 1 / 8.0))
        kwn = dict(max_iters=60, track_gaps=True)
        b0 = K.solve(An, None, bn, None, K.SolverConfig(method="pcg", **kwn))
        assert rec(K.solve(An, None, bn, None, K.SolverConfig(method="pcg_sh", shift=0.0, **kwn))) == rec(b0)


def test_criterion_06_exact_arithmetic_equivalence():
    """test_acceptance.py:200-230: five variants' iterates agree to 1e-10 over 10 iterations."""
    worst = 0.0
    for seed in (1, 2, 3):
        A = K.random_spd(50, cond=100.0, seed=seed)
        b = K.spmv(A, np.full(50, 1 / np.sqrt(50.0)))
        iterates = {}
        cfgs = {
            "cg": K.SolverConfig(method="cg", max_iters=10),
            "pcg": K.SolverConfig(method="pcg", max_iters=10),
            "pcg_sh": K.SolverConfig(method="pcg_sh", shift=1.0, max_iters=10),
            "pcg_var_sh": K.SolverConfig(method="pcg_var_sh", max_iters=10,
                                         shift_schedule=tuple(0.1 * k for k in range(11))),
            "pcg_rr": K.SolverConfig(method="pcg_rr", max_iters=10),
        }
        for tag, cfg in cfgs.items():
            store = iterates.setdefault(tag, [])
            K.solve(A, None, b, None, cfg, callback=lambda st, s=store: s.append(st.x.copy()))
        tags = list(cfgs)
        for a in tags:
            for c in tags:
                assert len(iterates[a]) == len(iterates[c]) == 11
                for xa, xc in zip(iterates[a], iterates[c]):
                    worst = max(worst, np.linalg.norm(xa - xc) / max(np.linalg.norm(xa), 1e-300))
    assert worst <= 1e-10, worst


def test_criterion_07_small_instance_oracle():
    """test_acceptance.py:233-260: 50 random systems n <= 12 vs a dense solve."""
    rng = np.random.default_rng(42)
    worst = 0.0
    for _ in range(50):
        n = int(rng.integers(2, 13))
        A = K.random_spd(n, cond=float(rng.uniform(2.0, 100.0)), seed=int(rng.integers(10**6)))
        xstar = rng.normal(size=n)
        b = K.spmv(A, xstar)
        xd = np.linalg.solve(A.to_dense(), b)
        for method, extra in (("cg", {}), ("pcg", {}), ("pcg_sh", {"shift": 1.0}),
                              ("pcg_var_sh", {"shift_schedule": tuple(0.2 * min(k, 5) for k in range(n + 11))}),
                              ("pcg_rr", {})):
            res = K.solve(A, None, b, None, K.SolverConfig(method=method, max_iters=n + 10, rtol=1e-12, **extra))
            assert res.converged, (method, n)
            err = np.linalg.norm(res.x - xd) / np.linalg.norm(xd)
            worst = max(worst, err)
            assert err <= 1e-9, (method, n, err)


def test_criterion_10_scaling_claims_substitute(finals):
    """test_acceptance.py:335-343."""
    assert finals["pcg_sh"] <= 10.0 * finals["cg"]
    assert finals["pcg"] >= 100.0 * finals["pcg_sh"]


def test_residual_replacement_restores_accuracy(lapl200, finals):
    """test_acceptance.py:346-354."""
    A, b = lapl200
    res = K.solve(A, None, b, None, K.SolverConfig(method="pcg_rr", max_iters=ITERS))
    assert res.history[-1].rnorm_true <= 10.0 * finals["cg"]
    assert 1 <= len(res.replacements) <= 50


def test_variable_shift_ramp_improves(lapl200, finals):
    """test_acceptance.py:398-409."""
    A, b = lapl200
    schedule = (0.0,) + tuple(SIGMA_STAR * min(1.0, i / 50.0) for i in range(ITERS))
    res = K.solve(A, None, b, None, K.SolverConfig(method="pcg_var_sh", shift_schedule=schedule,
                                                   max_iters=ITERS))
    assert res.history[-1].rnorm_true <= finals["pcg"]


def test_energy_norm_monotone():
    """test_solvers.py:184-195 via the device callback."""
    rng = np.random.default_rng(1234)
    n = 30
    q, _ = np.linalg.qr(rng.normal(size=(n, n)))
    a = (q * np.logspace(0, np.log10(80.0), n)) @ q.T
    a = (a + a.T) / 2.0
    A = K.SparseMatrix.from_dense(a)
    b = K.spmv(A, rng.normal(size=n))
    xs = []
    K.solve_cg(A, None, b, None, K.SolverConfig(max_iters=40, rtol=1e-12), callback=lambda st: xs.append(st.x.copy()))
    xd = np.linalg.solve(a, b)
    en = [float(np.sqrt((xd - x) @ a @ (xd - x))) for x in xs]
    for e0, e1 in zip(en, en[1:]):
        assert e1 <= e0 * (1 + 1e-12) + 1e-30
