"""Device edge cases the reference's own tests exercise (pkg/tests/test_solvers.py):
dimension mismatches, the smallest iteration budget, 1 x 1 systems, and
solve()'s dispatch vs the direct entry points -- each against the oracle in
the reference reduction order, bit for bit."""

import numpy as np
import pytest

from oracle import kpl_oracle as O
import paper_1706_05988_b200 as K

gpu = pytest.mark.gpu
METHODS = [("cg", {}), ("pcg", {}), ("pcg_sh", {"shift": 0.75}), ("pcg_rr", {}),
           ("pcg_var_sh", {"shift_schedule": tuple(0.1 * k for k in range(41))})]


def _need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _rows(res):
    return [(r.iter, r.alpha, r.beta, r.gamma, r.delta, r.rnorm_recursive, r.rnorm_true) for r in res.history]


def _orows(ores):
    h = ores.history
    return [tuple(None if (c == 6 and np.isnan(v)) else (int(v) if c == 0 else float(v)) for c, v in enumerate(row[:7]))
            for row in h]


@gpu
def test_dimension_mismatch_raises_value_error():
    """test_solvers.py::test_dimension_mismatch -- b or x0 of the wrong length."""
    _need_gpu()
    A = K.laplacian_2d(6, 5)
    cfg = K.SolverConfig(method="pcg_sh", shift=1.0, max_iters=5)
    with pytest.raises(ValueError):
        K.solve(A, None, np.ones(A.n + 1), None, cfg)
    with pytest.raises(ValueError):
        K.solve(A, None, np.ones(A.n), np.zeros(A.n - 1), cfg)


def test_zero_iteration_budget_rejected():
    """max_iters must be >= 1 (solvers.py:70-86, mirrored)."""
    with pytest.raises(ValueError):
        K.SolverConfig(method="pcg_sh", shift=1.0, max_iters=0)


@gpu
@pytest.mark.parametrize("method,extra", METHODS)
def test_one_iteration_budget(method, extra):
    """max_iters = 1: rows 0 and 1 (the last one with its true residual), x after one update."""
    _need_gpu()
    A = K.laplacian_2d(12, 9)
    b = K.spmv(A, np.linspace(0.1, 1.0, A.n))
    kw = dict(method=method, max_iters=1, rtol=0.0, **extra)
    if method == "pcg_var_sh":
        kw["shift_schedule"] = extra["shift_schedule"][:2]
    with K.reduction_order("reference"):
        res = K.solve(A, None, b, None, K.SolverConfig(**kw))
    ores = O.solve(O.as_oracle_operator(A), None, b, None, O.Config(**kw))
    assert res.iterations == ores.iterations == 1
    assert len(res.history) == 2
    assert _rows(res) == _orows(ores)
    assert np.asarray(res.x).tobytes() == ores.x.tobytes()


@gpu
@pytest.mark.parametrize("method,extra", METHODS)
def test_one_by_one_system(method, extra):
    """n = 1: the solve ends after one update; same record and x as the oracle."""
    _need_gpu()
    A = K.SparseMatrix(1, [0, 1], [0], [4.0])
    b = np.array([3.0])
    kw = dict(method=method, max_iters=5, rtol=1e-14, **extra)
    with K.reduction_order("reference"):
        res = K.solve(A, None, b, None, K.SolverConfig(**kw))
    ores = O.solve(O.as_oracle_operator(A), None, b, None, O.Config(**kw))
    assert res.iterations == ores.iterations and res.converged == ores.converged
    assert _rows(res) == _orows(ores)
    assert np.asarray(res.x).tobytes() == ores.x.tobytes()


@gpu
@pytest.mark.parametrize("method,extra", METHODS)
def test_dispatch_matches_direct_call(method, extra):
    """test_solvers.py::test_dispatch_matches_direct_call on the device."""
    _need_gpu()
    A = K.Stencil2D(20, 15)
    b = K.spmv(A, np.random.default_rng(4).random(A.n))
    cfg = K.SolverConfig(method=method, max_iters=40, rtol=1e-10, **extra)
    direct = {"cg": K.solve_cg, "pcg": K.solve_pcg, "pcg_sh": K.solve_pcg_shifted, "pcg_rr": K.solve_pcg_rr,
              "pcg_var_sh": K.solve_pcg_var_shifted}[method]
    a = K.solve(A, None, b, None, cfg)
    c = direct(A, None, b, None, cfg)
    assert _rows(a) == _rows(c)
    assert np.asarray(a.x).tobytes() == np.asarray(c.x).tobytes()
    assert a.replacements == c.replacements


@gpu
@pytest.mark.parametrize("form", ["stencil", "csr"])
@pytest.mark.parametrize("with_callback", [False, True])
def test_lazy_replacement_equals_eager(monkeypatch, form, with_callback):
    """p-CG-rr issues its replacement sweeps only when the device trigger fired
    (kpl_solver_iterate2 KPL_ITER_LAZY_REPLACE + kpl_solver_replace) instead of
    four predicated launches per iteration; every bit must be the same as the
    eager sequence (KPL_RR_EAGER=1), replacement list and callbacks included."""
    _need_gpu()
    A = K.Stencil2D(200, 200) if form == "stencil" else K.laplacian_2d(200, 200)
    b = np.full(A.n, 1 / np.sqrt(A.n))
    cfg = K.SolverConfig(method="pcg_rr", max_iters=500, rtol=0.0)
    out = {}
    for eager in ("1", "0"):
        monkeypatch.setenv("KPL_RR_EAGER", eager)
        seen = []
        cb = (lambda st: seen.append((st.iter, float(np.asarray(st.r)[7])))) if with_callback else None
        res = K.solve(A, None, b, None, cfg, callback=cb)
        out[eager] = (res, seen)
    (e, se), (l, sl) = out["1"], out["0"]
    assert len(e.replacements) >= 10 and e.replacements == l.replacements
    assert e.iterations == l.iterations
    for a, c in zip(e.history, l.history):
        assert (a.alpha, a.beta, a.gamma, a.delta, a.rnorm_recursive, a.rnorm_true) == \
               (c.alpha, c.beta, c.gamma, c.delta, c.rnorm_recursive, c.rnorm_true)
    assert np.asarray(e.x).tobytes() == np.asarray(l.x).tobytes()
    assert se == sl


@gpu
@pytest.mark.parametrize("n", [8_388_608 + 1, 25_000_003])
def test_pipelined_host_staging_round_trip(n):
    """Large numpy b / x (a kpl caller's types) go through the pinned staging ring
    (device.to_device_f64 / to_numpy_f64): every byte must arrive, ragged tail
    chunk included."""
    _need_gpu()
    import torch
    from paper_1706_05988_b200 import device as D
    a = np.random.default_rng(n).standard_normal(n)
    a[::7] = -0.0
    d, io = D.to_device_f64(a, n, D.require_cuda(), "vector")
    assert io == "numpy"
    assert d.cpu().numpy().tobytes() == a.tobytes()
    back = D.to_numpy_f64(d * 1.0)
    assert back.tobytes() == a.tobytes()
    torch.cuda.synchronize()
