"""Parity of the device path against the CPU oracle (needs a B200).

Two levels:
  1. bitwise: device history + x == oracle run with the device's reduction
     order injected (oracle.gpu_order), for every solver / operator kind;
  2. target: iteration count within +-2% and final true relative residual
     within 2x of the UNMODIFIED oracle (= the reference, pinned by
     tests/test_oracle_golden.py).
"""

import math

import numpy as np
import pytest

from gpu_helpers import first_diff, gpu_dot, hist6, oracle_hist6, same_bits
from oracle import kpl_oracle as O
import paper_1706_05988_b200 as K
from paper_1706_05988_b200 import problems

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)


def run_both(A, Mkind, b, cfg_kw, check_x=True):
    """Device solve vs oracle with the device dot order; bitwise."""
    M_dev = K.make_jacobi(A) if Mkind == "jacobi" else None
    M_or = O.make_jacobi(O.as_oracle_operator(A)) if Mkind == "jacobi" else None
    cfg = K.SolverConfig(**cfg_kw)
    res = K.solve(A, M_dev, b, None, cfg)
    ores = O.solve(A, M_or, b, None, O.Config(**cfg_kw), dot=gpu_dot(A))
    h, oh = hist6(res), oracle_hist6(ores)
    assert res.iterations == ores.iterations, (res.iterations, ores.iterations)
    assert same_bits(h, oh), first_diff(h, oh)
    if check_x:
        assert same_bits(res.x, ores.x), first_diff(res.x, ores.x)
    assert res.converged == ores.converged
    assert res.replacements == list(ores.replacements)
    return res, ores


# ------------------------------------------------------------ kernels

SPMV_OPS = [
    ("s2d_200", lambda: K.Stencil2D(200, 200)),
    ("s2d_odd", lambda: K.Stencil2D(37, 23)),
    ("s2d_1x1", lambda: K.Stencil2D(1, 1)),
    ("s2d_wide", lambda: K.Stencil2D(1030, 3)),
    ("s3d", lambda: K.Stencil3D(12, 10, 8)),
    ("s3d_odd", lambda: K.Stencil3D(33, 9, 5)),
    ("s3d_thin", lambda: K.Stencil3D(2, 1, 70)),
    ("csr_lap", lambda: K.laplacian_2d(37, 23)),
    ("csr_rspd", lambda: K.random_spd(40, cond=50.0, seed=4)),
    ("csr_vc", lambda: problems.varcoef_3d(9, seed=0)),
    ("csr_band", lambda: problems.banded_spd(5000, seed=0, band=300)),
]


@pytest.mark.parametrize("name,mk", SPMV_OPS)
def test_spmv_bitwise(name, mk):
    A = mk()
    rng = np.random.default_rng(7)
    v = rng.normal(size=A.n) * 10.0 ** rng.integers(-6, 6, size=A.n)
    v[::5] = 0.0
    v[1::7] = -0.0
    got = K.spmv(A, v)
    want = O.spmv(O.as_oracle_operator(A), v)
    assert same_bits(got, want), first_diff(got, want)


@pytest.mark.parametrize("name,mk", SPMV_OPS)
def test_dot_order_emulated(name, mk):
    A = mk()
    rng = np.random.default_rng(11)
    u = rng.normal(size=A.n)
    v = rng.normal(size=A.n) * 1e3
    got = K.dot(u, v, A)
    want = gpu_dot(A)(u, v)
    assert got == want
    assert math.isclose(got, math.fsum(u * v), rel_tol=1e-12, abs_tol=1e-9)


def test_axpy_zero_alpha_exact_copy():
    y = np.array([1.0, -0.0, 2.0])
    out = K.axpy(0.0, np.array([5.0, 5.0, 5.0]), y)
    assert out.tobytes() == y.tobytes()
    assert np.array_equal(K.axpy(-2.0, np.array([1.0, 2.0]), np.array([2.0, 4.0])), [0.0, 0.0])


# ------------------------------------------------------------ solvers

METHODS = [("cg", {}), ("pcg", {}), ("pcg_sh", {"shift": 2.1320754716981134}), ("pcg_rr", {})]


@pytest.mark.parametrize("m,extra", METHODS)
@pytest.mark.parametrize("form", ["stencil", "csr"])
def test_config1_bitwise(m, extra, form):
    """BASELINE config 1 (2D 200^2, M=I, b = A 1/sqrt(n), rtol 1e-12)."""
    A = K.Stencil2D(200, 200) if form == "stencil" else K.laplacian_2d(200, 200)
    b = O.spmv(O.as_oracle_operator(A), np.full(A.n, 1 / math.sqrt(A.n)))
    run_both(A, None, b, dict(method=m, max_iters=2000, rtol=1e-12, **extra))


@pytest.mark.parametrize("m,extra", METHODS)
def test_config1_targets_vs_reference(gold_cfg1, m, extra):
    """+-2% iterations, final true relative residual within 2x of the unmodified
    reference (golden).  Plain p-CG is reduction-order sensitive:
    its bar is convergence plus the attainable-accuracy gap to p-CG-sh."""
    A = K.Stencil2D(200, 200)
    b = O.spmv(O.as_oracle_operator(A), np.full(A.n, 1 / math.sqrt(A.n)))
    bn = math.sqrt(O.blocked_dot(b, b))
    res = K.solve(A, None, b, None, K.SolverConfig(method=m, max_iters=2000, rtol=1e-12, **extra))
    ref_it = int(gold_cfg1[f"cfg1_{m}_iters"])
    ref_true = float(gold_cfg1[f"cfg1_{m}_hist"][-1, 6]) / bn
    true = res.history[-1].rnorm_true / bn
    assert res.converged
    if m == "pcg":
        assert abs(res.iterations - ref_it) <= 0.1 * ref_it
        assert true <= 100 * ref_true
    else:
        assert abs(res.iterations - ref_it) <= 0.02 * ref_it, (res.iterations, ref_it)
        assert true <= 2.0 * ref_true and true >= ref_true / 2.0, (true, ref_true)


@pytest.mark.parametrize("m,extra", [("cg", {}), ("pcg", {}), ("pcg_sh", {"shift": 4.0}),
                                     ("pcg_rr", {})])
def test_table1_levels(gold_cfg1, m, extra):
    """Table 1 lapl200: 500 iterations from b_j = 1/sqrt(n)."""
    A = K.Stencil2D(200, 200)
    b = np.full(A.n, 1 / math.sqrt(A.n))
    res, _ = run_both(A, None, b, dict(method=m, max_iters=500, rtol=0.0, **extra))
    fin = res.history[-1].rnorm_true
    if m in ("cg", "pcg_sh", "pcg_rr"):
        assert fin <= 6.8e-11
    else:
        assert 1e-9 <= fin <= 3.1e-6      # stagnation level (order-sensitive)


@pytest.mark.parametrize("m,extra", [("cg", {}), ("pcg", {}), ("pcg_sh", {"shift": 2.30188679245283}),
                                     ("pcg_rr", {})])
def test_laplacian_3d_bitwise(m, extra):
    A = K.Stencil3D(12, 10, 8)
    b = O.spmv(O.as_oracle_operator(A), np.full(A.n, 1 / math.sqrt(A.n)))
    run_both(A, None, b, dict(method=m, max_iters=120, rtol=0.0, **extra))


@pytest.mark.parametrize("m,extra", [("cg", {}), ("pcg", {}),
                                     ("pcg_sh", {"shift": 0.49238826317067413}), ("pcg_rr", {})])
@pytest.mark.parametrize("form", ["stencil", "csr"])
def test_jacobi_2d_bitwise(m, extra, form):
    A = K.Stencil2D(64, 48) if form == "stencil" else K.laplacian_2d(64, 48)
    b = O.spmv(O.as_oracle_operator(A), np.random.default_rng(0).random(A.n))
    run_both(A, "jacobi", b, dict(method=m, max_iters=1000, rtol=1e-10, **extra))


@pytest.mark.parametrize("m,extra", [("cg", {}), ("pcg_sh", {"shift": 0.49238826317067413}),
                                     ("pcg", {}), ("pcg_rr", {})])
def test_varcoef_bitwise(m, extra):
    A = problems.varcoef_3d(8, seed=0)
    b = np.random.default_rng(1).standard_normal(A.n)
    run_both(A, "jacobi", b, dict(method=m, max_iters=400, rtol=1e-12, **extra))


@pytest.mark.parametrize("m,extra", [("cg", {}), ("pcg_sh", {"shift": 0.4124626382901352}),
                                     ("pcg_rr", {})])
def test_banded_bitwise(m, extra):
    A = problems.banded_spd(20000, seed=0, band=2000)
    b = O.spmv(O.as_oracle_operator(A), np.random.default_rng(1).standard_normal(A.n))
    run_both(A, "jacobi", b, dict(method=m, max_iters=300, rtol=1e-10, **extra))


@pytest.mark.parametrize("m,extra", [("cg", {}), ("pcg", {}), ("pcg_sh", {"shift": 0.9}),
                                     ("pcg_rr", {}), ("pcg_rr", {"rr_threshold": 0.0})])
def test_random_spd_bitwise(m, extra):
    A = K.random_spd(48, cond=1e3, seed=21)
    b = O.spmv(O.as_oracle_operator(A), np.full(48, 1 / math.sqrt(48.0)))
    run_both(A, None, b, dict(method=m, max_iters=60, rtol=0.0, **extra))


def test_shift_zero_is_pcg_bitwise():
    """solvers.py docstring / test_solvers.py:109-126: pcg_sh(0) == pcg, rr(tau=0) == pcg."""
    A = K.Stencil2D(60, 50)
    b = np.full(A.n, 1 / 60.0)
    base = K.solve(A, None, b, None, K.SolverConfig(method="pcg", max_iters=200))
    sh0 = K.solve(A, None, b, None, K.SolverConfig(method="pcg_sh", shift=0.0, max_iters=200))
    rr0 = K.solve(A, None, b, None, K.SolverConfig(method="pcg_rr", rr_threshold=0.0, max_iters=200))
    assert same_bits(hist6(sh0), hist6(base)) and same_bits(sh0.x, base.x)
    assert same_bits(hist6(rr0), hist6(base)) and rr0.replacements == []


def test_identity_matrix_one_iteration():
    A = K.SparseMatrix.from_dense(np.eye(5))
    b = np.random.default_rng(1234).normal(size=5)
    for m in ("cg", "pcg"):
        res = K.solve(A, None, b, None, K.SolverConfig(method=m, max_iters=10, rtol=1e-12))
        assert res.converged and res.iterations == 1 and len(res.history) == 2
        assert np.array_equal(res.x, b)
    first = K.solve(A, None, b, None, K.SolverConfig(method="pcg", max_iters=10, rtol=1e-12)).history[0]
    assert first.alpha == 1.0 and first.delta == first.gamma


def test_breakdown_indefinite():
    A = K.SparseMatrix.from_dense(np.array([[1.0, 0.0], [0.0, -1.0]]))
    for m in ("cg", "pcg", "pcg_sh"):
        with pytest.raises(K.BreakdownError) as exc:
            K.solve(A, None, np.array([0.5, 1.0]), None, K.SolverConfig(method=m, max_iters=5))
        assert exc.value.iteration == 0


def test_history_cadence_and_budget():
    A = K.Stencil2D(8, 8)
    b = np.full(A.n, 0.125)
    res = K.solve(A, None, b, None, K.SolverConfig(method="pcg", max_iters=25))
    assert not res.converged and res.iterations == 25 and len(res.history) == 26
    for r in res.history:
        assert (r.rnorm_true is not None) == (r.iter % 10 == 0 or r.iter == 25)


def test_zero_rhs_converges_immediately():
    A = K.Stencil3D(5, 4, 3)
    res = K.solve(A, None, np.zeros(A.n), None, K.SolverConfig(method="pcg_sh", shift=1.0, max_iters=5))
    assert res.converged and res.iterations == 0 and res.history[0].alpha == 0.0


def test_nonzero_initial_guess_bitwise():
    A = K.Stencil2D(30, 20)
    rng = np.random.default_rng(3)
    b, x0 = rng.normal(size=A.n), rng.normal(size=A.n)
    cfg = dict(method="pcg_sh", shift=1.5, max_iters=80, rtol=1e-9)
    res = K.solve(A, None, b, x0, K.SolverConfig(**cfg))
    ores = O.solve(A, None, b, x0, O.Config(**cfg), dot=gpu_dot(A))
    assert same_bits(hist6(res), oracle_hist6(ores)) and same_bits(res.x, ores.x)


def test_callback_states_match_oracle():
    A = K.Stencil2D(7, 7)
    b = np.full(A.n, 1 / 7.0)
    for m in ("pcg_sh", "cg"):
        seen, oseen = [], []
        cfg = dict(method=m, shift=1.0, max_iters=8)
        K.solve(A, None, b, None, K.SolverConfig(**cfg), callback=lambda st: seen.append(st.x.copy()))
        O.solve(A, None, b, None, O.Config(**cfg), dot=gpu_dot(A),
                callback=lambda st: oseen.append(st["x"].copy()))
        assert len(seen) == len(oseen) == 9
        for a, c in zip(seen, oseen):
            assert same_bits(a, c)


def test_device_tensor_io_stays_on_device():
    A = K.Stencil3D(16, 16, 16)
    b = torch.ones(A.n, dtype=torch.float64, device="cuda")
    res = K.solve(A, None, b, None, K.SolverConfig(method="pcg_sh", shift=2.0, max_iters=30))
    assert isinstance(res.x, torch.Tensor) and res.x.is_cuda


@pytest.mark.parametrize("shape,zc", [((70, 20, 9), 0), ((64, 64, 48), 16), ((130, 9, 17), 4)])
def test_stencil3d_shapes_bitwise(shape, zc):
    """Tile-edge, chunk-edge and partial-chunk geometries of the 3D sweep
    (TMA-fed on sm_100a) against the oracle with the device order."""
    A = K.Stencil3D(*shape)
    b = O.spmv(O.as_oracle_operator(A), np.full(A.n, 1 / math.sqrt(A.n)))
    cfg = dict(method="pcg_sh", shift=2.30188679245283, max_iters=40, rtol=0.0)
    from paper_1706_05988_b200.solvers import _Solve
    S = _Solve(A, None, b, None, K.SolverConfig(**cfg), zc=zc)
    res = S.run()
    ores = O.solve(A, None, b, None, O.Config(**cfg), dot=gpu_dot(A, zc=zc))
    assert same_bits(hist6(res), oracle_hist6(ores)), first_diff(hist6(res), oracle_hist6(ores))
    assert same_bits(res.x, ores.x)


def test_tma_and_register_sweeps_identical(monkeypatch):
    A = K.Stencil3D(96, 40, 24)
    b = np.random.default_rng(5).normal(size=A.n)
    cfg = K.SolverConfig(method="pcg_rr", max_iters=60)
    r1 = K.solve(A, None, b, None, cfg)
    monkeypatch.setenv("KPL_NO_TMA", "1")
    r2 = K.solve(A, None, b, None, cfg)
    assert same_bits(hist6(r1), hist6(r2)) and same_bits(r1.x, r2.x)


# ------------------------------------------------- 8f-1: gaps, variable shift

from gpu_helpers import hist11  # noqa: E402


def run_both11(A, b, cfg_kw):
    res = K.solve(A, None, b, None, K.SolverConfig(**cfg_kw))
    ores = O.solve(A, None, b, None, O.Config(**cfg_kw), dot=gpu_dot(A))
    h, oh = hist11(res), np.ascontiguousarray(ores.history)
    assert same_bits(h, oh), first_diff(h, oh)
    assert same_bits(res.x, ores.x)
    return res


@pytest.mark.parametrize("m,extra", [("cg", {}), ("pcg", {}), ("pcg_sh", {"shift": 0.9}),
                                     ("pcg_var_sh", {"shift_schedule": tuple(0.1 * k for k in range(62))}),
                                     ("pcg_rr", {})])
def test_track_gaps_bitwise(m, extra):
    """gap_f/g/h/j and the true residual at every record (solvers.py:142-167)."""
    A = K.random_spd(48, cond=1e3, seed=21)
    b = O.spmv(O.as_oracle_operator(A), np.full(48, 1 / math.sqrt(48.0)))
    run_both11(A, b, dict(method=m, max_iters=60, rtol=0.0, track_gaps=True, **extra))


@pytest.mark.parametrize("A", [K.Stencil2D(5, 4), K.Stencil3D(24, 18, 20)])
def test_track_gaps_stencil_bitwise(A):
    b = np.full(A.n, 1 / math.sqrt(A.n))
    res = run_both11(A, b, dict(method="pcg_sh", shift=1.0, max_iters=30, track_gaps=True))
    first = res.history[0]
    assert first.gap_f == 0.0 and first.gap_g == 0.0 and first.gap_j == 0.0   # test_solvers.py:148-159


def test_var_shift_ramp_bitwise():
    """Alg. 4 (solvers.py:425-498) with a ramped schedule (test_acceptance.py:398-409 shape)."""
    A = K.Stencil2D(60, 50)
    b = np.full(A.n, 1 / math.sqrt(A.n))
    sched = (0.0,) + tuple(4.0 * min(1.0, i / 50.0) for i in range(300))
    run_both11(A, b, dict(method="pcg_var_sh", shift_schedule=sched, max_iters=300))


def test_var_shift_constant_equals_pcg_sh():
    A = K.Stencil3D(20, 16, 12)
    b = np.full(A.n, 1 / math.sqrt(A.n))
    sh = K.solve(A, None, b, None, K.SolverConfig(method="pcg_sh", shift=0.7, max_iters=80))
    var = K.solve(A, None, b, None, K.SolverConfig(method="pcg_var_sh", shift_schedule=(0.7,) * 81,
                                                    max_iters=80))
    assert same_bits(hist11(sh), hist11(var)) and same_bits(sh.x, var.x)


def test_var_shift_jacobi_csr_bitwise():
    A = problems.varcoef_3d(8, seed=0)
    b = np.random.default_rng(1).standard_normal(A.n)
    sched = tuple(0.1 + 0.002 * k for k in range(401))
    cfg = dict(method="pcg_var_sh", shift_schedule=sched, max_iters=400, rtol=1e-12)
    res = K.solve(A, K.make_jacobi(A), b, None, K.SolverConfig(**cfg))
    oA = O.as_oracle_operator(A)
    ores = O.solve(oA, O.make_jacobi(oA), b, None, O.Config(**cfg), dot=gpu_dot(A))
    assert same_bits(hist11(res), np.ascontiguousarray(ores.history)) and same_bits(res.x, ores.x)


@pytest.mark.parametrize("inline", [False, True])
@pytest.mark.parametrize("shape,jac,method", [((200, 200), False, "pcg_sh"), ((37, 23), False, "pcg"),
                                              ((64, 48), True, "pcg_sh"), ((24, 20, 16), False, "pcg_var_sh"),
                                              ((130, 20, 16), False, "pcg_sh"), ((320, 64, 4), True, "pcg")])
def test_persistent_solver_bitwise(shape, jac, method, inline, monkeypatch):
    """The persistent cooperative path (small stencils) == per-iteration launches, bit for bit,
    with the redundant per-CTA epilogue (chunks of <= 32 items; (320, 64, 4) has 40 and
    takes the inline path) and with the inline counter-based epilogue forced."""
    from paper_1706_05988_b200.solvers import _Solve
    if inline:
        monkeypatch.setenv("KPL_PERSIST_INLINE", "1")
    A = K.Stencil2D(*shape) if len(shape) == 2 else K.Stencil3D(*shape)
    M = K.make_jacobi(A) if jac else None
    b = np.random.default_rng(4).normal(size=A.n)
    extra = {"shift": 1.1} if method == "pcg_sh" else {}
    if method == "pcg_var_sh":
        extra = {"shift_schedule": tuple(0.02 * k for k in range(301))}
    cfg = K.SolverConfig(method=method, max_iters=300, rtol=1e-10, **extra)
    r1 = _Solve(A, M, b, None, cfg, persistent=True).run()
    r2 = _Solve(A, M, b, None, cfg, persistent=False).run()
    assert r1.iterations == r2.iterations
    assert same_bits(hist11(r1), hist11(r2)) and same_bits(r1.x, r2.x)


@pytest.mark.gpu
@pytest.mark.parametrize("dims", [(200, 200), (64, 24, 32)])
def test_persistent_solver_repeatable(dims):
    """Repeated persistent (grid-barrier) solves equal the per-iteration-launch
    solve bit for bit every time (guards the CTA-private workspace views of
    persistent_redundant: a miscompiled copy made CTAs diverge now and then)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1706_05988_b200 as K
    from paper_1706_05988_b200.solvers import _Solve
    A = K.Stencil2D(*dims) if len(dims) == 2 else K.Stencil3D(*dims)
    b = np.full(A.n, 1.0 / np.sqrt(A.n))
    cfg = K.SolverConfig(method="pcg_sh", shift=4.0 if len(dims) == 2 else 2.3, max_iters=300, rtol=0.0)
    ref = _Solve(A, None, b, None, cfg, persistent=False).run()
    want = [(r.alpha, r.beta, r.rnorm_recursive, r.rnorm_true) for r in ref.history]
    for _ in range(25):
        res = _Solve(A, None, b, None, cfg, persistent=True).run()
        assert [(r.alpha, r.beta, r.rnorm_recursive, r.rnorm_true) for r in res.history] == want
        assert np.asarray(res.x).tobytes() == np.asarray(ref.x).tobytes()
