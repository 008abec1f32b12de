"""Device solves in the reference's own reduction order, checked bit for bit
against fixtures produced by the UNMODIFIED reference (tests/golden/*.npz).

With `reduction_order("reference")` every dot product and norm runs the
reference's blocked_dot order (pkg/src/kpl/_kernels.py:16-41) on the device
(kpl_op.order = KPL_ORDER_BLOCKED8: the fused sweeps store their products,
blocked_final_kernel folds them in 8 sequential lanes).  The update formulas
and SpMV term order already match the reference, so histories, iteration
counts, replacement lists and the solution x must equal the reference's own
output exactly -- no emulated oracle in between.
"""

import hashlib

import numpy as np
import pytest

from gpu_helpers import first_diff, hist11
import paper_1706_05988_b200 as K
from paper_1706_05988_b200 import problems

pytestmark = pytest.mark.gpu


def sha(x):
    return hashlib.sha256(np.ascontiguousarray(x, dtype=np.float64).tobytes()).hexdigest()


@pytest.fixture(autouse=True)
def _reference_order():
    with K.reduction_order("reference"):
        yield


def csr(g, tag):
    return K.SparseMatrix(int(g[f"{tag}_n"]), g[f"{tag}_row_ptr"], g[f"{tag}_col_idx"],
                          g[f"{tag}_values"])


def check(g, tag, res):
    h = hist11(res)
    want = g[f"{tag}_hist"]
    assert h.tobytes() == np.ascontiguousarray(want).tobytes(), f"{tag}: {first_diff(h, want)}"
    assert res.iterations == int(g[f"{tag}_iters"]), tag
    assert bool(res.converged) == bool(g[f"{tag}_converged"]), tag
    assert list(res.replacements) == list(g[f"{tag}_reps"]), tag
    assert sha(res.x) == str(g[f"{tag}_xsha"]), tag


@pytest.mark.parametrize("n", [1, 7, 8, 9, 15, 16, 17, 100, 1001, 4099])
def test_dot_reference_order(gold_kernels, n):
    g = gold_kernels
    got = K.dot(g[f"dot_{n}_u"], g[f"dot_{n}_v"])
    assert np.float64(got).tobytes() == np.float64(g[f"dot_{n}_r"]).tobytes()


def test_order_switch_is_scoped():
    assert K.get_reduction_order() == "reference"
    with K.reduction_order("tree"):
        assert K.get_reduction_order() == "tree"
    assert K.get_reduction_order() == "reference"
    with pytest.raises(ValueError):
        K.set_reduction_order("pairwise")


CFG1 = [("cg", {}), ("pcg", {}), ("pcg_sh", {"shift": 2.1320754716981134}), ("pcg_rr", {})]


@pytest.mark.parametrize("form", ["stencil", "csr"])
@pytest.mark.parametrize("m,extra", CFG1)
def test_config1_equals_reference(gold_cfg1, m, extra, form):
    """BASELINE config 1 (lapl200, rtol 1e-12): the device run IS the
    reference run -- e.g. p-CG stops at the reference's iteration count."""
    g = gold_cfg1
    A = K.Stencil2D(200, 200) if form == "stencil" else K.laplacian_2d(200, 200)
    b = K.build_rhs(A, "ones_solution")
    assert sha(b) == str(g["b_sha"])
    res = K.solve(A, None, b, None, K.SolverConfig(method=m, max_iters=2000, rtol=1e-12, **extra))
    check(g, f"cfg1_{m}", res)


@pytest.mark.parametrize("m,extra", [("cg", {}), ("pcg", {}), ("pcg_sh", {"shift": 4.0}),
                                     ("pcg_rr", {})])
def test_table1_lapl200_equals_reference(gold_cfg1, m, extra):
    g = gold_cfg1
    A = K.Stencil2D(200, 200)
    b = np.full(A.n, 1 / np.sqrt(A.n))
    res = K.solve(A, None, b, None, K.SolverConfig(method=m, max_iters=500, rtol=0.0, **extra))
    check(g, f"tab1_{m}", res)


SMALL = (("cg", {}), ("pcg", {}), ("pcg_sh", {"shift": 0.9}),
         ("pcg_var_sh", {"shift_schedule": tuple(0.1 * k for k in range(62))}),
         ("pcg_rr", {}), ("pcg_rr0", {"rr_threshold": 0.0}))


@pytest.mark.parametrize("pname", ["rspd48", "rspd64s3"])
@pytest.mark.parametrize("gaps", [False, True])
@pytest.mark.parametrize("mname,extra", SMALL)
def test_small_solvers_equal_reference(gold_small, pname, gaps, mname, extra):
    g = gold_small
    A = csr(g, pname)
    meth = "pcg_rr" if mname == "pcg_rr0" else mname
    cfg = K.SolverConfig(method=meth, max_iters=60, rtol=0.0, track_gaps=gaps, **extra)
    res = K.solve(A, None, g[f"{pname}_b"], None, cfg)
    tag = f"{pname}_{mname}_{'g' if gaps else 'n'}"
    check(g, tag, res)
    assert res.x.tobytes() == g[f"{tag}_x"].tobytes()


def test_identity_and_gap_cases_equal_reference(gold_small):
    g = gold_small
    A = K.SparseMatrix(5, np.arange(6), np.arange(5), np.ones(5))
    for m in ("cg", "pcg"):
        res = K.solve(A, None, g["eye5_b"], None, K.SolverConfig(method=m, max_iters=10, rtol=1e-12))
        check(g, f"eye5_{m}", res)
    for A in (K.laplacian_2d(5, 4), K.Stencil2D(5, 4)):
        res = K.solve(A, None, g["lap5x4_b"], None,
                      K.SolverConfig(method="pcg_sh", shift=1.0, max_iters=3, track_gaps=True))
        check(g, "lap5x4_pcgsh", res)


def test_breakdown_equals_reference(gold_small):
    A = K.SparseMatrix(2, np.array([0, 1, 2]), np.array([0, 1]), np.array([1.0, -1.0]))
    for m in ("cg", "pcg", "pcg_sh"):
        with pytest.raises(K.BreakdownError) as exc:
            K.solve(A, None, np.array([0.5, 1.0]), None, K.SolverConfig(method=m, max_iters=5))
        assert f"{exc.value.iteration}|{exc.value.what}" == str(gold_small[f"indef_{m}"])


@pytest.mark.parametrize("form", ["stencil", "csr"])
@pytest.mark.parametrize("m,extra", [("cg", {}), ("pcg", {}),
                                     ("pcg_sh", {"shift": 0.49238826317067413}), ("pcg_rr", {})])
def test_jacobi_2d_equals_reference(gold_j3d, m, extra, form):
    g = gold_j3d
    L = K.laplacian_2d(64, 48)
    A = K.Stencil2D(64, 48) if form == "stencil" else L
    M = K.make_jacobi(L)
    b = K.spmv(L, np.random.default_rng(0).random(L.n))
    assert sha(b) == str(g["j2d_b_sha"])
    res = K.solve(A, M, b, None, K.SolverConfig(method=m, max_iters=1000, rtol=1e-10, **extra))
    check(g, f"j2d_{m}", res)


@pytest.mark.parametrize("m,extra", [("pcg", {}), ("pcg_sh", {"shift": 2.30188679245283}), ("cg", {})])
def test_laplacian_3d_equals_reference(gold_j3d, m, extra):
    g = gold_j3d
    A = K.Stencil3D(12, 10, 8)
    b = K.build_rhs(A, "ones_solution")
    assert sha(b) == str(g["l3d_b_sha"])
    res = K.solve(A, None, b, None, K.SolverConfig(method=m, max_iters=120, rtol=0.0, **extra))
    check(g, f"l3d_{m}", res)


@pytest.mark.parametrize("m,extra", [("cg", {}), ("pcg_sh", {"shift": 0.49238826317067413}), ("pcg", {})])
def test_varcoef_equals_reference(gold_j3d, m, extra):
    g = gold_j3d
    A = problems.varcoef_3d(8, seed=0)
    M = K.make_jacobi(A)
    res = K.solve(A, M, g["vc8_b"], None, K.SolverConfig(method=m, max_iters=400, rtol=1e-12, **extra))
    check(g, f"vc8_{m}", res)
    assert res.x.tobytes() == g[f"vc8_{m}_x"].tobytes()


@pytest.mark.parametrize("m,extra", [("cg", {}), ("pcg_sh", {"shift": 0.4124626382901352}), ("pcg_rr", {})])
def test_banded_equals_reference(gold_j3d, m, extra):
    g = gold_j3d
    A = problems.banded_spd(20000, seed=0, band=2000)
    M = K.make_jacobi(A)
    b = K.spmv(A, np.random.default_rng(1).standard_normal(A.n))
    assert sha(b) == str(g["band20k_b_sha"])
    res = K.solve(A, M, b, None, K.SolverConfig(method=m, max_iters=300, rtol=1e-10, **extra))
    check(g, f"band20k_{m}", res)


def test_reference_order_refused_for_partitioned_solves():
    from paper_1706_05988_b200._lib import KplError
    from paper_1706_05988_b200.distributed import LocalComm, solve_distributed
    A = K.Stencil3D(8, 8, 8)
    with pytest.raises(KplError):
        solve_distributed(A, None, [np.ones(256), np.ones(256)], None,
                          K.SolverConfig(method="pcg_sh", shift=1.0, max_iters=5), comm=LocalComm(2))


@pytest.mark.parametrize("shape,m,extra", [((512, 256), "pcg_sh", {"shift": 1.5}), ((300, 301), "pcg_rr", {}),
                                            ((64, 48, 40), "pcg_sh", {"shift": 2.0}), ((257, 255), "cg", {})])
def test_streamed_fold_equals_the_oracle_chain(shape, m, extra):
    """n >= 65536 and even: the reference-order fold runs from a shared-memory ring
    of bulk copies (blocked_final_tma_kernel); odd n keeps the plain-load fold.  Both
    must reproduce the oracle's blocked_dot run (pinned to the reference) bit for bit."""
    from oracle import kpl_oracle as O
    A = K.Stencil3D(*shape) if len(shape) == 3 else K.Stencil2D(*shape)
    oA = O.as_oracle_operator(A)
    b = O.spmv(oA, np.random.default_rng(4).standard_normal(A.n))
    kw = dict(method=m, max_iters=25, rtol=0.0, **extra)
    res = K.solve(A, None, b, None, K.SolverConfig(**kw))
    ref = O.solve(oA, None, b, None, O.Config(**kw))
    got = np.array([[r.alpha, r.beta, r.gamma, r.delta, r.rnorm_recursive] for r in res.history])
    want = np.ascontiguousarray(ref.history[:, 1:6])
    assert got.tobytes() == want.tobytes(), first_diff(got, want)
    assert np.asarray(res.x).tobytes() == ref.x.tobytes()
