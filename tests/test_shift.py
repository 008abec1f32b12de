"""Shift selection: restated stability sweep + margin rule,
pinned bitwise to the reference's own sweep on the reference's histories."""

import numpy as np
import pytest

from conftest import golden
import paper_1706_05988_b200 as K
from paper_1706_05988_b200 import shift as S


@pytest.fixture(scope="module")
def gold_shift():
    return golden("shift")


@pytest.mark.parametrize("tag", ["cfg1", "j2d"])
def test_sweep_bitwise_vs_reference(gold_shift, tag):
    g = gold_shift
    hist = S.CoefficientHistory(g[f"{tag}_alphas"], g[f"{tag}_betas"])
    i = int(g[f"{tag}_i"])
    sw = S.select_shift(hist, i, g[f"{tag}_grid"])
    assert sw.psi_values.tobytes() == g[f"{tag}_psi"].tobytes()
    assert sw.argmin == float(g[f"{tag}_argmin"])
    assert S.margin_rule(sw) == float(g[f"{tag}_chosen"])


def test_default_grids_match_reference(gold_shift):
    assert S.default_sigma_grid(K.laplacian_2d(200, 200)).tobytes() == gold_shift["cfg1_grid"].tobytes()
    assert S.default_sigma_grid(K.Stencil2D(200, 200)).tobytes() == gold_shift["cfg1_grid"].tobytes()
    A = K.laplacian_2d(64, 48)
    assert S.default_sigma_grid(A, K.make_jacobi(A)).tobytes() == gold_shift["j2d_grid"].tobytes()
    As = K.Stencil2D(64, 48)
    assert S.default_sigma_grid(As, K.make_jacobi(As)).tobytes() == gold_shift["j2d_grid"].tobytes()


def test_selected_values_are_the_baseline_sigmas(gold_shift):
    """The values BASELINE.json's configs quote.  The rule's
    config-1 value is linspace(1, 16, 54)[4] = 2.132075471698113, one ulp below
    the survey's printed 1 + 4*15/53 = 2.1320754716981134."""
    assert np.nextafter(float(gold_shift["cfg1_chosen"]), 3.0) == 2.1320754716981134
    assert float(gold_shift["j2d_chosen"]) == 0.49238826317067413


def test_propagation_matrix_and_norm():
    P = S.propagation_matrix(0.5, 0.25, 0.0)
    assert P[0, 1] == -0.125 and P[2, 2] == 1.0
    assert abs(S.matrix_2norm(np.eye(4) * 3.0) - 3.0) < 1e-15
    assert S.matrix_2norm(np.full((4, 4), np.inf)) == float("inf")


@pytest.mark.gpu
def test_choose_shift_on_device_history():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import math
    A = K.Stencil2D(200, 200)
    b = K.spmv(A, np.full(A.n, 1 / math.sqrt(A.n)))
    sigma, sw, base = S.choose_shift(A, None, b, max_iters=2000, rtol=1e-12)
    assert sigma in set(sw.grid.tolist()) and sigma > 0.0
    res = K.solve(A, None, b, None, K.SolverConfig(method="pcg_sh", shift=sigma, max_iters=2000,
                                                   rtol=1e-12))
    ref = K.solve(A, None, b, None, K.SolverConfig(method="cg", max_iters=2000, rtol=1e-12))
    assert res.converged and abs(res.iterations - ref.iterations) <= 0.02 * ref.iterations
    assert res.history[-1].rnorm_true <= 2.0 * ref.history[-1].rnorm_true


@pytest.mark.gpu
def test_config3_rule_at_32cubed_reference_order():
    """Config 3's selection workflow (500 p-CG iterations, default grid, margin
    rule) on the device in the reference reduction order at 32^3 gives the
    sigma of SURVEY.md B.6 (2.30188679245283; argmin psi 9.245) -- the value
    bench.py uses at 512^3, where tools/sigma_config3.py recomputes it."""
    import math
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    A = K.Stencil3D(32, 32, 32)
    b = K.spmv(A, np.full(A.n, 1.0 / math.sqrt(A.n)))
    with K.reduction_order("reference"):
        sigma, sw, base = S.choose_shift(A, None, b, max_iters=500, rtol=0.0)
    assert base.iterations == 500
    assert sigma == 2.30188679245283
    assert abs(sw.argmin - 9.245) < 5e-4
