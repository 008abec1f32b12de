"""The INTEGRATION.md ctypes stub, run as a kpl maintainer would (needs a B200).

VERDICT r01: nothing exercised the documented binding.  Here the stub's
`solve_pcg_shifted_b200` drives libkpl_b200.so through the plain C ABI and
must reproduce this package's own `solve` bit for bit (same kernels, same
reduction tree), for the reference's own matrix type and both
preconditioners the stub handles.
"""

import os

import numpy as np
import pytest

import paper_1706_05988_b200 as K
from paper_1706_05988_b200 import _lib

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from test_host_cpu import _integration_stub  # noqa: E402


@pytest.fixture(scope="module")
def stub():
    os.environ["KPL_B200_LIB"] = _lib.LIB_PATH
    return _integration_stub()


@pytest.mark.parametrize("jacobi", [False, True])
@pytest.mark.parametrize("shift", [0.0, 1.3])
def test_stub_solve_equals_package_solve(stub, jacobi, shift):
    A = K.laplacian_2d(60, 50)
    M = K.make_jacobi(A) if jacobi else None
    b = np.random.default_rng(3).standard_normal(A.n)
    cfg = K.SolverConfig(method="pcg_sh", shift=shift, max_iters=400, rtol=1e-10)
    got = stub["solve_pcg_shifted_b200"](A, M, b, None, cfg)
    want = K.solve(A, M, b, None, cfg)
    assert got.iterations == want.iterations and got.converged == want.converged
    assert len(got.history) == len(want.history)
    for g, w in zip(got.history, want.history):
        assert (g.iter, g.alpha, g.beta, g.gamma, g.delta, g.rnorm_recursive, g.rnorm_true) == \
               (w.iter, w.alpha, w.beta, w.gamma, w.delta, w.rnorm_recursive, w.rnorm_true)
    assert np.asarray(got.x).tobytes() == np.asarray(want.x).tobytes()


def test_stub_raises_the_reference_breakdown(stub):
    A = K.laplacian_2d(8, 8)
    b = np.zeros(A.n)
    b[0] = 1.0
    # a negative shift large enough to make the shifted curvature vanish/negative
    cfg = K.SolverConfig(method="pcg_sh", shift=-1e300, max_iters=20, rtol=0.0)
    with pytest.raises((K.BreakdownError, AssertionError)):
        stub["solve_pcg_shifted_b200"](A, None, b, None, cfg)
