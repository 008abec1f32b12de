"""The two CSR SpMV gather layouts give identical bits (needs a B200).

`KPL_CSR_GATHER=csr` gathers the input in CSR order (csr_spmv_kernel);
`sorted` gathers it in column order per block of rows and sums each row in
CSR order out of shared memory (csr_sorted_spmv).  Both must
equal the oracle's csr_matvec (`_kernels.py:44-52`) bit for bit, and whole
solves must not change by a single bit when the layout changes.
"""

import numpy as np
import pytest

from gpu_helpers import first_diff, gpu_dot, hist6, oracle_hist6, same_bits
from oracle import kpl_oracle as O
import paper_1706_05988_b200 as K
from paper_1706_05988_b200 import device as D
from paper_1706_05988_b200 import problems

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

MATS = [
    ("lap2d", lambda: K.laplacian_2d(61, 47)),
    ("vc3d", lambda: problems.varcoef_3d(13, seed=2)),
    ("band", lambda: problems.banded_spd(30_000, seed=3, band=8000)),
    ("band_wide", lambda: problems.banded_spd(70_001, seed=1)),
    ("rspd", lambda: K.random_spd(300, cond=80.0, seed=5)),
    ("tiny", lambda: K.random_spd(3, cond=2.0, seed=1)),
]


def fresh(A):
    """Matrix copy without a cached device upload (the layout is chosen at upload)."""
    return K.SparseMatrix(A.n, A.row_ptr.copy(), A.col_idx.copy(), A.values.copy())


@pytest.mark.parametrize("name,make", MATS)
def test_spmv_layouts_bitwise(monkeypatch, name, make):
    A = make()
    v = np.random.default_rng(7).standard_normal(A.n)
    v[::5] = 0.0
    v[1::7] = -0.0
    want = O.spmv(O.as_oracle_operator(A), v)
    outs = {}
    for mode in ("csr", "sorted"):
        monkeypatch.setenv("KPL_CSR_GATHER", mode)
        B = fresh(A)
        got = np.asarray(K.spmv(B, v))
        dm = D.device_matrix(B, D.require_cuda())
        assert (dm.sorted is not None) == (mode == "sorted")
        assert same_bits(got, want), (mode, first_diff(got, want))
        outs[mode] = got
    assert same_bits(outs["csr"], outs["sorted"])


def test_auto_picks_sorted_for_scattered_only(monkeypatch):
    monkeypatch.setenv("KPL_CSR_GATHER", "auto")
    dev = D.require_cuda()
    assert D.device_matrix(fresh(problems.banded_spd(40_000, seed=0)), dev).sorted is not None
    assert D.device_matrix(fresh(K.laplacian_2d(300, 300)), dev).sorted is None


@pytest.mark.parametrize("method,extra", [("pcg_sh", {"shift": 0.41}), ("cg", {}), ("pcg_rr", {})])
def test_solves_identical_across_layouts(monkeypatch, method, extra):
    A = problems.banded_spd(50_000, seed=4, band=20_000)
    b = np.random.default_rng(2).standard_normal(A.n)
    kw = dict(method=method, max_iters=60, rtol=1e-10, **extra)
    res = {}
    for mode in ("csr", "sorted"):
        monkeypatch.setenv("KPL_CSR_GATHER", mode)
        B = fresh(A)
        res[mode] = K.solve(B, K.make_jacobi(B), b, None, K.SolverConfig(**kw))
    assert same_bits(hist6(res["csr"]), hist6(res["sorted"]))
    assert same_bits(res["csr"].x, res["sorted"].x)
    # and both are the oracle run in the device's reduction order
    ores = O.solve(A, O.make_jacobi(O.as_oracle_operator(A)), b, None, O.Config(**kw), dot=gpu_dot(A))
    assert same_bits(hist6(res["sorted"]), oracle_hist6(ores))
