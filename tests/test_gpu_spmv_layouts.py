"""The CSR SpMV gather layouts give identical bits (needs a B200).

`KPL_CSR_GATHER=csr` gathers the input in CSR order (csr_spmv_kernel);
`sorted` gathers it in column order per block of rows and sums each row in
CSR order out of shared memory (csr_sorted_spmv); `band` walks
shared-memory windows of the input per super-block of rows (csr_band_spmv,
kpl_spmv_band.cuh).  All must equal the oracle's csr_matvec (`_kernels.py:44-52`) bit for bit, and whole
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
    for mode in ("csr", "sorted", "band"):
        monkeypatch.setenv("KPL_CSR_GATHER", mode)
        B = fresh(A)
        got = np.asarray(K.spmv(B, v))
        dm = D.device_matrix(B, D.require_cuda())
        assert (dm.sorted is not None) == (mode == "sorted")
        # "rspd" is dense (300 nonzeros per row: a (row, window) segment over 255) -> no window layout
        assert (dm.band is not None) == (mode == "band" and name != "rspd")
        assert same_bits(got, want), (mode, first_diff(got, want))
        outs[mode] = got
    assert same_bits(outs["csr"], outs["sorted"])
    assert same_bits(outs["csr"], outs["band"])


@pytest.mark.parametrize("window,rows", [(2, 32), (64, 1024), (1000, 1056), (4096, 2400), (8192, 2400), (6144, 0),
                                         (512, 3072)])
def test_band_windows_and_block_heights_bitwise(monkeypatch, window, rows):
    """Many short passes, odd window tails (n odd), super-block heights that are and are
    not multiples of the 1024-slot rounds."""
    monkeypatch.setenv("KPL_CSR_GATHER", "band")
    monkeypatch.setenv("KPL_BAND_W", str(window))
    monkeypatch.setenv("KPL_BAND_ROWS", str(rows))
    A = problems.banded_spd(9_001 if window <= 64 else 70_001, seed=window, band=700 if window <= 64 else 30_000)
    v = np.random.default_rng(11).standard_normal(A.n)
    v[::3] = -0.0
    want = O.spmv(O.as_oracle_operator(A), v)
    B = fresh(A)
    got = np.asarray(K.spmv(B, v))
    lay = D.device_matrix(B, D.require_cuda()).band
    assert lay is not None and lay[5] == window and (rows == 0 or lay[4] == rows)
    assert same_bits(got, want), first_diff(got, want)


def test_auto_picks_the_window_layout_for_scattered_only(monkeypatch):
    monkeypatch.delenv("KPL_CSR_GATHER", raising=False)
    dev = D.require_cuda()
    dm = D.device_matrix(fresh(problems.banded_spd(400_000, seed=0)), dev)
    assert dm.band is not None and dm.sorted is None
    dm = D.device_matrix(fresh(K.laplacian_2d(300, 300)), dev)
    assert dm.band is None and dm.sorted is None


@pytest.mark.parametrize("method,extra", [("pcg_sh", {"shift": 0.41}), ("cg", {}), ("pcg_rr", {})])
def test_solves_identical_across_layouts(monkeypatch, method, extra):
    A = problems.banded_spd(50_000, seed=4, band=20_000)
    b = np.random.default_rng(2).standard_normal(A.n)
    kw = dict(method=method, max_iters=60, rtol=1e-10, **extra)
    res = {}
    for mode in ("csr", "sorted", "band"):
        monkeypatch.setenv("KPL_CSR_GATHER", mode)
        B = fresh(A)
        res[mode] = K.solve(B, K.make_jacobi(B), b, None, K.SolverConfig(**kw))
    for mode in ("sorted", "band"):
        assert same_bits(hist6(res["csr"]), hist6(res[mode])), mode
        assert same_bits(res["csr"].x, res[mode].x), mode
    # and both are the oracle run in the device's reduction order
    ores = O.solve(A, O.make_jacobi(O.as_oracle_operator(A)), b, None, O.Config(**kw), dot=gpu_dot(A))
    assert same_bits(hist6(res["sorted"]), oracle_hist6(ores))


def test_band_falls_back_for_inputs_bulk_copies_cannot_take(monkeypatch):
    """An input vector at an address that is not a multiple of 16 bytes cannot be bulk-copied
    into the window buffers: the CSR-order kernel runs instead, same bits."""
    monkeypatch.setenv("KPL_CSR_GATHER", "band")
    A = problems.banded_spd(30_001, seed=9, band=5000)
    B = fresh(A)
    rng = np.random.default_rng(3)
    host = rng.standard_normal(A.n + 1)
    dev = torch.as_tensor(host, device="cuda")
    assert D.device_matrix(B, D.require_cuda()).band is not None
    for off in (0, 1):                       # 16-byte aligned, then 8 bytes off
        v = dev[off:off + A.n]
        assert v.data_ptr() % 16 == 8 * off
        got = K.spmv(B, v).cpu().numpy()
        want = O.spmv(O.as_oracle_operator(A), host[off:off + A.n])
        assert same_bits(got, want), (off, first_diff(got, want))


@pytest.mark.parametrize("mode", ["band", "sorted", "csr"])
def test_repeated_launches_under_load_are_identical(monkeypatch, mode):
    """Races show up as rare wrong rows, not as a failing first launch: repeat the SpMV while another
    stream keeps the GPU busy (tools/stress_spmv.py is the long form; it caught the removed
    bulk-TMA column-sorted kernel failing ~2 % of its launches)."""
    monkeypatch.setenv("KPL_CSR_GATHER", mode)
    A = problems.banded_spd(70_001, seed=1)
    v = np.random.default_rng(7).standard_normal(A.n)
    want = O.spmv(O.as_oracle_operator(A), v)
    vd = torch.as_tensor(v, device="cuda")
    side = torch.cuda.Stream()
    junk = torch.empty(32 << 20, dtype=torch.float64, device="cuda")
    for rebuild in range(2):
        B = fresh(A)
        for rep in range(60):
            if rep % 3 == 0:
                with torch.cuda.stream(side):
                    junk.normal_()
            got = K.spmv(B, vd).cpu().numpy()
            assert same_bits(got, want), (mode, rebuild, rep, first_diff(got, want))
    torch.cuda.synchronize()
