"""Shared-memory-window SpMV layout (kpl_op.bd_*, device.py:band_layout): the
builder runs on the CPU here and a numpy walk of the layout in the kernel's
order must reproduce csr_matvec (_kernels.py:44-52) bit for bit."""
import numpy as np
import pytest
import torch

from oracle import kpl_oracle as O
from paper_1706_05988_b200 import device as D
from paper_1706_05988_b200 import problems
from paper_1706_05988_b200.sparse import SparseMatrix


def walk(layout, n, x):
    """What csr_band_spmv computes, one (super-block, pass, group, lane) at a time."""
    val, col, ln, grp, sb, rpt, W, round_max = layout
    val, col = val.numpy(), col.numpy().view(np.uint16)
    ln, grp, sb = ln.numpy(), grp.numpy(), sb.numpy()
    RB, G = 1024 * rpt, 32 * rpt
    out = np.zeros(n)
    for s in range(sb.shape[0]):
        pass0, npass, c_lo, _ = (int(v) for v in sb[s])
        acc = np.zeros(RB)                         # +0.0, as the reference's accumulator
        for j in range(npass):
            p = pass0 + j
            w0 = c_lo + j * W
            for g in range(G):
                lens = ln[p * RB + 32 * g: p * RB + 32 * g + 32].astype(np.int64)
                base = int(grp[p * G + g])
                for k in range(int(lens.max(initial=0))):
                    lanes = np.nonzero(lens > k)[0]
                    for rank, lane in enumerate(lanes):
                        e = base + rank
                        c = w0 + int(col[e])
                        assert c < n and int(col[e]) < W
                        acc[32 * g + lane] = acc[32 * g + lane] + val[e] * x[c]
                    base += len(lanes)
                assert base == int(grp[p * G + g + 1])
            for i in range(rpt):
                assert int(grp[p * G + 32 * i + 32]) - int(grp[p * G + 32 * i]) <= round_max
        r0 = s * RB
        m = min(RB, n - r0)
        out[r0:r0 + m] = acc[:m]
    return out


def build(A, **kw):
    rp = torch.from_numpy(np.ascontiguousarray(A.row_ptr, dtype=np.int32))
    ci = torch.from_numpy(np.ascontiguousarray(A.col_idx, dtype=np.int32))
    va = torch.from_numpy(np.ascontiguousarray(A.values, dtype=np.float64))
    return D.band_layout(A.row_ptr, A.col_idx, rp, ci, va, **kw)


@pytest.mark.parametrize("n,band,window,rpt", [(3000, 300, 64, 1), (2500, 2400, 128, 2), (1500, 40, 14336, 1),
                                                (1025, 500, 2, 1)])
def test_band_layout_walk_equals_csr_matvec(n, band, window, rpt):
    A = problems.banded_spd(n, seed=3, per_row=6, band=band)
    lay = build(A, mode="band", window=window, rpt=rpt)
    assert lay is not None
    x = np.random.default_rng(5).standard_normal(n)
    ref = O.spmv(O.as_oracle_operator(A), x)
    assert walk(lay, n, x).tobytes() == ref.tobytes()
    # every nonzero is stored exactly once
    assert int(lay[3][-8]) == len(A.values) and int(lay[3][-1]) == len(A.values)
    assert np.array_equal(np.sort(lay[0].numpy()[:-8]), np.sort(A.values))


def test_band_layout_handles_empty_rows_and_negative_zero():
    n = 1100
    # rows 0, 5, 700, 1099 hold entries (one of them -0.0); every other row is empty
    counts = np.zeros(n, dtype=np.int64)
    counts[[0, 5, 700, 1099]] = [2, 3, 1, 1]
    row_ptr = np.concatenate([[0], np.cumsum(counts)])
    cols = np.array([0, 900, 3, 5, 1000, 2, 1099])
    vals = np.array([1.0, -2.0, 0.5, 4.0, -1.0, -0.0, 3.0])
    A = SparseMatrix(n, row_ptr, cols, vals, check_symmetry=False)
    lay = build(A, mode="band", window=32, rpt=1)
    x = -np.ones(n)
    x[2] = 0.0
    ref = O.spmv(O.as_oracle_operator(A), x)
    assert walk(lay, n, x).tobytes() == ref.tobytes()


def test_band_layout_auto_rules():
    # a 5-point Laplacian (short structured rows) never takes the window layout in auto mode
    A = problems.Stencil2D(40, 30).to_csr()
    assert build(A, mode="auto") is None
    assert build(A, mode="csr") is None
    # a scattered band does
    B = problems.banded_spd(6000, seed=0, per_row=11, band=2000)
    assert build(B, mode="auto") is not None
    assert D.band_rows_per_thread(2_000_000) == 7
    assert D.band_rows_per_thread(20_000) == 1
