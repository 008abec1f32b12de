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


HEAD = 160 + 1024 + 2048


def walk(layout, n, x):
    """What csr_band_ring_spmv computes, one (super-block, pass, round record, group, lane) at a time."""
    stream, roff, sb, win, RB, W, round_max = layout
    raw = stream.numpy()
    roff, sb, win = roff.numpy().astype(np.int64) * 16, sb.numpy(), win.numpy()
    RP = -(-RB // 1024)
    out = np.zeros(n)
    seen = 0
    for s in range(sb.shape[0]):
        pass0, npass = int(sb[s][0]), int(sb[s][1])
        acc = np.zeros(RB)                         # +0.0, as the reference's accumulator
        for j in range(npass):
            p = pass0 + j
            w0 = int(win[p])
            assert w0 % 2 == 0 and (j == 0 or w0 > int(win[p - 1]))         # ascending windows
            rows_seen, pass_nnz = [], 0
            for i in range(RP):
                r = p * RP + i
                rec = raw[roff[r]:roff[r + 1]]
                grp = rec[:144].view(np.int32)
                cnt = int(grp[32] - grp[0])
                assert len(rec) == HEAD + 10 * cnt and cnt <= round_max and cnt % 32 == 0
                ln = rec[160:160 + 1024].astype(np.int64)
                rw = rec[160 + 1024:HEAD].view(np.uint16).astype(np.int64)
                col = rec[HEAD:HEAD + 2 * cnt].view(np.uint16)
                val = rec[HEAD + 2 * cnt:HEAD + 10 * cnt].view(np.float64)
                for g in range(32):
                    lens, rws = ln[32 * g:32 * g + 32], rw[32 * g:32 * g + 32]
                    base = int(grp[g] - grp[0])
                    L = int(lens.max(initial=0))
                    assert L == int(lens[0]) and np.all(np.diff(lens) <= 0)  # longest row first
                    assert int(grp[g + 1] - grp[g]) == 32 * L
                    for k in range(L):
                        for lane in range(32):
                            e = base + 32 * k + lane
                            if lens[lane] > k:
                                c = w0 + int(col[e])
                                assert c < n and int(col[e]) < W and rws[lane] < RB
                                acc[rws[lane]] = acc[rws[lane]] + val[e] * x[c]
                                seen += 1
                            else:
                                assert val[e] == 0.0 and col[e] == 0    # zero fill past the row's end
                    rows_seen.extend(rws[lens > 0].tolist())
                    pass_nnz += int(lens.sum())
            assert len(rows_seen) == len(set(rows_seen))              # a row has one slot per pass
            assert pass_nnz > 0                                       # no empty pass is stored
        r0 = s * RB
        m = min(RB, n - r0)
        out[r0:r0 + m] = acc[:m]
    return out, seen


def build(A, **kw):
    rp = torch.from_numpy(np.ascontiguousarray(A.row_ptr, dtype=np.int32))
    ci = torch.from_numpy(np.ascontiguousarray(A.col_idx, dtype=np.int32))
    va = torch.from_numpy(np.ascontiguousarray(A.values, dtype=np.float64))
    return D.band_layout(A.row_ptr, A.col_idx, rp, ci, va, **kw)


@pytest.mark.parametrize("n,band,window,rows", [(3000, 300, 64, 1024), (2500, 2400, 128, 1056), (1500, 40, 8192, 32),
                                                 (1025, 500, 2, 544), (5000, 900, 256, 2400)])
def test_band_layout_walk_equals_csr_matvec(n, band, window, rows):
    A = problems.banded_spd(n, seed=3, per_row=6, band=band)
    lay = build(A, mode="band", window=window, rows=rows)
    assert lay is not None
    x = np.random.default_rng(5).standard_normal(n)
    ref = O.spmv(O.as_oracle_operator(A), x)
    got, seen = walk(lay, n, x)
    assert got.tobytes() == ref.tobytes()
    assert seen == len(A.values)                                      # every nonzero exactly once


def test_band_layout_handles_empty_rows_and_negative_zero():
    n = 1100
    # rows 0, 5, 700, 1099 hold entries (one of them -0.0); every other row is empty
    counts = np.zeros(n, dtype=np.int64)
    counts[[0, 5, 700, 1099]] = [2, 3, 1, 1]
    row_ptr = np.concatenate([[0], np.cumsum(counts)])
    cols = np.array([0, 900, 3, 5, 1000, 2, 1099])
    vals = np.array([1.0, -2.0, 0.5, 4.0, -1.0, -0.0, 3.0])
    A = SparseMatrix(n, row_ptr, cols, vals, check_symmetry=False)
    lay = build(A, mode="band", window=32, rows=512)
    x = -np.ones(n)
    x[2] = 0.0
    ref = O.spmv(O.as_oracle_operator(A), x)
    assert walk(lay, n, x)[0].tobytes() == ref.tobytes()


def test_band_layout_auto_rules():
    # a 5-point Laplacian (short structured rows) never takes the window layout in auto mode
    A = problems.Stencil2D(40, 30).to_csr()
    assert build(A, mode="auto") is None
    assert build(A, mode="csr") is None
    # a scattered band does
    B = problems.banded_spd(6000, seed=0, per_row=11, band=2000)
    assert build(B, mode="auto") is not None
    assert D.band_rows(2_000_000) == 4512        # 444 CTAs = 3 waves of 148
    assert D.band_rows(20_000) == 160            # one wave
