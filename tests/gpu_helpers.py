"""Shared helpers for the GPU parity tests (test code: may use the oracle)."""

import ctypes

import numpy as np

from oracle import gpu_order
from oracle import kpl_oracle as O
from paper_1706_05988_b200 import _lib
from paper_1706_05988_b200.problems import _Stencil


def layout_op(A, zc=0, chunk_blocks=0):
    op = _lib.KplOp()
    op.n = A.n
    if isinstance(A, _Stencil) or hasattr(A, "stencil_spec"):
        op.kind = _lib.KPL_OP_STENCIL
        op.nx, op.ny, op.nz, op.diag = A.stencil_spec()
    else:
        op.kind = _lib.KPL_OP_CSR
    op.zc = zc
    op.chunk_blocks = chunk_blocks
    return op


def gpu_layout(A, zc=0, chunk_blocks=0):
    out = (ctypes.c_int64 * 8)()
    _lib.check(_lib.load().kpl_reduction_layout(layout_op(A, zc, chunk_blocks), out), "layout")
    return tuple(out)


def gpu_dot(A, zc=0, chunk_blocks=0):
    """dot(u, v) in the device's reduction order for operator A."""
    lay = gpu_layout(A, zc, chunk_blocks)
    if hasattr(A, "stencil_spec"):
        NX, NY, NZ, _ = A.stencil_spec()
        return gpu_order.make_dot("stencil", (NX, NY, NZ), lay)
    return gpu_order.make_dot("csr", A.n, lay)


def oracle_op(A):
    return O.as_oracle_operator(A)


def hist6(res_or_hist):
    """Device SolveResult -> [rows, 7] (iter, alpha, beta, gamma, delta, rnorm, true)."""
    rows = [[r.iter, r.alpha, r.beta, r.gamma, r.delta, r.rnorm_recursive,
             np.nan if r.rnorm_true is None else r.rnorm_true] for r in res_or_hist.history]
    return np.array(rows, dtype=np.float64)


def oracle_hist6(ores):
    return np.ascontiguousarray(ores.history[:, :7])


def same_bits(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return a.shape == b.shape and a.tobytes() == b.tobytes()


def first_diff(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape:
        return f"shape {a.shape} vs {b.shape}"
    bad = np.nonzero(a.view(np.int64) != b.view(np.int64))
    if not len(bad[0]):
        return "equal"
    idx = tuple(x[0] for x in bad)
    return f"first mismatch at {idx}: {a[idx]!r} vs {b[idx]!r}"


def hist11(res):
    """All IterationRecord fields (gaps included), NaN for None."""
    f = lambda v: np.nan if v is None else v
    return np.array([[r.iter, r.alpha, r.beta, r.gamma, r.delta, r.rnorm_recursive,
                      f(r.rnorm_true), f(r.gap_f), f(r.gap_g), f(r.gap_h), f(r.gap_j)]
                     for r in res.history], dtype=np.float64)
