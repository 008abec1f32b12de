"""Level-1/2 device operations of the drop-in API (mirror of pkg/src/kpl/sparse.py).

    spmv(A, v)      sparse.py:153-160  -> kpl_spmv   (reference term order)
    dot(u, v)       sparse.py:163-169  -> kpl_dot    (deterministic GPU tree order)
    axpy(a, x, y)   sparse.py:172-180  -> kpl_axpy   (a == 0 -> exact copy)
    norm2(v)        sparse.py:183-185

Inputs may be numpy arrays (results come back as numpy / float) or CUDA
tensors (results stay on the device).  All arithmetic runs on the GPU.
"""

from __future__ import annotations

import math

import numpy as np

from . import _lib, device as D


def _vec(v, n, dev, what="vector"):
    return D.to_device_f64(v, n, dev, what)


def spmv(A, v):
    dev = D.require_cuda()
    dm = D.device_matrix(A, dev)
    vd, host = _vec(v, dm.n, dev)
    out = D.torch().empty(dm.n, dtype=vd.dtype, device=dev)
    op = D.make_op(dm)
    _lib.check(_lib.load().kpl_spmv(op, D.ptr(vd), D.ptr(out), D.stream_handle()), "spmv")
    return D.to_numpy_f64(out) if host == "numpy" else (out.cpu() if host else out)


def _dot_dev(op, ud, vd, dev):
    t = D.torch()
    lib = _lib.load()
    ws = t.empty(int(lib.kpl_workspace_bytes(op, 0)), dtype=t.uint8, device=dev)
    res = t.empty(1, dtype=t.float64, device=dev)
    _lib.check(lib.kpl_dot(op, D.ptr(ud), D.ptr(vd), D.ptr(res), D.ptr(ws), D.stream_handle()), "dot")
    return res


def dot(u, v, A=None):
    """(u, v).  With `A` given, the reduction follows A's sweep layout (the
    order the solvers use for that operator); otherwise the plain-vector
    layout (256-element blocks)."""
    dev = D.require_cuda()
    n = len(u) if not hasattr(u, "numel") else u.numel()
    if (len(v) if not hasattr(v, "numel") else v.numel()) != n:
        raise ValueError("dimension mismatch in dot")
    ud, host = _vec(u, n, dev)
    vd, _ = _vec(v, n, dev)
    op = D.make_op(D.device_matrix(A, dev)) if A is not None else D.vector_op(n)
    return float(_dot_dev(op, ud, vd, dev).item())


def norm2(v, A=None):
    return math.sqrt(dot(v, v, A))


def axpy(alpha, x, y):
    dev = D.require_cuda()
    n = len(y) if not hasattr(y, "numel") else y.numel()
    xd, host = _vec(x, n, dev, "x")
    yd, _ = _vec(y, n, dev, "y")
    out = D.torch().empty_like(yd)
    _lib.check(_lib.load().kpl_axpy(n, float(alpha), D.ptr(xd), D.ptr(yd), D.ptr(out),
                                    D.stream_handle()), "axpy")
    return D.to_numpy_f64(out) if host == "numpy" else (out.cpu() if host else out)


def precond_apply(M, v):
    """m = M^-1 v through kpl_precond_apply (precond.py:82-94): Jacobi
    v * inv_diag, IC(0) the two substitution sweeps."""
    dev = D.require_cuda()
    t = D.torch()
    vd, host = _vec(v, M.n, dev, "preconditioner input")
    op = D.vector_op(M.n)
    if M.kind == "jacobi":
        if M.inv_const is not None:
            op.precond, op.pc_const = _lib.KPL_PC_JACOBI_CONST, float(M.inv_const)
        else:
            inv = getattr(M, "_device", None)
            if inv is None or inv.device != vd.device:
                inv = t.from_numpy(np.ascontiguousarray(M.inv_diag, dtype=np.float64)).to(dev)
                M._device = inv
            op.precond, op.inv_diag = _lib.KPL_PC_JACOBI_VEC, D.ptr(inv)
    elif M.kind == "ic0":
        op.precond = _lib.KPL_PC_IC0
        D.set_ic0(op, M.ic)
    else:
        raise ValueError(f"unknown preconditioner kind {M.kind!r}")
    lib = _lib.load()
    nb = lib.kpl_workspace_bytes(op, 0)
    _lib.check(nb if nb < 0 else 0, "workspace size")
    ws = t.empty(int(nb), dtype=t.uint8, device=dev)
    out = t.empty_like(vd)
    _lib.check(lib.kpl_precond_apply(op, D.ptr(vd), D.ptr(out), D.ptr(ws), D.stream_handle()),
               "preconditioner apply")
    return D.to_numpy_f64(out) if host == "numpy" else (out.cpu() if host else out)