"""CPU-only tests: C-ABI library loads and exports every declared symbol,
host-side API validation, generators, and the GPU-order emulator itself."""

import ctypes
import math

import numpy as np
import pytest

import paper_1706_05988_b200 as K
from paper_1706_05988_b200 import _lib, problems
from oracle import gpu_order
from oracle import kpl_oracle as O


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = _lib.header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.kpl_version() == 1


def test_library_layout_queries_without_gpu():
    lib = _lib.load()
    op = _lib.KplOp()
    op.kind, op.n, op.nx, op.ny, op.nz, op.diag = _lib.KPL_OP_STENCIL, 512 ** 3, 512, 512, 512, 6.0
    out = (ctypes.c_int64 * 8)()
    assert lib.kpl_reduction_layout(op, out) == 0
    vx, wx, wy, zc, ntx, nty, nch, T = out
    assert (vx, wx, wy) == (2, 1, 8) and ntx == 8 and nty == 64 and T == 512 and nch * zc == 512
    assert lib.kpl_workspace_bytes(op, 500) > 0
    op.nx = 0
    assert lib.kpl_reduction_layout(op, out) == _lib.KPL_EINVAL
    assert b"grid" in lib.kpl_last_error()


def test_ctypes_structs_match_the_c_header(tmp_path):
    """sizeof/offsetof of every ABI struct, compiled from include/kpl_b200.h
    with gcc, equal the ctypes mirrors the Python host side passes."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    structs = {"kpl_op": _lib.KplOp, "kpl_cfg": _lib.KplCfg, "kpl_vecs": _lib.KplVecs,
               "kpl_status": _lib.KplStatus, "kpl_copy": _lib.KplCopy, "kpl_post": _lib.KplPost,
               "kpl_peer_sweep": _lib.KplPeerSweep}
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "kpl_b200.h"', "int main(void) {"]
    for cname, cls in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines += ["return 0; }"]
    src = tmp_path / "abi.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "abi"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(root, "include"), str(src), "-o", str(exe)],
                   check=True)
    got = dict(ln.split() for ln in subprocess.run([str(exe)], capture_output=True, text=True,
                                                   check=True).stdout.splitlines())
    for cname, cls in structs.items():
        assert int(got[cname]) == ctypes.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(cls, fname).offset, f"{cname}.{fname}"


def _integration_stub():
    """The ctypes stub of INTEGRATION.md section 2, executed as written (its
    relative `from .solvers import` is satisfied by this package's types)."""
    import os
    import re
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    text = open(os.path.join(root, "INTEGRATION.md")).read()
    block = re.search(r"```python\n(# kpl/_b200.py.*?)```", text, re.S).group(1)
    code = block.replace("from .solvers import", "from paper_1706_05988_b200.solvers import")
    ns = {}
    exec(compile(code, "INTEGRATION.md:stub", "exec"), ns)
    return ns


def test_integration_stub_structs_match_the_abi():
    """the stub's structs must have the library's full layout
    (sizes and every field offset), so a maintainer copying it allocates and
    fills kpl_op / kpl_cfg / kpl_vecs / kpl_status correctly."""
    ns = _integration_stub()
    for stub, mine in ((ns["Op"], _lib.KplOp), (ns["Cfg"], _lib.KplCfg), (ns["Vecs"], _lib.KplVecs),
                       (ns["Status"], _lib.KplStatus)):
        assert ctypes.sizeof(stub) == ctypes.sizeof(mine), stub.__name__
        assert [f for f, _ in stub._fields_] == [f for f, _ in mine._fields_], stub.__name__
        for f, _ in mine._fields_:
            assert getattr(stub, f).offset == getattr(mine, f).offset, (stub.__name__, f)
            assert getattr(stub, f).size == getattr(mine, f).size, (stub.__name__, f)


def test_reduction_order_field_validation():
    lib = _lib.load()
    op = _lib.KplOp()
    op.kind, op.n = _lib.KPL_OP_CSR, 1000
    tree = lib.kpl_workspace_bytes(op, 10)
    op.order = _lib.KPL_ORDER_BLOCKED8
    assert lib.kpl_workspace_bytes(op, 10) >= tree + 4 * 8 * 1000      # product buffer
    op.chunks_global, op.chunk_offset = 8, 0
    assert lib.kpl_workspace_bytes(op, 10) < 0                          # single GPU only
    assert b"single-GPU" in lib.kpl_last_error()
    op.chunks_global, op.order = 0, 2
    assert lib.kpl_workspace_bytes(op, 10) == _lib.KPL_EINVAL
    with K.reduction_order("reference"):
        from paper_1706_05988_b200 import device
        assert device.vector_op(5).order == _lib.KPL_ORDER_BLOCKED8
    assert K.get_reduction_order() == "tree"


def test_breakdown_messages_match_reference():
    lib = _lib.load()
    msgs = [lib.kpl_breakdown_message(i).decode() for i in range(1, 7)]
    assert msgs == ["nonpositive (r, u)", "nonpositive curvature (w, u)", "vanishing (r, u)",
                    "vanishing alpha denominator", "non-finite coefficients",
                    "nonpositive curvature (s, p)"]


def test_solver_config_validation_mirrors_reference():
    with pytest.raises(ValueError):
        K.SolverConfig(method="sor")
    with pytest.raises(ValueError):
        K.SolverConfig(max_iters=0)
    with pytest.raises(ValueError):
        K.SolverConfig(rtol=-1.0)
    with pytest.raises(ValueError):
        K.SolverConfig(shift=float("inf"))
    with pytest.raises(ValueError):
        K.SolverConfig(method="pcg_var_sh", max_iters=5)
    with pytest.raises(ValueError):
        K.SolverConfig(method="pcg_var_sh", max_iters=5, shift_schedule=(0.0,) * 5)
    K.SolverConfig(method="pcg_var_sh", max_iters=5, shift_schedule=(0.0,) * 6)


def test_sparse_matrix_validation_mirrors_reference():
    with pytest.raises(ValueError):
        K.SparseMatrix(2, [0, 1, 2], [0, 0], [1.0, 1.0])          # asymmetric pattern
    with pytest.raises(ValueError):
        K.SparseMatrix.from_dense(np.array([[1.0, 2.0], [0.0, 1.0]]))
    with pytest.raises(ValueError):
        K.SparseMatrix(2, [0, 2, 2], [1, 0], [1.0, 1.0])           # unsorted columns
    A = K.laplacian_2d(200, 200)
    assert A.n == 40_000 and A.mu == 5 and A.norm_inf() == 8.0


def test_solver_without_gpu_fails_loudly():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(_lib.KplError):
        K.solve(K.Stencil2D(4, 4), None, np.ones(16), None, K.SolverConfig(method="pcg_sh"))


@pytest.mark.parametrize("shape", [(200, 200), (37, 23), (9, 1), (1, 1)])
def test_stencil2d_assembly_equals_laplacian_2d(shape):
    A = K.Stencil2D(*shape).to_csr()
    R = K.laplacian_2d(*shape)
    assert np.array_equal(A.row_ptr, R.row_ptr) and np.array_equal(A.col_idx, R.col_idx)
    assert A.values.tobytes() == R.values.tobytes()
    S = K.Stencil2D(*shape)
    assert S.mu == R.mu and S.norm_inf() == R.norm_inf() and S.nnz == R.nnz


@pytest.mark.parametrize("shape", [(12, 10, 8), (3, 1, 5), (1, 1, 1), (2, 2, 2)])
def test_stencil3d_metadata(shape):
    S = K.Stencil3D(*shape)
    R = S.to_csr()
    assert S.mu == R.mu and S.norm_inf() == R.norm_inf() and S.nnz == R.nnz


def test_config5_generator_statistics():
    # the full config (n=2e6, band 5e4) gives nnz 45,445,908, mu 42 -- the
    # survey's figures; checked here at reduced size
    A = problems.banded_spd(200_000, seed=0, band=5_000)
    per_row = A.nnz / A.n
    assert 22.0 < per_row < 23.0
    d = A.diagonal()
    rows = np.repeat(np.arange(A.n), np.diff(A.row_ptr))
    off = A.col_idx != rows
    assert np.all(np.abs(A.col_idx[off] - rows[off]) <= 5_000)
    absum = np.zeros(A.n)
    np.add.at(absum, rows[off], np.abs(A.values[off]))
    assert np.allclose(d - absum, 1e-3, atol=1e-9)


def test_jacobi_stencil_is_constant():
    M = K.make_jacobi(K.Stencil3D(4, 4, 4))
    assert M.inv_const == 1.0 / 6.0 and np.all(M.inv_diag == 1.0 / 6.0)
    M2 = K.make_jacobi(K.laplacian_2d(3, 3))
    assert np.all(M2.inv_diag == 0.25)
    # IC(0) is factored on the device: without a GPU it fails loudly (no CPU fallback)
    with pytest.raises(_lib.KplError, match="no CUDA device"):
        K.make_ic0(K.laplacian_2d(3, 3))
    with pytest.raises(ValueError):
        K.make_ic0(K.laplacian_2d(3, 3), eta=-1.0)


# ---------------------------------------------------- GPU-order emulator

@pytest.mark.parametrize("dims", [(200, 1, 200), (37, 1, 23), (12, 10, 8), (64, 64, 40)])
def test_emulated_stencil_dot_is_accurate(dims):
    rng = np.random.default_rng(1)
    n = dims[0] * dims[1] * dims[2]
    u, v = rng.normal(size=n), rng.normal(size=n)
    for vx in (1, 2):
        if dims[0] % 2 and vx == 2:
            continue
        wx, wy = (8, 1) if dims[1] == 1 else (1, 8)
        for zc in (1, 4, 16):
            d = gpu_order.stencil_dot_fn(*dims, vx, wx, wy, zc)(u, v)
            assert math.isclose(d, math.fsum(u * v), rel_tol=1e-12)


def test_emulated_csr_dot_is_accurate():
    rng = np.random.default_rng(2)
    for n in (1, 255, 256, 257, 70_001):
        u, v = rng.normal(size=n), rng.normal(size=n)
        for cb in (1, 16):
            d = gpu_order.csr_dot_fn(n, cb)(u, v)
            assert math.isclose(d, math.fsum(u * v), rel_tol=1e-12, abs_tol=1e-12)


def test_emulator_warp_tree_structure():
    """A single nonzero product lands unchanged in the sum; two products in
    the same warp add exactly once (structure sanity of the emulation)."""
    n = 300
    u = np.zeros(n)
    u[123] = 3.0
    assert gpu_order.csr_dot_fn(n, 16)(u, np.ones(n)) == 3.0
    u[5] = 2.0 ** -60
    assert gpu_order.csr_dot_fn(n, 16)(u, np.ones(n)) == 3.0 + 2.0 ** -60


def test_oracle_with_emulated_order_converges_like_reference(gold_cfg1):
    """p-CG-sh is reduction-order insensitive: the emulated
    GPU order gives the reference's 450 iterations on config 1."""
    A = O.StencilSpec(200, 1, 200, 4.0)
    b = O.spmv(A, np.full(A.n, 1 / math.sqrt(A.n)))
    dot = gpu_order.stencil_dot_fn(200, 1, 200, 2, 8, 1, 1)
    res = O.solve(A, None, b, None,
                  O.Config(method="pcg_sh", shift=2.1320754716981134, max_iters=2000, rtol=1e-12),
                  dot=dot)
    assert abs(res.iterations - int(gold_cfg1["cfg1_pcg_sh_iters"])) <= 9
