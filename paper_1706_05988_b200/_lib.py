"""ctypes binding of libkpl_b200.so (the C ABI declared in include/kpl_b200.h).

The library is built in-tree by `paper_1706_05988_b200.build` (nvcc,
sm_100a, --fmad=false).  There is no fallback: if the library or a CUDA
device is missing, every device entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KPL_LIB") or os.path.join(HERE, "lib", "libkpl_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "kpl_b200.h")

# constants mirrored from include/kpl_b200.h
KPL_OK, KPL_EINVAL, KPL_ECUDA, KPL_EUNSUPPORTED = 0, -1, -2, -3
KPL_OP_STENCIL, KPL_OP_CSR = 1, 2
KPL_PC_IDENTITY, KPL_PC_JACOBI_CONST, KPL_PC_JACOBI_VEC, KPL_PC_IC0 = 0, 1, 2, 3
KPL_M_CG, KPL_M_PCG, KPL_M_PCG_SH, KPL_M_PCG_VAR_SH, KPL_M_PCG_RR = 0, 1, 2, 3, 4
KPL_ST_RUNNING, KPL_ST_DONE, KPL_ST_BREAKDOWN = 0, 1, 2
KPL_HIST_COLS = 10
KPL_ORDER_TREE, KPL_ORDER_BLOCKED8 = 0, 1
(KPL_SW_BNORM, KPL_SW_INIT_R, KPL_SW_INIT_W, KPL_SW_ITER, KPL_SW_TRUE, KPL_SW_CG_P, KPL_SW_CG_X,
 KPL_SW_RR_R, KPL_SW_RR_W, KPL_SW_RR_S, KPL_SW_RR_Z,
 KPL_SW_GAP_F, KPL_SW_GAP_G, KPL_SW_GAP_H, KPL_SW_GAP_J) = range(1, 16)

_p = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_d = ctypes.c_double


class KplOp(ctypes.Structure):
    _fields_ = [("kind", _i32), ("precond", _i32), ("n", _i64),
                ("nx", _i64), ("ny", _i64), ("nz", _i64), ("diag", _d),
                ("zc", _i32), ("vx", _i32), ("halo_lo", _p), ("halo_hi", _p),
                ("row_ptr", _p), ("col_idx", _p), ("values", _p), ("nnz", _i64),
                ("chunk_blocks", _i32), ("zhalo", _i32), ("pc_const", _d), ("inv_diag", _p),
                ("chunk_offset", _i64), ("chunks_global", _i64), ("order", _i32), ("_reserved", _i32),
                ("ic_l_row_ptr", _p), ("ic_l_col_idx", _p), ("ic_l_values", _p),
                ("ic_u_row_ptr", _p), ("ic_u_col_idx", _p), ("ic_u_values", _p),
                ("ic_l_order", _p), ("ic_u_order", _p),
                ("sp_col", _p), ("sp_val", _p), ("sp_dest", _p), ("sp_rows", _i32), ("sp_max", _i32),
                ("bd_stream", _p), ("bd_roff", _p), ("bd_sb", _p), ("bd_win", _p),
                ("bd_rows", _i32), ("bd_w", _i32), ("bd_round_max", _i32), ("_reserved2", _i32)]


class KplCfg(ctypes.Structure):
    _fields_ = [("method", _i32), ("track_gaps", _i32), ("shift", _d), ("max_iters", _i64),
                ("rtol", _d), ("rr_threshold", _d), ("rr_coef", _d), ("shift_schedule", _p)]


class KplVecs(ctypes.Structure):
    _fields_ = [(n, _p) for n in ("x", "r", "u", "w0", "w1", "z", "q", "s", "t", "p", "p1", "b")]


class KplStatus(ctypes.Structure):
    _fields_ = [("state", _i64), ("iter", _i64), ("converged", _i64), ("bd_iter", _i64),
                ("bd_code", _i64), ("n_replacements", _i64), ("fire", _i64),
                ("_pad", _i64 * 9)]


KPL_PEER_MAX_COPIES, KPL_PEER_MAX_RANKS = 40, 16


class KplCopy(ctypes.Structure):
    _fields_ = [("src", _p), ("idx", _p), ("dst", _p), ("count", _i64)]


class KplPost(ctypes.Structure):
    _fields_ = [("ncopies", _i32), ("nsignals", _i32), ("copies", KplCopy * KPL_PEER_MAX_COPIES),
                ("signal", _p * KPL_PEER_MAX_RANKS), ("counter", _p), ("status", _p)]


KPL_PUSH_W, KPL_PUSH_X = 1, 2
KPL_ITER_LAZY_REPLACE = 1


class KplPeerSweep(ctypes.Structure):
    _fields_ = [("nranks", _i32), ("rank", _i32), ("table", (_p * KPL_PEER_MAX_RANKS) * 2),
                ("signal", _p * KPL_PEER_MAX_RANKS), ("w_src", _p * 2), ("w_lo", _p * 2), ("w_hi", _p * 2),
                ("x_src", _p), ("x_lo", _p), ("x_hi", _p), ("flags", _p)]


_SIGS = {
    "kpl_version": (_i32, []),
    "kpl_launch_count": (_i64, []),
    "kpl_last_error": (ctypes.c_char_p, []),
    "kpl_breakdown_message": (ctypes.c_char_p, [_i64]),
    "kpl_workspace_bytes": (_i64, [ctypes.POINTER(KplOp), _i64]),
    "kpl_history_offset": (_i64, [ctypes.POINTER(KplOp)]),
    "kpl_replacements_offset": (_i64, [ctypes.POINTER(KplOp), _i64]),
    "kpl_reduction_layout": (_i32, [ctypes.POINTER(KplOp), ctypes.POINTER(_i64)]),
    "kpl_spmv": (_i32, [ctypes.POINTER(KplOp), _p, _p, _p]),
    "kpl_dot": (_i32, [ctypes.POINTER(KplOp), _p, _p, _p, _p, _p]),
    "kpl_axpy": (_i32, [_i64, _d, _p, _p, _p, _p]),
    "kpl_gather": (_i32, [_i64, _p, _p, _p, _p]),
    "kpl_solver_init": (_i32, [ctypes.POINTER(KplOp), ctypes.POINTER(KplCfg),
                               ctypes.POINTER(KplVecs), _p, _p, _p]),
    "kpl_solver_iterate": (_i32, [ctypes.POINTER(KplOp), ctypes.POINTER(KplCfg),
                                  ctypes.POINTER(KplVecs), _i64, _i64, _p, _p]),
    "kpl_solver_iterate2": (_i32, [ctypes.POINTER(KplOp), ctypes.POINTER(KplCfg),
                                   ctypes.POINTER(KplVecs), _i64, _i64, _i32, _p, _p]),
    "kpl_solver_replace": (_i32, [ctypes.POINTER(KplOp), ctypes.POINTER(KplCfg),
                                  ctypes.POINTER(KplVecs), _p, _p]),
    "kpl_solver_iterate_persistent": (_i32, [ctypes.POINTER(KplOp), ctypes.POINTER(KplCfg),
                                             ctypes.POINTER(KplVecs), _i64, _i64, _p, _p]),
    "kpl_solver_cg_pass": (_i32, [ctypes.POINTER(KplOp), ctypes.POINTER(KplCfg),
                                  ctypes.POINTER(KplVecs), _i64, _i32, _p, _p]),
    "kpl_solver_finish": (_i32, [ctypes.POINTER(KplOp), ctypes.POINTER(KplCfg),
                                 ctypes.POINTER(KplVecs), _p, _p]),
    "kpl_read_status": (_i32, [_p, ctypes.POINTER(KplStatus), _p]),
    "kpl_finalize_global": (_i32, [ctypes.POINTER(KplOp), ctypes.POINTER(KplCfg), _i32, _i64, _p, _p]),
    "kpl_solver_prepare": (_i32, [ctypes.POINTER(KplOp), ctypes.POINTER(KplCfg),
                                  ctypes.POINTER(KplVecs), _p, _p]),
    "kpl_sweep": (_i32, [ctypes.POINTER(KplOp), ctypes.POINTER(KplCfg), ctypes.POINTER(KplVecs),
                         _i32, _i64, _p, _p]),
    "kpl_sweep_phase": (_i32, [_i32]),
    "kpl_ic0_scratch_bytes": (_i64, [_i64]),
    "kpl_ic0_levels": (_i32, [_i64, _p, _p, _i32, _p, _p, _p]),
    "kpl_ic0_factor": (_i32, [_i64, _p, _p, _p, _p, _d, _p, _p, ctypes.POINTER(_i64), _p]),
    "kpl_precond_apply": (_i32, [ctypes.POINTER(KplOp), _p, _p, _p, _p]),
    "kpl_peer_post": (_i32, [ctypes.POINTER(KplPost), ctypes.c_uint64, _p]),
    "kpl_peer_finalize": (_i32, [ctypes.POINTER(KplOp), ctypes.POINTER(KplCfg), _i32, _i64, _p, _p, _p, _i32,
                                 ctypes.c_uint64, _p]),
    "kpl_sweep_peer": (_i32, [ctypes.POINTER(KplOp), ctypes.POINTER(KplCfg), ctypes.POINTER(KplVecs), _i32,
                              _i64, _p, _p, ctypes.c_uint64, _i32, _i32, _i32, ctypes.c_uint64, _i32, _p]),
    "kpl_set_peer_timeout": (_i32, [_d]),
    "kpl_ipc_alloc": (_i32, [_i64, ctypes.POINTER(_p), _p]),
    "kpl_ipc_open": (_i32, [_p, ctypes.POINTER(_p)]),
    "kpl_ipc_close": (_i32, [_p]),
    "kpl_ipc_free": (_i32, [_p]),
    "kpl_chunk_table": (_i32, [ctypes.POINTER(KplOp), _p, ctypes.POINTER(_p), ctypes.POINTER(_p),
                               ctypes.POINTER(_i64)]),
}

_lib = None


class KplError(RuntimeError):
    pass


def header_symbols():
    """Function names declared in include/kpl_b200.h."""
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(kpl_\w+)\s*\(", src, re.M)))


def load():
    """Load the shared library (no CUDA device needed just to load it)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise KplError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1706_05988_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            if os.environ.get("KPL_LIB") and not hasattr(lib, name):
                continue          # an alternative (older) library under test: bind what it has
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc, what=""):
    if rc != KPL_OK:
        msg = load().kpl_last_error().decode()
        if rc == KPL_EINVAL:
            raise ValueError(f"{what}: {msg}")
        if rc == KPL_EUNSUPPORTED:
            raise NotImplementedError(f"{what}: {msg}")
        raise KplError(f"{what}: {msg} (rc={rc})")
