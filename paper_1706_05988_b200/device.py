"""Device residency: operators, preconditioners and vectors in HBM.

* CSR matrices are uploaded once as int32 `row_ptr`/`col_idx` + fp64
  `values` (the reference stores int64, sparse.py:48-50; every BASELINE
  config fits int32: nnz <= 2^31-1 is checked) and cached per matrix object.
* Stencil operators upload nothing.
* Jacobi uploads `inv_diag` (CSR) or passes the constant fl(1/diag)
  (stencils), cached per preconditioner object.

All device memory is owned by PyTorch's caching allocator; the C library
only receives raw pointers.
"""

from __future__ import annotations

import contextlib
import os
import weakref

import numpy as np

from . import _lib
from ._lib import KplError, KplOp

_torch = None

# Reduction order of dot products / norms (kpl_op.order):
#   "tree"      fixed tile/chunk tree, bandwidth-bound (default)
#   "reference" the reference's blocked_dot order (_kernels.py:16-41): device
#               results are bit-identical to the reference's own solvers, at
#               the cost of a sequential n/8-long fold after each reducing sweep
ORDERS = {"tree": _lib.KPL_ORDER_TREE, "reference": _lib.KPL_ORDER_BLOCKED8}
_order = os.environ.get("KPL_REDUCTION_ORDER", "tree")


def _check_order(name):
    if name not in ORDERS:
        raise ValueError(f"unknown reduction order {name!r} (expected one of {sorted(ORDERS)})")
    return name


def get_reduction_order() -> str:
    return _check_order(_order)


def set_reduction_order(name: str) -> str:
    """Set the process-wide reduction order; returns the previous one."""
    global _order
    prev, _order = _order, _check_order(name)
    return prev


@contextlib.contextmanager
def reduction_order(name: str):
    """`with reduction_order("reference"): solve(...)` -- scoped order."""
    prev = set_reduction_order(name)
    try:
        yield
    finally:
        set_reduction_order(prev)


def torch():
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise KplError("no CUDA device: the p-CG-sh path runs only on the GPU (no CPU fallback)")
    _lib.load()
    return t.device("cuda", t.cuda.current_device())


def stream_handle():
    return torch().cuda.current_stream().cuda_stream


def ptr(t):
    return None if t is None else t.data_ptr()


# Reference SparseMatrix objects use __slots__ without a cache slot; keep a
# small identity-keyed cache (strong refs, bounded) for those.
_foreign_cache: dict = {}
_FOREIGN_MAX = 4


class DeviceMatrix:
    """Device copy of an operator (CSR arrays or stencil geometry)."""

    def __init__(self, A, device):
        t = torch()
        self.n = int(A.n)
        self.device = t.device(device)
        self.stamp = _matrix_stamp(A)
        if hasattr(A, "stencil_spec"):
            self.kind = _lib.KPL_OP_STENCIL
            self.nx, self.ny, self.nz, self.diag = A.stencil_spec()
            self.row_ptr = self.col_idx = self.values = None
            self.nnz = 0
            self.sorted = None
            self.band = None
        else:
            self.kind = _lib.KPL_OP_CSR
            nnz = len(A.values)
            if nnz >= 2**31 or self.n >= 2**31:
                raise ValueError("matrix too large for int32 CSR indices")
            self.row_ptr = t.from_numpy(np.ascontiguousarray(A.row_ptr, dtype=np.int32)).to(device)
            self.col_idx = t.from_numpy(np.ascontiguousarray(A.col_idx, dtype=np.int32)).to(device)
            self.values = t.from_numpy(np.ascontiguousarray(A.values, dtype=np.float64)).to(device)
            self.nnz = nnz
            self.nx = self.ny = self.nz = 0
            self.diag = 0.0
            self.band = band_layout(A.row_ptr, A.col_idx, self.row_ptr, self.col_idx, self.values)
            self.sorted = None if self.band is not None else sorted_gather_layout(
                A.row_ptr, A.col_idx, self.row_ptr, self.col_idx, self.values)


def gather_mode():
    """KPL_CSR_GATHER: how the CSR SpMV reads its input vector.
    auto (default) -- the shared-memory-window layout (kpl_op.bd_*) for scattered
    banded matrices that qualify, CSR-order gathers otherwise; band -- the window
    layout whenever it can be built; sorted -- the column-sorted layout
    (kpl_op.sp_*); csr -- always gather in CSR order."""
    mode = os.environ.get("KPL_CSR_GATHER", "auto")
    if mode not in ("auto", "csr", "sorted", "band"):
        raise ValueError(f"KPL_CSR_GATHER={mode!r}: expected auto, csr, sorted or band")
    return mode


# Shared-memory-window SpMV (kpl_op.bd_*, csrc/kpl_spmv_band.cuh).  A CTA's shared
# memory holds the running sums of its super-block (8 B per row), two windows of
# the input vector (16 B per window column) and a ring of matrix-stream slots.
_BAND_SMEM = 227 * 1024
_BAND_MIN_LINES = 12.0               # auto: CSR-order warp gathers touching >= 12 lines ...
_BAND_MIN_ROW_NNZ = 16.0             # ... on rows longer than 16 nonzeros on average
_BAND_MAX_DESC_BYTES = 0.35          # the 3 B per (row, pass) descriptors stay under 35 % of the 10 B/nnz stream
_BAND_ROWS_MAX = 4608                # super-block height: 36 KiB of running sums at most
_BAND_WINDOWS = (8192, 7168, 6144, 5120, 4096, 3072, 2048)
_BAND_REC_HEAD = 160 + 1024 + 2048   # bytes of a round record before its entries: grp[36] + pad, len[1024], row[1024]
_SMS = 148


def band_rows(n):
    """Super-block height (a multiple of 32, <= 4608): the tallest whose CTA count is a
    whole number of waves of 148 SMs (one CTA per SM); small matrices: one wave."""
    waves = 1
    while True:
        rb = -(-n // (waves * _SMS))
        rb = -(-rb // 32) * 32
        if rb <= _BAND_ROWS_MAX:
            return max(32, rb)
        waves += 1


def band_ring_slots(rows, W, round_max):
    """Ring slots csr_band_ring_spmv gets next to the sums and the two windows
    (kpl_capi.cu:band_ring computes the same)."""
    cap = (round_max + 63) // 64 * 64
    room = _BAND_SMEM - 8 * rows - 16 * W - 128
    return max(0, min(12, room // (10 * cap + _BAND_REC_HEAD)))


def band_layout(row_ptr_h, col_idx_h, row_ptr, col_idx, values, mode=None, window=None, rows=None):
    """(bd_stream, bd_roff, bd_sb, bd_win, rows, W, round_max) or None --
    the layout include/kpl_b200.h documents under kpl_op.bd_*.  Index work only (the
    values are permuted, never combined), done once per matrix with torch on the device
    the CSR arrays live on."""
    mode = gather_mode() if mode is None else mode
    if mode in ("csr", "sorted"):
        return None
    t = torch()
    n = int(row_ptr.numel()) - 1
    nnz = int(col_idx.numel())
    if n < 1 or nnz < 1:
        return None
    if mode == "auto" and (nnz < _BAND_MIN_ROW_NNZ * n or csr_lines_per_warp(col_idx_h) < _BAND_MIN_LINES):
        return None
    RB = int(rows or int(os.environ.get("KPL_BAND_ROWS", 0)) or band_rows(n))
    if RB < 32 or RB % 32 or RB > _BAND_ROWS_MAX:
        raise ValueError(f"window SpMV: super-block height {RB} (expected a multiple of 32 in 32..{_BAND_ROWS_MAX})")
    RP = -(-RB // 1024)                  # rounds (1024 slots = 32 groups) per pass
    RBP = 1024 * RP                      # slots per pass (the tail slots are empty)
    nsb = -(-n // RB)
    dev = row_ptr.device
    counts = (row_ptr[1:] - row_ptr[:-1]).long()
    rowid = t.repeat_interleave(t.arange(n, device=dev), counts)
    sb = rowid // RB
    lrow = rowid - sb * RB
    col = col_idx.long()
    big = t.iinfo(t.int64).max
    c_lo = t.full((nsb,), big, dtype=t.int64, device=dev).scatter_reduce_(0, sb, col, "amin", include_self=True)
    c_hi = t.full((nsb,), -1, dtype=t.int64, device=dev).scatter_reduce_(0, sb, col, "amax", include_self=True)
    c_lo = t.where(c_hi < 0, t.zeros_like(c_lo), c_lo) & ~1          # even: 16-byte bulk copies
    c_hi = t.clamp(c_hi, min=0)
    rel = col - c_lo[sb]

    def plan(W):
        """Passes of window length W -- the windows of a super-block's span that hold
        nonzeros of its rows, in ascending column order; None when the pass table gets too large."""
        nwin = int(((c_hi - c_lo) // W + 1).max())
        wkey, p = t.unique(sb * nwin + rel // W, return_inverse=True)    # sorted: (super-block, window)
        NP = int(wkey.numel())
        if NP * RBP >= 2**31:
            return None
        psb = wkey // nwin
        npass = t.bincount(psb, minlength=nsb)
        pass0 = t.cumsum(npass, 0) - npass
        win = c_lo[psb] + (wkey % nwin) * W                               # first column of every pass
        lens = t.zeros(NP * RBP, dtype=t.int64, device=dev)
        lens.scatter_add_(0, p * RBP + lrow, t.ones_like(p))
        # slots of a pass: rows by length, longest first (stable); groups of 32 slots are
        # dealt to the pass's RP rounds in turn, so every round holds a mix of lengths
        ls, perm = t.sort(lens.view(NP, RBP), dim=1, descending=True, stable=True)
        gmax = ls.view(NP, RBP // 32, 32)[:, :, 0]                    # longest row of each group
        g = t.arange(RBP // 32, device=dev)
        rnd, m = g % RP, g // RP                                      # sorted group g -> round, position
        m = (m + 5 * rnd) % 32                                        # rotate: a warp sees every length class
        ring_g = rnd * 32 + m                                         # group index in ring order
        round_max = int(t.zeros(NP, RP, dtype=t.int64, device=dev).scatter_add_(
            1, rnd.expand(NP, -1), gmax * 32).max())
        return npass, pass0, NP, p, ls, perm, gmax, ring_g, round_max, win

    explicit = window or os.environ.get("KPL_BAND_W")
    if explicit:
        W = int(explicit)
        if W < 2 or W % 2 or W > 65536:
            raise ValueError(f"window SpMV: window length {W} (expected an even value in 2..65536)")
        pl = plan(W)
        if pl is None or band_ring_slots(RB, W, pl[8]) < 2:
            return None
    else:
        # the widest window that leaves room for two ring slots of the matrix stream (config 5,
        # ms/iteration: 8192 columns 0.260, 6144 0.266, 4096 0.286, 2048 0.412 -- passes cost more
        # than ring depth gains)
        pl = None
        for W in _BAND_WINDOWS:
            pl = plan(W)
            if pl is not None and band_ring_slots(RB, W, pl[8]) >= 2:
                break
        else:
            return None
    npass, pass0, NP, p, ls, perm, gmax, ring_g, round_max, win = pl
    if mode == "auto" and 3.0 * NP * RBP > _BAND_MAX_DESC_BYTES * 10.0 * nnz:
        return None                                                   # too wide a span for the window walk
    if int(ls.max()) > 255:
        return None
    G = RBP // 32
    # ring-order slot of every sorted slot, and the reverse map row -> slot
    spos = t.arange(RBP, device=dev)
    ring_slot = ring_g[spos // 32] * 32 + spos % 32                   # sorted position -> ring-order slot
    bd_row = t.empty(NP, RBP, dtype=t.int64, device=dev)
    bd_len = t.empty(NP, RBP, dtype=t.int64, device=dev)
    bd_row[:, ring_slot] = perm
    bd_len[:, ring_slot] = ls
    slot_of_row = t.empty(NP, RBP, dtype=t.int64, device=dev)
    slot_of_row.scatter_(1, perm, ring_slot.expand(NP, -1))
    # groups in ring order: each stored as (its longest row) full steps of 32 entries
    gsz = t.empty(NP, G, dtype=t.int64, device=dev)
    gsz[:, ring_g] = gmax * 32
    gstart = t.cumsum(gsz.view(-1), 0) - gsz.view(-1)
    S = int(gsz.sum())
    if S + 64 >= 2**31:
        return None
    # the k-th nonzero of a (pass, row) segment: segments are contiguous in CSR order
    idx = t.arange(nnz, device=dev)
    first = t.ones(nnz, dtype=t.bool, device=dev)
    first[1:] = (rowid[1:] != rowid[:-1]) | (p[1:] != p[:-1])
    k = idx - t.cummax(t.where(first, idx, t.zeros_like(idx)), 0)[0]
    slot = slot_of_row.view(-1)[p * RBP + lrow]
    pos = gstart[p * G + slot // 32] + k * 32 + slot % 32
    # one record per round (32 groups), copied by ONE bulk copy: a bulk copy costs ~0.3 us of the
    # SM's copy engine whatever its size (tools/bulk_stream_bench.cu), so five slices per round
    # (values, columns, rows, lengths, offsets) capped the stream at 3 TB/s
    NR = NP * RP
    gstart_r = gstart.view(NR, 32)
    rcnt = gsz.view(NR, 32).sum(1)                                     # entries per round
    rbytes = _BAND_REC_HEAD + 10 * rcnt
    roff = t.zeros(NR + 1, dtype=t.int64, device=dev)
    roff[1:] = t.cumsum(rbytes, 0)
    total = int(roff[-1])
    if total // 16 >= 2**31:
        return None
    stream = t.zeros(total + 64, dtype=t.uint8, device=dev)
    rbase = roff[:-1]
    # grp[36]: the 32 group starts, the round's end, padding
    s32 = stream.view(t.int32)
    gi = (rbase // 4).unsqueeze(1) + t.arange(33, device=dev)
    gv = t.cat([gstart_r, (gstart_r[:, :1] + rcnt.unsqueeze(1))], 1)
    s32[gi.reshape(-1)] = gv.reshape(-1).to(t.int32)
    # len[1024], row[1024]
    sl = t.arange(1024, device=dev)
    stream[((rbase + 160).unsqueeze(1) + sl).reshape(-1)] = bd_len.view(-1).to(t.uint8)
    s16 = stream.view(t.int16)
    s16[(((rbase + 160 + 1024) // 2).unsqueeze(1) + sl).reshape(-1)] = bd_row.view(-1).to(t.int32).to(t.int16)
    # col[cnt], val[cnt]: entry e of round r sits at e - (first entry of the round)
    rnd = (p * G + slot // 32) // 32
    local = pos - gstart_r[:, 0][rnd]
    s16[(rbase[rnd] + _BAND_REC_HEAD) // 2 + local] = (rel - (rel // W) * W).to(t.int32).to(t.int16)   # uint16 bits
    s64 = stream.view(t.float64)
    s64[(rbase[rnd] + _BAND_REC_HEAD + 2 * rcnt[rnd]) // 8 + local] = values
    bd_roff = (roff // 16).to(t.int32)
    bd_sb = t.stack([pass0, npass, t.zeros_like(c_lo), t.zeros_like(c_lo)], 1).to(t.int32).contiguous()
    return stream, bd_roff, bd_sb, win.to(t.int32).contiguous(), RB, W, round_max


# Column-sorted SpMV gathers (kpl_op.sp_*): meant for matrices whose CSR-order
# warp gathers touch many cache lines (config 5's random band: ~31 of 32 lanes
# on distinct 128-byte lines; a 7-point stencil matrix: ~6).  Measured on
# config 5 it only matches the pipelined CSR-order kernel (0.304 vs 0.287
# ms/iteration), so it is opt-in: KPL_CSR_GATHER = csr (default)
# | sorted | auto (sorted when a CSR-order warp gather touches >= 12 lines).
_SORTED_MIN_LINES = 12.0
# products of one block live in shared memory (8 bytes each; two CTAs per SM fit up to ~14,000)
_SORTED_MAX_NNZ = 21_800


def csr_lines_per_warp(col_idx, sample=1 << 16):
    """Mean distinct 128-byte lines of the input a 32-lane CSR-order gather touches
    (first `sample` nonzeros)."""
    c = np.asarray(col_idx[:sample], dtype=np.int64) // 16
    m = len(c) - len(c) % 32
    if m == 0:
        return 0.0
    w = np.sort(c[:m].reshape(-1, 32), axis=1)
    return float(1.0 + (np.diff(w, axis=1) != 0).sum(axis=1).mean())


def sorted_gather_layout(row_ptr_h, col_idx_h, row_ptr, col_idx, values):
    """(sp_col, sp_val, sp_dest, rows per block, max block nnz) or None.  Index
    work only (the values are permuted, never combined), done once per matrix
    with device sorts."""
    if gather_mode() != "sorted":
        return None
    rp = np.asarray(row_ptr_h, dtype=np.int64)
    n = len(rp) - 1
    R = 0
    for cand in list(range(1024, 0, -64)) + [32, 16, 8]:     # the largest block that fits
        ends = np.minimum(np.arange(0, n, cand) + cand, n)
        most = int((rp[ends] - rp[np.arange(0, n, cand)]).max()) if n else 0
        if most <= _SORTED_MAX_NNZ:
            R = cand
            break
    if R == 0 or most < 1:
        return None
    t = torch()
    counts = (row_ptr[1:] - row_ptr[:-1]).long()
    blk = t.repeat_interleave(t.arange(n, device=row_ptr.device) // R, counts)
    perm = t.argsort(blk * (1 << 31) + col_idx.long())
    del counts
    nnz = int(col_idx.numel())
    pad = lambda a: t.cat([a, a.new_zeros(8)])      # 8 entries: the last 16-byte bulk copy may over-read
    sp_col = pad(col_idx[perm])
    sp_val = pad(values[perm])
    first = row_ptr.long()[blk[perm] * R]
    sp_dest = pad((perm - first).to(t.int32).to(t.int16))             # < 65536: uint16 bits
    del blk, perm, first
    assert sp_col.numel() == nnz + 8
    return sp_col, sp_val, sp_dest, R, most


def _matrix_stamp(A):
    """What a cached upload must still match: the host arrays' identity and
    size (a matrix whose arrays were replaced, or resized, is re-uploaded)."""
    if hasattr(A, "stencil_spec"):
        return ("stencil",) + tuple(A.stencil_spec())
    v = A.values
    return ("csr", int(A.n), len(v), id(v), id(A.col_idx), id(A.row_ptr))


def _fresh(dm, device):
    """A cached device copy is usable only on the device it lives on and for
    the host arrays it was made from (keyed on the device)."""
    return dm is not None and dm.device == torch().device(device)


def device_matrix(A, device) -> DeviceMatrix:
    cached = getattr(A, "_device", None) if _has_slot(A) else None
    if _fresh(cached, device) and cached.stamp == _matrix_stamp(A):
        return cached
    if not _has_slot(A):
        hit = _foreign_cache.get(id(A))
        if hit is not None and hit[0] is A and _fresh(hit[1], device) and hit[1].stamp == _matrix_stamp(A):
            return hit[1]
    dm = DeviceMatrix(A, device)
    if _has_slot(A):
        A._device = dm
    else:
        if len(_foreign_cache) >= _FOREIGN_MAX:
            _foreign_cache.pop(next(iter(_foreign_cache)))
        _foreign_cache[id(A)] = (A, dm)
    return dm


def _has_slot(obj):
    try:
        getattr(obj, "_device")
        return True
    except AttributeError:
        return False


class DevicePrecond:
    def __init__(self, M, dm: DeviceMatrix, device):
        t = torch()
        kind = "identity" if M is None else getattr(M, "kind", "identity")
        self.inv_diag = None
        self.const = 0.0
        self.ic = None
        if kind == "identity":
            self.code = _lib.KPL_PC_IDENTITY
        elif kind == "jacobi":
            const = getattr(M, "inv_const", None)
            if const is None and dm.kind == _lib.KPL_OP_STENCIL:
                inv = np.asarray(M.inv_diag, dtype=np.float64)
                if not np.all(inv == inv[0]):
                    raise ValueError("stencil operators need a constant Jacobi diagonal")
                const = float(inv[0])
            if dm.kind == _lib.KPL_OP_STENCIL:
                self.code = _lib.KPL_PC_JACOBI_CONST
                self.const = float(const)
            else:
                self.code = _lib.KPL_PC_JACOBI_VEC
                inv = M.inv_diag
                if len(inv) != dm.n:
                    raise ValueError("dimension mismatch in preconditioner apply")
                self.inv_diag = t.from_numpy(np.ascontiguousarray(inv, dtype=np.float64)).to(device)
        elif kind == "ic0":
            if dm.kind != _lib.KPL_OP_CSR:
                raise NotImplementedError("IC(0) runs with CSR operators (use A.to_csr())")
            ic = getattr(M, "ic", None)
            if ic is None:
                # a reference kpl.make_ic0 object: host factor in _l, its transpose in _lt
                # (precond.py:64-70, :134-154) -> uploaded as they are
                from .precond import ic0_from_host
                ic = ic0_from_host(M._l, M._lt, device)
            if ic.n != dm.n:
                raise ValueError("dimension mismatch in preconditioner apply")
            self.code = _lib.KPL_PC_IC0
            self.ic = ic
        else:
            raise NotImplementedError(f"preconditioner kind {kind!r} is not on the device path")

    @property
    def identity(self):
        return self.code == _lib.KPL_PC_IDENTITY


_pc_cache: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def device_precond(M, dm, device) -> DevicePrecond:
    if M is None or getattr(M, "kind", "identity") == "identity":
        return DevicePrecond(None, dm, device)
    key = (id(dm), str(torch().device(device)))
    try:
        hit = _pc_cache.get(M)
    except TypeError:            # reference Preconditioner: __slots__, not weak-referenceable
        hit = _foreign_cache.get(("pc", id(M)))
        hit = hit[1:] if hit is not None and hit[0] is M else None
    if hit is not None and hit[0] == key:
        return hit[1]
    dp = DevicePrecond(M, dm, device)
    try:
        _pc_cache[M] = (key, dp)
    except TypeError:
        if len(_foreign_cache) >= _FOREIGN_MAX:
            _foreign_cache.pop(next(iter(_foreign_cache)))
        _foreign_cache[("pc", id(M))] = (M, key, dp)
    return dp


def make_op(dm: DeviceMatrix, dp: DevicePrecond | None = None, zc=0, vx=0, chunk_blocks=0,
            geometry=None) -> KplOp:
    """`geometry` overrides the stencil grid view (e.g. a 2D grid's slab view)."""
    op = KplOp()
    op.kind = dm.kind
    op.precond = dp.code if dp is not None else _lib.KPL_PC_IDENTITY
    op.n = dm.n
    if dm.kind == _lib.KPL_OP_STENCIL:
        op.nx, op.ny, op.nz, op.diag = dm.nx, dm.ny, dm.nz, float(dm.diag)
        if geometry is not None:
            op.nx, op.ny, op.nz = geometry
    else:
        op.row_ptr = ptr(dm.row_ptr)
        op.col_idx = ptr(dm.col_idx)
        op.values = ptr(dm.values)
        op.nnz = dm.nnz
        if dm.sorted is not None:
            sc, sv, sd, R, most = dm.sorted
            op.sp_col, op.sp_val, op.sp_dest = ptr(sc), ptr(sv), ptr(sd)
            op.sp_rows, op.sp_max = R, most
        if dm.band is not None:
            st, ro, bs, bw, rows, W, round_max = dm.band
            op.bd_stream, op.bd_roff, op.bd_sb, op.bd_win = ptr(st), ptr(ro), ptr(bs), ptr(bw)
            op.bd_rows, op.bd_w, op.bd_round_max = rows, W, round_max
    op.zc = zc
    op.vx = vx
    op.chunk_blocks = chunk_blocks
    op.order = ORDERS[get_reduction_order()]
    if dp is not None:
        op.pc_const = dp.const
        op.inv_diag = ptr(dp.inv_diag)
        if dp.ic is not None:
            set_ic0(op, dp.ic)
    return op


def set_ic0(op, ic):
    """Point kpl_op's IC(0) fields at a device factor (precond.Ic0Factor)."""
    op.ic_l_row_ptr, op.ic_l_col_idx, op.ic_l_values = ptr(ic.l_ptr), ptr(ic.l_col), ptr(ic.l_val)
    op.ic_u_row_ptr, op.ic_u_col_idx, op.ic_u_values = ptr(ic.u_ptr), ptr(ic.u_col), ptr(ic.u_val)
    op.ic_l_order, op.ic_u_order = ptr(ic.l_order), ptr(ic.u_order)


def vector_op(n) -> KplOp:
    """Layout descriptor for plain vectors (dot without an operator)."""
    op = KplOp()
    op.kind = _lib.KPL_OP_CSR
    op.n = n
    op.order = ORDERS[get_reduction_order()]
    return op


def to_device_f64(v, n, device, what):
    """Upload (or adopt) a length-n fp64 vector.

    Returns (tensor, io) with io = "numpy" (host array in, numpy out),
    "host" (CPU torch tensor in, e.g. pinned memory: CPU tensor out) or
    False (CUDA tensor in: result stays on the device)."""
    t = torch()
    if isinstance(v, t.Tensor):
        if v.dim() != 1 or v.numel() != n:
            raise ValueError(f"{what} dimension mismatch")
        io = "host" if v.device.type == "cpu" else False
        return v.to(device=device, dtype=t.float64, non_blocking=True).contiguous(), io
    a = np.asarray(v, dtype=np.float64)
    if a.shape != (n,):
        raise ValueError(f"{what} dimension mismatch")
    a = np.ascontiguousarray(a)
    if a.nbytes >= _STAGE_MIN:
        out = t.empty(n, dtype=t.float64, device=device)
        _staging(device).h2d(a, out)
        return out, "numpy"
    return t.from_numpy(a).to(device, non_blocking=False), "numpy"


def to_numpy_f64(d):
    """Device fp64 vector -> a new numpy array (pipelined pinned staging when large)."""
    if d.numel() * 8 >= _STAGE_MIN:
        out = np.empty(d.numel(), dtype=np.float64)
        _staging(d.device).d2h(d, out)
        return out
    return d.cpu().numpy()


# Host <-> device copies of large numpy vectors (a kpl caller's b and x): a
# pageable cudaMemcpy stages through one driver buffer at a time; here a ring
# of pinned chunks is filled / drained by host threads (numpy copies release
# the GIL) while the DMA engine moves the previous chunk, so the CPU memcpy
# and the PCIe transfer overlap.
_STAGE_MIN = 64 << 20          # below this the plain copy is as fast
_STAGE_CHUNK = 16 << 20        # bytes per pinned slot
_STAGE_SLOTS = 4
_stagers: dict = {}


def _staging(device):
    key = str(device)
    st = _stagers.get(key)
    if st is None:
        st = _stagers[key] = _HostStaging(device)
    return st


class _HostStaging:
    def __init__(self, device):
        import concurrent.futures
        t = torch()
        self.device = device
        per = _STAGE_CHUNK // 8
        self.slots = [t.empty(per, dtype=t.float64, pin_memory=True) for _ in range(_STAGE_SLOTS)]
        self.views = [s.numpy() for s in self.slots]
        self.events = [None] * _STAGE_SLOTS
        self.pool = concurrent.futures.ThreadPoolExecutor(max_workers=_STAGE_SLOTS)
        self.per = per

    def h2d(self, a, out):
        """out[:] = a (numpy, contiguous) on the current stream."""
        t = torch()
        stream = t.cuda.current_stream(self.device)
        n, per = a.size, self.per
        starts = list(range(0, n, per))
        fill = lambda i, k0: np.copyto(self.views[i][:min(per, n - k0)], a[k0:k0 + per])
        pending = {}
        for j, k0 in enumerate(starts[:_STAGE_SLOTS]):
            pending[j] = self.pool.submit(fill, j % _STAGE_SLOTS, k0)
        for j, k0 in enumerate(starts):
            i = j % _STAGE_SLOTS
            pending.pop(j).result()
            m = min(per, n - k0)
            out[k0:k0 + m].copy_(self.slots[i][:m], non_blocking=True)
            ev = t.cuda.Event()
            ev.record(stream)
            self.events[i] = ev
            nxt = j + _STAGE_SLOTS
            if nxt < len(starts):           # refill slot i once its DMA has left it
                def refill(i=i, k0=starts[nxt], ev=ev):
                    ev.synchronize()
                    fill(i, k0)
                pending[nxt] = self.pool.submit(refill)
        for ev in self.events:
            if ev is not None:
                ev.synchronize()            # the caller may reuse `a` right away

    def d2h(self, d, out):
        """out[:] = d (device, contiguous) -- waits for the current stream's work on d."""
        t = torch()
        stream = t.cuda.current_stream(self.device)
        n, per = d.numel(), self.per
        starts = list(range(0, n, per))
        drains = []
        for j, k0 in enumerate(starts):
            i = j % _STAGE_SLOTS
            if j >= _STAGE_SLOTS:
                drains[j - _STAGE_SLOTS].result()      # slot i's previous chunk is out
            m = min(per, n - k0)
            self.slots[i][:m].copy_(d[k0:k0 + m], non_blocking=True)
            ev = t.cuda.Event()
            ev.record(stream)

            def drain(i=i, k0=k0, m=m, ev=ev):
                ev.synchronize()
                np.copyto(out[k0:k0 + m], self.views[i][:m])
            drains.append(self.pool.submit(drain))
        for f in drains:
            f.result()
