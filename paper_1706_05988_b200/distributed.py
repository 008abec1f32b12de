"""Multi-GPU z-slab solver: one rank per GPU, NCCL for plumbing.

Partition.  A stencil grid (NX, NY, NZ) (2D grids are (nx, 1, ny)) is cut into
P z-slabs of NZ/P planes.  Each rank stores its slab of every vector plus one
halo plane below and above (`kpl_op.zhalo = 1`); global-boundary halos stay
zero (Dirichlet).  Slabs are whole reduction chunks (zc | NZ/P), so each
rank's chunk partials are exactly the partials a single GPU would compute for
those planes.

Per sweep.  halo exchange of the sweep's stencil input (plane 0 -> rank-1's
upper halo, plane nz-1 -> rank+1's lower halo; NCCL send/recv over NVLink) ->
the fused sweep on the local slab (writes this rank's slice of the chunk
table) -> all-gather of the chunk table (P x chunks x 32 bytes) -> the
level-4 fold + scalar epilogue on every rank (identical inputs, identical
scalars).  Because the chunk partials and the fold order do not depend on P,
a P-rank solve is bit-identical to the 1-GPU solve.

Communicators.  `TorchComm` wraps torch.distributed (NCCL on GPUs, gloo on
CPU for the plumbing tests).  `LocalComm` runs P ranks as P slab states in
one process on one device (exchanges and gathers become device copies; all
sweeps are launched sequentially, none waits on another) -- the single-GPU
stand-in used by the parity tests.

Row-block CSR.  `RowPlan` cuts the rows into chunk-aligned blocks; every
rank keeps its rows of the matrix with columns remapped to [local rows |
ghosts], where the ghosts are the sorted remote columns its rows touch.  Per
sweep the owners pack the requested rows (kpl_gather) and send them to the
ghost segments (NCCL send/recv); the Jacobi inverse diagonal of the ghosts is
static and copied once.

Scope: stencils (identity or constant-diagonal Jacobi) and CSR (identity or
Jacobi); every method (cg / pcg / pcg_sh / pcg_var_sh / pcg_rr) and
track_gaps.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _lib, device as D
from .solvers import (HC, BreakdownError, SolveResult, SolverConfig, make_kcfg, records_from)

_ZC_CHOICES = (16, 8, 4, 2, 1)
_BD_PEER_TIMEOUT = 7          # kpl_breakdown_message(7) == "peer exchange timeout"


class SlabPlan:
    """z-slab partition of an (NX, NY, NZ) grid over P ranks."""

    def __init__(self, NX, NY, NZ, P, zc=0):
        if NZ % P:
            raise ValueError(f"NZ={NZ} planes do not split evenly over {P} ranks")
        self.NX, self.NY, self.NZ, self.P = NX, NY, NZ, P
        self.nzl = NZ // P
        if zc <= 0:
            zc = next(c for c in _ZC_CHOICES if self.nzl % c == 0)
        if self.nzl % zc:
            raise ValueError(f"chunk length zc={zc} must divide the slab depth {self.nzl}")
        self.zc = zc
        self.sxy = NX * NY
        self.n_local = self.sxy * self.nzl
        self.chunks_local = self.nzl // zc
        self.chunks_global = self.chunks_local * P

    def z0(self, rank):
        return rank * self.nzl

    def local_slice(self, rank):
        """Slice of a global natural-order vector owned by `rank`."""
        a = rank * self.n_local
        return slice(a, a + self.n_local)


def storage_names(cfg, ident):
    """State vectors a rank stores (identity aliases u=r, q=s, p=t share storage)."""
    names = ["x", "r"]
    if not ident:
        names.append("u")
    if cfg.method == "cg":
        names += ["p", "p1", "s"]
    else:
        names += ["w0", "w1", "z", "s", "t"]
        if not ident:
            names += ["q", "p"]
    return names


_ALIGN = 256


def _align(v):
    return (v + _ALIGN - 1) // _ALIGN * _ALIGN


class PeerLayout:
    """Byte layout of one rank's peer-shareable region (device-initiated
    exchange): flag words (one uint64 per rank, written by that rank's posts),
    the post completion counter, the double-buffered exchange table
    [2][chunks_global][4] fp64, then every stored state vector (interior +
    halo planes / ghost rows).  Every rank computes every rank's layout."""

    FLAGS = 0
    COUNTER = 8 * _lib.KPL_PEER_MAX_RANKS

    def __init__(self, names, n_total, chunks_global):
        self.chunks_global = chunks_global
        off = _align(self.COUNTER + 8)
        self.px = off                       # device copy of kpl_peer_sweep (fused sweeps)
        off += _align(ctypes.sizeof(_lib.KplPeerSweep))
        self.table = off
        off += _align(2 * 4 * 8 * chunks_global)
        self.vec = {}
        for nm in names:
            self.vec[nm] = off
            off += _align(8 * n_total)
        self.bytes = off

    def table_slot(self, parity):
        return self.table + parity * 4 * 8 * self.chunks_global


class _RankState:
    """Device state of one rank: vectors (interior + halo/ghost storage), op,
    kcfg, workspace and its chunk-table views.  Subclasses define the layout."""

    VEC_NAMES = ("x", "r", "u", "w0", "w1", "z", "q", "s", "t", "p", "p1")

    def _alloc_vectors(self, cfg, ident, n, extra, device, region=None, layout=None):
        """Every state vector as one tensor of n + extra values (extra = halo
        or ghost storage); identity aliases u=r, q=s, p=t as on one GPU.
        With a peer region (device-initiated exchange) the vectors are views
        into it at the offsets of `layout`."""
        t = D.torch()
        f64 = dict(dtype=t.float64, device=device)
        self.full = {}
        names = storage_names(cfg, ident)
        for nm in names:
            if region is None:
                self.full[nm] = t.zeros(n + extra, **f64)
            else:
                o = layout.vec[nm]
                self.full[nm] = region[o:o + 8 * (n + extra)].view(t.float64)
                self.full[nm].zero_()
        self.alias = {nm: nm for nm in names}
        if ident:
            self.full["u"] = self.full["r"]
            self.alias["u"] = "r"
            if cfg.method != "cg":
                self.full["q"] = self.full["s"]
                self.full["p"] = self.full["t"]
                self.alias["q"], self.alias["p"] = "s", "t"
        self.b = t.zeros(n, **f64)

    def _finish(self, op, cfg, kcfg, device, chunks_local):
        t = D.torch()
        self.op, self.kcfg, self.cfg = op, kcfg, cfg
        v = _lib.KplVecs()
        for nm in self.VEC_NAMES:
            setattr(v, nm, D.ptr(self.interior(nm)) if nm in self.full else None)
        v.b = D.ptr(self.b)
        self.vecs = v
        lib = _lib.load()
        nbytes = lib.kpl_workspace_bytes(op, cfg.max_iters)
        _lib.check(nbytes if nbytes < 0 else 0, "workspace size")
        self.ws = t.empty(int(nbytes), dtype=t.uint8, device=device)
        loc, glob, lbytes = _lib._p(), _lib._p(), _lib._i64()
        _lib.check(lib.kpl_chunk_table(op, D.ptr(self.ws), loc, glob, lbytes), "chunk table")
        base = self.ws.data_ptr()
        g0 = glob.value - base
        nb = 8 * 4 * int(op.chunks_global)
        self.table = self.ws[g0:g0 + nb].view(t.float64)
        self.chunk_offset = int(op.chunk_offset)
        self.chunks_local = chunks_local
        self.table_local = self.table[4 * self.chunk_offset:4 * (self.chunk_offset + chunks_local)]
        self.hist_off = lib.kpl_history_offset(op)
        self.reps_off = lib.kpl_replacements_offset(op, cfg.max_iters)
        self.status = _lib.KplStatus()

    # -- device calls (on this rank's stream: the current stream, or its own
    #    stream when a LocalPeerComm runs the ranks concurrently)
    stream = None

    def hs(self):
        return self.stream.cuda_stream if self.stream is not None else D.stream_handle()

    def prepare(self):
        _lib.check(_lib.load().kpl_solver_prepare(self.op, self.kcfg, self.vecs, D.ptr(self.ws),
                                                  self.hs()), "prepare")

    def sweep(self, kind, row=0):
        _lib.check(_lib.load().kpl_sweep(self.op, self.kcfg, self.vecs, kind, row, D.ptr(self.ws),
                                         self.hs()), f"sweep {kind}")

    def finalize(self, kind, row=0):
        _lib.check(_lib.load().kpl_finalize_global(self.op, self.kcfg, kind, row, D.ptr(self.ws),
                                                   self.hs()), f"finalize {kind}")

    def read_status(self):
        _lib.check(_lib.load().kpl_read_status(D.ptr(self.ws), self.status, self.hs()), "status")
        return self.status

    def history(self, rows):
        t = D.torch()
        raw = self.ws[self.hist_off:self.hist_off + 8 * HC * rows]
        return raw.view(t.float64).reshape(rows, HC).cpu().numpy()


class _SlabState(_RankState):
    """z-slab of a stencil grid: vectors carry one halo plane on each side."""

    def __init__(self, plan: SlabPlan, rank, diag, pc_code, pc_const, cfg, device, kcfg, region=None,
                 layout=None):
        self.plan, self.rank, self.device = plan, rank, device
        self.ident = pc_code == _lib.KPL_PC_IDENTITY
        n, sxy = plan.n_local, plan.sxy
        self._alloc_vectors(cfg, self.ident, n, 2 * sxy, device, region, layout)
        op = _lib.KplOp()
        op.kind = _lib.KPL_OP_STENCIL
        op.precond = pc_code
        op.n = n
        op.nx, op.ny, op.nz, op.diag = plan.NX, plan.NY, plan.nzl, float(diag)
        op.zc = plan.zc
        op.zhalo = 1
        op.pc_const = pc_const
        op.chunk_offset = rank * plan.chunks_local
        op.chunks_global = plan.chunks_global
        self._finish(op, cfg, kcfg, device, plan.chunks_local)

    def interior(self, name):
        sxy = self.plan.sxy
        return self.full[name][sxy:sxy + self.plan.n_local]

    def planes(self, name):
        """(lower halo, first plane, last plane, upper halo) views."""
        f, sxy, n = self.full[name], self.plan.sxy, self.plan.n_local
        return f[:sxy], f[sxy:2 * sxy], f[n:n + sxy], f[n + sxy:]


class RowPlan:
    """Row-block partition of a CSR matrix over P ranks with general halo
    (ghost) gathers.  Block boundaries are multiples of one reduction chunk
    (chunk_blocks x 256 rows), so every rank's chunk partials are the ones a
    single GPU computes for those rows and the gathered fold is bit-identical.

    Every rank holds the host matrix, so every rank derives every rank's ghost
    and send lists locally -- no setup communication."""

    def __init__(self, A, P, chunk_blocks=8):
        n = int(A.n)
        self.n, self.P = n, P
        self.chunk_rows = 256 * chunk_blocks
        self.chunk_blocks = chunk_blocks
        al = self.chunk_rows
        starts = [min(n, ((r * n) // P) // al * al) for r in range(P)] + [n]
        if any(starts[r + 1] <= starts[r] for r in range(P)):
            raise ValueError(f"{n} rows are too few for {P} ranks of {al}-row chunks")
        self.starts = starts
        self.chunks_global = -(-n // al)
        rp = np.asarray(A.row_ptr, dtype=np.int64)
        ci = np.asarray(A.col_idx, dtype=np.int64)
        self.ranks = []
        for r in range(P):
            r0, r1 = starts[r], starts[r + 1]
            k0, k1 = int(rp[r0]), int(rp[r1])
            cols = ci[k0:k1]
            remote = (cols < r0) | (cols >= r1)
            ghosts = np.unique(cols[remote])
            owner = np.searchsorted(np.asarray(starts), ghosts, side="right") - 1
            local = np.where(remote, 0, cols - r0)
            gpos = np.searchsorted(ghosts, cols[remote])
            local[remote] = (r1 - r0) + gpos
            recv = {}
            for q in np.unique(owner):
                sel = np.nonzero(owner == q)[0]
                recv[int(q)] = (int(sel[0]), len(sel), ghosts[sel] - starts[q])   # offset, count, q-local rows
            self.ranks.append(dict(r0=r0, r1=r1, k0=k0, k1=k1, ghosts=ghosts, recv=recv,
                                   row_ptr=(rp[r0:r1 + 1] - k0).astype(np.int32),
                                   col_idx=local.astype(np.int32)))
        # send lists: rank q sends to r the q-local rows listed in r's recv[q]
        for r in range(P):
            self.ranks[r]["send"] = {}
        for r in range(P):
            for q, (off, cnt, qrows) in self.ranks[r]["recv"].items():
                self.ranks[q]["send"][r] = qrows

    def local_slice(self, rank):
        return slice(self.starts[rank], self.starts[rank + 1])

    def chunk_offset(self, rank):
        return self.starts[rank] // self.chunk_rows

    def chunks_local(self, rank):
        return -(-(self.starts[rank + 1] - self.starts[rank]) // self.chunk_rows)


class _RowState(_RankState):
    """Row block of a CSR matrix: vectors = [local rows | ghost values]."""

    def __init__(self, plan: RowPlan, rank, A, M, pc_code, cfg, device, kcfg, region=None, layout=None):
        t = D.torch()
        self.plan, self.rank, self.device = plan, rank, device
        self.ident = pc_code == _lib.KPL_PC_IDENTITY
        info = plan.ranks[rank]
        n = info["r1"] - info["r0"]
        self.n_local, self.n_ghost = n, len(info["ghosts"])
        self._alloc_vectors(cfg, self.ident, n, self.n_ghost, device, region, layout)
        up = lambda a, dt: t.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(device)
        self.row_ptr = up(info["row_ptr"], np.int32)
        self.col_idx = up(info["col_idx"], np.int32)
        self.values = up(np.asarray(A.values)[info["k0"]:info["k1"]], np.float64)
        op = _lib.KplOp()
        op.kind = _lib.KPL_OP_CSR
        op.precond = pc_code
        op.n = n
        op.row_ptr, op.col_idx, op.values = D.ptr(self.row_ptr), D.ptr(self.col_idx), D.ptr(self.values)
        op.nnz = info["k1"] - info["k0"]
        op.chunk_blocks = plan.chunk_blocks
        self.dinv = None
        if pc_code == _lib.KPL_PC_JACOBI_VEC:
            inv = np.asarray(M.inv_diag, dtype=np.float64)
            # inverse diagonal of the local rows followed by the ghosts' (static, no exchange)
            self.dinv = up(np.concatenate([inv[info["r0"]:info["r1"]], inv[info["ghosts"]]]), np.float64)
            op.inv_diag = D.ptr(self.dinv)
        op.chunk_offset = plan.chunk_offset(rank)
        op.chunks_global = plan.chunks_global
        self.recv = {q: (off, cnt) for q, (off, cnt, _) in info["recv"].items()}
        self.send_idx = {q: up(rows, np.int32) for q, rows in info["send"].items()}
        self.send_buf = {q: t.empty(len(rows), dtype=t.float64, device=device)
                         for q, rows in info["send"].items()}
        self._finish(op, cfg, kcfg, device, plan.chunks_local(rank))

    def interior(self, name):
        return self.full[name][:self.n_local]

    def ghost(self, name, q):
        off, cnt = self.recv[q]
        return self.full[name][self.n_local + off:self.n_local + off + cnt]


def _gather(idx, src, dst):
    """dst[k] = src[idx[k]] on the device (kpl_gather)."""
    _lib.check(_lib.load().kpl_gather(idx.numel(), D.ptr(idx), D.ptr(src), D.ptr(dst),
                                      D.stream_handle()), "gather")


class LocalComm:
    """P ranks as P states in one process on one device (parity tests)."""

    def __init__(self, P):
        self.size = P
        self.rank = None                 # all ranks are local

    def local_ranks(self):
        return list(range(self.size))

    def solve_barrier(self):
        pass

    def exchange(self, states, name):
        for s in states:
            r = s.rank
            if isinstance(s, _SlabState):
                lo, first, last, hi = s.planes(name)
                if r > 0:
                    lo.copy_(states[r - 1].planes(name)[2])
                if r < self.size - 1:
                    hi.copy_(states[r + 1].planes(name)[1])
            else:
                for q in s.recv:
                    src = states[q]
                    _gather(src.send_idx[r], src.interior(name), s.ghost(name, q))

    def allgather(self, states):
        for dst in states:
            for src in states:
                if src is not dst:
                    o, n = 4 * src.chunk_offset, 4 * src.chunks_local
                    dst.table[o:o + n].copy_(src.table_local)


class TorchComm:
    """torch.distributed process group (NCCL over NVLink on GPUs; gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.size = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self._counts = {}          # per partition plan: every rank's chunk count
        # gloo moves CUDA tensors for collectives but not point-to-point: stage
        # those through host memory (used to run the multi-process path on a
        # single GPU; NCCL is the production backend)
        self.stage_p2p = dist.get_backend(group) == "gloo"

    def _p2p(self, sends, recvs):
        """sends/recvs: lists of (tensor, peer)."""
        dist = self.dist
        if self.stage_p2p:
            host_s = [(t.cpu(), q) for t, q in sends]
            host_r = [(t.new_empty(t.shape, device="cpu"), q) for t, q in recvs]
            ops = [dist.P2POp(dist.isend, t, q, self.group) for t, q in host_s]
            ops += [dist.P2POp(dist.irecv, t, q, self.group) for t, q in host_r]
            if ops:
                for req in dist.batch_isend_irecv(ops):
                    req.wait()
            for (dst, _), (src, _) in zip(recvs, host_r):
                dst.copy_(src)
            return
        ops = [dist.P2POp(dist.isend, t, q, self.group) for t, q in sends]
        ops += [dist.P2POp(dist.irecv, t, q, self.group) for t, q in recvs]
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def local_ranks(self):
        return [self.rank]

    def solve_barrier(self):
        """Host barrier at the start of every solve: a reused peer
        region must not receive pushes from a rank that is already in the
        next solve while this rank is still zeroing its state."""
        self.dist.barrier(group=self.group)

    def exchange(self, states, name):
        (s,) = states
        sends, recvs = [], []
        if isinstance(s, _SlabState):
            lo, first, last, hi = s.planes(name)
            if s.rank > 0:
                sends.append((first, s.rank - 1))
                recvs.append((lo, s.rank - 1))
            if s.rank < self.size - 1:
                sends.append((last, s.rank + 1))
                recvs.append((hi, s.rank + 1))
        else:
            for q, idx in s.send_idx.items():          # pack the rows each peer needs
                _gather(idx, s.interior(name), s.send_buf[q])
                sends.append((s.send_buf[q], q))
            for q in s.recv:
                recvs.append((s.ghost(name, q), q))
        self._p2p(sends, recvs)

    def allgather(self, states):
        (s,) = states
        t = D.torch()
        key = (s.chunk_offset, s.chunks_local, int(s.table.numel()) // 4)
        counts = self._counts.get(key)
        if counts is None:          # a new partition (never reuse another plan's counts)
            dev = "cpu" if self.stage_p2p else s.table.device
            c = t.tensor([s.chunks_local], dtype=t.int64, device=dev)
            allc = [t.zeros_like(c) for _ in range(self.size)]
            self.dist.all_gather(allc, c, group=self.group)
            counts = self._counts[key] = [int(v.item()) for v in allc]
        if self.stage_p2p:                       # gloo: host-staged, equal-size (padded) all-gather
            mx = max(counts)
            mine = t.zeros(4 * mx, dtype=t.float64)
            mine[:4 * counts[self.rank]].copy_(s.table_local.cpu())
            parts = [t.zeros(4 * mx, dtype=t.float64) for _ in counts]
            self.dist.all_gather(parts, mine, group=self.group)
            s.table.copy_(t.cat([p[:4 * cq] for p, cq in zip(parts, counts)]))
            return
        if all(c == counts[0] for c in counts):
            # in-place all-gather: this rank's slice sits at offset rank*count
            self.dist.all_gather_into_tensor(s.table, s.table_local.clone(), group=self.group)
            return
        # uneven row blocks: gather padded slices, then compact in rank order
        mx = max(counts)
        buf = t.zeros(4 * mx * self.size, dtype=t.float64, device=s.table.device)
        mine = t.zeros(4 * mx, dtype=t.float64, device=s.table.device)
        mine[:s.table_local.numel()].copy_(s.table_local)
        self.dist.all_gather_into_tensor(buf, mine, group=self.group)
        off = 0
        for q, cq in enumerate(counts):
            s.table[4 * off:4 * (off + cq)].copy_(buf[4 * mx * q:4 * mx * q + 4 * cq])
            off += cq


class _CudaArray:
    """__cuda_array_interface__ view of raw device bytes (wraps an IPC region
    as a torch tensor without copying)."""

    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None}


class _Regions:
    """Peer-shareable regions of one layout set: this process's tensors, every
    rank's base address, and the epoch counter of its flag words (flags are
    never reset, so epochs keep increasing across the solves that reuse it)."""

    def __init__(self, tensors, bases, owned=(), opened=()):
        self.tensors, self.bases = tensors, bases
        self.epoch = 0          # last signalled flag value
        self.red = 0            # reductions exchanged (table slot = red & 1)
        self._owned, self._opened = list(owned), list(opened)

    def close(self, barrier=None):
        """Unmap the peers' regions, then (after `barrier`, so no rank still has
        this rank's region mapped -- freeing an exported allocation while it is
        open elsewhere is undefined) free this rank's own."""
        lib = _lib.load()
        for p in self._opened:
            lib.kpl_ipc_close(p)
        if barrier is not None and self._owned:
            barrier()
        for p in self._owned:
            lib.kpl_ipc_free(p)
        self._owned, self._opened, self.tensors = [], [], {}


class LocalPeerComm(LocalComm):
    """P ranks on one device exchanging through the device-initiated peer path
    (kpl_peer_post / kpl_peer_finalize) with plain device pointers as the peer
    pointers.  By default every rank's sweep, post and finalize are launched
    in rank order on one stream, so each wait is already satisfied when its
    kernel starts.  `concurrent=True` gives every rank its own CUDA stream:
    the ranks' kernels then run at the same time and the flag waits really
    block -- only for problems whose grids are co-resident
    on the one device (a waiting CTA must not starve the kernel it waits for)."""

    peer = True

    def __init__(self, P, fused=True, concurrent=False, fold=True):
        super().__init__(P)
        self.fused = fused
        self.fold = fold
        self.concurrent = concurrent
        self._cache = {}

    def regions(self, sizes, device):
        key = tuple(sizes)
        if key not in self._cache:
            t = D.torch()
            tens = {q: t.zeros(sz, dtype=t.uint8, device=device) for q, sz in enumerate(sizes)}
            self._cache = {key: _Regions(tens, [tens[q].data_ptr() for q in range(len(sizes))])}
        return self._cache[key]


def LocalPeerCommNoFold(P):
    """LocalPeerComm with a kpl_peer_finalize launch between consecutive fused
    iteration sweeps (no deferred fold) -- the parity tests run both forms."""
    return LocalPeerComm(P, fold=False)


def LocalPeerCommPostOnly(P):
    """LocalPeerComm without the fused sweep exchange (every sweep is followed
    by a kpl_peer_post kernel) -- the parity tests run both forms."""
    return LocalPeerComm(P, fused=False)


class PeerComm(TorchComm):
    """One process per GPU, exchanging through peer memory over NVLink: each
    rank allocates its region with kpl_ipc_alloc, the 64-byte IPC handles are
    all-gathered once through torch.distributed, and every rank maps the
    others' regions (kpl_ipc_open).  Per sweep there is no host-side
    collective: kpl_peer_post pushes halos + partials and signals,
    kpl_peer_finalize waits and folds."""

    peer = True

    def __init__(self, group=None, fused=True):
        super().__init__(group)
        self.fused = fused
        self._cache = {}

    def regions(self, sizes, device):
        key = tuple(sizes)
        if key in self._cache:
            return self._cache[key]
        for r in self._cache.values():
            r.close(barrier=lambda: self.dist.barrier(group=self.group))
        self._cache = {}
        import ctypes
        lib = _lib.load()
        me, P = self.rank, self.size
        ptr = ctypes.c_void_p()
        h = ctypes.create_string_buffer(64)
        _lib.check(lib.kpl_ipc_alloc(int(sizes[me]), ctypes.byref(ptr), h), "IPC region")
        handles = [None] * P
        self.dist.all_gather_object(handles, bytes(h.raw), group=self.group)
        bases, opened, why = [], [], ""
        for q in range(P):
            if q == me:
                bases.append(ptr.value)
                continue
            p = ctypes.c_void_p()
            if lib.kpl_ipc_open(ctypes.create_string_buffer(handles[q], 64), ctypes.byref(p)) != 0:
                why = f"rank {me}: IPC open of rank {q}: {lib.kpl_last_error().decode()}"
                break
            bases.append(p.value)
            opened.append(p.value)
        # one collective verdict, so every rank takes the same path
        verdicts = [None] * P
        self.dist.all_gather_object(verdicts, why, group=self.group)
        bad = [v for v in verdicts if v]
        if bad:
            _Regions({}, [], owned=[ptr.value], opened=opened).close(
                barrier=lambda: self.dist.barrier(group=self.group))
            raise _lib.KplError("peer exchange unavailable: " + "; ".join(bad))
        t = D.torch()
        tens = {me: t.as_tensor(_CudaArray(ptr.value, int(sizes[me])), device=device)}
        self._cache[key] = _Regions(tens, bases, owned=[ptr.value], opened=opened)
        # every rank has mapped every region before any rank pushes into one
        self.dist.barrier(group=self.group)
        return self._cache[key]


class DistributedSolve:
    """Drive one partitioned solve (stencil z-slabs or CSR row blocks);
    `comm` decides which ranks are local."""

    def __init__(self, A, M, cfg: SolverConfig, comm, zc=0, chunk_blocks=8):
        self.device = D.require_cuda()
        self.A, self.cfg, self.comm = A, cfg, comm
        kind = "identity" if M is None else getattr(M, "kind", "identity")
        self.limit = cfg.max_iters + (1 if cfg.method == "cg" else 0)
        if not hasattr(A, "stencil_spec"):
            if kind not in ("identity", "jacobi"):
                raise NotImplementedError(f"preconditioner {kind!r} not on the device path")
            pc = _lib.KPL_PC_IDENTITY if kind == "identity" else _lib.KPL_PC_JACOBI_VEC
            self.plan = RowPlan(A, comm.size, chunk_blocks)
            self.kcfg, self._keep = make_kcfg(cfg, A, self, self.device)
            n_tot = [info["r1"] - info["r0"] + len(info["ghosts"]) for info in self.plan.ranks]
            self._peer_regions(cfg, kind == "identity", n_tot)
            self.states = [_RowState(self.plan, r, A, M, pc, cfg, self.device, self.kcfg, *self._region(r))
                           for r in comm.local_ranks()]
            self._peer_ready()
            return
        NX, NY, NZ, diag = A.slab_spec() if hasattr(A, "slab_spec") else A.stencil_spec()
        self.plan = SlabPlan(NX, NY, NZ, comm.size, zc)
        if kind == "identity":
            pc, c = _lib.KPL_PC_IDENTITY, 0.0
        elif kind == "jacobi":
            c = getattr(M, "inv_const", None)
            if c is None:
                inv = np.asarray(M.inv_diag)
                if not np.all(inv == inv[0]):
                    raise ValueError("stencil operators need a constant Jacobi diagonal")
                c = float(inv[0])
            pc = _lib.KPL_PC_JACOBI_CONST
        else:
            raise NotImplementedError(f"preconditioner {kind!r} not on the device path")
        self.kcfg, self._keep = make_kcfg(cfg, A, self, self.device)
        self._peer_regions(cfg, kind == "identity", [self.plan.n_local + 2 * self.plan.sxy] * comm.size)
        self.states = [_SlabState(self.plan, r, diag, pc, c, cfg, self.device, self.kcfg, *self._region(r))
                       for r in comm.local_ranks()]
        self._peer_ready()

    # -- device-initiated exchange (peer comms)
    def _peer_regions(self, cfg, ident, n_tot):
        self.peer = bool(getattr(self.comm, "peer", False))
        self._pending = None
        self.fused = False
        self.fold = False
        if not self.peer:
            return
        # fused exchange inside the iteration sweep: stencil slabs, pipelined methods
        self.fused = (bool(getattr(self.comm, "fused", True)) and isinstance(self.plan, SlabPlan)
                      and cfg.method != "cg")
        # ... and the deferred fold of one iteration sweep's exchange inside the next
        # (KPL_PEER_FOLD=0 keeps a kpl_peer_finalize launch between them)
        self.fold = (self.fused and cfg.method in ("pcg", "pcg_sh", "pcg_var_sh") and not cfg.track_gaps
                     and bool(getattr(self.comm, "fold", True))
                     and os.environ.get("KPL_PEER_FOLD", "1") != "0")
        if self.comm.size > _lib.KPL_PEER_MAX_RANKS:
            raise ValueError(f"peer exchange supports up to {_lib.KPL_PEER_MAX_RANKS} ranks")
        self._names = storage_names(cfg, ident)
        self.layouts = [PeerLayout(self._names, n, self.plan.chunks_global) for n in n_tot]
        self.reg = self.comm.regions([L.bytes for L in self.layouts], self.device)
        self._posts = {}

    def _region(self, r):
        if not self.peer:
            return (None, None)
        return (self.reg.tensors[r], self.layouts[r])

    def _peer_ready(self):
        if not self.peer:
            return
        self._dirty = set(self._names)
        if self.fused:
            t = D.torch()
            for s in self.states:
                px = self._peer_sweep_struct(s)
                raw = t.frombuffer(bytearray(bytes(px)), dtype=t.uint8)
                o = self.layouts[s.rank].px
                self.reg.tensors[s.rank][o:o + len(raw)].copy_(raw)     # stream-ordered before any sweep

    def _peer_sweep_struct(self, s):
        """kpl_peer_sweep of rank s: every rank's table slots and flag word for
        s, and the neighbour halo planes of w0, w1 and x."""
        P, r = self.comm.size, s.rank
        sxy, n = self.plan.sxy, self.plan.n_local
        px = _lib.KplPeerSweep()
        px.nranks = P
        px.rank = r
        px.flags = self.reg.bases[r] + PeerLayout.FLAGS
        for par in (0, 1):
            for q in range(P):
                px.table[par][q] = self.reg.bases[q] + self.layouts[q].table_slot(par)
        for q in range(P):
            px.signal[q] = self.reg.bases[q] + PeerLayout.FLAGS + 8 * r

        def halos(name):
            lo = self._addr(r - 1, name, sxy + n) if r > 0 else None
            hi = self._addr(r + 1, name, 0) if r < P - 1 else None
            return s.interior(name).data_ptr(), lo, hi

        for k, nm in enumerate(("w0", "w1")):
            px.w_src[k], px.w_lo[k], px.w_hi[k] = halos(nm)
        px.x_src, px.x_lo, px.x_hi = halos("x")
        return px

    def _addr(self, q, name, elem_off=0):
        """Device address of element `elem_off` of rank q's stored vector `name`."""
        return self.reg.bases[q] + self.layouts[q].vec[name] + 8 * elem_off

    def _halo_copies(self, s, name):
        """(src, idx, dst, count) of the rows peers read of this rank's `name`."""
        out = []
        full = s.full[name].data_ptr()
        if isinstance(s, _SlabState):
            sxy, n = self.plan.sxy, self.plan.n_local
            if s.rank > 0:                         # first plane -> rank-1's upper halo
                out.append((full + 8 * sxy, None, self._addr(s.rank - 1, name, sxy + n), sxy))
            if s.rank < self.comm.size - 1:        # last plane -> rank+1's lower halo
                out.append((full + 8 * n, None, self._addr(s.rank + 1, name, 0), sxy))
        else:
            for q, idx in s.send_idx.items():      # packed rows -> q's ghost segment for this rank
                info = self.plan.ranks[q]
                off, cnt, _ = info["recv"][s.rank]
                out.append((full, idx.data_ptr(), self._addr(q, name, info["r1"] - info["r0"] + off), cnt))
        return out

    def _post_struct(self, s, push, reducing, parity):
        key = (s.rank, push, reducing, parity)
        post = self._posts.get(key)
        if post is not None:
            return post
        copies = []
        for nm in push:
            copies += self._halo_copies(s, nm)
        P = self.comm.size
        if reducing:                               # my chunk partials -> every rank's table slot
            src = s.table_local.data_ptr()
            for q in range(P):
                dst = self.reg.bases[q] + self.layouts[q].table_slot(parity) + 32 * s.chunk_offset
                copies.append((src, None, dst, 4 * s.chunks_local))
        if len(copies) > _lib.KPL_PEER_MAX_COPIES:
            raise ValueError(f"{len(copies)} peer copies exceed KPL_PEER_MAX_COPIES")
        post = _lib.KplPost()
        post.ncopies, post.nsignals = len(copies), P
        for i, (src, idx, dst, cnt) in enumerate(copies):
            c = post.copies[i]
            c.src, c.idx, c.dst, c.count = src, idx, dst, cnt
        for q in range(P):
            post.signal[q] = self.reg.bases[q] + PeerLayout.FLAGS + 8 * s.rank
        post.counter = self.reg.bases[s.rank] + PeerLayout.COUNTER
        post.status = D.ptr(s.ws)            # this rank's head: poison once its exchange failed
        self._posts[key] = post
        return post

    def _flush(self, inputs=()):
        """Issue the deferred post + finalize of the last sweep: push the halos
        of `inputs` (the next sweep's stencil inputs) that changed since their
        last push, this rank's chunk partials if the sweep reduces, signal,
        then wait for every rank and fold."""
        push = []
        for nm in inputs:
            st = self.states[0].alias[nm]
            if st in self._dirty and st not in push:
                push.append(st)
        if self._pending is None and not push:
            return
        kind, row, e, par = self._pending if self._pending is not None else (0, 0, None, 0)
        lib = _lib.load()
        reducing = kind != 0 and lib.kpl_sweep_phase(kind) != 0
        if e is None or push:
            # a post kernel: the halos, plus the partials unless the sweep pushed them itself
            partials = reducing and e is None
            if partials:
                self.reg.red += 1
                par = self.reg.red & 1
            self.reg.epoch += 1
            e = self.reg.epoch
            for s in self.states:
                _lib.check(lib.kpl_peer_post(self._post_struct(s, tuple(push), partials, par), e, s.hs()),
                           "peer post")
        for s in self.states:
            L = self.layouts[s.rank]
            table = self.reg.bases[s.rank] + L.table_slot(par)
            _lib.check(lib.kpl_peer_finalize(s.op, s.kcfg, kind, row, D.ptr(s.ws), table,
                                             self.reg.bases[s.rank] + PeerLayout.FLAGS, self.comm.size, e,
                                             s.hs()), "peer finalize")
        self._dirty.difference_update(push)
        self._pending = None

    def _status(self):
        if self.peer:
            self._flush()
        return self.states[0].read_status()

    # -- collective building blocks
    def _all(self, fn):
        for s in self.states:
            fn(s)

    def exchange(self, name):
        self.comm.exchange(self.states, name)

    def _can_fold(self, kind, inputs):
        """The deferred fold (kpl_sweep_peer wait_epoch): the pending sweep is a
        fused iteration sweep whose exchange has not been finalised, this sweep
        is the next fused iteration sweep, and it needs no halo push first --
        then its CTAs fold the previous exchange themselves and no finalize
        launch sits between the two sweeps."""
        if not (self.fold and kind == _lib.KPL_SW_ITER and self._pending is not None):
            return False
        pk, _, pe, _ = self._pending
        if pk != _lib.KPL_SW_ITER or pe is None:
            return False
        return not any(self.states[0].alias[nm] in self._dirty for nm in inputs)

    def sweep(self, kind, row=0, inputs=(), push_x=False):
        if self.peer:
            wait_e = wait_par = 0
            if self.fused and self._can_fold(kind, inputs):
                _, _, wait_e, wait_par = self._pending
                self._pending = None
            else:
                self._flush(inputs)
            kept = {self.states[0].alias[nm] for nm in inputs}
            if self.fused and kind == _lib.KPL_SW_ITER:
                # the sweep pushes its w output (and x for the next cadence record)
                # and its partials itself, then signals
                self.reg.red += 1
                self.reg.epoch += 1
                e, par = self.reg.epoch, self.reg.red & 1
                wout = "w0" if inputs[0] == "w1" else "w1"
                push = _lib.KPL_PUSH_W | (_lib.KPL_PUSH_X if push_x else 0)
                lib = _lib.load()
                for s in self.states:
                    pxd = self.reg.bases[s.rank] + self.layouts[s.rank].px
                    _lib.check(lib.kpl_sweep_peer(s.op, s.kcfg, s.vecs, kind, row, D.ptr(s.ws), pxd, e, par, push,
                                                  1 if wout == "w1" else 0, wait_e, wait_par, s.hs()),
                               "fused sweep")
                clean = {wout} | ({"x"} if push_x else set())
                self._dirty.update(nm for nm in self._names if nm not in kept)
                self._dirty.difference_update(clean)
                self._pending = (kind, row, e, par)
                return
            self._all(lambda s: s.sweep(kind, row))
            self._dirty.update(nm for nm in self._names if nm not in kept)
            self._pending = (kind, row, None, 0)
            return
        for nm in inputs:
            self.exchange(nm)
        self._all(lambda s: s.sweep(kind, row))
        if _lib.load().kpl_sweep_phase(kind) != 0:
            self.comm.allgather(self.states)
            self._all(lambda s: s.finalize(kind, row))

    # -- public
    def load_rhs(self, b_local_list, x0_local_list=None):
        """Per local rank: its slab of b (and x0), any array-like of length n_local."""
        t = D.torch()
        for i, s in enumerate(self.states):
            s.b.copy_(t.as_tensor(np.asarray(b_local_list[i]) if not isinstance(b_local_list[i], t.Tensor)
                                  else b_local_list[i], dtype=t.float64))
            x = s.interior("x")
            if x0_local_list is None:
                x.zero_()
            else:
                v = x0_local_list[i]
                x.copy_(v if isinstance(v, t.Tensor) else t.as_tensor(np.asarray(v), dtype=t.float64))

    def init(self):
        m = self.cfg.method
        if self.peer:
            self.comm.solve_barrier()
        if getattr(self.comm, "concurrent", False):
            t = D.torch()
            cur = t.cuda.current_stream()
            for s in self.states:
                if s.stream is None:
                    s.stream = t.cuda.Stream(device=self.device)
                s.stream.wait_stream(cur)          # setup, regions and rhs copies come first
        self._all(lambda s: s.prepare())
        if self.peer:
            self._pending = (0, 0, None, 0)    # barrier: no peer pushes into this rank before its prepare
        self.sweep(_lib.KPL_SW_BNORM)
        self.sweep(_lib.KPL_SW_INIT_R, inputs=("x",))
        if m != "cg":
            self.sweep(_lib.KPL_SW_INIT_W, inputs=("u",))
        self.issued = 0

    def step(self):
        """One iteration (host index j = self.issued)."""
        j = self.issued
        m = self.cfg.method
        self.record(j, cadence_only=True)
        if m == "cg":
            par = "p1" if (j & 1) else "p"
            self.sweep(_lib.KPL_SW_CG_P, inputs=(par, "u"))
            self.sweep(_lib.KPL_SW_CG_X)
        else:
            # x goes to the neighbours with the sweep when the next record reads it
            px = not self.cfg.track_gaps and (j + 1) % 10 == 0
            self.sweep(_lib.KPL_SW_ITER, inputs=("w1" if (j & 1) else "w0",), push_x=px)
            if m == "pcg_rr":
                self.sweep(_lib.KPL_SW_RR_R, inputs=("x",))
                self.sweep(_lib.KPL_SW_RR_W, inputs=("u",))
                self.sweep(_lib.KPL_SW_RR_S, inputs=("p",))
                self.sweep(_lib.KPL_SW_RR_Z, inputs=("q",))
        self.issued += 1

    def record(self, j, cadence_only):
        """Record-point sweeps of row j (solvers.py:398-402): gap norms with
        track_gaps, else the true residual on the i % 10 cadence."""
        if self.cfg.track_gaps:
            self.sweep(_lib.KPL_SW_GAP_F, row=j, inputs=("x",))
            if self.cfg.method != "cg":
                self.sweep(_lib.KPL_SW_GAP_G, row=j, inputs=("p",))
                self.sweep(_lib.KPL_SW_GAP_H, row=j, inputs=("u",))
                self.sweep(_lib.KPL_SW_GAP_J, row=j, inputs=("q",))
        elif not cadence_only or j % 10 == 0:
            self.sweep(_lib.KPL_SW_TRUE, row=j, inputs=("x",))

    def run(self, poll=16):
        self.init()
        st = self._status()
        while st.state == _lib.KPL_ST_RUNNING and self.issued < self.limit:
            for _ in range(min(poll, self.limit - self.issued)):
                self.step()
            st = self._status()
        return self.result()

    def _join(self):
        """The current stream waits for every rank stream (concurrent ranks)."""
        cur = D.torch().cuda.current_stream()
        for s in self.states:
            if s.stream is not None:
                cur.wait_stream(s.stream)

    def result(self):
        s0 = self.states[0]
        st = self._status()
        if st.state == _lib.KPL_ST_BREAKDOWN:
            msg = _lib.load().kpl_breakdown_message(st.bd_code).decode()
            if st.bd_code >= _BD_PEER_TIMEOUT:
                raise _lib.KplError(f"multi-GPU exchange failed: {msg}")
            raise BreakdownError(int(st.bd_iter), msg)
        if st.state != _lib.KPL_ST_DONE:
            raise _lib.KplError(f"distributed solve ended in state {st.state}")
        rows = int(st.iter) + 1
        if np.isnan(s0.history(rows)[-1, 5]):
            if self.peer:
                # sweeps issued past convergence were predicated off on the device,
                # so the halos a fused sweep would have pushed were never sent:
                # re-push whatever the final record reads
                self._dirty.update(self._names)
            self.record(int(st.iter), cadence_only=False)
            if self.peer:
                self._flush()
        self._join()
        history = records_from(s0.history(rows), rows)
        reps = []
        if st.n_replacements:
            t = D.torch()
            raw = s0.ws[s0.reps_off:s0.reps_off + 8 * int(st.n_replacements)]
            reps = [int(v) for v in raw.view(t.int64).cpu().numpy()]
        xs = [s.interior("x").clone() for s in self.states]
        return SolveResult(xs, bool(st.converged), rows - 1, history, reps)


DistributedStencilSolve = DistributedSolve       # earlier name


def solve_distributed(A, M, b_local, x0_local, cfg: SolverConfig, comm=None, zc=0, chunk_blocks=8):
    """Partitioned solve on the ranks of `comm` (default: the torch.distributed
    world): stencils by z-slabs (`SlabPlan`), CSR matrices by row blocks with
    general ghost gathers (`RowPlan`).

    `b_local` / `x0_local`: this rank's rows (plan.local_slice(rank)), or, with
    a LocalComm, a list with one block per rank.  Returns a SolveResult whose
    `x` is the list of local blocks and whose history is global."""
    if D.get_reduction_order() != "tree":
        raise _lib.KplError("the reference (blocked) reduction order is single-GPU only; "
                            "partitioned solves use the P-invariant chunk tree")
    if comm is None:
        comm = TorchComm()
    S = DistributedSolve(A, M, cfg, comm, zc=zc, chunk_blocks=chunk_blocks)
    if not isinstance(comm, LocalComm):
        b_local = [b_local]
        x0_local = None if x0_local is None else [x0_local]
    S.load_rhs(b_local, x0_local)
    return S.run()
