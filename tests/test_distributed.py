"""Multi-GPU z-slab path.

CPU (gloo, world_size 2): partition plan, the halo exchange + chunk-table
all-gather plumbing of TorchComm, and the partition invariance of the
reduction order (per-rank chunk partials + gathered level-4 fold == the
single-GPU tree).

GPU (one device, P virtual ranks via LocalComm): a P-rank solve is bit-identical
to the 1-GPU solve, for every method, 2D and 3D, identity and Jacobi.
"""

import ctypes
import math
import os
import socket

import numpy as np
import pytest
import torch

from oracle import gpu_order
from paper_1706_05988_b200 import _lib, distributed as dmod
from paper_1706_05988_b200.distributed import RowPlan, SlabPlan, TorchComm


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_slab_plan():
    p = SlabPlan(512, 512, 512, 8)
    assert p.nzl == 64 and p.zc == 16 and p.chunks_local == 4 and p.chunks_global == 32
    assert p.local_slice(3) == slice(3 * 512 * 512 * 64, 4 * 512 * 512 * 64)
    with pytest.raises(ValueError):
        SlabPlan(8, 8, 10, 4)
    with pytest.raises(ValueError):
        SlabPlan(8, 8, 16, 2, zc=16)
    assert SlabPlan(8, 8, 24, 2).zc == 4


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("dims,vx,wx,wy", [((64, 10, 32), 2, 1, 8), ((200, 1, 64), 2, 8, 1)])
def test_reduction_partition_invariant(P, dims, vx, wx, wy):
    """Level 1-3 per slab, gather, level 4 == the single-GPU tree (bitwise)."""
    NX, NY, NZ = dims
    rng = np.random.default_rng(0)
    u, v = rng.normal(size=NX * NY * NZ), rng.normal(size=NX * NY * NZ)
    zc = 4
    whole = gpu_order.stencil_dot_fn(NX, NY, NZ, vx, wx, wy, zc)(u, v)
    plan = SlabPlan(NX, NY, NZ, P, zc)
    chunks = []
    for r in range(P):
        sl = plan.local_slice(r)
        items = gpu_order.stencil_item_partials(u[sl] * v[sl], NX, NY, plan.nzl, vx, wx, wy, zc)
        chunks += list(items)
    assert gpu_order.reduce_items(chunks) == whole


class _FakeState(dmod._SlabState):
    """Stand-in slab state with CPU tensors (plumbing test only)."""

    def __init__(self, rank, P, sxy, nzl, chunks):
        self.rank = rank
        self.chunk_offset, self.chunks_local = rank * chunks, chunks
        self.sxy, self.nzl = sxy, nzl
        self.full = {"w0": torch.zeros((nzl + 2) * sxy, dtype=torch.float64)}
        self.full["w0"][sxy:(nzl + 1) * sxy] = torch.arange(nzl * sxy, dtype=torch.float64) + 1000 * rank
        self.table = torch.zeros(P * chunks * 4, dtype=torch.float64)
        self.table_local = self.table[rank * chunks * 4:(rank + 1) * chunks * 4]
        self.table_local.copy_(torch.arange(chunks * 4, dtype=torch.float64) + 100 * rank)

    def planes(self, name):
        f, sxy, n = self.full[name], self.sxy, self.sxy * self.nzl
        return f[:sxy], f[sxy:2 * sxy], f[n:n + sxy], f[n + sxy:]


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = TorchComm()
        sxy, nzl, chunks = 6, 3, 2
        s = _FakeState(rank, world, sxy, nzl, chunks)
        comm.exchange([s], "w0")
        comm.allgather([s])
        lo, first, last, hi = s.planes("w0")
        q.put((rank, lo.tolist(), hi.tolist(), s.table.tolist()))
    finally:
        dist.destroy_process_group()


def test_gloo_halo_exchange_and_table_allgather():
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, lo, hi, table = q.get(timeout=120)
        out[r] = (lo, hi, table)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sxy, nzl = 6, 3
    # rank 0: lower halo is the Dirichlet zero plane, upper halo = rank 1's first plane
    assert out[0][0] == [0.0] * sxy
    assert out[0][1] == [1000.0 + k for k in range(sxy)]
    # rank 1: lower halo = rank 0's last plane, upper halo zero
    assert out[1][0] == [float((nzl - 1) * sxy + k) for k in range(sxy)]
    assert out[1][1] == [0.0] * sxy
    want = [float(k) for k in range(8)] + [100.0 + k for k in range(8)]
    assert out[0][2] == want and out[1][2] == want


# ----------------------------------------------------------------- GPU

gpu = pytest.mark.gpu


def _one_gpu(A, M, b, cfg, zc):
    """1-GPU solve in the geometry the slab partition uses (2D grids: (nx, 1, ny))."""
    from paper_1706_05988_b200.solvers import _Solve
    return _Solve(A, M, b, None, cfg, zc=zc, slab_view=True).run()


COMMS = ["LocalComm", "LocalPeerComm", "LocalPeerCommPostOnly", "LocalPeerCommNoFold"]


@gpu
@pytest.mark.parametrize("comm", COMMS)
@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("method,extra", [("pcg_sh", {"shift": 2.30188679245283}), ("pcg", {}),
                                          ("cg", {}), ("pcg_rr", {})])
def test_local_ranks_bitwise_3d(P, method, extra, comm):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1706_05988_b200 as K
    from paper_1706_05988_b200.distributed import LocalComm, SlabPlan, solve_distributed
    A = K.Stencil3D(64, 24, 32)
    b = K.spmv(A, np.random.default_rng(2).normal(size=A.n))
    cfg = K.SolverConfig(method=method, max_iters=80, rtol=1e-10, **extra)
    zc = 4
    ref = _one_gpu(A, None, b, cfg, zc)
    plan = SlabPlan(64, 24, 32, P, zc)
    res = solve_distributed(A, None, [b[plan.local_slice(r)] for r in range(P)], None, cfg,
                            comm=getattr(dmod, comm)(P), zc=zc)
    x = np.concatenate([xi.cpu().numpy() for xi in res.x])
    assert res.iterations == ref.iterations
    for a, c in zip(res.history, ref.history):
        assert (a.alpha, a.beta, a.gamma, a.delta, a.rnorm_recursive, a.rnorm_true) == \
               (c.alpha, c.beta, c.gamma, c.delta, c.rnorm_recursive, c.rnorm_true)
    assert x.tobytes() == ref.x.tobytes()
    assert res.replacements == ref.replacements


@gpu
@pytest.mark.parametrize("comm", COMMS)
@pytest.mark.parametrize("P", [2, 3])
def test_local_ranks_bitwise_2d_jacobi(P, comm):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1706_05988_b200 as K
    from paper_1706_05988_b200.distributed import LocalComm, SlabPlan, solve_distributed
    A = K.Stencil2D(96, 48)
    M = K.make_jacobi(A)
    b = K.spmv(A, np.random.default_rng(0).random(A.n))
    cfg = K.SolverConfig(method="pcg_sh", shift=0.49238826317067413, max_iters=300, rtol=1e-10)
    zc = 2
    ref = _one_gpu(A, M, b, cfg, zc)
    plan = SlabPlan(96, 1, 48, P, zc)
    res = solve_distributed(A, M, [b[plan.local_slice(r)] for r in range(P)], None, cfg,
                            comm=getattr(dmod, comm)(P), zc=zc)
    x = np.concatenate([xi.cpu().numpy() for xi in res.x])
    assert res.iterations == ref.iterations and res.converged
    assert [r.alpha for r in res.history] == [r.alpha for r in ref.history]
    assert x.tobytes() == ref.x.tobytes()


@gpu
@pytest.mark.parametrize("comm", COMMS)
@pytest.mark.parametrize("method,extra", [("pcg_sh", {"shift": 1.0}),
                                          ("pcg_var_sh", {"shift_schedule": tuple(0.05 * k for k in range(41))})])
def test_local_ranks_gaps_bitwise(method, extra, comm):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1706_05988_b200 as K
    from paper_1706_05988_b200.distributed import LocalComm, SlabPlan, solve_distributed
    A = K.Stencil3D(64, 16, 16)
    b = np.full(A.n, 1 / math.sqrt(A.n))
    cfg = K.SolverConfig(method=method, max_iters=40, track_gaps=True, **extra)
    ref = _one_gpu(A, None, b, cfg, 4)
    plan = SlabPlan(64, 16, 16, 2, 4)
    res = solve_distributed(A, None, [b[plan.local_slice(r)] for r in range(2)], None, cfg,
                            comm=getattr(dmod, comm)(2), zc=4)
    for a, c in zip(res.history, ref.history):
        assert (a.gap_f, a.gap_g, a.gap_h, a.gap_j, a.rnorm_true) == \
               (c.gap_f, c.gap_g, c.gap_h, c.gap_j, c.rnorm_true)
        assert (a.alpha, a.beta) == (c.alpha, c.beta)


def test_row_plan_ghost_mapping_reproduces_global_spmv():
    """Local rows with remapped columns [local | ghosts] and the plan's
    send/recv lists reproduce the global csr_matvec bit for bit."""
    from oracle import kpl_oracle as O
    from paper_1706_05988_b200 import problems
    A = problems.banded_spd(20000, seed=0, band=3000)
    v = np.random.default_rng(3).normal(size=A.n)
    want = O.spmv(O.CSR(A.n, A.row_ptr, A.col_idx, A.values), v)
    for P in (2, 3, 5):
        plan = RowPlan(A, P, chunk_blocks=2)
        for r in range(P):
            info = plan.ranks[r]
            ext = np.concatenate([v[plan.local_slice(r)], v[info["ghosts"]]])
            # the ghost segment from each owner equals that owner's packed send list
            for q, (off, cnt, qrows) in info["recv"].items():
                sent = v[plan.local_slice(q)][plan.ranks[q]["send"][r]]
                assert sent.tobytes() == ext[len(ext) - len(info["ghosts"]) + off:][:cnt].tobytes()
            n_loc = info["r1"] - info["r0"]
            Aloc = O.CSR(n_loc, info["row_ptr"], info["col_idx"],
                         np.asarray(A.values)[info["k0"]:info["k1"]])
            got = O.spmv(Aloc, ext) if n_loc else np.zeros(0)
            assert got.tobytes() == want[plan.local_slice(r)].tobytes()
        assert plan.starts[0] == 0 and all(s % plan.chunk_rows == 0 for s in plan.starts[:-1])


@gpu
@pytest.mark.parametrize("comm", COMMS)
@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("method,extra", [("pcg_sh", {"shift": 0.4124626382901352}), ("cg", {}),
                                          ("pcg_rr", {})])
def test_local_ranks_csr_bitwise(P, method, extra, comm):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1706_05988_b200 as K
    from paper_1706_05988_b200 import problems
    from paper_1706_05988_b200.distributed import LocalComm, solve_distributed
    A = problems.banded_spd(20000, seed=0, band=2000)
    M = K.make_jacobi(A)
    b = K.spmv(A, np.random.default_rng(1).standard_normal(A.n))
    cfg = K.SolverConfig(method=method, max_iters=300, rtol=1e-10, **extra)
    ref = K.solve(A, M, b, None, cfg)
    plan = RowPlan(A, P)
    res = solve_distributed(A, M, [b[plan.local_slice(r)] for r in range(P)], None, cfg,
                            comm=getattr(dmod, comm)(P))
    x = np.concatenate([xi.cpu().numpy() for xi in res.x])
    assert res.iterations == ref.iterations and res.converged == ref.converged
    for a, c in zip(res.history, ref.history):
        assert (a.alpha, a.beta, a.gamma, a.delta, a.rnorm_recursive, a.rnorm_true) == \
               (c.alpha, c.beta, c.gamma, c.delta, c.rnorm_recursive, c.rnorm_true)
    assert x.tobytes() == ref.x.tobytes()
    assert res.replacements == ref.replacements


@gpu
@pytest.mark.parametrize("comm", COMMS)
def test_local_ranks_csr_varcoef_identity_bitwise(comm):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1706_05988_b200 as K
    from paper_1706_05988_b200 import problems
    from paper_1706_05988_b200.distributed import LocalComm, solve_distributed
    A = problems.varcoef_3d(24, seed=0)          # 13824 rows
    b = np.random.default_rng(1).standard_normal(A.n)
    cfg = K.SolverConfig(method="pcg_sh", shift=0.3, max_iters=150, rtol=0.0, track_gaps=True)
    ref = K.solve(A, None, b, None, cfg)
    plan = RowPlan(A, 2)
    res = solve_distributed(A, None, [b[plan.local_slice(r)] for r in range(2)], None, cfg,
                            comm=getattr(dmod, comm)(2))
    for a, c in zip(res.history, ref.history):
        assert (a.alpha, a.gap_f, a.gap_g, a.gap_h, a.gap_j) == (c.alpha, c.gap_f, c.gap_g, c.gap_h, c.gap_j)


class _FakeRowState(dmod._RowState):
    """Row-block state with CPU tensors built from a real RowPlan (plumbing only)."""

    def __init__(self, plan, rank, v):
        info = plan.ranks[rank]
        self.plan, self.rank = plan, rank
        self.n_local, self.n_ghost = info["r1"] - info["r0"], len(info["ghosts"])
        self.full = {"w0": torch.zeros(self.n_local + self.n_ghost, dtype=torch.float64)}
        self.full["w0"][:self.n_local] = torch.as_tensor(v[plan.local_slice(rank)])
        self.recv = {q: (off, cnt) for q, (off, cnt, _) in info["recv"].items()}
        self.send_idx = {q: torch.as_tensor(rows.astype(np.int64)) for q, rows in info["send"].items()}
        self.send_buf = {q: torch.zeros(len(rows), dtype=torch.float64) for q, rows in info["send"].items()}


def _gloo_row_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1706_05988_b200 import problems
        dmod._gather = lambda idx, src, dst: dst.copy_(src[idx])      # CPU stand-in for kpl_gather
        A = problems.banded_spd(12000, seed=0, band=1500)
        plan = RowPlan(A, world, chunk_blocks=2)
        v = np.arange(A.n, dtype=np.float64) * 0.5
        s = _FakeRowState(plan, rank, v)
        TorchComm().exchange([s], "w0")
        ghosts = s.full["w0"][s.n_local:].numpy()
        q.put((rank, bool(np.array_equal(ghosts, v[plan.ranks[rank]["ghosts"]])), len(ghosts)))
    finally:
        dist.destroy_process_group()


def test_gloo_row_ghost_exchange():
    """TorchComm's general ghost gather (pack -> send/recv -> ghost segments), world_size 2."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_gloo_row_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, ng in res:
        assert ok and ng > 0, (rank, ng)


def _gloo_gpu_worker(rank, world, port, q, kind):
    """One rank of a real multi-process solve: gloo for plumbing, all ranks on cuda:0."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1706_05988_b200 as K
        from paper_1706_05988_b200 import problems
        from paper_1706_05988_b200.distributed import RowPlan, SlabPlan, solve_distributed
        torch.cuda.set_device(0)
        if kind == "slab":
            A = K.Stencil3D(64, 24, 32)
            b = np.random.default_rng(2).normal(size=A.n)
            plan = SlabPlan(64, 24, 32, world, 4)
            cfg = K.SolverConfig(method="pcg_sh", shift=2.3, max_iters=60)
            M = None
            res = solve_distributed(A, M, b[plan.local_slice(rank)], None, cfg, zc=4)
        else:
            A = problems.banded_spd(20000, seed=0, band=2000)
            M = K.make_jacobi(A)
            b = np.random.default_rng(1).standard_normal(A.n)
            plan = RowPlan(A, world)
            cfg = K.SolverConfig(method="pcg_sh", shift=0.41, max_iters=60, rtol=1e-10)
            res = solve_distributed(A, M, b[plan.local_slice(rank)], None, cfg)
        q.put((rank, res.iterations, [r.alpha for r in res.history], res.x[0].cpu().numpy().tobytes()))
    except Exception as exc:                      # report, don't hang the parent
        q.put((rank, "error", repr(exc), b""))
    finally:
        dist.destroy_process_group()


@gpu
@pytest.mark.parametrize("kind", ["slab", "rows"])
def test_multiprocess_gloo_on_one_gpu_bitwise(kind):
    """TorchComm + the sweep-level C ABI in real separate processes (2 ranks
    sharing cuda:0, gloo for the exchanges); bit-identical to one GPU."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import torch.multiprocessing as mp
    import paper_1706_05988_b200 as K
    from paper_1706_05988_b200 import problems
    from paper_1706_05988_b200.distributed import RowPlan, SlabPlan
    from paper_1706_05988_b200.solvers import _Solve
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_gloo_gpu_worker, args=(r, 2, port, q, kind)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(2):
        r, its, alphas, xb = q.get(timeout=300)
        assert its != "error", alphas
        out[r] = (its, alphas, xb)
    for p in procs:
        p.join(timeout=120)
    if kind == "slab":
        A = K.Stencil3D(64, 24, 32)
        b = np.random.default_rng(2).normal(size=A.n)
        ref = _Solve(A, None, b, None, K.SolverConfig(method="pcg_sh", shift=2.3, max_iters=60), zc=4).run()
        plan = SlabPlan(64, 24, 32, 2, 4)
    else:
        A = problems.banded_spd(20000, seed=0, band=2000)
        b = np.random.default_rng(1).standard_normal(A.n)
        ref = K.solve(A, K.make_jacobi(A), b, None,
                      K.SolverConfig(method="pcg_sh", shift=0.41, max_iters=60, rtol=1e-10))
        plan = RowPlan(A, 2)
    for r in range(2):
        its, alphas, xb = out[r]
        assert its == ref.iterations
        assert alphas == [h.alpha for h in ref.history]
        assert xb == ref.x[plan.local_slice(r)].tobytes()


# ------------------------------------------- device-initiated peer exchange

def _host_execute_post(post, epoch):
    """What peer_post_kernel does, on host memory: every copy, then the signals
    (the addresses in `post` are CPU addresses when the regions are CPU tensors)."""
    import ctypes
    for i in range(post.ncopies):
        c = post.copies[i]
        n = int(c.count)
        dst = np.frombuffer((ctypes.c_double * n).from_address(c.dst), dtype=np.float64)
        if c.idx:
            idx = np.frombuffer((ctypes.c_int32 * n).from_address(c.idx), dtype=np.int32)
            m = int(idx.max()) + 1 if n else 0
            src = np.frombuffer((ctypes.c_double * m).from_address(c.src), dtype=np.float64)
            dst[:] = src[idx]
        else:
            dst[:] = np.frombuffer((ctypes.c_double * n).from_address(c.src), dtype=np.float64)
    for q in range(post.nsignals):
        ctypes.c_uint64.from_address(post.signal[q]).value = epoch


def _cpu_peer_solve(monkeypatch, A, M, cfg, P, **kw):
    from paper_1706_05988_b200 import device as Dv
    monkeypatch.setattr(Dv, "require_cuda", lambda: torch.device("cpu"))
    return dmod.DistributedSolve(A, M, cfg, dmod.LocalPeerComm(P), **kw)


@pytest.mark.parametrize("P", [2, 3])
def test_peer_post_plan_slab_cpu(monkeypatch, P):
    """Peer-exchange plan of z-slabs (regions as CPU tensors, copies executed
    on the host): halos = the neighbours' boundary planes (zero at the global
    boundary), every rank's table slot = all ranks' partials in rank order,
    every flag word = the epoch."""
    import paper_1706_05988_b200 as K
    NX, NY, NZ = 8, 5, 12
    A = K.Stencil3D(NX, NY, NZ)
    cfg = K.SolverConfig(method="pcg_sh", shift=1.0, max_iters=10)
    S = _cpu_peer_solve(monkeypatch, A, None, cfg, P, zc=2)
    g = np.arange(A.n, dtype=np.float64) + 0.5
    for s in S.states:
        s.interior("w1").copy_(torch.from_numpy(g[S.plan.local_slice(s.rank)]))
        s.table_local.copy_(torch.arange(s.table_local.numel(), dtype=torch.float64) + 1000 * s.rank)
    for s in S.states:
        _host_execute_post(S._post_struct(s, ("w1",), True, 1), 7)
    sxy, nzl = NX * NY, NZ // P
    want_table = np.concatenate([np.arange(4 * S.plan.chunks_local) + 1000.0 * r for r in range(P)])
    for s in S.states:
        lo, first, last, hi = (v.numpy() for v in s.planes("w1"))
        z0 = s.rank * nzl
        assert lo.tobytes() == (g[(z0 - 1) * sxy:z0 * sxy] if s.rank else np.zeros(sxy)).tobytes()
        z1 = z0 + nzl
        assert hi.tobytes() == (g[z1 * sxy:(z1 + 1) * sxy] if s.rank < P - 1 else np.zeros(sxy)).tobytes()
        reg = S.reg.tensors[s.rank]
        L = S.layouts[s.rank]
        slot = reg[L.table_slot(1):L.table_slot(1) + 32 * S.plan.chunks_global].view(torch.float64).numpy()
        assert slot.tobytes() == want_table.tobytes()
        flags = reg[:8 * P].view(torch.int64).numpy()
        assert list(flags) == [7] * P
        # the other slot and the other vectors are untouched
        other = reg[L.table_slot(0):L.table_slot(0) + 32 * S.plan.chunks_global]
        assert int(other.sum()) == 0
        assert float(s.full["w0"].abs().sum()) == 0.0


def test_peer_post_plan_rows_cpu(monkeypatch):
    """Peer-exchange plan of CSR row blocks: every ghost value = the global
    vector at that column, delivered by its owner's packed send list."""
    import paper_1706_05988_b200 as K
    from paper_1706_05988_b200 import problems
    A = problems.banded_spd(12000, seed=0, band=1500)
    M = K.make_jacobi(A)
    cfg = K.SolverConfig(method="pcg_sh", shift=0.4, max_iters=10)
    P = 3
    S = _cpu_peer_solve(monkeypatch, A, M, cfg, P, chunk_blocks=2)
    g = np.arange(A.n, dtype=np.float64) * 0.25
    for s in S.states:
        s.interior("w0").copy_(torch.from_numpy(g[S.plan.local_slice(s.rank)]))
        # CPU stand-ins for the int32 device send lists
        s.send_idx = {q: v.to(torch.int32) for q, v in s.send_idx.items()}
    S._posts.clear()
    for s in S.states:
        _host_execute_post(S._post_struct(s, ("w0",), False, 0), 3)
    for s in S.states:
        ghosts = s.full["w0"][s.n_local:].numpy()
        assert ghosts.tobytes() == g[S.plan.ranks[s.rank]["ghosts"]].tobytes()
        assert list(S.reg.tensors[s.rank][:8 * P].view(torch.int64).numpy()) == [3] * P


def _ipc_post_worker(rank, world, port, q):
    """One process of the IPC plumbing check: map the other rank's region
    (cudaIpc on the same device), push halos + partials + signal with
    kpl_peer_post, host barrier, then read this rank's region.  No kernel
    waits on another process (the barrier orders them on the host)."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1706_05988_b200 as K
        from paper_1706_05988_b200 import _lib, device as Dv
        torch.cuda.set_device(0)
        NX, NY, NZ = 16, 6, 8
        A = K.Stencil3D(NX, NY, NZ)
        cfg = K.SolverConfig(method="pcg_sh", shift=1.0, max_iters=10)
        S = dmod.DistributedSolve(A, None, cfg, dmod.PeerComm(), zc=2)
        (s,) = S.states
        g = torch.arange(A.n, dtype=torch.float64, device="cuda") + 0.5
        s.interior("w0").copy_(g[S.plan.local_slice(rank)])
        s.table_local.copy_(torch.arange(s.table_local.numel(), dtype=torch.float64) + 100 * rank)
        torch.cuda.synchronize()
        dist.barrier()
        lib = _lib.load()
        _lib.check(lib.kpl_peer_post(S._post_struct(s, ("w0",), True, 0), 5, Dv.stream_handle()), "post")
        torch.cuda.synchronize()
        dist.barrier()
        sxy, nzl = NX * NY, NZ // world
        lo, _, _, hi = s.planes("w0")
        gh = g.cpu().numpy()
        z0 = rank * nzl
        ok_lo = lo.cpu().numpy().tobytes() == (gh[(z0 - 1) * sxy:z0 * sxy] if rank else np.zeros(sxy)).tobytes()
        z1 = z0 + nzl
        ok_hi = hi.cpu().numpy().tobytes() == (gh[z1 * sxy:(z1 + 1) * sxy] if rank < world - 1
                                               else np.zeros(sxy)).tobytes()
        L = S.layouts[rank]
        reg = S.reg.tensors[rank]
        slot = reg[L.table_slot(0):L.table_slot(0) + 32 * S.plan.chunks_global].view(torch.float64).cpu().numpy()
        want = np.concatenate([np.arange(4 * S.plan.chunks_local) + 100.0 * r for r in range(world)])
        flags = reg[:8 * world].view(torch.int64).cpu().numpy().tolist()
        q.put((rank, ok_lo, ok_hi, slot.tobytes() == want.tobytes(), flags))
        dist.barrier()
        S.reg.close(barrier=dist.barrier)
    except Exception as exc:
        q.put((rank, "error", repr(exc), None, None))
    finally:
        dist.destroy_process_group()


@gpu
def test_ipc_peer_post_two_processes_one_gpu():
    """PeerComm's IPC regions (kpl_ipc_alloc / kpl_ipc_open) and kpl_peer_post
    across two real processes sharing cuda:0."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_ipc_post_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
    for rank, ok_lo, ok_hi, ok_table, flags in res:
        assert ok_lo != "error", ok_hi
        assert ok_lo and ok_hi and ok_table, (rank, ok_lo, ok_hi, ok_table)
        assert flags == [5, 5]


def test_peer_sweep_struct_cpu(monkeypatch):
    """The fused sweep's device descriptor: table slots and flag words of every
    rank, and the neighbour halo planes of w0/w1/x (none at the global boundary)."""
    import paper_1706_05988_b200 as K
    A = K.Stencil3D(8, 4, 12)
    cfg = K.SolverConfig(method="pcg_sh", shift=1.0, max_iters=10)
    P = 3
    S = _cpu_peer_solve(monkeypatch, A, None, cfg, P, zc=2)
    assert S.fused
    sxy, n = 32, 32 * 4
    for s in S.states:
        o = S.layouts[s.rank].px
        raw = bytes(S.reg.tensors[s.rank][o:o + ctypes.sizeof(_lib.KplPeerSweep)].numpy())
        px = _lib.KplPeerSweep.from_buffer_copy(raw)
        assert px.nranks == P
        for q in range(P):
            assert px.signal[q] == S.reg.bases[q] + 8 * s.rank
            for par in (0, 1):
                assert px.table[par][q] == S.reg.bases[q] + S.layouts[q].table_slot(par)
        for k, nm in enumerate(("w0", "w1")):
            assert px.w_src[k] == s.interior(nm).data_ptr()
            lo = None if s.rank == 0 else S.states[s.rank - 1].full[nm][sxy + n:].data_ptr()
            hi = None if s.rank == P - 1 else S.states[s.rank + 1].full[nm].data_ptr()
            assert (px.w_lo[k], px.w_hi[k]) == (lo, hi)
        assert px.x_src == s.interior("x").data_ptr()


# Writes of each sweep kind (storage names before aliasing; kpl_capi.cu do_sweep):
# ITER j writes w[(j+1)&1], CG_P j writes p[(j+1)&1]; RR_W is taken to write both w.
def _writes(kind, j):
    L = _lib
    if kind == L.KPL_SW_INIT_R or kind == L.KPL_SW_RR_R:
        return {"r", "u"}
    if kind == L.KPL_SW_INIT_W:
        return {"w0"}
    if kind == L.KPL_SW_ITER:
        return {"x", "r", "u", "z", "q", "s", "t", "p", "w1" if j % 2 == 0 else "w0"}
    if kind == L.KPL_SW_CG_P:
        return {"p1" if j % 2 == 0 else "p", "s"}
    if kind == L.KPL_SW_CG_X:
        return {"x", "r", "u"}
    if kind == L.KPL_SW_RR_W:
        return {"w0", "w1"}
    if kind == L.KPL_SW_RR_S:
        return {"s", "q"}
    if kind == L.KPL_SW_RR_Z:
        return {"z"}
    return set()


@pytest.mark.parametrize("method,extra,gaps,fused", [
    ("pcg_sh", {"shift": 1.0}, False, True), ("pcg_sh", {"shift": 1.0}, False, False),
    ("pcg_sh", {"shift": 1.0}, True, True), ("pcg", {}, False, True), ("pcg_rr", {}, False, True),
    ("cg", {}, False, True), ("cg", {}, True, False)])
@pytest.mark.parametrize("jacobi", [False, True])
def test_peer_exchange_schedule_is_fresh_and_race_free(monkeypatch, method, extra, gaps, fused, jacobi):
    """Replays the distributed driver's sweep / post / finalize sequence with a
    recording stand-in for the device calls and checks, against the write sets
    of every sweep kind: (1) every halo a sweep reads was pushed after the last
    write of that vector; (2) no push issued during or after sweep s targets a
    vector sweep s reads (a peer may still be running sweep s); (3) a finalize
    (wait) separates every two sweeps."""
    import paper_1706_05988_b200 as K
    from paper_1706_05988_b200 import device as Dv
    monkeypatch.setattr(Dv, "require_cuda", lambda: torch.device("cpu"))
    A = K.Stencil3D(8, 4, 8)
    M = K.make_jacobi(A) if jacobi else None
    cfg = K.SolverConfig(method=method, max_iters=40, track_gaps=gaps, **extra)
    comm = dmod.LocalPeerComm(2, fused=fused)
    S = dmod.DistributedSolve(A, M, cfg, comm, zc=2)
    ev = []
    real = _lib.load()

    class FakeLib:
        def kpl_sweep_phase(self, kind):
            return real.kpl_sweep_phase(kind)

        def kpl_peer_post(self, post, e, hs):
            return 0

        def kpl_peer_finalize(self, *a):
            ev.append(("fin",))
            return 0

        def kpl_sweep_peer(self, op, kcfg, vecs, kind, row, ws, pxd, e, par, push, wpar, wait_e, wait_par, hs):
            if ws == D0[0]:
                if wait_e:             # deferred fold: the sweep's CTAs wait (and fold) first
                    ev.append(("fin",))
                ev.append(("sweep",) + cur[0])
            pushed = set()
            if push & _lib.KPL_PUSH_W:
                pushed.add("w1" if wpar else "w0")
            if push & _lib.KPL_PUSH_X:
                pushed.add("x")
            if ws == D0[0]:
                ev.append(("fused", kind, pushed))
            return 0

    monkeypatch.setattr(_lib, "load", lambda: FakeLib())
    orig_post = dmod.DistributedSolve._post_struct

    def rec_post(self, s, push, reducing, parity):
        if s.rank == 0:
            ev.append(("post", set(push)))
        return orig_post(self, s, push, reducing, parity)

    monkeypatch.setattr(dmod.DistributedSolve, "_post_struct", rec_post)
    orig_sweep = dmod.DistributedSolve.sweep

    cur = [None]
    D0 = [S.states[0].ws.data_ptr()]

    def rec_sweep(self, kind, row=0, inputs=(), push_x=False):
        cur[0] = (kind, {self.states[0].alias[n] for n in inputs}, getattr(self, "issued", 0))
        return orig_sweep(self, kind, row, inputs, push_x)

    def rank_sweep(self, kind, row=0):
        if self.rank == 0:
            ev.append(("sweep",) + cur[0])

    monkeypatch.setattr(dmod.DistributedSolve, "sweep", rec_sweep)
    monkeypatch.setattr(dmod._RankState, "sweep", rank_sweep)
    monkeypatch.setattr(dmod._RankState, "prepare", lambda self: None)
    monkeypatch.setattr(Dv, "stream_handle", lambda: None)
    S.init()
    for _ in range(23):
        S.step()
    S._flush()
    alias = S.states[0].alias
    version = {n: 0 for n in S._names}
    pushed = {n: 0 for n in S._names}
    prev_inputs, since_fin = set(), True
    last_kind = last_j = None
    for e in ev:
        if e[0] == "sweep":
            _, kind, inputs, j = e
            assert since_fin, f"two sweeps without a finalize between them ({kind})"
            for n in inputs:
                assert pushed[n] == version[n], f"sweep {kind} at step {j} reads a stale halo of {n}"
            for n in _writes(kind, j):
                version[alias.get(n, n)] += 1
            prev_inputs, since_fin = inputs, False
            last_kind, last_j = kind, j
        elif e[0] == "fused":
            _, kind, push = e
            assert not (push & prev_inputs), f"fused push {push} overlaps the sweep's inputs"
            for n in push:
                pushed[n] = version[n]
        elif e[0] == "post":
            assert not (e[1] & prev_inputs), f"post {e[1]} overlaps the inputs of sweep {last_kind} at step {last_j}: {ev[max(0, ev.index(e) - 8):ev.index(e) + 1]}"
            for n in e[1]:
                pushed[n] = version[n]
        elif e[0] == "fin":
            since_fin = True
    assert since_fin


@gpu
@pytest.mark.parametrize("kind", ["slab", "rows"])
def test_local_peer_eight_ranks_bitwise(kind):
    """Eight virtual ranks (the 8 x B200 box layout) through the peer exchange:
    bit-identical to one GPU for a z-slab stencil and a CSR row-block matrix."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1706_05988_b200 as K
    from paper_1706_05988_b200 import problems
    from paper_1706_05988_b200.distributed import LocalPeerComm, solve_distributed
    P = 8
    if kind == "slab":
        A = K.Stencil3D(64, 24, 32)
        b = K.spmv(A, np.random.default_rng(2).normal(size=A.n))
        cfg = K.SolverConfig(method="pcg_sh", shift=2.30188679245283, max_iters=80, rtol=1e-10)
        ref = _one_gpu(A, None, b, cfg, 4)
        plan = SlabPlan(64, 24, 32, P, 4)
        res = solve_distributed(A, None, [b[plan.local_slice(r)] for r in range(P)], None, cfg,
                                comm=LocalPeerComm(P), zc=4)
        M = None
    else:
        A = problems.banded_spd(20000, seed=0, band=2000)
        M = K.make_jacobi(A)
        b = K.spmv(A, np.random.default_rng(1).standard_normal(A.n))
        cfg = K.SolverConfig(method="pcg_sh", shift=0.4124626382901352, max_iters=300, rtol=1e-10)
        ref = K.solve(A, M, b, None, cfg)
        plan = RowPlan(A, P)
        res = solve_distributed(A, M, [b[plan.local_slice(r)] for r in range(P)], None, cfg,
                                comm=LocalPeerComm(P))
    x = np.concatenate([xi.cpu().numpy() for xi in res.x])
    assert res.iterations == ref.iterations
    assert [(h.alpha, h.beta, h.rnorm_true) for h in res.history] == \
           [(h.alpha, h.beta, h.rnorm_true) for h in ref.history]
    assert x.tobytes() == np.asarray(ref.x).tobytes()


@gpu
def test_fused_final_record_after_predicated_sweeps():
    """Regression (found by tools/fuzz_parity.py dist): sweeps enqueued past
    convergence are predicated off on the device, so the x halo a fused sweep
    would push for the next cadence row never arrives; the final true-residual
    record must re-push it.  Converges at row 67, not a cadence row."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1706_05988_b200 as K
    from paper_1706_05988_b200.distributed import LocalPeerComm, solve_distributed
    A = K.Stencil3D(16, 9, 9)
    b = np.random.default_rng(0).standard_normal(A.n)
    cfg = K.SolverConfig(method="pcg_sh", shift=0.75, max_iters=110, rtol=1e-12)
    ref = _one_gpu(A, None, b, cfg, 1)
    plan = SlabPlan(16, 9, 9, 3, 1)
    res = solve_distributed(A, None, [b[plan.local_slice(r)] for r in range(3)], None, cfg,
                            comm=LocalPeerComm(3), zc=1)
    assert res.iterations == ref.iterations and ref.iterations % 10 != 0
    assert [(h.alpha, h.rnorm_true) for h in res.history] == [(h.alpha, h.rnorm_true) for h in ref.history]


# ---------------------------------------------------------------- concurrency
# the ranks' kernels run AT THE SAME TIME (one CUDA stream
# per virtual rank), so every device flag wait really blocks on a kernel of
# another rank that is still running.  Grids are small enough to be
# co-resident on the one GPU (a spinning CTA must not starve the kernel it
# waits for).  A push that raced a peer's read, a fold of a stale table slot
# or a missed wait would change bits against the 1-GPU solve; the solve is
# repeated to give a race many chances.  A short device timeout turns a
# protocol deadlock into an error instead of a hang.

@pytest.fixture
def short_peer_timeout():
    lib = _lib.load()
    assert lib.kpl_set_peer_timeout(10.0) == 0
    yield
    lib.kpl_set_peer_timeout(20.0)


def _check_same(res, ref, x):
    assert res.iterations == ref.iterations and res.converged == ref.converged
    for a, c in zip(res.history, ref.history):
        assert (a.alpha, a.beta, a.gamma, a.delta, a.rnorm_recursive, a.rnorm_true) == \
               (c.alpha, c.beta, c.gamma, c.delta, c.rnorm_recursive, c.rnorm_true)
    assert x.tobytes() == np.asarray(ref.x).tobytes()


@gpu
@pytest.mark.parametrize("fused,fold", [(True, True), (True, False), (False, False)])
@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("method,extra", [("pcg_sh", {"shift": 2.30188679245283}), ("pcg_rr", {}), ("cg", {})])
def test_concurrent_ranks_slab_bitwise(short_peer_timeout, P, method, extra, fused, fold):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1706_05988_b200 as K
    from paper_1706_05988_b200.distributed import LocalPeerComm, solve_distributed
    A = K.Stencil3D(128, 64, 32)                       # <= 64 items per rank: co-resident
    b = K.spmv(A, np.random.default_rng(5).normal(size=A.n))
    cfg = K.SolverConfig(method=method, max_iters=120, rtol=1e-11, **extra)
    zc = 4
    ref = _one_gpu(A, None, b, cfg, zc)
    plan = SlabPlan(128, 64, 32, P, zc)
    for rep in range(4):
        res = solve_distributed(A, None, [b[plan.local_slice(r)] for r in range(P)], None, cfg,
                                comm=LocalPeerComm(P, fused=fused, concurrent=True, fold=fold), zc=zc)
        torch.cuda.synchronize()
        _check_same(res, ref, np.concatenate([xi.cpu().numpy() for xi in res.x]))


@gpu
@pytest.mark.parametrize("P", [2, 3])
def test_concurrent_ranks_rows_bitwise(short_peer_timeout, P):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1706_05988_b200 as K
    from paper_1706_05988_b200 import problems
    from paper_1706_05988_b200.distributed import LocalPeerComm, solve_distributed
    A = problems.banded_spd(20000, seed=0, band=2000)
    M = K.make_jacobi(A)
    b = K.spmv(A, np.random.default_rng(1).standard_normal(A.n))
    cfg = K.SolverConfig(method="pcg_sh", shift=0.4124626382901352, max_iters=300, rtol=1e-10)
    ref = K.solve(A, M, b, None, cfg)
    plan = RowPlan(A, P)
    for rep in range(4):
        res = solve_distributed(A, M, [b[plan.local_slice(r)] for r in range(P)], None, cfg,
                                comm=LocalPeerComm(P, concurrent=True))
        torch.cuda.synchronize()
        _check_same(res, ref, np.concatenate([xi.cpu().numpy() for xi in res.x]))


@gpu
def test_fold_removes_the_finalize_launches(monkeypatch):
    """With the deferred fold, consecutive fused iteration sweeps have no
    kpl_peer_finalize between them: only cadence records, polls and the end
    of the solve still finalize (DESIGN.md 6.1 cost model)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1706_05988_b200 as K
    from paper_1706_05988_b200.distributed import LocalPeerComm, solve_distributed
    A = K.Stencil3D(64, 32, 32)
    b = K.spmv(A, np.random.default_rng(5).normal(size=A.n))
    cfg = K.SolverConfig(method="pcg_sh", shift=1.0, max_iters=100, rtol=0.0)
    plan = SlabPlan(64, 32, 32, 2, 4)
    counts = {}
    for fold in (True, False):
        lib = _lib.load()
        calls = {"fin": 0, "sweep": 0}
        real_fin, real_sw = lib.kpl_peer_finalize, lib.kpl_sweep_peer

        class Spy:
            def __getattr__(self, name):
                return getattr(lib, name)

            def kpl_peer_finalize(self, *a):
                calls["fin"] += 1
                return real_fin(*a)

            def kpl_sweep_peer(self, *a):
                calls["sweep"] += 1
                return real_sw(*a)

        spy = Spy()
        monkeypatch.setattr(_lib, "load", lambda: spy)
        solve_distributed(A, None, [b[plan.local_slice(r)] for r in range(2)], None, cfg,
                          comm=LocalPeerComm(2, fold=fold), zc=4)
        monkeypatch.setattr(_lib, "load", lambda: lib)
        counts[fold] = dict(calls)
    assert counts[True]["sweep"] == counts[False]["sweep"]
    # 100 iterations: without the fold one finalize per fused sweep; with it only
    # the cadence rows (every 10th) and the host polls keep one
    assert counts[False]["fin"] >= 2 * 100
    assert counts[True]["fin"] <= counts[False]["fin"] - 2 * 60
