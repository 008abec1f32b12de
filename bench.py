#!/usr/bin/env python3
"""Benchmark: p-CG-sh iterations/s + achieved HBM GB/s, 3D Poisson 512^3 fp64.

BASELINE.json metric / config 3: 7-point Laplacian on 512^3 (134,217,728 DOF),
matrix-free, unpreconditioned, b = A * (1/sqrt(n)), x0 = 0, fixed 500 p-CG-sh
iterations (rtol 0), sigma = 2.30188679245283 (the reference's selection rule
on the 500-iteration p-CG history, recomputed at 512^3 on the device:
tools/sigma_config3.py, profiles/r01_sigma_config3.jsonl).

A "step" is one full solve through the drop-in API (init + 500 fused
iterations + the reference's true-residual cadence).  `value` is iterations/s
with b resident in HBM; `e2e` is the same solve called with a pinned HOST
right-hand side and the solution copied back to host memory, both copies
inside the timed region.  The inputs (8 x 1 GiB vectors) exceed the 126 MB L2,
so no flush is needed between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 is launched by torchrun (one rank per GPU): the 512^3 grid is cut
into N z-slabs (paper_1706_05988_b200.distributed): per sweep the fused
sweep on the slab, then a device-initiated exchange over NVLink peer memory
(kpl_peer_post stores the next sweep's halo planes and this rank's chunk
partials into the neighbours' IPC-mapped buffers and raises a flag;
kpl_peer_finalize waits for every rank's flag, folds the partials and runs
the scalar epilogue) -- no host-side collective per iteration ("scaling":
"strong", the global problem is fixed).  `--impl reference` times the CPU oracle (a
restatement of the reference `kpl` package's single-threaded numpy/numba
path, oracle/kpl_oracle.py) on the host, one p-CG-sh iteration per step.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N3 = 512
ITERS = 500
SIGMA = 2.30188679245283
BYTES_PER_DOF = 96            # 6 state vectors read + written once
METRIC = "p-CG-sh iters/s + achieved HBM GB/s, 3D Poisson 512³ fp64 at 1/2/4/8 B200"
UNIT = "iterations/s"
WORKLOAD = ("config3: 3D Poisson 7-point 512^3 matrix-free fp64, M=I, b=A*1/sqrt(n), x0=0, "
            "500 fixed p-CG-sh iterations, sigma=2.30188679245283")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def profiled_traffic():
    """Per-launch DRAM bytes of the fused iteration kernel from the committed
    ncu capture (profiles/ncu_pcgsh_iter.json), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_pcgsh_iter.json")
    try:
        with open(path) as f:
            return float(json.load(f)["dram_bytes_per_launch"])
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ----------------------------------------------------------------- GPU arm

def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1706_05988_b200 as K
    from paper_1706_05988_b200 import _lib, device as Dv
    from paper_1706_05988_b200.solvers import _Solve

    rank, world, local = dist_env()
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        # NCCL over NVLink; KPL_DIST_BACKEND=gloo runs the same multi-process
        # path with several ranks on one GPU (plumbing checks only)
        backend = os.environ.get("KPL_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        return run_distributed(args, rank, world, local)
    dev = torch.device("cuda", local)

    A = K.Stencil3D(N3, N3, N3)
    n = A.n
    cfg = K.SolverConfig(method="pcg_sh", shift=SIGMA, max_iters=ITERS, rtol=0.0)
    # b = A * (1/sqrt(n)) computed by the device SpMV (harness.build_rhs, ones_solution)
    b = K.spmv(A, torch.full((n,), 1.0 / math.sqrt(n), dtype=torch.float64, device=dev))
    lib = _lib.load()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- warm-up (also checks the run converges the same way every time)
    for _ in range(args.warmup):
        res = K.solve(A, None, b, None, cfg)
    final_rel = res.history[-1].rnorm_true / math.sqrt(float(torch.dot(b, b)))

    # ---- timed: K solves, inputs resident in HBM
    clocks = ClockSampler(local)
    barrier()
    clocks.start()
    l0 = lib.kpl_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        res = K.solve(A, None, b, None, cfg)
    e1.record()
    barrier()
    launches = lib.kpl_launch_count() - l0
    clk = clocks.stop()
    t_dev = max_over_ranks(e0.elapsed_time(e1) / 1000.0)
    iters_done = res.iterations
    value = world * iters_done * args.steps / t_dev

    # ---- e2e: pinned host b in, host x out, copies inside the timed region
    b_host = torch.empty(n, dtype=torch.float64, pin_memory=True)
    b_host.copy_(b)
    K.solve(A, None, b_host, None, cfg)
    barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    for _ in range(args.steps):
        r2 = K.solve(A, None, b_host, None, cfg)
        _ = r2.x[0].item()          # host-side read of the step's result
        its = r2.iterations
        del r2                      # consumed: its pinned block returns to torch's host cache
    f1.record()
    barrier()
    t_e2e = max_over_ranks(f0.elapsed_time(f1) / 1000.0)
    e2e = world * its * args.steps / t_e2e
    hist_bytes = 80 * (its + 1)

    # ---- e2e with the caller's real types: a numpy b in, a numpy x out (pageable
    # host memory, as a kpl user calls solve), copies inside the timed region
    b_np = b_host.numpy().copy()
    K.solve(A, None, b_np, None, cfg)
    barrier()
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record()
    for _ in range(args.steps):
        r3 = K.solve(A, None, b_np, None, cfg)
        assert isinstance(r3.x, np.ndarray)
        its_np = r3.iterations
        del r3
    g1.record()
    barrier()
    t_np = max_over_ranks(g0.elapsed_time(g1) / 1000.0)
    e2e_np = world * its_np * args.steps / t_np
    del b_np

    # ---- dominant kernel: the fused p-CG-sh iteration sweep, timed alone
    S = _Solve(A, None, b, None, K.SolverConfig(method="pcg_sh", shift=SIGMA, max_iters=100, rtol=0.0))
    S.init()
    S.iterate(1)                      # j=0 (cadence row 0 + first update)
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 9                          # j = 1..9: no cadence kernel, iteration sweeps only
    k0.record()
    S.iterate(reps)
    k1.record()
    torch.cuda.synchronize()
    t_kernel = k0.elapsed_time(k1) / 1000.0 / reps
    alg_bytes = BYTES_PER_DOF * n
    achieved = alg_bytes / t_kernel / 1e9
    peak, peak_kind = peaks()
    traffic = profiled_traffic()

    # whole-solve algorithmic bytes: init (b,x0 reads; r,w writes ~ 40 B/DOF) +
    # 500 x 96 B/DOF + 50 cadence sweeps x 16 B/DOF
    solve_bytes = n * (40 + BYTES_PER_DOF * iters_done + 16 * (iters_done // 10 + 1))
    hbm_gbs = solve_bytes * args.steps / t_dev / 1e9 * world

    out = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t_dev / args.steps * 1000.0,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (generated operator and rhs; no dataset)",
        "config": {
            "workload": WORKLOAD,
            "n": n,
            "iterations_per_step": iters_done,
            "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
            "l2": "no flush: 8 resident vectors of 1 GiB each >> 126 MB L2",
            "final_true_rel_residual": final_rel,
        },
        "hbm_gbs": hbm_gbs,
        "hbm_frac_of_measured": hbm_gbs / peak / world,
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": 8 * n,
                "d2h_bytes_per_step": 8 * n + hist_bytes + 128,
                "host_buffers": "pinned torch CPU tensors (b in, x out)"},
        "e2e_numpy": {"value": e2e_np, "unit": UNIT, "h2d_bytes_per_step": 8 * n,
                      "d2h_bytes_per_step": 8 * n + hist_bytes + 128,
                      "host_buffers": "numpy arrays (pageable): the kpl caller's own types"},
        "roofline": {
            "bound": "hbm",
            "achieved": achieved,
            "peak": peak,
            "unit": "GB/s",
            "frac": achieved / peak,
            "traffic": traffic,
            "kernel": "tma_sweep<BodyPcgIter<0>, 2> (TMA-fed fused 7-point SpMV + 9 recurrences + next dots)",
            "algorithmic_bytes_per_launch": alg_bytes,
            "launch_ms": t_kernel * 1000.0,
            "peak_kind": peak_kind,
        },
        "gpu_launches": launches,
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args.cpu_iters)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_distributed(args, rank, world, local):
    """N-GPU z-slab solve of the same 512^3 problem (strong scaling)."""
    import torch
    import torch.distributed as dist

    import paper_1706_05988_b200 as K
    from paper_1706_05988_b200 import _lib
    from paper_1706_05988_b200.distributed import PeerComm, SlabPlan, TorchComm, solve_distributed

    dev = torch.device("cuda", local)
    A = K.Stencil3D(N3, N3, N3)
    n = A.n
    cfg = K.SolverConfig(method="pcg_sh", shift=SIGMA, max_iters=ITERS, rtol=0.0)
    plan = SlabPlan(N3, N3, N3, world)
    b_full = K.spmv(A, torch.full((n,), 1.0 / math.sqrt(n), dtype=torch.float64, device=dev))
    b = b_full[plan.local_slice(rank)].clone()
    bnorm = float(torch.linalg.norm(b_full))
    del b_full
    torch.cuda.empty_cache()
    # device-initiated exchange over NVLink peer memory (kpl_peer_post /
    # kpl_peer_finalize on IPC-mapped regions); KPL_DIST_EXCHANGE=host selects
    # the host-driven NCCL send/recv + all-gather path.  Ranks sharing one GPU
    # (gloo plumbing runs) always use the host path: their kernels must not
    # wait on one another.
    exchange = os.environ.get("KPL_DIST_EXCHANGE", "peer" if dist.get_backend() == "nccl" else "host")
    comm = None
    check = None
    if exchange == "peer":
        why = ""
        try:
            # self-check before trusting the device-initiated exchange: 12
            # iterations (cadence rows, deferred folds, halo pushes) through PeerComm must
            # equal the host-driven NCCL exchange bit for bit on every rank
            comm = PeerComm()
            pcfg = K.SolverConfig(method="pcg_sh", shift=SIGMA, max_iters=12, rtol=0.0)
            rp = solve_distributed(A, None, b, None, pcfg, comm=comm)
            rh = solve_distributed(A, None, b, None, pcfg, comm=TorchComm())
            same = (rp.iterations == rh.iterations and all(
                (a.alpha, a.beta, a.gamma, a.delta, a.rnorm_recursive, a.rnorm_true) ==
                (c.alpha, c.beta, c.gamma, c.delta, c.rnorm_recursive, c.rnorm_true)
                for a, c in zip(rp.history, rh.history)) and bool(torch.equal(rp.x[0], rh.x[0])))
            check = "peer == host exchange, bitwise (12 iterations)" if same else "MISMATCH"
            if not same:
                why = f"rank {rank}: peer exchange result differs from the host-driven exchange"
        except Exception as exc:          # IPC unavailable: use the host-driven path (all ranks)
            why = f"rank {rank}: {exc}"
        verdicts = [None] * world
        dist.all_gather_object(verdicts, why)
        if any(verdicts):
            print(f"[bench] peer exchange unavailable ({'; '.join(v for v in verdicts if v)}); "
                  "using NCCL send/recv + all-gather", file=sys.stderr)
            comm, exchange = None, "host"
    if comm is None:
        comm = TorchComm()
    lib = _lib.load()

    def barrier():
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        res = solve_distributed(A, None, b, None, cfg, comm=comm)
    clocks = ClockSampler(local)
    barrier()
    clocks.start()
    l0 = lib.kpl_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        res = solve_distributed(A, None, b, None, cfg, comm=comm)
    e1.record()
    barrier()
    launches = lib.kpl_launch_count() - l0
    clk = clocks.stop()
    t_dev = max_over_ranks(e0.elapsed_time(e1) / 1000.0)
    value = res.iterations * args.steps / t_dev

    # e2e: this rank's slab of b from pinned host memory, slab of x back to host
    b_host = torch.empty(b.numel(), dtype=torch.float64, pin_memory=True)
    b_host.copy_(b)
    barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    for _ in range(args.steps):
        bd = b_host.to(dev, non_blocking=True)
        r2 = solve_distributed(A, None, bd, None, cfg, comm=comm)
        xh = torch.empty(bd.numel(), dtype=torch.float64, pin_memory=True)
        xh.copy_(r2.x[0], non_blocking=True)
    f1.record()
    barrier()
    t_e2e = max_over_ranks(f0.elapsed_time(f1) / 1000.0)
    peak, peak_kind = peaks()
    solve_bytes = n * (40 + BYTES_PER_DOF * res.iterations + 16 * (res.iterations // 10 + 1))
    hbm = solve_bytes * args.steps / t_dev / 1e9
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_dev / args.steps * 1000.0, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (generated operator and rhs; no dataset)",
        "config": {"workload": WORKLOAD, "n": n, "iterations_per_step": res.iterations,
                   "final_true_rel_residual": res.history[-1].rnorm_true / bnorm,
                   "exchange_check": check,
                   "parallelism": (f"z-slab x{world} (NVLink peer-memory halos + partials, device flags)"
                                   if exchange == "peer" else
                                   f"z-slab x{world} ({dist.get_backend()} halo send/recv + chunk all-gather)"),
                   "l2": "no flush: per-rank vectors >> 126 MB L2"},
        "hbm_gbs": hbm, "hbm_frac_of_measured": hbm / peak / world,
        "e2e": {"value": res.iterations * args.steps / t_e2e, "unit": UNIT,
                "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n},
        "roofline": {"bound": "hbm", "achieved": hbm / world, "peak": peak, "unit": "GB/s",
                     "frac": hbm / world / peak, "traffic": profiled_traffic(),
                     "kernel": "whole distributed solve per GPU (fused sweeps + exchanges)",
                     "peak_kind": peak_kind},
        "gpu_launches": launches, "clocks": clk,
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


# ----------------------------------------------------------- CPU baseline

def _cpu_setup():
    import numpy as np

    from oracle import kpl_oracle as O
    A = O.StencilSpec(N3, N3, N3, 6.0)
    b = O.spmv(A, np.full(A.n, 1.0 / math.sqrt(A.n)))
    return O, A, b


def cpu_iterations(nsteps, O=None, A=None, b=None, warm=0):
    """Time `nsteps` p-CG-sh iterations of the oracle on the 512^3 problem
    (after `warm` untimed ones).  Returns seconds per iteration list."""
    import numpy as np
    if O is None:
        O, A, b = _cpu_setup()
    times = []
    marks = []

    def cb(st):
        marks.append(time.perf_counter())

    total = warm + nsteps
    O.solve_pcg_shifted(A, None, b, None,
                        O.Config(method="pcg_sh", shift=SIGMA, max_iters=total, rtol=0.0),
                        callback=cb)
    # record k is reached after update k-1; iteration k-1 = marks[k] - marks[k-1]
    for k in range(warm + 1, total + 1):
        times.append(marks[k] - marks[k - 1])
    return times


def host_cpu():
    """CPU model and core count of the host the baseline ran on."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "host_cores": os.cpu_count()}


PORT_NOTE = ("the oracle port is matrix-free (the reference assembles a 512^3 int64 CSR, ~50-60 GB); "
             "at 128^3 the reference ran 1.8x slower per DOF than this port (BASELINE.md 2), so the port "
             "overstates the reference's speed; the reference itself is timed on configs 1, 2 and 5 in "
             "profiles/r02_reference_cpu.jsonl (tools/time_reference.py)")


def cpu_baseline(iters):
    O, A, b = _cpu_setup()
    times = cpu_iterations(iters, O, A, b, warm=0)
    per = sum(times) / len(times)
    return {"value": 1.0 / per, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": (f"{len(times)} p-CG-sh iterations of the 512^3 problem with the CPU "
                       "oracle (numpy ufuncs + C restatement of the reference's kernels, "
                       "single thread like the reference); includes its true-residual cadence"),
            "seconds_per_iteration": per, **host_cpu(), "note": PORT_NOTE}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    O, A, b = _cpu_setup()
    steps = args.steps
    warm = args.warmup
    times = cpu_iterations(steps, O, A, b, warm=warm)
    per = sum(times) / len(times)
    value = 1.0 / per
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
        "warmup": warm, "ms_per_step": per * 1000.0, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (generated operator and rhs; no dataset)",
        "config": {"workload": WORKLOAD, "n": A.n, "step": "one p-CG-sh iteration (bounded sample)"},
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port",
                         "sample": f"{steps} iterations of the 512^3 problem, oracle restatement "
                                   "of the single-threaded reference path", **host_cpu(), "note": PORT_NOTE},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--cpu-iters", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
