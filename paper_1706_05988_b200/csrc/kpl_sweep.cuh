// kpl_sweep.cuh -- the two traversal skeletons every kernel is built from.
//
//  * stencil_sweep: one CTA per (x-y tile, z-chunk) item.  8 warps; warp
//    (wx, wy) owns 32*VX consecutive x-elements of tile row wy.  The CTA
//    marches through the chunk's planes: the stencil input's own column is a
//    register queue (z-1, z, z+1, z+2), its x/y neighbours come from a
//    double-buffered shared-memory plane with a one-element x halo and a
//    one-row y halo, and the body's streams for plane z+1 are prefetched into
//    registers while plane z is computed.  One __syncthreads per plane.
//
//  * csr_spmv_kernel + csr_chunk_sweep (CSR): the SpMV in the reference's
//    csr_matvec order (_kernels.py:44-52), then the body's update + reductions
//    one reduction chunk per CTA (see the block comment below).
//
// Both end with the same deterministic reduction: per-element accumulators
// (sequential over z for stencils), per-thread pair sum (VX=2), warp xor
// butterfly, 8-warp halving tree -> item partial; complete_item() folds items
// into chunks and chunks into the final value.
#pragma once
#include "kpl_core.cuh"

namespace kpl {

struct SGeo {
    long long NX, NY, NZ;
    double diag;
    const double *halo_lo, *halo_hi;   // raw stencil-input planes z=-1 / z=NZ (or null)
    int zhalo;                         // 1: the input vector itself carries planes -1 and NZ
};

struct CGeo {
    long long n;
    const int *row_ptr, *col_idx;
    const double *values;
};

// Largest smem plane: 3D tile (1x8 warps, VX=2): 10 rows x (128+4); 2D tile
// (8x1 warps, VX=2): 3 rows x (512+4).
constexpr int SMEM_PLANE = 1548;
#ifndef KPL_CSR_WIN
#define KPL_CSR_WIN 1024
#endif
#ifndef KPL_SPMV_MINB
#define KPL_SPMV_MINB 8
#endif
constexpr int CSR_WIN = KPL_CSR_WIN;   // staged nonzeros per window

// One pass of a stencil sweep over all items (grid-stride), callable from the
// one-launch-per-sweep kernel below and from the persistent solver kernel.
// `spbuf` (2 * SMEM_PLANE doubles) and `sred` (NQ * NWARP) are the caller's
// shared memory, so several passes in one kernel share it.
template <int VX, class In, class Body, bool FOLD = true>
__device__ __forceinline__ void stencil_pass(const SGeo &g, const Layout &L, In in, Body body, const Ws &ws,
                                             const Cfg &cfg, int phase, double *spbuf, double *sred) {
    constexpr int Q = Body::NQ;
    double (*sp)[SMEM_PLANE] = reinterpret_cast<double (*)[SMEM_PLANE]>(spbuf);

    body.setup(ws);
    in.setup(ws);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wx = warp % L.wx, wy = warp / L.wx;
    const int TX = 32 * VX * L.wx, TY = L.wy;
    // one item per CTA normally; rarely-active sweeps (replacement path) launch a
    // small grid that strides over the items so an idle launch costs a few CTAs
    for (long long item = blockIdx.x; item < L.items; item += gridDim.x) {
    const long long c = item / L.T;
    const int tile = (int)(item - c * L.T);
    const int tyi = tile / L.ntx, txi = tile - tyi * L.ntx;
    const long long x0 = (long long)txi * TX, y0 = (long long)tyi * TY;
    const int xl = wx * 32 * VX + lane * VX;          // x inside the tile
    const long long x = x0 + xl, y = y0 + wy;
    const bool ok = (y < g.NY) && (x < g.NX);         // VX=2 => NX even => pair all-or-none
    const long long NX = g.NX, sxy = g.NX * g.NY;
    const long long z0 = c * L.zc;
    const long long z1 = min(z0 + (long long)L.zc, g.NZ);
    const int rowlen = TX + 4;                         // [1]=x0-1, [2..TX+1]=tile, [TX+2]=x0+TX
    const int cidx = (wy + 1) * rowlen + 2 + xl;       // own element in the smem plane

    double acc[Q > 0 ? Q : 1][VX];
#pragma unroll
    for (int q = 0; q < (Q > 0 ? Q : 1); ++q)
#pragma unroll
        for (int v = 0; v < VX; ++v) acc[q][v] = 0.0;

    // raw stencil-input loaders with Dirichlet ghosts / slab halos
    auto plane_ptr = [&](long long zz, long long &off) -> const double * {
        if (!g.zhalo) {
            if (zz < 0) { off = 0; return g.halo_lo; }
            if (zz >= g.NZ) { off = 0; return g.halo_hi; }
        }
        off = zz * sxy;                                // zhalo: planes -1 and NZ are real memory
        return in.base();
    };
    auto ld_own = [&](long long zz, double (&o)[VX]) {
#pragma unroll
        for (int v = 0; v < VX; ++v) o[v] = 0.0;
        long long off;
        const double *p = plane_ptr(zz, off);
        if (ok && p) in.template raw<VX>(p, off + x + NX * y, o);
    };
    // halo values of plane zz: [0] x0-1, [1] x0+TX (row y), [2..] y0-1 row, y0+TY row
    struct Halo { double xl, xr, yl[VX], yh[VX]; };
    auto ld_halo = [&](long long zz, Halo &hh) {
        hh.xl = 0.0; hh.xr = 0.0;
#pragma unroll
        for (int v = 0; v < VX; ++v) { hh.yl[v] = 0.0; hh.yh[v] = 0.0; }
        long long off;
        const double *p = plane_ptr(zz, off);
        if (!p) return;
        if (y < g.NY) {
            if (wx == 0 && lane == 0 && x0 > 0) {
                double t[1]; in.template raw<1>(p, off + (x0 - 1) + NX * y, t); hh.xl = t[0];
            }
            if (wx == L.wx - 1 && lane == 31 && x0 + TX < NX) {
                double t[1]; in.template raw<1>(p, off + (x0 + TX) + NX * y, t); hh.xr = t[0];
            }
        }
        if (x < NX) {
            if (wy == 0 && y0 > 0) in.template raw<VX>(p, off + x + NX * (y0 - 1), hh.yl);
            if (wy == TY - 1 && y0 + TY < g.NY) in.template raw<VX>(p, off + x + NX * (y0 + TY), hh.yh);
        }
    };
    auto stage = [&](double *P, const double (&cen)[VX], const Halo &hh) {
#pragma unroll
        for (int v = 0; v < VX; ++v) P[cidx + v] = cen[v];
        if (wx == 0 && lane == 0) P[(wy + 1) * rowlen + 1] = hh.xl;
        if (wx == L.wx - 1 && lane == 31) P[(wy + 1) * rowlen + TX + 2] = hh.xr;
        if (wy == 0) {
#pragma unroll
            for (int v = 0; v < VX; ++v) P[2 + xl + v] = hh.yl[v];
        }
        if (wy == TY - 1) {
#pragma unroll
            for (int v = 0; v < VX; ++v) P[(TY + 1) * rowlen + 2 + xl + v] = hh.yh[v];
        }
    };

    typename Body::template Regs<VX> cur, nxt;
    double qm[VX], qc[VX], qp[VX], qn[VX];
    Halo h1, h2;
    if (z0 < z1) {
        if constexpr (Body::kStencil) {
            ld_own(z0 - 1, qm);
            ld_own(z0, qc);
            ld_own(z0 + 1, qp);
            Halo h0;
            ld_halo(z0, h0);
            ld_halo(z0 + 1, h1);
            stage(sp[0], qc, h0);
        }
        if (ok) body.template load<VX>(z0 * sxy + x + NX * y, cur);
    }
    for (long long z = z0; z < z1; ++z) {
        const int kb = (int)((z - z0) & 1);
        const long long k = z * sxy + x + NX * y;
        if constexpr (Body::kStencil) {
            if (z + 1 < z1) {
                ld_own(z + 2, qn);
                ld_halo(z + 2, h2);
            }
        }
        if (z + 1 < z1 && ok) body.template load<VX>(k + sxy, nxt);
        double n[VX];
        if constexpr (Body::kStencil) {
            __syncthreads();
            const double *P = sp[kb];
            // terms in ascending column order: z-1, y-1, x-1, diag, x+1, y+1, z+1
            double ym[VX], yp[VX], xm[VX], xp[VX];
#pragma unroll
            for (int v = 0; v < VX; ++v) {
                ym[v] = P[cidx - rowlen + v];
                yp[v] = P[cidx + rowlen + v];
            }
            xm[0] = P[cidx - 1];
            xp[VX - 1] = P[cidx + VX];
            if constexpr (VX == 2) { xm[1] = qc[0]; xp[0] = qc[1]; }
#pragma unroll
            for (int v = 0; v < VX; ++v) {
                const long long kv = k + v;
                double a = 0.0;
                a = __dadd_rn(a, -in.xf(qm[v], kv - sxy));
                a = __dadd_rn(a, -in.xf(ym[v], kv - NX));
                a = __dadd_rn(a, -in.xf(xm[v], kv - 1));
                a = __dadd_rn(a, __dmul_rn(g.diag, in.xf(qc[v], kv)));
                a = __dadd_rn(a, -in.xf(xp[v], kv + 1));
                a = __dadd_rn(a, -in.xf(yp[v], kv + NX));
                a = __dadd_rn(a, -in.xf(qp[v], kv + sxy));
                n[v] = a;
            }
        } else {
#pragma unroll
            for (int v = 0; v < VX; ++v) n[v] = 0.0;
        }
        if (ok) body.template compute<VX>(k, cur, n, qc, acc);
        if constexpr (Body::kStencil) {
            if (z + 1 < z1) {
                stage(sp[kb ^ 1], qp, h1);
                h1 = h2;
            }
#pragma unroll
            for (int v = 0; v < VX; ++v) { qm[v] = qc[v]; qc[v] = qp[v]; qp[v] = qn[v]; }
        }
        cur = nxt;
    }
    if constexpr (FOLD) peer_halo_push<VX>(ws, c, L.nch, g.NZ, sxy, x + NX * y, ok);   // (never in persistent passes)

    if constexpr (Q > 0) {
        double t[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            t[q] = acc[q][0];
            if constexpr (VX == 2) t[q] = __dadd_rn(acc[q][0], acc[q][1]);
        }
        block_sum<Q>(t, sred);
        if (tid == 0) {
#pragma unroll
            for (int q = 0; q < Q; ++q) ws.items[item * NQ + q] = t[q];
        }
        if constexpr (FOLD) complete_item<Q>(ws, cfg, L, phase, c, sred);
    }
    __syncthreads();           // smem planes are restaged by the next item
    }
}

template <int VX, class In, class Body, bool FOLD = false>
__global__ void __launch_bounds__(NT, 2)
stencil_sweep(SGeo g, Layout L, In in, Body body, Ws ws, Cfg cfg, int phase, int pred, long long row) {
    __shared__ __align__(16) double sp[Body::kStencil ? 2 * SMEM_PLANE : 2];
    __shared__ double sred[NQ * NWARP];
    pdl_wait();
    pdl_launch_dependents();
    if constexpr (FOLD) {                                   // deferred fold of the previous sweep
        __shared__ FoldSmem fsm;
        peer_fold_start(ws, cfg, fsm, sred);
        const Ws view = ws_fold_view(ws, &fsm.head, fsm.row, true);
        if (!pred_ok(view.head, pred, row)) { peer_signal_idle(view); return; }
        stencil_pass<VX, In, Body>(g, L, in, body, view, cfg, phase, sp, sred);
    } else {
        if (!pred_ok(ws.head, pred, row)) { peer_signal_idle(ws); return; }
        stencil_pass<VX, In, Body>(g, L, in, body, ws, cfg, phase, sp, sred);
    }
}

// ---------------------------------------------------------------------------
// Persistent solver for small stencil problems: one cooperative launch runs
// up to `count` p-CG(-sh) iterations; a grid barrier replaces the kernel
// boundary after every pass (the last CTA's scalar epilogue must be visible
// before anybody reads alpha/beta).  Same passes, items and trees as the
// per-iteration launches, so results are bit-identical.  Stencil-input loads
// go through L2 (InVec<PC, 1>) because neighbours' values were written
// earlier in the same kernel.
__device__ __forceinline__ void grid_sync(WsHead *h) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned gen = atomicAdd(&h->bar_gen, 0u);
        __threadfence();
        if (atomicAdd(&h->bar_cnt, 1u) == gridDim.x - 1) {
            atomicExch(&h->bar_cnt, 0u);
            __threadfence();
            atomicAdd(&h->bar_gen, 1u);
        } else {
            volatile unsigned *g = &h->bar_gen;          // poll through L2 without atomics
            unsigned long long t0 = 0, t;
            for (unsigned n = 1; *g == gen; ++n) {
                if ((n & 4095u) == 0u) {                  // watchdog: a broken barrier traps, not hangs
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                    if (t0 == 0) t0 = t;
                    else if (t - t0 > 10000000000ull) __trap();
                }
            }
        }
        __threadfence();
    }
    __syncthreads();
}

template <int VX, class InW, class BodyIt, class InX>
__global__ void __launch_bounds__(NT, 2)
persistent_pipelined(SGeo g, Layout L, InW in_w, BodyIt body, InX in_x, BodyTrue tbody, Ws ws, Cfg cfg,
                     long long first, long long count) {
    __shared__ __align__(16) double sp[2 * SMEM_PLANE];
    __shared__ double sred[NQ * NWARP];
    for (long long j = first; j < first + count; ++j) {
        if (ld_head(&ws.head->state) != KPL_ST_RUNNING) break;    // uniform: read after a barrier
        if (j % 10 == 0) {                                           // true-residual cadence (row j)
            if (ld_head(&ws.head->iter) == j)
                stencil_pass<VX, InX, BodyTrue>(g, L, in_x, tbody, ws, cfg, PH_TRUE, sp, sred);
            grid_sync(ws.head);
        }
        stencil_pass<VX, InW, BodyIt>(g, L, in_w, body, ws, cfg, PH_PIPE, sp, sred);
        grid_sync(ws.head);
    }
}

// One-phase grid barrier: a monotone 64-bit arrival counter; barrier k of a
// launch completes when the counter reaches base + k*grid.  One release
// atomic to arrive, relaxed polling (an acquire load per poll would also
// invalidate L1), one acquire load to leave.  `base` is the counter at
// launch, rounded down to a multiple of the grid (every completed barrier
// adds exactly one grid, and fewer than a grid of arrivals can precede any
// CTA's first read).
struct GridBarrier {
    unsigned long long *cnt;
    unsigned long long target;
    __device__ void init(unsigned long long *c) {
        cnt = c;
        if (threadIdx.x == 0) {
            unsigned long long v;
            asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(c) : "memory");
            target = v - v % gridDim.x;
        }
    }
    // false: the barrier did not complete within 3 s (a bug, never a wait a
    // correct run needs): the real head is marked BREAKDOWN / "device barrier
    // timeout" and the caller leaves the kernel instead of hanging the GPU
    __device__ bool sync(WsHead *real) {
        __shared__ int s_ok;
        __syncthreads();
        if (threadIdx.x == 0) {
            target += gridDim.x;
            unsigned long long v, t0, t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
            asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;" : "=l"(v) : "l"(cnt) : "memory");
            int ok = 1;
            for (unsigned spin = 1; v < target; ++spin) {
                asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(cnt) : "memory");
                if ((spin & 1023) == 0) {                       // the clock only now and then
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                    if (t - t0 > 3000000000ull) { ok = 0; break; }
                }
            }
            if (!ok) {
                real->bd_code = BD_BARRIER_TIMEOUT;
                real->bd_iter = -1;
                atomicExch(reinterpret_cast<unsigned long long *>(&real->state), (unsigned long long)KPL_ST_BREAKDOWN);
            }
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(cnt) : "memory");
            s_ok = ok;
        }
        __syncthreads();
        return s_ok;
    }
};

// Redundant epilogue (small problems): after one grid barrier every CTA folds
// all item partials itself -- level 3 one warp per chunk (chunks of <= 32
// items: the block tree of complete_item reduces to warp 0's butterfly, the
// other warps adding +0.0, which is exact because no partial of the form
// 0.0 + x is -0.0), level 4 the same strided tree over the chunk values in
// shared memory -- and runs the scalar epilogue on its own copy of the head.
// Every CTA therefore holds the same alpha, beta, state as the inline path
// without the chunk/final counter round trips or a second barrier.
template <int Q>
__device__ void fold_redundant(const Ws &wl, const Cfg &cfg, const Layout &L, int phase, double *sitems,
                               double *schunk, double *sred) {
    // one parallel, coalesced copy of the item table (a single L2 round trip)
    const long long nitem = L.items * NQ;
    for (long long k = threadIdx.x; k < nitem; k += blockDim.x) sitems[k] = __ldcg(wl.items + k);
    __syncthreads();
    // level 3, packed: with P = pow2 >= T, lanes [gP, gP+P) hold chunk g of the
    // warp's group; the butterfly restricted to offsets < P gives lane gP exactly
    // lane 0's value of the full 32-lane butterfly (the lanes >= P only add +0.0)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int P = 1;
    while (P < L.T) P <<= 1;
    const int per = 32 / P, sub = lane / P, idx = lane - sub * P;
    for (long long c0 = (long long)warp * per; c0 < L.nch; c0 += (long long)NWARP * per) {
        const long long c = c0 + sub;
        const long long i0 = c * L.T;
        const int cnt = c < L.nch ? (int)min((long long)L.T, L.items - i0) : 0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            double v = idx < cnt ? __dadd_rn(0.0, sitems[(i0 + idx) * NQ + q]) : 0.0;
            for (int off = P >> 1; off > 0; off >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
            if (idx == 0 && c < L.nch) schunk[c * NQ + q] = v;
        }
    }
    __syncthreads();
    double f[Q];
    strided_sum<Q, true>(schunk, L.nch, NQ, f, sred);
    if (threadIdx.x == 0) {
        double full[NQ] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int q = 0; q < Q; ++q) full[q] = f[q];
        finalize(wl, cfg, phase, full);
    }
    __syncthreads();           // the CTA's head is read by every thread of the next pass
}

// A CTA-private view of the workspace, built field by field.  (Copying the
// by-value kernel parameter `Ws ws` into a local and then changing fields of
// the copy was miscompiled: nvcc 12.9 forwarded some reads of the copy to the
// parameter, so private-head CTAs read CTA 0's head and the shared item
// buffer -- the intermittent divergence/hang of the redundant-epilogue solver.)
__device__ __forceinline__ Ws ws_view(const Ws &ws, WsHead *head, double *hist, int scratch, double *items) {
    Ws w;
    w.head = head; w.items = items; w.chunks = ws.chunks; w.chunk_cnt = ws.chunk_cnt; w.hist = hist;
    w.reps = ws.reps; w.nbuf = ws.nbuf; w.mbuf = ws.mbuf; w.chunk_offset = ws.chunk_offset;
    w.chunks_global = ws.chunks_global; w.inline_final = ws.inline_final; w.prod = ws.prod; w.nprod = ws.nprod;
    w.hist_scratch = scratch; w.px = nullptr; w.epoch = 0; w.tpar = 0; w.push = 0; w.wpar = 0;
    w.wait_epoch = 0; w.wait_tpar = 0; w.timeout_ns = ws.timeout_ns; w.final_cnt = ws.final_cnt;
    return w;
}

template <int VX, class InW, class BodyIt, class InX>
__global__ void __launch_bounds__(NT, 2)
persistent_redundant(SGeo g, Layout L, InW in_w, BodyIt body, InX in_x, BodyTrue tbody, Ws ws, Cfg cfg,
                     long long first, long long count, char *pheads) {
    __shared__ __align__(16) double sp[2 * SMEM_PLANE];
    __shared__ double sred[NQ * NWARP];
    extern __shared__ double sdyn[];                   // item table [items][NQ], chunk table [nch][NQ]
    double *const sitems = sdyn, *const schunk = sdyn + NQ * L.items;
    WsHead *head = ws.head;
    double *hist = ws.hist;
    int scratch = 0;
    if (blockIdx.x > 0) {                              // private head + scratch history row
        char *slot = pheads + (blockIdx.x - 1) * (1024 + 256);
        WsHead *mine = reinterpret_cast<WsHead *>(slot);
        const unsigned long long *src = reinterpret_cast<const unsigned long long *>(ws.head);
        unsigned long long *dst = reinterpret_cast<unsigned long long *>(mine);
        for (int k = threadIdx.x; k < (int)(sizeof(WsHead) / 8); k += blockDim.x) dst[k] = __ldcg(src + k);
        head = mine;
        hist = reinterpret_cast<double *>(slot + 1024);
        scratch = 1;
        __syncthreads();
    }
    // two views, one per item buffer (passes alternate them)
    const Ws w0 = ws_view(ws, head, hist, scratch, ws.items);
    const Ws w1 = ws_view(ws, head, hist, scratch, ws.items + NQ * L.items);
    long long pass = 0;
    GridBarrier bar;
    bar.init(&ws.head->bar_arrive);
    for (long long j = first; j < first + count; ++j) {
        if (ld_head(&head->state) != KPL_ST_RUNNING) break;        // identical in every CTA
        if (j % 10 == 0 && ld_head(&head->iter) == j) {             // true-residual cadence (row j)
            const Ws &wl = (pass++ & 1) ? w1 : w0;
            stencil_pass<VX, InX, BodyTrue, false>(g, L, in_x, tbody, wl, cfg, PH_TRUE, sp, sred);
            if (!bar.sync(ws.head)) return;
            fold_redundant<1>(wl, cfg, L, PH_TRUE, sitems, schunk, sred);
        }
        const Ws &wl = (pass++ & 1) ? w1 : w0;
        stencil_pass<VX, InW, BodyIt, false>(g, L, in_w, body, wl, cfg, PH_PIPE, sp, sred);
        if (!bar.sync(ws.head)) return;
        fold_redundant<BodyIt::NQ>(wl, cfg, L, PH_PIPE, sitems, schunk, sred);
    }
}

// ---------------------------------------------------------------------------
// CSR, split form (the production CSR path).
//
//  csr_spmv_kernel   n = A * xf(input): one CTA per 256-row block, the block's
//                    nonzeros staged through shared memory (coalesced
//                    col_idx/values loads, gathered input, products), each
//                    thread summing its row left to right from +0.0 -- the
//                    reference csr_matvec order.  No reductions, small register
//                    and smem footprint -> high occupancy for the gathers.
//  csr_chunk_sweep   one CTA per reduction chunk (chunk_blocks 256-row items):
//                    the body's update for every row of the chunk with n read
//                    back from memory, item partials kept in shared memory, the
//                    chunk fold (level 3) done in-CTA, one completion atomic per
//                    chunk.  The item (256 rows) and chunk trees are the ones
//                    oracle/gpu_order.py emulates.
// WIN: staged nonzeros per window (1024 for short rows; 512 for long, randomly
// gathered rows, where more resident warps beat longer windows); 8 CTAs/SM.
template <class In, int WIN = CSR_WIN, bool L2G = false>
__global__ void __launch_bounds__(NT, KPL_SPMV_MINB)
csr_spmv_kernel(CGeo g, In in, double *__restrict__ out, Ws ws, int pred, long long row) {
    constexpr int PER = WIN / NT;
    __shared__ double sprod[WIN];
    pdl_wait();
    pdl_launch_dependents();
    if (ws.head && !pred_ok(ws.head, pred, row)) return;
    if (ws.head) in.setup(ws);
    const int tid = threadIdx.x;
    const long long nblk = (g.n + RB - 1) / RB;
    for (long long blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const long long r0 = blk * RB;
    const long long r = r0 + tid;
    const bool ok = r < g.n;
    const long long rend = min(r0 + RB, g.n);
    const long long k0 = __ldg(g.row_ptr + r0), k1 = __ldg(g.row_ptr + rend);
    long long lo = 0, hi = 0;
    if (ok) { lo = __ldg(g.row_ptr + r); hi = __ldg(g.row_ptr + r + 1); }
    double a = 0.0;
    for (long long wk = k0; wk < k1; wk += WIN) {
        const long long we = min(wk + (long long)WIN, k1);
        int col[PER];
        double val[PER], raw[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const long long kk = wk + tid + (long long)j * NT;
            col[j] = 0; val[j] = 0.0;
            if (kk < we) { col[j] = __ldcs(g.col_idx + kk); val[j] = __ldcs(g.values + kk); }
        }
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const long long kk = wk + tid + (long long)j * NT;
            raw[j] = 0.0;
            if (kk < we) raw[j] = load1<L2G>(in, in.base(), col[j]);
        }
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const long long kk = wk + tid + (long long)j * NT;
            if (kk < we) sprod[kk - wk] = __dmul_rn(val[j], in.xf(raw[j], col[j]));
        }
        __syncthreads();
        const long long a0 = max(lo, wk), a1 = min(hi, we);
        for (long long kk = a0; kk < a1; ++kk) a = __dadd_rn(a, sprod[kk - wk]);   // csr_matvec order
        __syncthreads();
    }
    if (ok) out[r] = a;
    }
}

// Software-pipelined form of csr_spmv_kernel: the products of window k go to
// one of two shared-memory buffers, then window k+1's col/val loads and
// gathers are issued BEFORE the barrier and the row sums of window k, so they
// are in flight while the CTA sums (one __syncthreads per window instead of
// two).  Same products, same csr_matvec order: bitwise equal.
template <class In, int WIN, bool L2G, int MINB>
__global__ void __launch_bounds__(NT, MINB)
csr_spmv_pipe(CGeo g, In in, double *__restrict__ out, Ws ws, int pred, long long row) {
    constexpr int PER = WIN / NT;
    __shared__ double sprod[2][WIN];
    pdl_wait();
    pdl_launch_dependents();
    if (ws.head && !pred_ok(ws.head, pred, row)) return;
    if (ws.head) in.setup(ws);
    const int tid = threadIdx.x;
    const long long nblk = (g.n + RB - 1) / RB;
    const double *base = in.base();
    for (long long blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        const long long r0 = blk * RB;
        const long long r = r0 + tid;
        const bool ok = r < g.n;
        const long long rend = min(r0 + RB, g.n);
        const long long k0 = __ldg(g.row_ptr + r0), k1 = __ldg(g.row_ptr + rend);
        long long lo = 0, hi = 0;
        if (ok) { lo = __ldg(g.row_ptr + r); hi = __ldg(g.row_ptr + r + 1); }
        int col[PER];
        double val[PER], raw[PER];
        auto issue = [&](long long wk) {          // col/val of window wk, then its gathers
            const long long we = min(wk + (long long)WIN, k1);
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                const long long kk = wk + tid + (long long)j * NT;
                col[j] = 0; val[j] = 0.0;
                if (kk < we) { col[j] = __ldcs(g.col_idx + kk); val[j] = __ldcs(g.values + kk); }
            }
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                const long long kk = wk + tid + (long long)j * NT;
                raw[j] = kk < we ? load1<L2G>(in, base, col[j]) : 0.0;
            }
        };
        double a = 0.0;
        if (k0 < k1) issue(k0);
        int buf = 0;
        for (long long wk = k0; wk < k1; wk += WIN, buf ^= 1) {
            const long long we = min(wk + (long long)WIN, k1);
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                const long long kk = wk + tid + (long long)j * NT;
                if (kk < we) sprod[buf][kk - wk] = __dmul_rn(val[j], in.xf(raw[j], col[j]));
            }
            if (we < k1) issue(we);                  // next window in flight during the sums
            __syncthreads();
            const long long a0 = max(lo, wk), a1 = min(hi, we);
            for (long long kk = a0; kk < a1; ++kk) a = __dadd_rn(a, sprod[buf][kk - wk]);   // csr_matvec order
        }
        if (ok) out[r] = a;
        __syncthreads();          // the next block reuses both buffers
    }
}

// Column-sorted gather form of csr_spmv_kernel (kpl_op.sp_*; scattered
// matrices such as config 5's random band, where a CSR-order warp gather
// touches ~31 cache lines and the SpMV is bound by L1 wavefronts).  One CTA
// per block of S.R rows: phase 1 streams the block's nonzeros in column order
// (coalesced col/val/dest, gathers whose lanes share lines: ~9 lines per warp
// at 1024 rows) and stores each product at its CSR position in shared memory;
// phase 2 sums every row left to right from +0.0 out of shared memory -- the
// csr_matvec order, so n is bit-identical to csr_spmv_kernel's.
struct SGather {
    const int *col;
    const double *val;
    const unsigned short *dest;
    int R;                    // rows per block
};

template <class In, int NTS, int PER, bool L2G = false>
__global__ void __launch_bounds__(NTS, 1)
csr_sorted_spmv(CGeo g, SGather S, In in, double *__restrict__ out, Ws ws, int pred, long long row) {
    extern __shared__ double sprod[];
    pdl_wait();
    pdl_launch_dependents();
    if (ws.head && !pred_ok(ws.head, pred, row)) return;
    if (ws.head) in.setup(ws);
    const int tid = threadIdx.x;
    const long long nblk = (g.n + S.R - 1) / S.R;
    const double *base = in.base();
    constexpr long long STEP = (long long)NTS * PER;
    // software pipeline: the (col, val, dest) stream of round k+1 -- or of the
    // next block's first round -- is in flight while round k's gathers are
    int col[PER], d[PER], ncol[PER], nd[PER];
    double val[PER], nval[PER];
    auto fetch = [&](long long kb, long long k1, int (&c)[PER], double (&v)[PER], int (&dd)[PER]) {
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const long long kk = kb + (long long)j * NTS;
            c[j] = 0; dd[j] = 0; v[j] = 0.0;
            if (kk < k1) { c[j] = __ldcs(S.col + kk); v[j] = __ldcs(S.val + kk); dd[j] = __ldcs(S.dest + kk); }
        }
    };
    long long blk = blockIdx.x;
    long long k0 = 0, k1 = 0;
    if (blk < nblk) {
        k0 = __ldg(g.row_ptr + blk * S.R);
        k1 = __ldg(g.row_ptr + min(blk * S.R + S.R, g.n));
        fetch(k0 + tid, k1, col, val, d);
    }
    for (; blk < nblk; blk += gridDim.x) {
        const long long r0 = blk * S.R, r1 = min(r0 + (long long)S.R, g.n);
        const long long nb = blk + gridDim.x;
        long long nk0 = 0, nk1 = 0;
        if (nb < nblk) { nk0 = __ldg(g.row_ptr + nb * S.R); nk1 = __ldg(g.row_ptr + min(nb * S.R + S.R, g.n)); }
        for (long long kb = k0 + tid; kb < k1; kb += STEP) {
            const bool more = kb + STEP < k1;
            if (more) fetch(kb + STEP, k1, ncol, nval, nd);
            else if (nb < nblk) fetch(nk0 + tid, nk1, ncol, nval, nd);      // next block's first round
            double raw[PER];
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                raw[j] = 0.0;
                if (kb + (long long)j * NTS < k1) raw[j] = load1<L2G>(in, base, col[j]);
            }
#pragma unroll
            for (int j = 0; j < PER; ++j)
                if (kb + (long long)j * NTS < k1) sprod[d[j]] = __dmul_rn(val[j], in.xf(raw[j], col[j]));
#pragma unroll
            for (int j = 0; j < PER; ++j) { col[j] = ncol[j]; val[j] = nval[j]; d[j] = nd[j]; }
        }
        if (k0 + tid >= k1 && nb < nblk) fetch(nk0 + tid, nk1, col, val, d);  // no round this block
        __syncthreads();
        for (long long r = r0 + tid; r < r1; r += NTS) {
            const int a0 = __ldg(g.row_ptr + r) - (int)k0, a1 = __ldg(g.row_ptr + r + 1) - (int)k0;
            double a = 0.0;
            for (int kk = a0; kk < a1; ++kk) a = __dadd_rn(a, sprod[kk]);   // csr_matvec order
            out[r] = a;
        }
        __syncthreads();
        k0 = nk0; k1 = nk1;
    }
}

template <class In, class Body, bool L2G = false>
__global__ void __launch_bounds__(NT, 3)
csr_chunk_sweep(CGeo g, Layout L, In in, Body body, const double *__restrict__ nin, Ws ws, Cfg cfg, int phase,
                int pred, long long row) {
    constexpr int Q = Body::NQ;
    __shared__ double sred[NQ * NWARP];
    __shared__ double sitem[Q > 0 ? Q : 1][64];
    pdl_wait();
    pdl_launch_dependents();
    if (!pred_ok(ws.head, pred, row)) return;
    body.setup(ws);
    in.setup(ws);
    const int tid = threadIdx.x;
    __shared__ int s_last;
    for (long long chunk = blockIdx.x; chunk < L.nch; chunk += gridDim.x) {
    const long long it0 = chunk * L.T;
    const int nit = (int)min((long long)L.T, L.items - it0);
    // software pipeline over the chunk's items: streams of item i+1 in flight while i computes
    typename Body::template Regs<1> R, Rn;
    double nn = 0.0, cen = 0.0, nn_n = 0.0, cen_n = 0.0;
    auto fetch = [&](long long item, typename Body::template Regs<1> &RR, double &n1, double &c1) {
        const long long r = item * RB + tid;
        if (r < g.n) {
            body.template load<1>(r, RR);
            if constexpr (Body::kStencil) {
                n1 = __ldcs(nin + r);
                c1 = load1<L2G>(in, in.base(), r);
            }
        }
    };
    fetch(it0, R, nn, cen);
    for (int i = 0; i < nit; ++i) {
        const long long item = it0 + i;
        if (i + 1 < nit) fetch(item + 1, Rn, nn_n, cen_n);
        const long long r = item * RB + tid;
        double acc[Q > 0 ? Q : 1][1];
#pragma unroll
        for (int q = 0; q < (Q > 0 ? Q : 1); ++q) acc[q][0] = 0.0;
        if (r < g.n) {
            const double n1[1] = {nn}, c1[1] = {cen};
            body.template compute<1>(r, R, n1, c1, acc);
        }
        if constexpr (Q > 0) {
            double t[Q];
#pragma unroll
            for (int q = 0; q < Q; ++q) t[q] = acc[q][0];
            block_sum<Q>(t, sred);                    // item partial (levels 2b, 2c)
            if (tid == 0) {
#pragma unroll
                for (int q = 0; q < Q; ++q) { sitem[q][i] = t[q]; ws.items[item * NQ + q] = t[q]; }
            }
        }
        R = Rn; nn = nn_n; cen = cen_n;
    }
    if constexpr (Q > 0) {
        __syncthreads();
        // level 3 in-CTA: thread t adds items t, t+256, ... (nit <= 64) then block_sum
        double v[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) v[q] = (tid < nit) ? __dadd_rn(0.0, sitem[q][tid]) : 0.0;
        block_sum<Q>(v, sred);
        const long long cg = ws.chunk_offset + chunk;
        if (tid == 0) {
#pragma unroll
            for (int q = 0; q < Q; ++q) ws.chunks[cg * NQ + q] = v[q];
        }
        if (ws.inline_final) {
            if (tid == 0) {
                __threadfence();
                const unsigned prev = atomicAdd(ws.final_cnt, 1u);
                s_last = (prev == (unsigned)(L.nch - 1));
                if (s_last) __threadfence();
            }
            __syncthreads();
            if (s_last) {          // the globally last chunk (necessarily this CTA's last)
                double f[Q];
                strided_sum<Q>(ws.chunks, ws.chunks_global, NQ, f, sred);
                if (tid == 0) {
                    double full[NQ] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                    for (int q = 0; q < Q; ++q) full[q] = f[q];
                    finalize(ws, cfg, phase, full);
                    *ws.final_cnt = 0u;
                    __threadfence();
                }
            }
        }
    }
    __syncthreads();
    }
}

// Tiny single-CTA kernel: level-4 fold of the (gathered) chunk table + epilogue.
__global__ void __launch_bounds__(NT) finalize_kernel(Ws ws, Cfg cfg, int phase, int pred, long long row) {
    __shared__ double sred[NQ * NWARP];
    if (!pred_ok(ws.head, pred, row)) return;
    double f[NQ];
    strided_sum<NQ>(ws.chunks, ws.chunks_global, NQ, f, sred);
    if (threadIdx.x == 0) finalize(ws, cfg, phase, f);
}

// Reference-order fold (KPL_ORDER_BLOCKED8): one warp, thread (q, lane) runs
// lane `lane` of _kernels.py:16-41 over products prod[q][lane + 8j] -- the
// same sequential chain a0 += u[k]*v[k] -- then the pairwise lane fold and
// the tail, and the epilogue of `phase` on the result.  The products were
// stored by the sweep that just ran (accp), so the values are bit-identical
// to the reference's blocked_dot of the same vectors.
__global__ void __launch_bounds__(32) blocked_final_kernel(Ws ws, Cfg cfg, int phase, int pred, long long row,
                                                           int nq) {
    __shared__ double lanes[NQ][8];
    __shared__ double tails[NQ];
    if (!pred_ok(ws.head, pred, row)) return;
    const int q = threadIdx.x >> 3, lane = threadIdx.x & 7;
    const long long n = ws.nprod, lim = n - n % 8;
    if (q < nq) {
        const double *p = ws.prod + q * n + lane;
        double a = 0.0;
        long long k = 0;
        constexpr int U = 16;
        for (; k + 8LL * U <= lim; k += 8LL * U) {
            double t[U];
#pragma unroll
            for (int j = 0; j < U; ++j) t[j] = __ldcg(p + k + 8LL * j);
#pragma unroll
            for (int j = 0; j < U; ++j) a = __dadd_rn(a, t[j]);
        }
        for (; k < lim; k += 8) a = __dadd_rn(a, __ldcg(p + k));
        lanes[q][lane] = a;
        if (lane == 0) {
            double t = 0.0;
            for (long long j = lim; j < n; ++j) t = __dadd_rn(t, __ldcg(ws.prod + q * n + j));
            tails[q] = t;
        }
    }
    __syncwarp();
    if (threadIdx.x == 0) {
        double v[NQ] = {0.0, 0.0, 0.0, 0.0};
        for (int i = 0; i < nq; ++i) {
            const double *l = lanes[i];
            v[i] = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(l[0], l[1]), __dadd_rn(l[2], l[3])),
                                       __dadd_rn(__dadd_rn(l[4], l[5]), __dadd_rn(l[6], l[7]))),
                             tails[i]);
        }
        finalize(ws, cfg, phase, v);
    }
}

}  // namespace kpl
