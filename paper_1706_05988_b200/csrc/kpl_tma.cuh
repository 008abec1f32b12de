// kpl_tma.cuh -- TMA-fed, warp-specialised version of the fused p-CG-sh
// stencil sweep (3D grids, 2 elements per thread, tile 64 x 8).
//
// Same traversal, element mapping and reduction order as stencil_sweep<2>
// (so results are bit-identical), but the operands arrive in shared memory
// through cp.async.bulk.tensor (TMA) instead of per-thread loads:
//
//   warp 8 (producer, one elected lane)     warps 0..7 (consumers, one tile row each)
//   ---------------------------------       -----------------------------------------
//   for each plane of the chunk:            for each plane z:
//     wait empty[slot]                        wait full[w slot of z+1], full[stream slot of z]
//     expect_tx + TMA w box (68x10)           7-point stencil from the w ring (z-1, z, z+1)
//     expect_tx + TMA 5 stream boxes (64x8)   9 recurrences, stores to HBM (st.global.cs)
//                                             arrive empty[...] (slot free)
//
// The w ring holds SW = D+3 planes (stencil needs z-1..z+1, D planes ahead);
// the stream ring SS = D+1 stages.  Dirichlet ghosts (x,y,z out of range) are
// the TMA out-of-bounds zero fill, so the consumer has no boundary logic.
// With D = 2 and the 5 streams of the p-CG-sh update: 5 x 5.4 KB + 3 x 20 KB
// ~ 89 KB smem per CTA, 2 CTAs per SM,
// ~100 KB of loads in flight per SM (vs ~49 KB for the register-prefetch sweep).
#pragma once
#include <cuda.h>
#include "kpl_bodies.cuh"
#include "kpl_sweep.cuh"

namespace kpl {

struct TmaMaps {
    CUtensorMap w[2];      // ping-pong stencil input, box (68, 10, 1) at (x0-2, y0-1, z)
    CUtensorMap s[5];      // x, r, z, s, t: box (64, 8, 1) at (x0, y0, z)
};

constexpr int TMA_TX = 64, TMA_TY = 8;
constexpr int TMA_WX = TMA_TX + 4, TMA_WY = TMA_TY + 2;       // 68 x 10
constexpr int TMA_WPLANE = 688;                               // 68*10 = 680 doubles, padded to 128 B
constexpr int TMA_SPLANE = TMA_TX * TMA_TY;                   // 512 doubles
constexpr int TMA_NS = 5;
constexpr unsigned TMA_WBYTES = TMA_WX * TMA_WY * 8;          // 5440
constexpr unsigned TMA_SBYTES = TMA_NS * TMA_SPLANE * 8;      // 20480

__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long *b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *b, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load3d(void *dst, const CUtensorMap *map, int c0, int c1, int c2,
                                           unsigned long long *bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

template <int D, int NSTR>
struct TmaRing {
    static constexpr int SW = D + 3, SS = D + 1;
    static constexpr size_t bytes() {
        return (size_t)SW * TMA_WPLANE * 8 + (size_t)SS * NSTR * TMA_SPLANE * 8 + 8 * 2 * (SW + SS);
    }
};

// Generic over bodies that declare kTmaStreams (<= 5) and load_tma(); the
// stencil input ring is maps.w[wsel ? iter & 1 : 0].  Identity preconditioner
// only (the stencil input is used raw).
template <class Body, int D>
__global__ void __launch_bounds__(NT + 32, 2)
tma_sweep(const __grid_constant__ TmaMaps maps, SGeo g, Layout L, Body body, Ws ws, Cfg cfg, int phase,
          int pred, long long row, int wsel, int wzoff) {
    constexpr int NSTR = Body::kTmaStreams;
    constexpr int SW = TmaRing<D, NSTR>::SW, SS = TmaRing<D, NSTR>::SS;
    constexpr int Q = Body::NQ > 0 ? Body::NQ : 1;
    constexpr unsigned SBYTES = NSTR * TMA_SPLANE * 8;
    extern __shared__ __align__(128) unsigned char smem[];
    double *wring = reinterpret_cast<double *>(smem);
    double *sring = wring + SW * TMA_WPLANE;
    unsigned long long *wfull = reinterpret_cast<unsigned long long *>(sring + SS * NSTR * TMA_SPLANE);
    unsigned long long *sfull = wfull + SW;
    unsigned long long *wempty = sfull + SS;
    unsigned long long *sempty = wempty + SW;
    __shared__ double sred[NQ * NWARP];

    if (!pred_ok(ws.head, pred, row)) return;
    body.setup(ws);
    const long long par = wsel ? (ws.head->iter & 1) : 0;    // w_in = w[iter & 1] (ping-pong) or fixed

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long item = blockIdx.x;
    const long long c = item / L.T;
    const int tile = (int)(item - c * L.T);
    const int tyi = tile / L.ntx, txi = tile - tyi * L.ntx;
    const int x0 = txi * TMA_TX, y0 = tyi * TMA_TY;
    const int z0 = (int)(c * L.zc);
    const int z1 = (int)min((long long)z0 + L.zc, g.NZ);
    const int ns = z1 - z0;            // planes computed
    const int nw = ns + 2;             // w planes z0-1 .. z1

    if (tid == 0) {
        for (int j = 0; j < SW; ++j) { mbar_init(&wfull[j], 1); mbar_init(&wempty[j], NWARP); }
        for (int j = 0; j < SS; ++j) { mbar_init(&sfull[j], 1); mbar_init(&sempty[j], NWARP); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    double acc[Q][2];
#pragma unroll
    for (int q = 0; q < Q; ++q) acc[q][0] = acc[q][1] = 0.0;

    if (warp == NWARP) {
        // ------------------------------------------------------ producer
        if (lane == 0) {
            const CUtensorMap *wm = par ? &maps.w[1] : &maps.w[0];
            int p = 0, q = 0;
            while (p < nw || q < ns) {
                if (p < nw && (p <= q + 2 || q >= ns)) {
                    const int slot = p % SW;
                    if (p >= SW) mbar_wait(&wempty[slot], ((p / SW) - 1) & 1);
                    mbar_expect_tx(&wfull[slot], TMA_WBYTES);
                    tma_load3d(wring + slot * TMA_WPLANE, wm, x0 - 2, y0 - 1, z0 - 1 + p + wzoff, &wfull[slot]);
                    ++p;
                } else {
                    const int slot = q % SS;
                    if (q >= SS) mbar_wait(&sempty[slot], ((q / SS) - 1) & 1);
                    mbar_expect_tx(&sfull[slot], SBYTES);
#pragma unroll
                    for (int s = 0; s < NSTR; ++s)
                        tma_load3d(sring + (slot * NSTR + s) * TMA_SPLANE, &maps.s[s], x0, y0, z0 + q,
                                   &sfull[slot]);
                    ++q;
                }
            }
        }
    } else {
        // ------------------------------------------------------ consumers
        const int wy = warp;
        const int xl = 2 * lane;
        const long long x = x0 + xl, y = y0 + wy;
        const bool ok = (y < g.NY) && (x < g.NX);
        const long long NX = g.NX, sxy = g.NX * g.NY;
        const int cw = (wy + 1) * TMA_WX + 2 + xl;           // own pair in a w plane
        const int cs = wy * TMA_TX + xl;                     // own pair in a stream plane
        mbar_wait(&wfull[0], 0);
        mbar_wait(&wfull[1 % SW], (1 / SW) & 1);
        for (int k = 0; k < ns; ++k) {
            const int z = z0 + k;
            const int pz = k + 2;                            // w plane z+1
            mbar_wait(&wfull[pz % SW], (pz / SW) & 1);
            mbar_wait(&sfull[k % SS], (k / SS) & 1);
            const double *Wm = wring + (k % SW) * TMA_WPLANE;
            const double *Wc = wring + ((k + 1) % SW) * TMA_WPLANE;
            const double *Wp = wring + (pz % SW) * TMA_WPLANE;
            const double *Sp = sring + (k % SS) * NSTR * TMA_SPLANE;
            if (ok) {
                const double2 qm = *reinterpret_cast<const double2 *>(Wm + cw);
                const double2 qc = *reinterpret_cast<const double2 *>(Wc + cw);
                const double2 qp = *reinterpret_cast<const double2 *>(Wp + cw);
                const double2 ym = *reinterpret_cast<const double2 *>(Wc + cw - TMA_WX);
                const double2 yp = *reinterpret_cast<const double2 *>(Wc + cw + TMA_WX);
                const double xm0 = Wc[cw - 1], xp1 = Wc[cw + 2];
                typename Body::template Regs<2> R;
                body.load_tma(Sp, cs, R);
                // 7-point stencil, terms in ascending column order (as csr_matvec)
                const double zmv[2] = {qm.x, qm.y}, ymv[2] = {ym.x, ym.y}, xmv[2] = {xm0, qc.x};
                const double cv[2] = {qc.x, qc.y}, xpv[2] = {qc.y, xp1}, ypv[2] = {yp.x, yp.y},
                             zpv[2] = {qp.x, qp.y};
                double n[2];
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    double a = 0.0;
                    a = __dadd_rn(a, -zmv[v]);
                    a = __dadd_rn(a, -ymv[v]);
                    a = __dadd_rn(a, -xmv[v]);
                    a = __dadd_rn(a, __dmul_rn(g.diag, cv[v]));
                    a = __dadd_rn(a, -xpv[v]);
                    a = __dadd_rn(a, -ypv[v]);
                    a = __dadd_rn(a, -zpv[v]);
                    n[v] = a;
                }
                const long long kk = (long long)z * sxy + x + NX * y;
                body.template compute<2>(kk, R, n, cv, acc);
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&wempty[k % SW]);     // plane z-1 is dead after this step
                mbar_arrive(&sempty[k % SS]);
            }
        }
    }

    if constexpr (Body::NQ > 0) {
        double t[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) t[q] = __dadd_rn(acc[q][0], acc[q][1]);
        block_sum<Q>(t, sred);
        if (tid == 0) {
#pragma unroll
            for (int q = 0; q < Q; ++q) ws.items[item * NQ + q] = t[q];
        }
        complete_item<Q>(ws, cfg, L, phase, c, sred);
    }
}

}  // namespace kpl
