// kpl_spmv_band.cuh -- shared-memory-window SpMV for scattered banded matrices
// (kpl_op.bd_*; config 5: random columns within +-50,000 of the row).
//
// A CSR-order warp gather from global memory touches ~31 distinct cache lines
// and the L1 tag stage takes one line per cycle: config 5's 45.4 M gathers cost
// 170 us on their own (tools/gather_bench.cu), which bounds csr_spmv_pipe at
// ~237 us.  Shared memory has no tag stage.  Here one CTA owns a super-block of
// RPT*1024 rows and walks the super-block's column span in windows of W columns;
// each window's slice of the input vector is staged in shared memory by bulk
// copies (cp.async.bulk, double-buffered: window j+2 lands while window j+1 is
// used), and the gathers become shared-memory loads.
//
// Order of the sums: thread t keeps the accumulators of rows t, t+1024, ... in
// registers across the passes.  The windows are visited in ascending column
// order and a row's nonzeros inside a window keep their CSR order, so every row
// is summed left to right from +0.0: csr_matvec (_kernels.py:44-52) bit for bit.
//
// Stream layout (built once per matrix, device.py:band_layout): inside a
// (pass, 32-row group) the nonzeros are stored in jagged-diagonal order -- step
// k of every row that has a k-th nonzero in the window, in lane order -- so the
// lanes that take step k read consecutive entries (coalesced), each its own
// row's next nonzero; the position comes from a ballot over the row lengths.
// 10 bytes per nonzero (fp64 value + uint16 window-relative column) + 1 byte
// per (row, pass) against CSR's 12.
#pragma once
#include "kpl_spmv_tma.cuh"

namespace kpl {

struct BandGeo {
    const double *val;
    const unsigned short *col;
    const unsigned char *len;
    const int *grp;
    const int4 *sb;           // {first pass, passes, first column (even), -}
    int W;
};

template <class In, int RPT, int UN>
__global__ void __launch_bounds__(1024, 1)
csr_band_spmv(long long n, BandGeo B, In in, double *__restrict__ out, Ws ws, int pred, long long row) {
    constexpr int RBS = RPT * 1024, G = RBS / 32;
    extern __shared__ __align__(128) unsigned char smem[];
    double *xs0 = reinterpret_cast<double *>(smem);
    double *xs1 = xs0 + B.W;
    unsigned long long *full = reinterpret_cast<unsigned long long *>(smem + 16 * (size_t)B.W);
    pdl_wait();
    pdl_launch_dependents();
    if (ws.head && !pred_ok(ws.head, pred, row)) return;
    if (ws.head) in.setup(ws);
    const double *x = in.base();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const unsigned ltmask = (1u << lane) - 1u;
    const int4 info = __ldg(B.sb + blockIdx.x);
    const int pass0 = info.x, npass = info.y;
    const long long row0 = (long long)blockIdx.x * RBS;
    if (tid == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // window j -> buffer j & 1; an odd tail element goes in with a plain store
    // (made visible by the release of the expect_tx arrive that follows it)
    auto issue = [&](int j) {
        double *dst = (j & 1) ? xs1 : xs0;
        const long long w0 = info.z + (long long)j * B.W;
        const long long len = min((long long)B.W, n - w0);
        if (len & 1) dst[len - 1] = x[w0 + len - 1];
        const unsigned bytes = (unsigned)((len & ~1LL) * 8);
        mbar_expect_tx(&full[j & 1], bytes);
        for (unsigned o = 0; o < bytes; o += 32768u)
            bulk_g2s(reinterpret_cast<unsigned char *>(dst) + o, reinterpret_cast<const unsigned char *>(x + w0) + o,
                     min(32768u, bytes - o), &full[j & 1]);
    };
    if (tid == 0) {
        issue(0);
        if (npass > 1) issue(1);
    }
    double acc[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) acc[i] = 0.0;
    for (int j = 0; j < npass; ++j) {
        const long long p = pass0 + j;
        unsigned L[RPT];
        int gb[RPT];
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            L[i] = __ldg(B.len + p * RBS + i * 1024 + tid);
            gb[i] = __ldg(B.grp + p * G + i * 32 + warp);
        }
        mbar_wait(&full[j & 1], (unsigned)((j >> 1) & 1));
        const double *xs = (j & 1) ? xs1 : xs0;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            const unsigned len = L[i];
            const unsigned maxl = __reduce_max_sync(0xffffffffu, len);
            int base = gb[i];
            for (unsigned k = 0; k < maxl; k += UN) {
                double v[UN];
                int c[UN];
                bool act[UN];
#pragma unroll
                for (int u = 0; u < UN; ++u) {
                    act[u] = len > k + u;
                    const unsigned m = __ballot_sync(0xffffffffu, act[u]);
                    const int idx = base + __popc(m & ltmask);
                    base += __popc(m);
                    v[u] = 0.0;
                    c[u] = 0;
                    if (act[u]) {
                        v[u] = __ldcs(B.val + idx);
                        c[u] = __ldcs(B.col + idx);
                    }
                }
                double xv[UN];
#pragma unroll
                for (int u = 0; u < UN; ++u) xv[u] = xs[c[u]];
#pragma unroll
                for (int u = 0; u < UN; ++u)
                    if (act[u]) acc[i] = __dadd_rn(acc[i], __dmul_rn(v[u], in.xf(xv[u], 0)));   // csr_matvec order
            }
        }
        __syncthreads();                        // every warp is done with buffer j & 1
        if (tid == 0 && j + 2 < npass) issue(j + 2);
    }
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
        const long long r = row0 + i * 1024 + tid;
        if (r < n) out[r] = acc[i];
    }
}

// ---------------------------------------------------------------------------
// Ring-fed form.  With ~224 KB of the SM's 256 KB carved out as shared memory
// almost no L1 is left, and the value/column stream of csr_band_spmv (plain
// loads) runs out of L1 miss slots long before it reaches the DRAM rate: the
// kernel is latency-bound (ncu: 17 of 32 warps on the long scoreboard, DRAM at
// 40 %).  Here the stream never touches the LSU's global path: a producer warp
// moves it with cp.async.bulk into a ring of shared-memory slots, one slot per
// "round" (32 consecutive groups of a pass: their values, columns, row lengths
// and group offsets -- four contiguous slices of the bd_* arrays), and the 16
// consumer warps (two groups of a round each) read values, columns and the
// input window from shared memory only.  Same walk, same sums: bit-identical
// to csr_band_spmv.
//
//   slot = | val[cap] | col[cap] | len[1024] | grp[36] |     cap % 64 == 0
//   barriers: xfull[2] (input windows), full[ns] (1 arrival + bytes), empty[ns] (16 arrivals)
//
//   warp 16 (producer)                           warps 0..15 (consumers), thread t: rows t + 512 h + 1024 i
//   ------------------------------------        ---------------------------------------------------------
//   round boundaries 32 at a time (one per       per pass: wait the window; per round: wait full[slot],
//   lane); per round: wait empty[slot],          walk groups w and w + 16 (two independent chains),
//   expect_tx, 4 bulk copies                     arrive on empty[slot]; bar.sync among consumers, window j+2
//
// (A CTA cannot exceed 1024 threads.  Measured alternatives on config 5: all 32
// warps consuming with the producer role rotating among them -- every round then
// waits for the slowest warp, 0.51 ms/iteration -- or with warp 0 feeding the
// ring between its own groups without blocking -- fills lag, 0.37; this form: 0.27.)
struct BandRing {
    int cap, ns;
    __host__ __device__ size_t slot() const { return 10 * (size_t)cap + 1024 + 144; }
    __host__ __device__ size_t bytes(int W) const { return 16 * (size_t)W + ns * slot() + 8 * (2 + 2 * (size_t)ns); }
};

// try_wait with a suspend-time hint: a waiting warp sleeps instead of spinning on the barrier word
__device__ __forceinline__ void mbar_wait_sleep(unsigned long long *b, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAITS_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra WAITS_%=;\n"
        "}\n" ::"r"(smem_u32(b)),
        "r"(parity), "r"(2000u)
        : "memory");
}

constexpr int BAND_CW = 16;                        // consumer warps

template <class In, int RPT>
__global__ void __launch_bounds__(BAND_CW * 32 + 32, 1)
csr_band_ring_spmv(long long n, BandGeo B, BandRing R, In in, double *__restrict__ out, Ws ws, int pred,
                   long long row) {
    constexpr int RBS = RPT * 1024, G = RBS / 32, NC = BAND_CW * 32;
    extern __shared__ __align__(128) unsigned char smem[];
    double *xs0 = reinterpret_cast<double *>(smem);
    double *xs1 = xs0 + B.W;
    unsigned char *ring = smem + 16 * (size_t)B.W;
    const size_t SLOT = R.slot();
    unsigned long long *xfull = reinterpret_cast<unsigned long long *>(ring + R.ns * SLOT);
    unsigned long long *full = xfull + 2;
    unsigned long long *empty = full + R.ns;
    pdl_wait();
    pdl_launch_dependents();
    if (ws.head && !pred_ok(ws.head, pred, row)) return;
    if (ws.head) in.setup(ws);
    const double *x = in.base();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int4 info = __ldg(B.sb + blockIdx.x);
    const int pass0 = info.x, npass = info.y;
    if (tid == 0) {
        mbar_init(&xfull[0], 1);
        mbar_init(&xfull[1], 1);
        for (int s = 0; s < R.ns; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], BAND_CW); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == BAND_CW) {
        // ------------------------------------------------------------ producer
        const int nq = npass * RPT;                    // rounds of this super-block
        const long long g0 = (long long)pass0 * G;     // its first group
        int s = 0, wrap = 0;
        for (int qb = 0; qb < nq; qb += 32) {
            // round boundaries of the next 32 rounds, one per lane
            const int q = min(qb + lane, nq - 1);
            const int eb = __ldg(B.grp + g0 + 32LL * q), ee = __ldg(B.grp + g0 + 32LL * q + 32);
            const int m = min(32, nq - qb);
            for (int l = 0; l < m; ++l) {
                const int e0 = __shfl_sync(0xffffffffu, eb, l), e1 = __shfl_sync(0xffffffffu, ee, l);
                if (lane == 0) {
                    if (wrap) mbar_wait_sleep(&empty[s], (unsigned)((wrap - 1) & 1));
                    unsigned char *slot = ring + s * SLOT;
                    const long long a0 = e0 & ~7, a1 = ((long long)e1 + 7) & ~7LL;   // 16-byte bounds of both streams
                    const unsigned cnt = (unsigned)(a1 - a0);
                    const long long gq = g0 + 32LL * (qb + l);
                    mbar_expect_tx(&full[s], cnt * 10u + 1024u + 144u);
                    if (cnt) {
                        bulk_g2s(slot, B.val + a0, cnt * 8u, &full[s]);
                        bulk_g2s(slot + 8 * (size_t)R.cap, B.col + a0, cnt * 2u, &full[s]);
                    }
                    bulk_g2s(slot + 10 * (size_t)R.cap, B.len + gq * 32, 1024u, &full[s]);
                    bulk_g2s(slot + 10 * (size_t)R.cap + 1024, B.grp + gq, 144u, &full[s]);
                }
                if (++s == R.ns) { s = 0; ++wrap; }
            }
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    const unsigned ltmask = (1u << lane) - 1u;
    const long long row0 = (long long)blockIdx.x * RBS;
    auto issue = [&](int j) {
        double *dst = (j & 1) ? xs1 : xs0;
        const long long w0 = info.z + (long long)j * B.W;
        const long long len = min((long long)B.W, n - w0);
        if (len & 1) dst[len - 1] = x[w0 + len - 1];
        const unsigned bytes = (unsigned)((len & ~1LL) * 8);
        mbar_expect_tx(&xfull[j & 1], bytes);
        for (unsigned o = 0; o < bytes; o += 32768u)
            bulk_g2s(reinterpret_cast<unsigned char *>(dst) + o, reinterpret_cast<const unsigned char *>(x + w0) + o,
                     min(32768u, bytes - o), &xfull[j & 1]);
    };
    if (tid == 0) {
        issue(0);
        if (npass > 1) issue(1);
    }
    double acc[RPT][2];
#pragma unroll
    for (int i = 0; i < RPT; ++i) acc[i][0] = acc[i][1] = 0.0;
    int s = 0;
    unsigned ph = 0;
    for (int j = 0; j < npass; ++j) {
        mbar_wait_sleep(&xfull[j & 1], (unsigned)((j >> 1) & 1));
        const double *xs = (j & 1) ? xs1 : xs0;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            mbar_wait_sleep(&full[s], ph);
            const unsigned char *slot = ring + s * SLOT;
            const double *sval = reinterpret_cast<const double *>(slot);
            const unsigned short *scol = reinterpret_cast<const unsigned short *>(slot + 8 * (size_t)R.cap);
            const int *sgrp = reinterpret_cast<const int *>(slot + 10 * (size_t)R.cap + 1024);
            const int e0 = sgrp[0] & ~7;
            // groups w and w + 16 of the round: two independent chains, interleaved
            const unsigned la = slot[10 * (size_t)R.cap + tid], lb = slot[10 * (size_t)R.cap + NC + tid];
            int ba = sgrp[warp] - e0, bb = sgrp[warp + BAND_CW] - e0;
            const unsigned maxl = __reduce_max_sync(0xffffffffu, max(la, lb));
            double ra = acc[i][0], rb = acc[i][1];
            // branch-free steps: a lane whose row has no k-th nonzero reads entry 0 / column 0
            // (broadcast reads) and keeps its sum
            for (unsigned k = 0; k < maxl; ++k) {
                const bool pa = la > k, pb = lb > k;
                const unsigned ma = __ballot_sync(0xffffffffu, pa), mb = __ballot_sync(0xffffffffu, pb);
                const int ia = pa ? ba + __popc(ma & ltmask) : 0, ib = pb ? bb + __popc(mb & ltmask) : 0;
                ba += __popc(ma);
                bb += __popc(mb);
                const double va = sval[ia], vb = sval[ib];
                const unsigned ca = pa ? scol[ia] : 0u, cb = pb ? scol[ib] : 0u;
                const double ta = __dadd_rn(ra, __dmul_rn(va, in.xf(xs[ca], 0)));       // csr_matvec order
                const double tb = __dadd_rn(rb, __dmul_rn(vb, in.xf(xs[cb], 0)));
                ra = pa ? ta : ra;
                rb = pb ? tb : rb;
            }
            acc[i][0] = ra;
            acc[i][1] = rb;
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == R.ns) { s = 0; ph ^= 1; }
        }
        consumer_sync(NC);                          // every consumer warp is done with window buffer j & 1
        if (tid == 0 && j + 2 < npass) issue(j + 2);
    }
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const long long r = row0 + i * 1024 + h * NC + tid;
            if (r < n) out[r] = acc[i][h];
        }
    }
}

// ---------------------------------------------------------------------------
// Reference-order fold (KPL_ORDER_BLOCKED8) for large n: blocked_final_kernel's
// chain -- lane l of quantity q adds prod[q][l + 8 j] for j = 0, 1, ... -- fed
// from shared memory.  One warp reading 4 GiB straight from HBM with 16 loads in
// flight per thread is bound by memory latency (~0.7 s per fold at 512^3); here
// a producer thread streams the product arrays through a ring of bulk copies
// and the 32 chain threads only see shared-memory latency, so the fold runs at
// the speed of its dependent fp64 adds.  Same chain, same bits.
constexpr int BF_T = 2048;                         // elements per quantity per stage
constexpr int BF_NS = 3;                           // stages
constexpr int BF_QS = BF_T + 8;                    // quantity stride (64 bytes of padding: bank spread)
constexpr size_t BF_SMEM = sizeof(double) * BF_NS * NQ * BF_QS + 16 * BF_NS;

__global__ void __launch_bounds__(64) blocked_final_tma_kernel(Ws ws, Cfg cfg, int phase, int pred, long long row,
                                                               int nq) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ double lanes[NQ][8];
    __shared__ double tails[NQ];
    double *stage = reinterpret_cast<double *>(smem);
    unsigned long long *full = reinterpret_cast<unsigned long long *>(smem + sizeof(double) * BF_NS * NQ * BF_QS);
    unsigned long long *empty = full + BF_NS;
    if (!pred_ok(ws.head, pred, row)) return;
    const long long n = ws.nprod, lim = n - n % 8;
    const long long nst = (lim + BF_T - 1) / BF_T;
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < BF_NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid >= 32) {
        if (tid == 32) {
            for (long long st = 0; st < nst; ++st) {
                const int s = (int)(st % BF_NS);
                if (st >= BF_NS) mbar_wait(&empty[s], (unsigned)(((st / BF_NS) - 1) & 1));
                const unsigned m = (unsigned)min((long long)BF_T, lim - st * BF_T);
                mbar_expect_tx(&full[s], (unsigned)nq * m * 8u);
                for (int q = 0; q < nq; ++q)
                    bulk_g2s(stage + ((size_t)s * NQ + q) * BF_QS, ws.prod + q * n + st * BF_T, m * 8u, &full[s]);
            }
        }
        return;
    }
    const int q = tid >> 3, lane = tid & 7;
    double a = 0.0;
    for (long long st = 0; st < nst; ++st) {
        const int s = (int)(st % BF_NS);
        mbar_wait(&full[s], (unsigned)((st / BF_NS) & 1));
        if (q < nq) {
            const double *p = stage + ((size_t)s * NQ + q) * BF_QS + lane;
            const int m = (int)min((long long)BF_T, lim - st * BF_T);
            constexpr int U = 16;
            int k = 0;
            for (; k + 8 * U <= m; k += 8 * U) {
                double t[U];
#pragma unroll
                for (int j = 0; j < U; ++j) t[j] = p[k + 8 * j];
#pragma unroll
                for (int j = 0; j < U; ++j) a = __dadd_rn(a, t[j]);
            }
            for (; k < m; k += 8) a = __dadd_rn(a, p[k]);
        }
        __syncwarp();
        if (tid == 0) mbar_arrive(&empty[s]);
    }
    if (q < nq) {
        lanes[q][lane] = a;
        if (lane == 0) {
            double t = 0.0;
            for (long long j = lim; j < n; ++j) t = __dadd_rn(t, __ldcg(ws.prod + q * n + j));
            tails[q] = t;
        }
    }
    __syncwarp();
    if (tid == 0) {
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

// Classic CG with the window SpMV: p_new = axpy(beta, p_old, u) (solvers.py:269) written
// out first, so the SpMV reads a plain vector (the CSR-order kernels evaluate it per
// gathered column instead: two gathers per nonzero).  Same expression as InCgP::raw,
// and csr_chunk_sweep's BodyCgP stores the same values again.
__global__ void __launch_bounds__(256) cg_p_materialise_kernel(long long n, InCgP in, double *p0, double *p1, Ws ws,
                                                               int pred, long long row) {
    pdl_wait();
    pdl_launch_dependents();
    if (!pred_ok(ws.head, pred, row)) return;
    in.setup(ws);
    double *pout = const_cast<double *>(pick(ws.head, SEL_ITER1, p0, p1));
    for (long long k = blockIdx.x * 256LL + threadIdx.x; k < n; k += 256LL * gridDim.x) {
        double o[1];
        in.template raw<1>(in.base(), k, o);
        pout[k] = o[0];
    }
}

}  // namespace kpl
