// kpl_spmv_band.cuh -- shared-memory-window SpMV for scattered banded matrices
// (kpl_op.bd_*; config 5: random columns within +-50,000 of the row).
//
// A CSR-order warp gather from global memory touches ~31 distinct cache lines
// and the L1 tag stage takes one line per cycle: config 5's 45.4 M gathers cost
// 170 us on their own (tools/gather_bench.cu), which bounds csr_spmv_pipe at
// ~231 us.  Shared memory has no tag stage.  Here one CTA owns a super-block of
// bd_rows rows and walks the super-block's column span in windows of W columns;
// each window's slice of the input vector is staged in shared memory by bulk
// copies (cp.async.bulk, double-buffered: window j+2 lands while window j+1 is
// used), and the gathers become shared-memory loads.
//
// Order of the sums: the running sum of every row of the super-block lives in
// shared memory.  The windows are visited in ascending column order and a row's
// nonzeros inside a window keep their CSR order, so every row is summed left to
// right from +0.0: csr_matvec (_kernels.py:44-52) bit for bit.
//
// Lane use: inside a window a row holds only ~2 of its ~23 nonzeros, with a wide
// spread (0..6), so a warp that takes 32 consecutive rows idles most lanes most
// steps (measured: 41 % lane use, the kernel bound by instruction issue).  The
// layout (device.py:band_layout) therefore sorts the rows of a pass by their
// length inside the window: a group's 32 slots hold rows of (nearly) equal
// length and are stored as L full steps of 32 entries -- lane l's k-th nonzero at
// entry 32 k + l, no index arithmetic beyond that, ~100 % lane use.  The price is
// the slot -> row indirection (2 bytes per row and pass) and the running sums in
// shared memory instead of registers.
//
// The matrix stream never touches the LSU's global path: with ~220 KB of the
// SM's 256 KB carved out as shared memory almost no L1 is left, and plain loads
// run out of L1 miss slots long before the DRAM rate (measured on the first
// form of this kernel: 17 of 32 warps on the long scoreboard, DRAM at 40 %).  A
// producer warp moves the stream with cp.async.bulk into a ring of shared-memory
// slots, one slot per "round" (32 groups).  A bulk copy occupies the SM's copy
// engine for ~0.3 us whatever its size (tools/bulk_stream_bench.cu: 8 KB copies
// stream at 21 GB/s per SM, 24 KB ones at 47), so a round is ONE record of the
// byte stream bd_stream -- group offsets, slot lengths, slot rows, columns, values
// -- and one copy; with five slices per round the stream was capped at 3 TB/s.
//
//   smem = | sums[rows] | window 0 [W] | window 1 [W] | ring[ns] | barriers |
//   slot = record = | grp[36] pad | len[1024] | row[1024] | col[cnt] | val[cnt] |   cnt <= cap
//   barriers: xfull[2] (input windows), full[ns] (1 arrival + bytes), empty[ns] (16 arrivals)
//
//   warp 16 (producer)                           warps 0..15 (consumers)
//   ------------------------------------        ---------------------------------------------------------
//   round boundaries 32 at a time (one per       per pass: wait the window; per round: wait full[slot],
//   lane); per round: wait empty[slot],          walk groups w and w + 16 (two independent chains),
//   expect_tx, 1 bulk copy                       arrive on empty[slot]; bar.sync among consumers, window j+2
#pragma once
#include "kpl_tma.cuh"

namespace kpl {

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// barrier among the consumer threads only (the producer warp does not take part)
__device__ __forceinline__ void consumer_sync(int nthreads) {
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

constexpr int BAND_HEAD = 160 + 1024 + 2048;       // record bytes before the entries

struct BandGeo {
    const unsigned char *stream;  // round records
    const int *roff;              // record r = bytes 16 roff[r] .. 16 roff[r+1]
    const int4 *sb;           // {first pass, passes, -, -}
    const int *win;           // first column of every pass (even)
    int W, rows;
};

struct BandRing {
    int cap, ns;
    __host__ __device__ size_t slot() const { return 10 * (size_t)cap + BAND_HEAD; }
    __host__ __device__ size_t bytes(int rows, int W) const {
        return 8 * (size_t)rows + 16 * (size_t)W + ns * slot() + 8 * (2 + 2 * (size_t)ns);
    }
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

template <class In>
__global__ void __launch_bounds__(BAND_CW * 32 + 32, 1)
csr_band_ring_spmv(long long n, BandGeo B, BandRing R, In in, double *__restrict__ out, Ws ws, int pred,
                   long long row) {
    constexpr int NC = BAND_CW * 32;
    extern __shared__ __align__(128) unsigned char smem[];
    const int RB = B.rows, RP = (RB + 1023) >> 10;     // rows, rounds per pass
    double *sums = reinterpret_cast<double *>(smem);
    double *xs0 = sums + RB;
    double *xs1 = xs0 + B.W;
    unsigned char *ring = reinterpret_cast<unsigned char *>(xs1 + B.W);
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
    for (int t = tid; t < RB; t += NC + 32) sums[t] = 0.0;      // +0.0: the reference's accumulator
    __syncthreads();

    if (warp == BAND_CW) {
        // ------------------------------------------------------------ producer
        const int nq = npass * RP;                     // rounds of this super-block
        const long long r0 = (long long)pass0 * RP;    // its first round
        int s = 0, wrap = 0;
        for (int qb = 0; qb < nq; qb += 32) {
            // record bounds of the next 32 rounds, one per lane
            const int q = min(qb + lane, nq - 1);
            const int ob = __ldg(B.roff + r0 + q), oe = __ldg(B.roff + r0 + q + 1);
            const int m = min(32, nq - qb);
            for (int l = 0; l < m; ++l) {
                const int o0 = __shfl_sync(0xffffffffu, ob, l), o1 = __shfl_sync(0xffffffffu, oe, l);
                if (lane == 0) {
                    if (wrap) mbar_wait_sleep(&empty[s], (unsigned)((wrap - 1) & 1));
                    const unsigned bytes = (unsigned)(o1 - o0) * 16u;
                    mbar_expect_tx(&full[s], bytes);
                    bulk_g2s(ring + s * SLOT, B.stream + 16LL * o0, bytes, &full[s]);
                }
                if (++s == R.ns) { s = 0; ++wrap; }
            }
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    // window j -> buffer j & 1; an odd tail element goes in with a plain store
    // (made visible by the release of the expect_tx arrive that follows it)
    auto issue = [&](int j) {
        double *dst = (j & 1) ? xs1 : xs0;
        const long long w0 = __ldg(B.win + pass0 + j);
        const long long len = min((long long)B.W, n - w0);
        if (len & 1) dst[len - 1] = x[w0 + len - 1];
        const unsigned bytes = (unsigned)((len & ~1LL) * 8);
        mbar_expect_tx(&xfull[j & 1], bytes);
        for (unsigned o = 0; o < bytes; o += 65536u)          // few, large copies (see above)
            bulk_g2s(reinterpret_cast<unsigned char *>(dst) + o, reinterpret_cast<const unsigned char *>(x + w0) + o,
                     min(65536u, bytes - o), &xfull[j & 1]);
    };
    if (tid == 0) {
        issue(0);
        if (npass > 1) issue(1);
    }
    int s = 0;
    unsigned ph = 0;
    for (int j = 0; j < npass; ++j) {
        mbar_wait_sleep(&xfull[j & 1], (unsigned)((j >> 1) & 1));
        const double *xs = (j & 1) ? xs1 : xs0;
        for (int i = 0; i < RP; ++i) {
            mbar_wait_sleep(&full[s], ph);
            const unsigned char *slot = ring + s * SLOT;
            const int *sgrp = reinterpret_cast<const int *>(slot);
            const unsigned char *slen = slot + 160;
            const unsigned short *srow = reinterpret_cast<const unsigned short *>(slot + 160 + 1024);
            const unsigned short *scol = reinterpret_cast<const unsigned short *>(slot + BAND_HEAD);
            const int e0 = sgrp[0];
            const double *sval = reinterpret_cast<const double *>(slot + BAND_HEAD + 2 * (size_t)(sgrp[32] - e0));
            // groups w and w + 16 of the round: two independent chains, interleaved.  Lane 0 holds
            // the group's longest row, lane 31 its shortest.
            const unsigned la = slen[tid], lb = slen[NC + tid];
            const unsigned ra_i = srow[tid], rb_i = srow[NC + tid];
            const double *pa = sval + (sgrp[warp] - e0) + lane, *pb = sval + (sgrp[warp + BAND_CW] - e0) + lane;
            const unsigned short *ca = scol + (sgrp[warp] - e0) + lane, *cb = scol + (sgrp[warp + BAND_CW] - e0) + lane;
            const unsigned maxa = __shfl_sync(0xffffffffu, la, 0), maxb = __shfl_sync(0xffffffffu, lb, 0);
            const unsigned mina = __shfl_sync(0xffffffffu, la, 31), minb = __shfl_sync(0xffffffffu, lb, 31);
            double ra = la ? sums[ra_i] : 0.0, rb = lb ? sums[rb_i] : 0.0;
            const unsigned both = min(mina, minb);
            unsigned k = 0;
            for (; k < both; ++k) {                    // steps every lane of both groups takes
                const double va = pa[32 * k], vb = pb[32 * k];
                const unsigned xa = ca[32 * k], xb = cb[32 * k];
                ra = __dadd_rn(ra, __dmul_rn(va, in.xf(xs[xa], 0)));                    // csr_matvec order
                rb = __dadd_rn(rb, __dmul_rn(vb, in.xf(xs[xb], 0)));
            }
            for (; k < maxa; ++k) {                    // the rest: zero-filled entries are read and dropped
                const double t = __dadd_rn(ra, __dmul_rn(pa[32 * k], in.xf(xs[ca[32 * k]], 0)));
                ra = k < la ? t : ra;
            }
            for (k = both; k < maxb; ++k) {
                const double t = __dadd_rn(rb, __dmul_rn(pb[32 * k], in.xf(xs[cb[32 * k]], 0)));
                rb = k < lb ? t : rb;
            }
            if (la) sums[ra_i] = ra;
            if (lb) sums[rb_i] = rb;
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == R.ns) { s = 0; ph ^= 1; }
        }
        consumer_sync(NC);                          // every consumer warp is done with window buffer j & 1
        if (tid == 0 && j + 2 < npass) issue(j + 2);
    }
    const long long row0 = (long long)blockIdx.x * RB;
    for (int t = tid; t < RB; t += NC) {
        const long long r = row0 + t;
        if (r < n) out[r] = sums[t];
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
