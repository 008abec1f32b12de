// kpl_spmv_tma.cuh -- column-sorted CSR SpMV fed by bulk TMA copies.
//
// For scattered matrices (config 5: every CSR-order warp gather touches ~31
// cache lines) the SpMV is bound by the L1 miss requests one SM can keep in
// flight.  The column-sorted layout (kpl_op.sp_*) cuts a warp gather to ~9
// lines (tools/gather_bench.cu: 170 -> 60 us for config 5's 45.4 M gathers),
// but only if the gathers are not queued behind DRAM-latency loads: the LSU
// returns loads in issue order, so the matrix stream (col, val, dest: 14 B per
// nonzero, DRAM-resident) must not share that FIFO.  Here the stream arrives
// through cp.async.bulk (the TMA engine) into a shared-memory ring, and the
// LSU carries only the L2-resident gathers:
//
//   warp NC/32 (producer, one lane)          warps 0..NC/32-1 (consumers)
//   ------------------------------           -------------------------------------------
//   per block, per chunk of CH nonzeros:     per chunk: wait full, read (col, val, dest)
//     wait empty[slot], expect_tx,             into registers, release the slot, issue the
//     3 bulk copies (val, col, dest)           gathers; then multiply the PREVIOUS chunk's
//                                              gathers and store the products at their CSR
//                                              positions in shared memory (one chunk of lag)
//                                            block complete: row sums in CSR order from
//                                              shared memory (csr_matvec order, bitwise)
//
// Each CTA owns a contiguous range of row blocks (one CTA per SM).  Chunks are
// aligned to 8 nonzeros (16-byte bulk copies); the sp_* arrays carry 8 padding
// entries so the last chunk may over-read.
#pragma once
#include "kpl_tma.cuh"

namespace kpl {

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void consumer_sync(int nthreads) {
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

template <int CH, int NS>
struct SpRing {
    static constexpr int STAGE = CH * (8 + 4 + 2);                    // val | col | dest
    static constexpr int BARS = 2 * NS * 8;
    static constexpr int PROD_OFF = ((NS * STAGE + BARS) + 127) / 128 * 128;
    static constexpr size_t bytes(long long smax) { return PROD_OFF + 8 * (size_t)smax; }
};

template <class In, int NC, int CH, int NS, int LAG = 1, bool L2G = false>
__global__ void __launch_bounds__(NC + 32, 1)
csr_sorted_tma_spmv(CGeo g, SGather S, In in, double *__restrict__ out, Ws ws, int pred, long long row) {
    using RG = SpRing<CH, NS>;
    constexpr int PER = CH / NC;
    static_assert(CH % NC == 0 && CH % 8 == 0, "chunk shape");
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned long long *full = reinterpret_cast<unsigned long long *>(smem + NS * RG::STAGE);
    unsigned long long *empty = full + NS;
    double *sprod = reinterpret_cast<double *>(smem + RG::PROD_OFF);
    auto sval = [&](int s) { return reinterpret_cast<const double *>(smem + s * RG::STAGE); };
    auto scol = [&](int s) { return reinterpret_cast<const int *>(smem + s * RG::STAGE + CH * 8); };
    auto sdst = [&](int s) { return reinterpret_cast<const unsigned short *>(smem + s * RG::STAGE + CH * 12); };

    pdl_wait();
    pdl_launch_dependents();
    if (ws.head && !pred_ok(ws.head, pred, row)) return;
    if (ws.head) in.setup(ws);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const long long nblk = (g.n + S.R - 1) / S.R;
    const long long b0 = blockIdx.x * nblk / gridDim.x, b1 = (blockIdx.x + 1) * nblk / gridDim.x;
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NC / 32); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto krange = [&](long long blk, long long &k0, long long &k1) {
        k0 = __ldg(g.row_ptr + blk * S.R);
        k1 = __ldg(g.row_ptr + min(blk * S.R + S.R, g.n));
    };

    if (warp == NC / 32) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            long long it = 0;
            for (long long blk = b0; blk < b1; ++blk) {
                long long k0, k1;
                krange(blk, k0, k1);
                const long long e1 = (k1 + 7) & ~7LL;
                for (long long c = k0 & ~7LL; c < e1; c += CH, ++it) {
                    const int s = (int)(it % NS);
                    if (it >= NS) mbar_wait(&empty[s], (unsigned)(((it / NS) - 1) & 1));
                    const unsigned len = (unsigned)min((long long)CH, e1 - c);
                    mbar_expect_tx(&full[s], len * 14u);
                    bulk_g2s(smem + s * RG::STAGE, S.val + c, len * 8u, &full[s]);
                    bulk_g2s(smem + s * RG::STAGE + CH * 8, S.col + c, len * 4u, &full[s]);
                    bulk_g2s(smem + s * RG::STAGE + CH * 12, S.dest + c, len * 2u, &full[s]);
                }
            }
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    const double *base = in.base();
    // LAG chunks whose gathers are in flight; slot LAG-1 is the oldest
    struct Pend {
        double raw[PER], val[PER];
        int col[PER], dst[PER];
        bool ok[PER];
        bool valid;
        long long blk, k0;
    };
    Pend pq[LAG];
#pragma unroll
    for (int l = 0; l < LAG; ++l) pq[l].valid = false;
    auto consume = [&](const Pend &p) {
#pragma unroll
        for (int j = 0; j < PER; ++j)
            if (p.ok[j]) sprod[p.dst[j]] = __dmul_rn(p.val[j], in.xf(p.raw[j], p.col[j]));
    };
    auto rowsums = [&](long long blk, long long k0) {
        consumer_sync(NC);                          // every product of the block is stored
        const long long r0 = blk * S.R, r1 = min(r0 + (long long)S.R, g.n);
        for (long long r = r0 + tid; r < r1; r += NC) {
            const int a0 = __ldg(g.row_ptr + r) - (int)k0, a1 = __ldg(g.row_ptr + r + 1) - (int)k0;
            double a = 0.0;
            for (int kk = a0; kk < a1; ++kk) a = __dadd_rn(a, sprod[kk]);    // csr_matvec order
            out[r] = a;
        }
        consumer_sync(NC);                          // sprod is rewritten by the next block
    };
    // retire the oldest pending chunk; its block is complete when the next
    // chunk in flight (or `next_blk`, the block about to start) is a later one
    auto retire = [&](long long next_blk) {
        Pend &o = pq[LAG - 1];
        if (!o.valid) return;
        consume(o);
        long long nb = next_blk;
#pragma unroll
        for (int l = LAG - 2; l >= 0; --l)
            if (pq[l].valid) { nb = pq[l].blk; break; }
        if (nb != o.blk) rowsums(o.blk, o.k0);
        o.valid = false;
    };
    auto shift = [&]() {
#pragma unroll
        for (int l = LAG - 1; l > 0; --l) pq[l] = pq[l - 1];
        pq[0].valid = false;
    };
    long long it = 0;
    for (long long blk = b0; blk < b1; ++blk) {
        long long k0, k1;
        krange(blk, k0, k1);
        const long long e1 = (k1 + 7) & ~7LL;
        bool had = false;
        for (long long c = k0 & ~7LL; c < e1; c += CH, ++it) {
            had = true;
            const int s = (int)(it % NS);
            mbar_wait(&full[s], (unsigned)((it / NS) & 1));
            const long long len = min((long long)CH, e1 - c);
            Pend p;
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                const int idx = tid + j * NC;
                const long long kk = c + idx;
                p.ok[j] = idx < len && kk >= k0 && kk < k1;
                p.col[j] = p.ok[j] ? scol(s)[idx] : 0;
                p.dst[j] = p.ok[j] ? (int)sdst(s)[idx] : 0;
                p.val[j] = p.ok[j] ? sval(s)[idx] : 0.0;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);   // the slot is free: values are in registers
#pragma unroll
            for (int j = 0; j < PER; ++j) p.raw[j] = p.ok[j] ? load1<L2G>(in, base, p.col[j]) : 0.0;
            p.valid = true;
            p.blk = blk;
            p.k0 = k0;
            retire(blk);                            // the oldest chunk, while this one's gathers fly
            shift();
            pq[0] = p;
        }
        if (!had) {                                 // no nonzeros: its rows are +0.0
#pragma unroll
            for (int l = 0; l < LAG; ++l) { retire(blk); shift(); }
            rowsums(blk, k0);
        }
    }
#pragma unroll
    for (int l = 0; l < LAG; ++l) { retire(-1); shift(); }
}

}  // namespace kpl
