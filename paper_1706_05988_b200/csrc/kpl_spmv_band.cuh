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

}  // namespace kpl
