// kpl_peer.cuh -- device-initiated exchange over peer memory (NVLink P2P).
//
// The multi-GPU exchange of one sweep without a host-driven
// collective: after a sweep, `peer_post_kernel` stores
//   * the halo planes (z-slabs) / packed ghost rows (CSR row blocks) of the
//     vectors the next sweep reads at neighbours, directly into the
//     neighbours' halo / ghost storage (peer pointers, IPC-mapped), and
//   * this rank's chunk partials into every rank's exchange table slot
//     (double-buffered by epoch parity),
// then its last CTA publishes `epoch` into every rank's flag word for this
// rank (st.release.sys after a system-scope fence).  `peer_finalize_kernel`
// waits until every rank's flag reached `epoch` (ld.acquire.sys), then folds
// the gathered table (the level-4 tree of a single GPU, so results stay
// bit-identical to one GPU) and runs the scalar epilogue.
//
// Ordering argument (why one flag per sweep is enough): a rank
// only pushes into a peer after passing the wait of the previous sweep, which
// the peer signalled after finishing that sweep; the halos pushed after sweep
// s are those of vectors sweep s+1 reads and sweep s did not read, so no push
// overwrites data a concurrently running sweep reads; the partial tables
// alternate by epoch parity.
#pragma once
#include "kpl_core.cuh"

namespace kpl {

// Copies (grid-stride over every copy in turn), then the completion count and
// the signals.  `cnt` is a device word of this rank, zero before the first
// post; atomicInc wraps it back to zero in the last CTA.
__global__ void __launch_bounds__(NT) peer_post_kernel(kpl_post post, unsigned long long epoch) {
    const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long nthr = (long long)gridDim.x * blockDim.x;
    for (int c = 0; c < post.ncopies; ++c) {
        const kpl_copy cp = post.copies[c];
        if (cp.idx) {
            for (long long k = tid; k < cp.count; k += nthr) cp.dst[k] = __ldg(cp.src + cp.idx[k]);
        } else {
            for (long long k = tid; k < cp.count; k += nthr) cp.dst[k] = __ldcg(cp.src + k);
        }
    }
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();                 // this CTA's stores before the count (cumulative)
        const unsigned prev = atomicInc(post.counter, gridDim.x - 1);
        s_last = prev == gridDim.x - 1;
        if (s_last) __threadfence_system();
    }
    __syncthreads();
    if (!s_last) return;
    // a rank whose exchange failed signals poison, so no peer folds stale partials
    const unsigned long long v = peer_signal_value(reinterpret_cast<const WsHead *>(post.status), epoch);
    for (int p = threadIdx.x; p < post.nsignals; p += blockDim.x)
        st_release_sys_u64(reinterpret_cast<unsigned long long *>(post.signal[p]), v);
}

// Wait for every rank's flag >= epoch, then (reducing sweeps) fold the
// exchange table in ws.chunks and run the epilogue of `phase`.
__global__ void __launch_bounds__(NT) peer_finalize_kernel(Ws ws, Cfg cfg, int phase, int pred, long long row,
                                                           const unsigned long long *flags, int nranks,
                                                           unsigned long long epoch) {
    __shared__ double sred[NQ * NWARP];
    __shared__ int s_ok;
    if (threadIdx.x == 0) {
        // after a failure the exchange is dead: later waits return at once (and
        // this rank's posts signal poison from now on)
        int code = peer_failed(ws.head) ? BD_PEER_FAILED : peer_wait(flags, nranks, epoch, ws.timeout_ns, nullptr);
        if (code && ws.head && ws.head->state == KPL_ST_RUNNING) set_breakdown(ws.head, -1, code);
        __threadfence_system();
        s_ok = code == 0;
    }
    __syncthreads();
    if (!s_ok || phase == PH_NONE || !ws.head) return;
    if (!pred_ok(ws.head, pred, row)) return;
    double f[NQ];
    strided_sum<NQ>(ws.chunks, ws.chunks_global, NQ, f, sred);
    if (threadIdx.x == 0) finalize(ws, cfg, phase, f);
}

}  // namespace kpl
