// kpl_core.cuh -- device-side building blocks shared by every sweep:
// workspace layout, streaming loads/stores, the deterministic reduction tree,
// and the scalar recurrences of the reference solvers.
//
// Compiled with --fmad=false: every a*b+c below is two IEEE roundings, the
// same as the reference's numba kernels and numpy ufuncs.
// The hot update formulas additionally use __dmul_rn/__dadd_rn/__dsub_rn so
// contraction is impossible even if the flag were dropped.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "../../include/kpl_b200.h"

namespace kpl {

constexpr int NT = 256;          // threads per CTA for every sweep
constexpr int NWARP = NT / 32;   // 8 warps
constexpr int NQ = 4;            // reduced quantities per item (max)
constexpr int RB = 256;          // CSR rows per item (one row per thread)
constexpr int HC = 10;           // history columns: alpha beta gamma delta |r| true f g h j

// ---------------------------------------------------------------- workspace
// Offset 0: head (1 KiB).  Mirrors kpl_status in its first 16 int64.
struct WsHead {
    long long state, iter, converged, bd_iter, bd_code, n_rep, fire, _st_pad[9];
    double alpha, beta, gamma_prev, alpha_prev;  // pipelined coefficients
    double bnorm, dot_result;
    double rr_e, rr_xnorm;                        // residual-replacement trigger
    long long rr_held, rr_started;
    double cg_gamma, cg_beta, cg_rnorm, cg_alpha; // classic CG head -> delta
    long long cg_last, _cg_pad;
    unsigned long long bar_arrive;                // one-phase grid barrier (persistent_redundant)
    double dsig_pad[3];
    unsigned int final_cnt, bar_cnt, bar_gen;     // completion count; grid barrier
    unsigned int fold_cnt, fold_fail, _cnt_pad[3];  // deferred peer fold: readers done; a failed wait
};
static_assert(sizeof(WsHead) <= 1024, "head too large");

enum Phase : int {
    PH_NONE = 0,      // no reduction (spmv, replacement intermediates)
    PH_DOT = 1,       // result -> head.dot_result
    PH_BNORM = 2,     // head.bnorm = sqrt(v0)
    PH_INITR = 3,     // r = b - A x0: pcg_rr trigger.start(|x|, |r|)  (+ CG head of row 0)
    PH_PIPE = 4,      // pipelined record: gamma, delta, rho (+xi for rr)
    PH_RRFINAL = 5,   // after an explicit replacement: trigger.reset + record
    PH_TRUE = 6,      // ||b - A x|| into the current history row
    PH_CGHEAD = 7,    // classic CG: gamma, rho -> beta, convergence, last
    PH_CGDELTA = 8,   // classic CG: delta -> alpha, record, done
    PH_GAPF = 9,      // track_gaps: ||b - A x||, ||f|| = ||(b - A x) - r||      (solvers.py:148-149)
    PH_GAPG = 10,     // ||axpy(-sigma_prev, t, A p) - s||                      (:153)
    PH_GAPH = 11,     // ||axpy(-sigma_prev, r, A u) - w||                      (:152)
    PH_GAPJ = 12,     // ||A q - z||                                            (:154)
};

// Launch predicate evaluated uniformly by every CTA at kernel start.
enum Pred : int {
    PRED_ALWAYS = 0,
    PRED_RUNNING = 1,        // state == RUNNING
    PRED_FIRE = 2,           // state == RUNNING && fire  (pcg_rr replacement)
    PRED_ROW = 3,            // head.iter == row (explicit true-residual row)
    PRED_NOFIRE = 4,         // state == RUNNING && !fire  (an iteration waits for a pending replacement)
};

struct Layout {               // identical on host and device
    int vx, wx, wy, zc;       // stencil tile: TX = 32*vx*wx, TY = wy
    int ntx, nty;             // tiles per plane
    long long nch;            // chunks owned by this launch (local)
    long long items;          // CTAs of a sweep
    int T;                    // items per chunk
};

struct Ws {                   // device view of the caller's workspace
    WsHead *head;
    double *items;            // [items][NQ]
    double *chunks;           // [chunks_global][NQ] (global table)
    unsigned int *chunk_cnt;  // [nch_local]
    double *hist;             // [max_iters+1][HC]
    long long *reps;          // [max_iters+1]
    double *nbuf;             // CSR: n = A m of the current sweep (split SpMV / update)
    double *mbuf;             // CSR + vector Jacobi (1 GPU): m = w * inv_diag, written with w
    long long chunk_offset;   // first global chunk of this rank
    long long chunks_global;
    int inline_final;         // 1: last CTA finalises (single GPU)
    double *prod;             // KPL_ORDER_BLOCKED8: products [NQ][nprod] for blocked_final_kernel
    long long nprod;
    int hist_scratch;         // 1: history writes go to the single scratch row `hist` (redundant epilogues)
    // fused multi-GPU exchange (kpl_sweep_peer; px == nullptr otherwise)
    const kpl_peer_sweep *px;
    unsigned long long epoch; // value signalled to every rank when this rank's sweep is done
    int tpar;                 // exchange-table slot the chunk partials go to
    int push;                 // KPL_PUSH_* outputs whose boundary planes go to the neighbours
    int wpar;                 // which ping-pong w is the output
    // deferred fold (kpl_sweep_peer, wait_epoch != 0): every CTA first waits for
    // the previous sweep's exchange (flags >= wait_epoch), folds table slot
    // wait_tpar and runs its epilogue on a private copy of the head
    unsigned long long wait_epoch;
    int wait_tpar;
    unsigned long long timeout_ns;   // peer waits: give up after this long
    unsigned int *final_cnt;  // chunk-completion count (on the real head, also in a private view)
};

// Product sink of the reference-order mode: bodies accumulate through accp(),
// which also stores each product when the workspace carries a product buffer.
struct Sink {
    double *p = nullptr;
    long long n = 0;
    __device__ __forceinline__ void set(const Ws &ws) { p = ws.prod; n = ws.nprod; }
};

template <int Q, int V>
__device__ __forceinline__ void accp(double (&acc)[Q][V], int q, int v, const Sink &sk, long long k,
                                     double prod) {
    acc[q][v] = __dadd_rn(acc[q][v], prod);
    if (sk.p) sk.p[q * sk.n + k + v] = prod;
}

struct Cfg {                  // scalar view of kpl_cfg
    int method;
    int track_gaps;
    double shift, rtol, tau, coef;
    long long max_iters;
    const double *schedule;   // pcg_var_sh: shift_schedule on the device (max_iters+1 values)
};

// ------------------------------------------------------------- memory ops

// streaming (evict-first) loads/stores for the vectors touched once per sweep
template <int V>
__device__ __forceinline__ void ld_cs(const double *p, long long k, double (&o)[V]) {
    if constexpr (V == 2) {
        double2 t = __ldcs(reinterpret_cast<const double2 *>(p + k));
        o[0] = t.x; o[1] = t.y;
    } else {
        o[0] = __ldcs(p + k);
    }
}
template <int V>
__device__ __forceinline__ void st_cs(double *p, long long k, const double (&o)[V]) {
    if constexpr (V == 2) {
        __stcs(reinterpret_cast<double2 *>(p + k), make_double2(o[0], o[1]));
    } else {
        __stcs(p + k, o[0]);
    }
}
// read-only loads of the stencil input (re-read by neighbouring tiles: keep in L2)
template <int V>
__device__ __forceinline__ void ld_ro(const double *p, long long k, double (&o)[V]) {
    if constexpr (V == 2) {
        double2 t = __ldg(reinterpret_cast<const double2 *>(p + k));
        o[0] = t.x; o[1] = t.y;
    } else {
        o[0] = __ldg(p + k);
    }
}

// Reads of the workspace head (state, iteration, alpha, beta ...): a strong
// GPU-scope load whose asm carries a "memory" clobber, so the compiler keeps
// it after the barrier / epilogue stores that precede it in program order
// (__ldcg's asm has no clobber, so nothing but the barrier orders it).
// Generic address: the head is global memory, or a CTA's private copy in
// shared memory (deferred peer fold).
__device__ __forceinline__ long long ld_head(const long long *p) { return *(const volatile long long *)p; }
__device__ __forceinline__ double ld_head(const double *p) { return *(const volatile double *)p; }

// Programmatic dependent launch: sweeps may be launched while the previous
// kernel in the stream is still draining (cudaLaunchAttributeProgrammatic-
// StreamSerialization); they wait here -- before touching anything the
// previous kernel wrote -- and let their own dependents launch early.  Both
// are no-ops for a normal launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ------------------------------------------------------------ arithmetic
// axpy(alpha, x, y) of sparse.py:172-180: alpha == 0 -> exact copy of y.
__device__ __forceinline__ double axpy1(double a, double x, double y) {
    return a == 0.0 ? y : __dadd_rn(__dmul_rn(a, x), y);
}
// _sub2(base, a, xv, c, yv) of solvers.py:170-178.
__device__ __forceinline__ double sub2(double base, double a, double xv, double c, double yv) {
    return c == 0.0 ? __dsub_rn(base, __dmul_rn(a, xv))
                    : __dsub_rn(base, __dadd_rn(__dmul_rn(a, xv), __dmul_rn(c, yv)));
}

// ------------------------------------------------------- reduction tree
// Level 2b: xor butterfly over the 32 lanes (every lane ends with the sum).
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
    return v;
}

// Level 2c: the NWARP warp totals combined by a halving tree (s[0:4]+s[4:8], ...).
// Returns the block total in thread 0 (all threads of warp 0 hold it).
template <int Q>
__device__ __forceinline__ void block_sum(double (&v)[Q], double *sm /* >= NWARP*Q */) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < Q; ++q) v[q] = warp_sum(v[q]);
    if (lane == 0 && warp < NWARP) {      // extra (producer) warps never contribute
#pragma unroll
        for (int q = 0; q < Q; ++q) sm[q * NWARP + warp] = v[q];
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            double t = lane < NWARP ? sm[q * NWARP + lane] : 0.0;
            t = __dadd_rn(t, __shfl_xor_sync(0xffffffffu, t, 4));
            t = __dadd_rn(t, __shfl_xor_sync(0xffffffffu, t, 2));
            t = __dadd_rn(t, __shfl_xor_sync(0xffffffffu, t, 1));
            v[q] = t;
        }
    }
    __syncthreads();
}

// Levels 3/4: sum src[j*stride + q] for j in [0, count) -- thread t adds
// j = t, t+256, ... sequentially from +0.0, then block_sum.  Loads bypass L1
// (the values were written by other CTAs of this grid).
template <int Q, bool SHARED = false>
__device__ __forceinline__ void strided_sum(const double *src, long long count, int stride,
                                            double (&v)[Q], double *sm) {
#pragma unroll
    for (int q = 0; q < Q; ++q) v[q] = 0.0;
    for (long long j = threadIdx.x; j < count && threadIdx.x < NT; j += NT) {
#pragma unroll
        for (int q = 0; q < Q; ++q)
            v[q] = __dadd_rn(v[q], SHARED ? src[j * stride + q] : __ldcg(src + j * stride + q));
    }
    block_sum<Q>(v, sm);
}

// ---------------------------------------------------- scalar recurrences
enum Breakdown : int {
    BD_NONPOS_RU = 1,        // "nonpositive (r, u)"
    BD_NONPOS_WU = 2,        // "nonpositive curvature (w, u)"
    BD_VANISH_RU = 3,        // "vanishing (r, u)"
    BD_VANISH_DEN = 4,       // "vanishing alpha denominator"
    BD_NONFINITE = 5,        // "non-finite coefficients"
    BD_NONPOS_SP = 6,        // "nonpositive curvature (s, p)"
    BD_PEER_TIMEOUT = 7,     // "peer exchange timeout"
    BD_BARRIER_TIMEOUT = 8,  // "device barrier timeout" (persistent solver)
    BD_PEER_FAILED = 9,      // "peer rank failed" (a peer signalled poison)
};

__device__ __forceinline__ void set_breakdown(WsHead *h, long long i, int code) {
    h->state = KPL_ST_BREAKDOWN;
    h->bd_iter = i;
    h->bd_code = code;
}

// solvers.py:194-230 _pipelined_scalars.  Returns false on breakdown.
__device__ bool pipelined_scalars(WsHead *h, long long i, double gamma, double delta, bool last,
                                  double &beta, double &alpha) {
    const double gamma_prev = h->gamma_prev, alpha_prev = h->alpha_prev;
    if (i == 0) {
        beta = 0.0;
        if (delta > 0.0) {
            alpha = gamma / delta;
        } else if (last) {
            alpha = 0.0;
        } else if (gamma <= 0.0) {
            set_breakdown(h, i, BD_NONPOS_RU); return false;
        } else {
            set_breakdown(h, i, BD_NONPOS_WU); return false;
        }
        return true;
    }
    beta = gamma_prev != 0.0 ? gamma / gamma_prev : 0.0;
    if (last) {
        if (gamma == 0.0 || delta == 0.0) { alpha = 0.0; return true; }
        const double denom = __dsub_rn(delta / gamma, beta / alpha_prev);
        double a = denom != 0.0 ? 1.0 / denom : 0.0;
        alpha = isfinite(a) ? a : 0.0;
        return true;
    }
    if (gamma == 0.0) { set_breakdown(h, i, BD_VANISH_RU); return false; }
    const double denom = __dsub_rn(delta / gamma, beta / alpha_prev);
    if (denom == 0.0) { set_breakdown(h, i, BD_VANISH_DEN); return false; }
    alpha = 1.0 / denom;
    if (!(isfinite(alpha) && isfinite(beta))) { set_breakdown(h, i, BD_NONFINITE); return false; }
    return true;
}

__device__ __forceinline__ double *hist_row(const Ws &ws, long long i) {
    return ws.hist_scratch ? ws.hist : ws.hist + HC * i;
}

__device__ __forceinline__ bool converged_test(const Cfg &cfg, const WsHead *h, double rnorm) {
    // solvers.py:391
    return rnorm == 0.0 || (cfg.rtol > 0.0 && rnorm <= cfg.rtol * h->bnorm);
}

// Pipelined record of row i (solvers.py:388-403 minus the cadence column).
__device__ void pipe_record(const Ws &ws, const Cfg &cfg, long long i, double gamma, double delta,
                            double rho) {
    WsHead *h = ws.head;
    const double rnorm = sqrt(rho);
    const bool conv = converged_test(cfg, h, rnorm);
    const bool last = conv || i == cfg.max_iters;
    double beta, alpha;
    if (!pipelined_scalars(h, i, gamma, delta, last, beta, alpha)) return;
    double *row = hist_row(ws, i);
    row[0] = alpha; row[1] = beta; row[2] = gamma; row[3] = delta; row[4] = rnorm;
    h->alpha = alpha;
    h->beta = beta;
    h->gamma_prev = gamma;     // solvers.py:420-421 (consumed by row i+1)
    h->alpha_prev = alpha;
    h->iter = i;
    if (last) {
        h->converged = conv ? 1 : 0;
        h->state = KPL_ST_DONE;
    }
}

// _ReplacementTrigger (solvers.py:501-532); eps = unit roundoff.
constexpr double UNIT_ROUNDOFF = 1.1102230246251565e-16;

// The scalar epilogue run once per sweep by one thread after the reduction.
__device__ void finalize(const Ws &ws, const Cfg &cfg, int phase, const double (&v)[NQ]) {
    WsHead *h = ws.head;
    switch (phase) {
    case PH_DOT:
        h->dot_result = v[0];
        break;
    case PH_BNORM:
        h->bnorm = sqrt(v[0]);
        break;
    case PH_INITR: {
        // v = {(x,x), (r,r), (r,u)}
        if (cfg.method == KPL_M_PCG_RR) {      // trigger.start (solvers.py:519-521, :558)
            const double xnorm = sqrt(v[0]), rnorm = sqrt(v[1]);
            h->rr_e = UNIT_ROUNDOFF * (cfg.coef * xnorm + h->bnorm);
            h->rr_held = h->rr_e <= cfg.tau * rnorm;
        }
        if (cfg.method == KPL_M_CG) {          // classic CG head of row 0 (solvers.py:258-268)
            const double gamma = v[2], rnorm = sqrt(v[1]);
            const bool conv = converged_test(cfg, h, rnorm);
            const bool last = conv || 0 == cfg.max_iters;
            h->cg_gamma = gamma; h->cg_rnorm = rnorm; h->cg_beta = 0.0;
            h->cg_last = last; h->converged = conv; h->iter = 0;
            if (!last && gamma <= 0.0) set_breakdown(h, 0, BD_NONPOS_RU);
        }
        break;
    }
    case PH_PIPE: {
        // v = {gamma, delta, rho, xi}; the row index is iter+1 except for init (iter = -1)
        const long long i = h->iter + 1;
        if (cfg.method == KPL_M_PCG_RR && i > 0) {   // trigger.update (solvers.py:523-528, :599)
            const double xnorm = sqrt(v[3]), rnorm = sqrt(v[2]);
            h->rr_e = h->rr_e + UNIT_ROUNDOFF * (cfg.coef * xnorm + rnorm);
            const bool ok = h->rr_e <= cfg.tau * rnorm;
            const bool fire = h->rr_held && !ok && cfg.tau > 0.0;
            h->rr_held = ok;
            if (fire) {
                h->fire = 1;
                h->rr_xnorm = xnorm;
                ws.reps[h->n_rep] = i;           // replacements.append(i + 1)
                h->n_rep += 1;
                return;                          // record after the replacement sweeps
            }
        }
        pipe_record(ws, cfg, i, v[0], v[1], v[2]);
        break;
    }
    case PH_RRFINAL: {
        // trigger.reset(|x|, |r|) with the replaced r (solvers.py:530-532, :607)
        const long long i = h->iter + 1;
        const double rnorm = sqrt(v[2]);
        h->rr_e = UNIT_ROUNDOFF * (cfg.coef * h->rr_xnorm + rnorm);
        h->rr_held = h->rr_e <= cfg.tau * rnorm;
        h->fire = 0;
        pipe_record(ws, cfg, i, v[0], v[1], v[2]);
        break;
    }
    case PH_TRUE:
        hist_row(ws, h->iter)[5] = sqrt(v[0]);
        break;
    case PH_GAPF:
        hist_row(ws, h->iter)[5] = sqrt(v[0]);
        hist_row(ws, h->iter)[6] = sqrt(v[1]);
        break;
    case PH_GAPG:
        hist_row(ws, h->iter)[7] = sqrt(v[0]);
        break;
    case PH_GAPH:
        hist_row(ws, h->iter)[8] = sqrt(v[0]);
        break;
    case PH_GAPJ:
        hist_row(ws, h->iter)[9] = sqrt(v[0]);
        break;
    case PH_CGHEAD: {
        // v = {(r,u), (r,r)} of the updated vectors: row i = iter + 1 (solvers.py:258-268)
        const long long i = h->iter + 1;
        const double gamma = v[0], rnorm = sqrt(v[1]);
        const bool conv = converged_test(cfg, h, rnorm);
        const bool last = conv || i == cfg.max_iters;
        const double gamma_prev = h->cg_gamma;
        h->cg_beta = gamma_prev > 0.0 ? gamma / gamma_prev : 0.0;
        h->cg_gamma = gamma; h->cg_rnorm = rnorm;
        h->cg_last = last; h->converged = conv; h->iter = i;
        if (!last && gamma <= 0.0) set_breakdown(h, i, BD_NONPOS_RU);
        break;
    }
    case PH_CGDELTA: {
        // v = {(s,p)} (solvers.py:271-289)
        const long long i = h->iter;
        const double delta = v[0], gamma = h->cg_gamma;
        double alpha;
        if (h->cg_last) {
            alpha = delta > 0.0 ? gamma / delta : 0.0;
        } else if (delta <= 0.0) {
            set_breakdown(h, i, BD_NONPOS_SP);
            return;
        } else {
            alpha = gamma / delta;
        }
        double *row = hist_row(ws, i);
        row[0] = alpha; row[1] = h->cg_beta; row[2] = gamma; row[3] = delta; row[4] = h->cg_rnorm;
        h->cg_alpha = alpha;
        h->alpha = alpha;
        if (h->cg_last) h->state = KPL_ST_DONE;
        break;
    }
    default:
        break;
    }
}

// Per-kernel uniform predicate.
__device__ __forceinline__ bool pred_ok(const WsHead *h, int pred, long long row) {
    if (pred == PRED_ALWAYS) return true;          // (plain spmv launches carry no workspace)
    // both words are requested before either is tested: one L2 round trip, not two in series
    const long long state = ld_head(&h->state);
    const long long second = pred == PRED_ROW ? ld_head(&h->iter)
                             : (pred == PRED_FIRE || pred == PRED_NOFIRE) ? ld_head(&h->fire) : 0;
    switch (pred) {
    case PRED_RUNNING: return state == KPL_ST_RUNNING;
    case PRED_FIRE: return state == KPL_ST_RUNNING && second != 0;
    case PRED_ROW: return second == row && state != KPL_ST_BREAKDOWN;
    case PRED_NOFIRE: return state == KPL_ST_RUNNING && second == 0;
    default: return true;
    }
}

// ---------------------------------------------------- fused peer exchange
// Flags are monotone epochs; a rank whose exchange failed (a wait timed out,
// or a peer's poison was seen) signals epoch | PEER_POISON from then on, so
// every peer fails its next wait at once instead of folding stale partials.
constexpr unsigned long long PEER_POISON = 1ull << 63;

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ bool peer_failed(const WsHead *h) {
    if (!h || ld_head(&h->state) != KPL_ST_BREAKDOWN) return false;
    const long long c = ld_head(&h->bd_code);
    return c == BD_PEER_TIMEOUT || c == BD_PEER_FAILED;
}
__device__ __forceinline__ unsigned long long peer_signal_value(const WsHead *h, unsigned long long epoch) {
    return epoch | (peer_failed(h) ? PEER_POISON : 0ull);
}

// Wait until flags[0..nranks) >= epoch (acquire, system scope).  Returns 0,
// or BD_PEER_FAILED (a peer's poison) / BD_PEER_TIMEOUT.  `abort` (optional):
// a word another CTA of this rank sets when its own wait failed.
__device__ __noinline__ int peer_wait(const unsigned long long *flags, int nranks, unsigned long long epoch,
                                      unsigned long long timeout_ns, const unsigned *abort) {
    const unsigned long long t0 = globaltimer_ns();
    for (int p = 0; p < nranks; ++p) {
        for (;;) {
            const unsigned long long v = ld_acquire_sys(flags + p);
            if (v & PEER_POISON) return BD_PEER_FAILED;
            if (v >= epoch) break;
            __nanosleep(64);
            if (abort && *(const volatile unsigned *)abort) return BD_PEER_FAILED;
            if (globaltimer_ns() - t0 > timeout_ns) return BD_PEER_TIMEOUT;
        }
    }
    return 0;
}

__device__ __forceinline__ void peer_signal_all(const Ws &ws) {
    const unsigned long long v = peer_signal_value(ws.head, ws.epoch);
    for (int p = 0; p < ws.px->nranks; ++p)
        st_release_sys_u64(reinterpret_cast<unsigned long long *>(ws.px->signal[p]), v);
}

// A predicated-off fused sweep still signals (the finalize skips its fold by
// the same predicate), so the ranks' epochs stay in step.
__device__ __forceinline__ void peer_signal_idle(const Ws &ws) {
    if (ws.px && blockIdx.x == 0 && threadIdx.x == 0) {
        __threadfence_system();
        peer_signal_all(ws);
    }
}

// ---- deferred fold: the reduction exchange of sweep i-1 folded inside sweep i
// (the paper's overlap: no finalize launch between sweeps).
struct FoldSmem {
    WsHead head;              // this CTA's private copy of the head (epilogue applied)
    double row[HC];           // its history row (scratch)
};

// The view every later part of the sweep uses: scalars from `h` (the private
// head) and history into `row`; counters stay on the real head.  Built field
// by field (see ws_view in kpl_sweep.cuh for why).
__device__ __forceinline__ Ws ws_fold_view(const Ws &ws, WsHead *h, double *row, bool fold) {
    Ws w;
    w.head = fold ? h : ws.head; w.items = ws.items; w.chunks = ws.chunks; w.chunk_cnt = ws.chunk_cnt;
    w.hist = fold ? row : ws.hist; w.reps = ws.reps; w.nbuf = ws.nbuf; w.mbuf = ws.mbuf;
    w.chunk_offset = ws.chunk_offset; w.chunks_global = ws.chunks_global; w.inline_final = ws.inline_final;
    w.prod = ws.prod; w.nprod = ws.nprod; w.hist_scratch = fold ? 1 : ws.hist_scratch;
    w.px = ws.px; w.epoch = ws.epoch; w.tpar = ws.tpar; w.push = ws.push; w.wpar = ws.wpar;
    w.wait_epoch = ws.wait_epoch; w.wait_tpar = ws.wait_tpar; w.timeout_ns = ws.timeout_ns;
    w.final_cnt = ws.final_cnt;
    return w;
}

// Every CTA (all threads): wait for every rank's flag of the previous sweep,
// copy the head, fold this rank's table slot (the level-4 tree of a single
// GPU: strided_sum over chunks_global, as peer_finalize_kernel) and run the
// pipelined epilogue on the copy -- every CTA computes the same alpha_i,
// beta_i bit for bit.  The last CTA to finish reading the real head publishes
// its copy (scalars + history row) there.  Only for PH_PIPE sweeps that
// follow a fused iteration sweep of the same solve (the host decides).
__device__ __noinline__ void peer_fold_start(const Ws &ws, const Cfg &cfg, FoldSmem &fs, double *sred) {
    __shared__ int s_fail;
    if (threadIdx.x == 0)       // nothing to wait for once the solve has stopped
        s_fail = ld_head(&ws.head->state) != KPL_ST_RUNNING
                     ? 0 : peer_wait(reinterpret_cast<const unsigned long long *>(ws.px->flags), ws.px->nranks, ws.wait_epoch, ws.timeout_ns, &ws.head->fold_fail);
    {
        const unsigned long long *src = reinterpret_cast<const unsigned long long *>(ws.head);
        unsigned long long *dst = reinterpret_cast<unsigned long long *>(&fs.head);
        for (int k = threadIdx.x; k < (int)(sizeof(WsHead) / 8); k += blockDim.x) dst[k] = __ldcg(src + k);
    }
    if (threadIdx.x == 0) __threadfence_system();
    __syncthreads();
    const bool running = fs.head.state == KPL_ST_RUNNING;   // the finalize's PRED_RUNNING
    double f[NQ];
    strided_sum<NQ>(ws.px->table[ws.wait_tpar][ws.px->rank], ws.chunks_global, NQ, f, sred);
    if (threadIdx.x == 0) {
        for (int c = 0; c < HC; ++c) fs.row[c] = __longlong_as_double(0x7ff8000000000000LL);
        const Ws v = ws_fold_view(ws, &fs.head, fs.row, true);
        if (s_fail) {
            if (running) set_breakdown(&fs.head, -1, s_fail);
            atomicOr(&ws.head->fold_fail, 1u << s_fail);
        } else if (running) {
            finalize(v, cfg, PH_PIPE, f);
        }
        __threadfence();
        const unsigned prev = atomicAdd(&ws.head->fold_cnt, 1u);
        if (prev == gridDim.x - 1) {               // every CTA has read the real head
            __threadfence();
            const unsigned fail = atomicExch(&ws.head->fold_fail, 0u);
            WsHead *h = ws.head;
            if (fail && running && fs.head.state != KPL_ST_BREAKDOWN)
                set_breakdown(&fs.head, -1, (fail >> BD_PEER_FAILED) & 1 ? BD_PEER_FAILED : BD_PEER_TIMEOUT);
            // scalars only: the counters (from bar_arrive on) belong to running sweeps
            const size_t nsc = offsetof(WsHead, bar_arrive) / 8;
            const unsigned long long *src = reinterpret_cast<const unsigned long long *>(&fs.head);
            unsigned long long *dst = reinterpret_cast<unsigned long long *>(h);
            for (size_t k = 0; k < nsc; ++k) dst[k] = src[k];
            if (running && !s_fail && fs.head.state != KPL_ST_BREAKDOWN) {
                double *row = ws.hist + HC * fs.head.iter;
                for (int c = 0; c < 5; ++c) row[c] = fs.row[c];
            }
            h->fold_cnt = 0u;
            __threadfence();
        }
    }
    __syncthreads();
}

// Halo part of the fused exchange: CTAs of the slab's first / last chunk copy
// their tile of plane 0 / NZ-1 of each pushed output into the neighbour's
// halo plane.  Each thread re-reads the elements it has just stored itself
// (program order), k0 = x + NX*y of its first element.  Ends with a CTA
// barrier and a system-scope fence, before the chunk completion count.
template <int V>
__device__ __forceinline__ void peer_halo_push(const Ws &ws, long long c, long long nch, long long NZ,
                                               long long sxy, long long k0, bool ok) {
    if (!ws.px || !ws.push) return;
    const bool first = c == 0, last = c == nch - 1;
    if (!first && !last) return;
    const kpl_peer_sweep *px = ws.px;
    if (ok) {
#pragma unroll
        for (int m = 0; m < 2; ++m) {
            if (!(ws.push & (1 << m))) continue;
            const double *src = m == 0 ? px->w_src[ws.wpar] : px->x_src;
            double *lo = m == 0 ? px->w_lo[ws.wpar] : px->x_lo;
            double *hi = m == 0 ? px->w_hi[ws.wpar] : px->x_hi;
            if (first && lo) {
#pragma unroll
                for (int v = 0; v < V; ++v) lo[k0 + v] = src[k0 + v];
            }
            if (last && hi) {
                const long long kz = (NZ - 1) * sxy + k0;
#pragma unroll
                for (int v = 0; v < V; ++v) hi[k0 + v] = src[kz + v];
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) __threadfence_system();
}

// After a CTA has written its item partial (thread 0, before the call):
// chunk-completion and grid-completion counting; the last CTA of a chunk
// folds the chunk (level 3), the last chunk folds the grid (level 4) and runs
// the scalar epilogue.  Every CTA of the grid must call this.
template <int Q>
__device__ void complete_item(const Ws &ws, const Cfg &cfg, const Layout &L, int phase,
                              long long chunk_local, double *sm) {
    // Only thread 0 wrote the item partial, so only thread 0 fences (release)
    // before counting, and fences again (acquire) once it knows it is last.
    __shared__ int s_last;
    const long long item0 = chunk_local * L.T;
    const long long expect = min((long long)L.T, L.items - item0);   // last CSR chunk may be short
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned prev = atomicAdd(&ws.chunk_cnt[chunk_local], 1u);
        s_last = (prev == (unsigned)(expect - 1));
        if (s_last) __threadfence();
    }
    __syncthreads();
    if (!s_last) return;
    double v[Q];
    strided_sum<Q>(ws.items + item0 * NQ, expect, NQ, v, sm);
    const long long cg = ws.chunk_offset + chunk_local;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < Q; ++q) ws.chunks[cg * NQ + q] = v[q];
        ws.chunk_cnt[chunk_local] = 0u;
        if (ws.px) {
            // fused exchange: this chunk's partial into every rank's table slot;
            // the rank's last chunk signals every rank
            for (int p = 0; p < ws.px->nranks; ++p) {
                double *dst = ws.px->table[ws.tpar][p] + cg * NQ;
#pragma unroll
                for (int q = 0; q < NQ; ++q) dst[q] = q < Q ? v[q] : 0.0;
            }
            __threadfence_system();
            const unsigned prev = atomicAdd(ws.final_cnt, 1u);
            if (prev == (unsigned)(L.nch - 1)) {
                *ws.final_cnt = 0u;
                __threadfence_system();
                peer_signal_all(ws);
            }
        }
    }
    if (!ws.inline_final) return;
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned prev = atomicAdd(ws.final_cnt, 1u);
        s_last = (prev == (unsigned)(L.nch - 1));
        if (s_last) __threadfence();
    }
    __syncthreads();
    if (!s_last) return;
    double f[Q];
    strided_sum<Q>(ws.chunks, ws.chunks_global, NQ, f, sm);
    if (threadIdx.x == 0) {
        double full[NQ] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int q = 0; q < Q; ++q) full[q] = f[q];
        finalize(ws, cfg, phase, full);
        *ws.final_cnt = 0u;
        __threadfence();
    }
}

}  // namespace kpl
