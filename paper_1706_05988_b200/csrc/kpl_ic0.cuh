// kpl_ic0.cuh -- IC(0) preconditioner on the device:
// the factorisation (_kernels.py:77-115) and the forward / backward
// substitutions of its apply (_kernels.py:55-74, precond.py:90-94).
//
// All three are row-sequential recurrences whose dependencies follow the
// sparsity pattern.  They run as *sync-free* sweeps: one thread per row, each
// row waits until every row it reads has been published, then publishes its
// own (the substitutions: the value itself, see kIcEmpty; the factor: a
// per-row flag with release/acquire, since a row there is many values).  Rows are handed to CTAs by an atomic ticket
// in a topological order -- the rows sorted by dependency level (computed
// once per factor by ic0_levels_kernel), so the resident CTAs hold whole
// wavefronts instead of a contiguous band of rows, and a CTA only ever waits
// on rows owned by CTAs that are already resident: no deadlock regardless of
// grid size.  (NULL order = natural order, ascending for L, descending for
// L^T, also topological.)  Inside a row the arithmetic is the
// reference's, term for term (--fmad=false, explicit __d*_rn), so the factor
// and every apply are bit-identical to the reference.
// Each sweep re-arms the other's ticket (the other sweep is complete by
// stream order), so nothing is reset between applies.
#pragma once
#include "kpl_bodies.cuh"

namespace kpl {

__device__ __forceinline__ int ld_acquire(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(int *p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

#ifndef KPL_IC0_SPIN_NS
#define KPL_IC0_SPIN_NS 20
#endif

__device__ __forceinline__ int ld_relaxed(const int *p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Spin with relaxed loads, then one acquire load: an acquire load also
// invalidates the SM's L1 (CCTL.IVALL), so spinning on it would evict the
// data every other warp on the SM is reading.
// Watchdog of the dependency spins: a wait that a correct sweep satisfies in
// microseconds; after ~10 s something is broken -- trap (the launch fails with
// an error) rather than leave the GPU spinning.
__device__ __forceinline__ void spin_watchdog(unsigned &n, unsigned long long &t0) {
    if ((++n & 4095u) != 0u) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t0 == 0) t0 = t;
    else if (t - t0 > 10000000000ull) __trap();
}

__device__ __forceinline__ void wait_flag(const int *f) {
    unsigned n = 0;
    unsigned long long t0 = 0;
    while (ld_relaxed(f) == 0) {
        if (KPL_IC0_SPIN_NS > 0) __nanosleep(KPL_IC0_SPIN_NS);
        spin_watchdog(n, t0);
    }
    (void)ld_acquire(f);
}

struct Tri {                // CSR triangle, int32 indices
    const int *rp, *ci;
    const double *v;
    const int *order;       // processing order (topological), NULL = natural
};

// Row handled by slot t of a sweep (upper sweeps run the natural order backwards).
__device__ __forceinline__ long long tri_row(const Tri &T, long long t, long long n, bool upper) {
    if (T.order) return __ldg(T.order + t);
    return upper ? n - 1 - t : t;
}

struct Ic0Ws {              // apply scratch inside the solver workspace
    double *y;              // L^-1 v (holds kIcEmpty between applies)
    unsigned int *tickets;  // [0] forward, [1] backward
};

// The substitution sweeps publish each row's value by storing the value
// itself: every not-yet-computed entry holds kIcEmpty, a *signalling* NaN.
// IEEE arithmetic never returns a signalling NaN (an sNaN operand comes back
// quieted), and every published value is a quotient, so a reader that sees
// anything else sees the final value -- one relaxed 8-byte store per row, no
// flag, no fence, no second load.  The forward sweep empties `out` row by row
// for the backward sweep; the backward sweep empties y for the next forward
// sweep (each after reading its own entry).
constexpr unsigned long long kIcEmpty = 0x7ff4000000b1c0deULL;

__device__ __forceinline__ double ld_relaxed_f64(const double *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return __longlong_as_double((long long)v);
}

__device__ __forceinline__ void st_relaxed_f64(double *p, double x) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(__double_as_longlong(x)) : "memory");
}

__device__ __forceinline__ double wait_value(const double *p) {
    double x = ld_relaxed_f64(p);
    unsigned n = 0;
    unsigned long long t0 = 0;
    while ((unsigned long long)__double_as_longlong(x) == kIcEmpty) {
        if (KPL_IC0_SPIN_NS > 0) __nanosleep(KPL_IC0_SPIN_NS);
        spin_watchdog(n, t0);
        x = ld_relaxed_f64(p);
    }
    return x;
}

__device__ __forceinline__ double ic_empty() { return __longlong_as_double((long long)kIcEmpty); }

// y = L^-1 v  (lower_solve, _kernels.py:55-63): acc = v[i]; acc -= l*y[c] in
// stored order; y[i] = acc / l[diag].  `v` = pick(head, sel, v0, v1).
__global__ void __launch_bounds__(NT) ic0_lower_kernel(long long n, Tri L, const double *v0, const double *v1,
                                                       int sel, double *out, Ic0Ws s, const WsHead *head,
                                                       int pred, long long row) {
    if (!pred_ok(head, pred, row)) return;
    __shared__ unsigned int s_blk;
    if (threadIdx.x == 0) {
        s_blk = atomicAdd(&s.tickets[0], 1u);
        if (s_blk == 0) s.tickets[1] = 0u;             // re-arm the backward sweep
    }
    __syncthreads();
    const long long t = (long long)s_blk * NT + threadIdx.x;
    if (t >= n) return;
    const long long i = tri_row(L, t, n, false);
    const double *v = pick(head, sel, v0, v1);
    const int lo = L.rp[i], di = L.rp[i + 1] - 1;
    double acc = v[i];
    out[i] = ic_empty();                               // (after reading v[i]: out may alias v)
    for (int k = lo; k < di; ++k)
        acc = __dsub_rn(acc, __dmul_rn(L.v[k], wait_value(s.y + L.ci[k])));
    st_relaxed_f64(s.y + i, __ddiv_rn(acc, L.v[di]));
}

// out = U^-1 y with U = L^T stored by rows, diagonal first (upper_solve,
// _kernels.py:66-74), rows from n-1 down.
__global__ void __launch_bounds__(NT) ic0_upper_kernel(long long n, Tri U, double *out, Ic0Ws s,
                                                       const WsHead *head, int pred, long long row) {
    if (!pred_ok(head, pred, row)) return;
    __shared__ unsigned int s_blk;
    if (threadIdx.x == 0) {
        s_blk = atomicAdd(&s.tickets[1], 1u);
        if (s_blk == 0) s.tickets[0] = 0u;             // re-arm the forward sweep
    }
    __syncthreads();
    const long long t = (long long)s_blk * NT + threadIdx.x;
    if (t >= n) return;
    const long long i = tri_row(U, t, n, true);
    const int di = U.rp[i], hi = U.rp[i + 1];
    double acc = __ldcg(s.y + i);
    s.y[i] = ic_empty();
    for (int k = di + 1; k < hi; ++k)
        acc = __dsub_rn(acc, __dmul_rn(U.v[k], wait_value(out + U.ci[k])));
    st_relaxed_f64(out + i, __ddiv_rn(acc, U.v[di]));
}

// Fill y with kIcEmpty (workspace preparation).
__global__ void ic0_empty_kernel(long long n, double *y) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += gridDim.x * (long long)blockDim.x)
        y[k] = ic_empty();
}

// IC(0) factor (ic0_factor, _kernels.py:77-115) on the lower pattern of A
// (`a`, diagonal last per row; diagonal scaled by dscale = 1 + eta).  Row i needs the finished
// rows c of its strictly-lower columns; the merge walk over the shared
// columns, the division by l[c,c] and the pivot sum run in the reference's
// order.  A non-positive pivot records min(row) in `bad` and publishes NaN,
// so dependants still finish; rows before the first failure are exact.
__global__ void __launch_bounds__(NT) ic0_factor_kernel(long long n, Tri P, const double *a, double dscale,
                                                        double *l, int *flag, unsigned int *ticket,
                                                        unsigned long long *bad) {
    __shared__ unsigned int s_blk;
    if (threadIdx.x == 0) s_blk = atomicAdd(ticket, 1u);
    __syncthreads();
    const long long t = (long long)s_blk * NT + threadIdx.x;
    if (t >= n) return;
    const long long i = tri_row(P, t, n, false);
    const int lo = P.rp[i], di = P.rp[i + 1] - 1;
    for (int kk = lo; kk < di; ++kk) {
        const int c = P.ci[kk];
        wait_flag(flag + c);
        const int dc = P.rp[c + 1] - 1;
        double s = a[kk];
        int p = lo, q = P.rp[c];
        while (p < kk && q < dc) {
            const int cp = P.ci[p], cq = P.ci[q];
            if (cp == cq) {
                s = __dsub_rn(s, __dmul_rn(l[p], __ldcg(l + q)));
                ++p; ++q;
            } else if (cp < cq) {
                ++p;
            } else {
                ++q;
            }
        }
        l[kk] = __ddiv_rn(s, __ldcg(l + dc));
    }
    double d = __dmul_rn(a[di], dscale);               // vals[diag] *= 1 + eta (precond.py:41-42)
    for (int kk = lo; kk < di; ++kk) d = __dsub_rn(d, __dmul_rn(l[kk], l[kk]));
    if (d <= 0.0) {                                   // _kernels.py:112-113 (NaN passes, as there)
        atomicMin(bad, (unsigned long long)i);
        d = __longlong_as_double(0x7ff8000000000000LL);
    } else {
        d = __dsqrt_rn(d);
    }
    __stcg(l + di, d);
    st_release(flag + i, 1);
}

// Dependency levels of a triangle's rows: level[i] = 1 + max level of the
// rows it reads (0 if none), natural order, sync-free.  upper = 0: row i of
// L reads columns < i (diagonal last); upper = 1: row i of L^T reads columns
// > i (diagonal first), rows visited from n-1 down.
__global__ void __launch_bounds__(NT) ic0_levels_kernel(long long n, Tri P, int upper, int *level, int *flag,
                                                        unsigned int *ticket) {
    __shared__ unsigned int s_blk;
    if (threadIdx.x == 0) s_blk = atomicAdd(ticket, 1u);
    __syncthreads();
    const long long t = (long long)s_blk * NT + threadIdx.x;
    if (t >= n) return;
    const long long i = upper ? n - 1 - t : t;
    const int lo = upper ? P.rp[i] + 1 : P.rp[i], hi = upper ? P.rp[i + 1] : P.rp[i + 1] - 1;
    int lv = 0;
    for (int k = lo; k < hi; ++k) {
        const int c = P.ci[k];
        wait_flag(flag + c);
        lv = max(lv, __ldcg(level + c) + 1);
    }
    __stcg(level + i, lv);
    st_release(flag + i, 1);
}

}  // namespace kpl
