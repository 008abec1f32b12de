// kpl_ic0.cuh -- IC(0) preconditioner on the device:
// the factorisation (_kernels.py:77-115) and the forward / backward
// substitutions of its apply (_kernels.py:55-74, precond.py:90-94).
//
// All three are row-sequential recurrences whose dependencies follow the
// sparsity pattern.  They run as *sync-free* sweeps: one thread per row, each
// row waits (acquire-spin) on a per-row ready flag of every row it reads, then
// publishes its own value with a release store.  Rows are handed to CTAs by
// an atomic ticket in dependency order (ascending for L, descending for L^T),
// so a CTA only ever waits on rows owned by CTAs that are already resident --
// no deadlock regardless of grid size.  Inside a row the arithmetic is the
// reference's, term for term (--fmad=false, explicit __d*_rn), so the factor
// and every apply are bit-identical to the reference.
//
// Flags are never reset by a separate pass: the forward sweep clears the
// backward flags of the rows it finishes and vice versa (the other sweep is
// complete by stream order), and each sweep re-arms the other's ticket.
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

__device__ __forceinline__ void wait_flag(const int *f) {
    while (ld_acquire(f) == 0) __nanosleep(20);
}

struct Tri {                // CSR triangle, int32 indices
    const int *rp, *ci;
    const double *v;
};

struct Ic0Ws {              // apply scratch inside the solver workspace
    double *y;              // L^-1 v
    int *fflag, *bflag;     // per-row ready flags of the two sweeps
    unsigned int *tickets;  // [0] forward, [1] backward
};

// y = L^-1 v  (lower_solve, _kernels.py:55-63): acc = v[i]; acc -= l*y[c] in
// stored order; y[i] = acc / l[diag].  `v` = pick(head, sel, v0, v1).
__global__ void __launch_bounds__(NT) ic0_lower_kernel(long long n, Tri L, const double *v0, const double *v1,
                                                       int sel, Ic0Ws s, const WsHead *head, int pred,
                                                       long long row) {
    if (!pred_ok(head, pred, row)) return;
    __shared__ unsigned int s_blk;
    if (threadIdx.x == 0) {
        s_blk = atomicAdd(&s.tickets[0], 1u);
        if (s_blk == 0) s.tickets[1] = 0u;             // re-arm the backward sweep
    }
    __syncthreads();
    const long long i = (long long)s_blk * NT + threadIdx.x;
    if (i >= n) return;
    const double *v = pick(head, sel, v0, v1);
    const int lo = L.rp[i], di = L.rp[i + 1] - 1;
    double acc = v[i];
    for (int k = lo; k < di; ++k) {
        const int c = L.ci[k];
        wait_flag(s.fflag + c);
        acc = __dsub_rn(acc, __dmul_rn(L.v[k], __ldcg(s.y + c)));
    }
    __stcg(s.y + i, __ddiv_rn(acc, L.v[di]));
    s.bflag[i] = 0;
    st_release(s.fflag + i, 1);
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
    const long long j = (long long)s_blk * NT + threadIdx.x;
    if (j >= n) return;
    const long long i = n - 1 - j;
    const int di = U.rp[i], hi = U.rp[i + 1];
    double acc = __ldcg(s.y + i);
    for (int k = di + 1; k < hi; ++k) {
        const int c = U.ci[k];
        wait_flag(s.bflag + c);
        acc = __dsub_rn(acc, __dmul_rn(U.v[k], __ldcg(out + c)));
    }
    __stcg(out + i, __ddiv_rn(acc, U.v[di]));
    s.fflag[i] = 0;
    st_release(s.bflag + i, 1);
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
    const long long i = (long long)s_blk * NT + threadIdx.x;
    if (i >= n) return;
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

}  // namespace kpl
