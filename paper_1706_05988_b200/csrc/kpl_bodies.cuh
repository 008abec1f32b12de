// kpl_bodies.cuh -- per-element work of each sweep (the loop bodies of the
// reference solvers, pkg/src/kpl/solvers.py), plus the stencil-input
// adapters that apply the preconditioner on the fly (m = M^-1 w).
//
// A Body provides:
//   NQ          number of reduced quantities (0 = no reduction)
//   kStencil    whether the sweep computes n = A * xf(input)
//   Regs<V>     the per-element streams it loads
//   setup(ws)   read uniform scalars (alpha, beta, parity) from the workspace
//   load<V>(k, R)                       issue loads of the streams at k..k+V-1
//   compute<V>(k, R, n, cen, acc)       update + accumulate products
// `cen` is the raw stencil input at k (the register queue's centre), so the
// update never re-reads it from memory.
#pragma once
#include <type_traits>
#include "kpl_core.cuh"

namespace kpl {

enum Sel : int { SEL_FIXED = 0, SEL_ITER = 1, SEL_ITER1 = 2 };

// Scalars and the iteration counter are read with ld_head (strong, GPU scope,
// compiler-ordered): inside a persistent kernel they were written after a barrier.
__device__ __forceinline__ const double *pick(const WsHead *h, int sel, const double *a0,
                                              const double *a1) {
    if (sel == SEL_FIXED) return a0;
    const long long par = (ld_head(&h->iter) + (sel == SEL_ITER1 ? 1 : 0)) & 1;
    return par ? a1 : a0;
}

// ----------------------------------------------------- stencil inputs
struct InNone {
    __device__ void setup(const Ws &) {}
    __device__ const double *base() const { return nullptr; }
    template <int V> __device__ void raw(const double *, long long, double (&o)[V]) const {
#pragma unroll
        for (int v = 0; v < V; ++v) o[v] = 0.0;
    }
    __device__ double xf(double r, long long) const { return r; }
};

// Raw vector (optionally a ping-pong pair); PC selects the transform:
//   KPL_PC_IDENTITY: m = w;  KPL_PC_JACOBI_CONST: m = w*c;  KPL_PC_JACOBI_VEC: m = w*d[k]
// (precond.py:88-89 computes v * inv_diag elementwise: one rounding).
// COH (compile time): 0 = read-only path (ld.global.nc); 1 = through L2 only
// (ld.global.cg) -- for vectors written earlier in the same kernel (persistent
// solvers).  A compile-time choice: a runtime flag tested per load kept the
// compiler from batching the loads (the CSR gathers ran 7 % slower with it).
template <int PC, int COH = 0>
struct InVec {
    const double *a0, *a1;
    int sel;
    double c;
    const double *dinv;
    const double *a;
    __device__ void setup(const Ws &ws) { a = pick(ws.head, sel, a0, a1); }
    __device__ const double *base() const { return a; }
    template <int V> __device__ void raw(const double *p, long long k, double (&o)[V]) const {
        if constexpr (COH == 1) {
            if constexpr (V == 2) {
                const double2 t = __ldcg(reinterpret_cast<const double2 *>(p + k));
                o[0] = t.x; o[1] = t.y;
            } else {
                o[0] = __ldcg(p + k);
            }
        } else {
            ld_ro<V>(p, k, o);
        }
    }
    __device__ double xf(double r, long long k) const {
        if constexpr (PC == KPL_PC_JACOBI_CONST) return __dmul_rn(r, c);
        else if constexpr (PC == KPL_PC_JACOBI_VEC) return __dmul_rn(r, __ldg(dinv + k));
        else return r;
    }
};

// One-element load of a CSR operand (gather or row centre).  L2G: plain
// vectors are read L2-direct (ld.global.cg) with no runtime branch on
// the cache policy; other inputs (e.g. classic CG's p = axpy(beta, p, u)) use raw().
template <class T> struct is_invec : std::false_type {};
template <int PC, int COH> struct is_invec<InVec<PC, COH>> : std::true_type {};
template <bool L2G, class In>
__device__ __forceinline__ double load1(const In &in, const double *p, long long k) {
    if constexpr (L2G && is_invec<In>::value) {
        return __ldcg(p + k);
    } else {
        double t[1];
        in.template raw<1>(p, k, t);
        return t[0];
    }
}

// Classic CG direction evaluated where the stencil needs it:
// p_new = axpy(beta, p_old, u) = beta*p_old + u (beta == 0 -> u), solvers.py:269.
struct InCgP {
    const double *p0, *p1, *u;
    const double *p;
    double beta;
    __device__ void setup(const Ws &ws) {
        p = pick(ws.head, SEL_ITER, p0, p1);
        beta = ws.head->cg_beta;
    }
    __device__ const double *base() const { return p; }
    template <int V> __device__ void raw(const double *b, long long k, double (&o)[V]) const {
        if (b != p) { ld_ro<V>(b, k, o); return; }       // halo plane holds p_new
        double pu[V], po[V];
        ld_ro<V>(u, k, pu);
        ld_ro<V>(p, k, po);
#pragma unroll
        for (int v = 0; v < V; ++v) o[v] = axpy1(beta, po[v], pu[v]);
    }
    __device__ double xf(double r, long long) const { return r; }
};

// Shared-memory stream plane accessor for the TMA sweep: stream s of the
// stage at S + s*512, own pair at offset cs.
__device__ __forceinline__ void sm2(const double *S, int s, int cs, double (&o)[2]) {
    const double2 t = *reinterpret_cast<const double2 *>(S + s * 512 + cs);
    o[0] = t.x; o[1] = t.y;
}

// ---------------------------------------------------------------- bodies
// out = A v  (sparse.py:153-160)
struct BodySpmv {
    static constexpr int NQ = 0;
    static constexpr bool kStencil = true;
    double *out;
    template <int V> struct Regs { double d; };
    __device__ void setup(const Ws &) {}
    template <int V> __device__ void load(long long, Regs<V> &) const {}
    template <int V>
    __device__ void compute(long long k, const Regs<V> &, const double (&n)[V], const double (&)[V],
                            double (&)[1][V]) const {
        st_cs<V>(out, k, n);
    }
};

// (a, b) in the tile/chunk tree order (sparse.py:163-169 replacement)
struct BodyDot {
    static constexpr int NQ = 1;
    static constexpr bool kStencil = false;
    Sink sk;              // reference-order product sink
    const double *a, *b;
    template <int V> struct Regs { double a[V], b[V]; };
    __device__ void setup(const Ws &ws) { sk.set(ws); }
    template <int V> __device__ void load(long long k, Regs<V> &R) const {
        ld_cs<V>(a, k, R.a);
        ld_cs<V>(b, k, R.b);
    }
    template <int V>
    __device__ void compute(long long k, const Regs<V> &R, const double (&)[V], const double (&)[V],
                            double (&acc)[1][V]) const {
#pragma unroll
        for (int v = 0; v < V; ++v) accp(acc, 0, v, sk, k, __dmul_rn(R.a[v], R.b[v]));
    }
};

// r = b - A x_in; u = M r; x = x_in (copy when x != x_in).
// Partials (x,x), (r,r), (r,u).  solvers.py:373-375 / :600-601.
template <int PC>
struct BodyInitR {
    static constexpr int NQ = 3;
    static constexpr bool kStencil = true;
    Sink sk;              // reference-order product sink
    const double *b;
    double *x, *r, *u;
    const double *dinv;
    double c;
    int copy_x;
    template <int V> struct Regs { double b[V], d[V]; };
    static constexpr int kTmaStreams = 1;                 // b
    __device__ void setup(const Ws &ws) { sk.set(ws); }
    template <int V> __device__ void load(long long k, Regs<V> &R) const {
        ld_cs<V>(b, k, R.b);
        if constexpr (PC == KPL_PC_JACOBI_VEC) ld_cs<V>(dinv, k, R.d);
    }
    __device__ void load_tma(const double *S, int cs, Regs<2> &R) const { sm2(S, 0, cs, R.b); }
    template <int V>
    __device__ void compute(long long k, const Regs<V> &R, const double (&n)[V], const double (&xin)[V],
                            double (&acc)[NQ][V]) const {
        double rr[V], uu[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            rr[v] = __dsub_rn(R.b[v], n[v]);
            if constexpr (PC == KPL_PC_IDENTITY) uu[v] = rr[v];
            else if constexpr (PC == KPL_PC_JACOBI_CONST) uu[v] = __dmul_rn(rr[v], c);
            else if constexpr (PC == KPL_PC_JACOBI_VEC) uu[v] = __dmul_rn(rr[v], R.d[v]);
            else uu[v] = 0.0;                 // IC(0): u = M r by the substitution sweeps after
            accp(acc, 0, v, sk, k, __dmul_rn(xin[v], xin[v]));
            accp(acc, 1, v, sk, k, __dmul_rn(rr[v], rr[v]));
            accp(acc, 2, v, sk, k, __dmul_rn(rr[v], uu[v]));
        }
        st_cs<V>(r, k, rr);
        if constexpr (PC != KPL_PC_IDENTITY && PC != KPL_PC_IC0) st_cs<V>(u, k, uu);
        if (copy_x) st_cs<V>(x, k, xin);
    }
};

// ||b - A x||^2 (the true-residual cadence, solvers.py:233-234, :401-402)
struct BodyTrue {
    static constexpr int NQ = 1;
    static constexpr bool kStencil = true;
    Sink sk;              // reference-order product sink
    const double *b;
    template <int V> struct Regs { double b[V]; };
    static constexpr int kTmaStreams = 1;                 // b
    __device__ void setup(const Ws &ws) { sk.set(ws); }
    template <int V> __device__ void load(long long k, Regs<V> &R) const { ld_cs<V>(b, k, R.b); }
    __device__ void load_tma(const double *S, int cs, Regs<2> &R) const { sm2(S, 0, cs, R.b); }
    template <int V>
    __device__ void compute(long long k, const Regs<V> &R, const double (&n)[V], const double (&)[V],
                            double (&acc)[1][V]) const {
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const double t = __dsub_rn(R.b[v], n[v]);
            accp(acc, 0, v, sk, k, __dmul_rn(t, t));
        }
    }
};

// w = axpy(-sigma, r, A u); partials gamma=(r,u), delta=(axpy(sigma,r,w),u), rho=(r,r).
// solvers.py:376 and :388-390 for i = 0 (and :312 for pcg / pcg_rr, sigma = 0).
struct BodyInitW {
    static constexpr int NQ = 3;
    static constexpr bool kStencil = true;
    Sink sk;              // reference-order product sink
    const double *r, *u;
    double *w;
    double sigma;
    int ident;
    const double *dinv;    // with mout: m = w * inv_diag for the CSR SpMV
    double *mout;
    template <int V> struct Regs { double r[V], u[V], d[V]; };
    static constexpr int kTmaStreams = 1;                 // r (identity preconditioner: u == r)
    __device__ void setup(const Ws &ws) { sk.set(ws); }
    template <int V> __device__ void load(long long k, Regs<V> &R) const {
        ld_cs<V>(r, k, R.r);
        if (!ident) ld_cs<V>(u, k, R.u);
        if (mout) ld_cs<V>(dinv, k, R.d);
    }
    __device__ void load_tma(const double *S, int cs, Regs<2> &R) const { sm2(S, 0, cs, R.r); }
    template <int V>
    __device__ void compute(long long k, const Regs<V> &R, const double (&n)[V], const double (&uc)[V],
                            double (&acc)[NQ][V]) const {
        double ww[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const double uu = uc[v];
            ww[v] = axpy1(-sigma, R.r[v], n[v]);
            const double dv = axpy1(sigma, R.r[v], ww[v]);
            accp(acc, 0, v, sk, k, __dmul_rn(R.r[v], uu));
            accp(acc, 1, v, sk, k, __dmul_rn(dv, uu));
            accp(acc, 2, v, sk, k, __dmul_rn(R.r[v], R.r[v]));
        }
        st_cs<V>(w, k, ww);
        if (mout) {
            double mm[V];
#pragma unroll
            for (int v = 0; v < V; ++v) mm[v] = __dmul_rn(ww[v], R.d[v]);
            st_cs<V>(mout, k, mm);
        }
    }
};

// One p-CG-sh update (solvers.py:408-421) fused with the next iteration's
// reductions (solvers.py:388-390) -- the hot path.  m = M^-1 w is applied by
// the stencil input; n = A m arrives in `n`; `wc` is this element's w.
// PC == IDENTITY: u, q, p alias r, s, t (bitwise equal in the reference) and
// are neither loaded nor stored.  Partials: gamma=(r,u), delta=(sigma r + w, u),
// rho=(r,r), xi=(x,x) (pcg_rr trigger only).
//
// VAR (pcg_var_sh, solvers.py:479-495): the shift changes from sigma_prev =
// schedule[i] to sigma_cur = schedule[i+1]; dsig = sigma_cur - sigma_prev
// enters the s, q, z and w recurrences with the reference's evaluation order
// (t, p first; s, q; z; x; w before r, which it reads).
template <int PC, bool VAR = false>
struct BodyPcgIter {
    static constexpr int NQ = 4;
    static constexpr bool kStencil = true;
    Sink sk;              // reference-order product sink
    double *x, *r, *u, *z, *q, *s, *t, *p;
    double *w0, *w1;
    const double *dinv;
    double c, sigma;
    int want_xi;
    double alpha, beta, asig;
    double *wout;
    const double *schedule;
    double dsig;
    double *mout;          // CSR + vector Jacobi: also store m = w * inv_diag (next SpMV input)
    const double *mld;     // IC(0): m = M^-1 w, materialised by the substitution sweeps
    template <int V> struct Regs { double x[V], r[V], z[V], s[V], t[V], u[V], q[V], p[V], d[V]; };
    // x, r, z, s, t (+ u, q, p with a constant-diagonal Jacobi)
    static constexpr int kTmaStreams = PC == KPL_PC_IDENTITY ? 5 : 8;
    __device__ void load_tma(const double *S, int cs, Regs<2> &R) const {
        sm2(S, 0, cs, R.x); sm2(S, 1, cs, R.r); sm2(S, 2, cs, R.z); sm2(S, 3, cs, R.s); sm2(S, 4, cs, R.t);
        if constexpr (PC != KPL_PC_IDENTITY) { sm2(S, 5, cs, R.u); sm2(S, 6, cs, R.q); sm2(S, 7, cs, R.p); }
    }
    __device__ void setup(const Ws &ws) {
        sk.set(ws);
        alpha = ld_head(&ws.head->alpha);
        beta = ld_head(&ws.head->beta);
        if constexpr (VAR) {
            const long long i = ld_head(&ws.head->iter);
            const double sp = schedule[i];
            sigma = schedule[i + 1];                    // sigma_cur; also the next delta's shift
            dsig = __dsub_rn(sigma, sp);                // solvers.py:481
        }
        asig = __dmul_rn(alpha, sigma);                 // solvers.py:416 / :493
        wout = const_cast<double *>(pick(ws.head, SEL_ITER1, w0, w1));
    }
    template <int V> __device__ void load(long long k, Regs<V> &R) const {
        ld_cs<V>(x, k, R.x);
        ld_cs<V>(r, k, R.r);
        ld_cs<V>(z, k, R.z);
        ld_cs<V>(s, k, R.s);
        ld_cs<V>(t, k, R.t);
        if constexpr (PC != KPL_PC_IDENTITY) {
            ld_cs<V>(u, k, R.u);
            ld_cs<V>(q, k, R.q);
            ld_cs<V>(p, k, R.p);
        }
        if constexpr (PC == KPL_PC_JACOBI_VEC) ld_cs<V>(dinv, k, R.d);
        if constexpr (PC == KPL_PC_IC0) ld_cs<V>(mld, k, R.d);
    }
    template <int V>
    __device__ void compute(long long k, const Regs<V> &R, const double (&n)[V], const double (&wc)[V],
                            double (&acc)[NQ][V]) const {
        double xo[V], ro[V], zo[V], so[V], to[V], wo[V], uo[V], qo[V], po[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const double w = wc[v];
            double m;
            if constexpr (PC == KPL_PC_IDENTITY) m = w;
            else if constexpr (PC == KPL_PC_JACOBI_CONST) m = __dmul_rn(w, c);
            else if constexpr (PC == KPL_PC_JACOBI_VEC) m = __dmul_rn(w, R.d[v]);
            else m = R.d[v];                                   // IC(0): loaded m
            const double uin = (PC == KPL_PC_IDENTITY) ? R.r[v] : R.u[v];
            double qn, pn;
            if constexpr (!VAR) {
                zo[v] = axpy1(beta, R.z[v], n[v]);              // z = axpy(beta, z, n)
                so[v] = axpy1(beta, R.s[v], w);                 // s = axpy(beta, s, w)
                to[v] = axpy1(beta, R.t[v], R.r[v]);            // t = axpy(beta, t, r)
                if constexpr (PC == KPL_PC_IDENTITY) { qn = so[v]; pn = to[v]; }
                else {
                    qn = axpy1(beta, R.q[v], m);                // q = axpy(beta, q, m)
                    pn = axpy1(beta, R.p[v], uin);              // p = axpy(beta, p, u)
                }
            } else {
                const double md = -dsig;
                to[v] = axpy1(beta, R.t[v], R.r[v]);            // t = axpy(beta, t, r)
                pn = (PC == KPL_PC_IDENTITY) ? to[v] : axpy1(beta, R.p[v], uin);   // p = axpy(beta, p, u)
                so[v] = axpy1(md, to[v], axpy1(beta, R.s[v], w));                  // s = axpy(-dsig, t, axpy(beta, s, w))
                qn = (PC == KPL_PC_IDENTITY) ? so[v] : axpy1(md, pn, axpy1(beta, R.q[v], m));
                const double zb = axpy1(beta, R.z[v], n[v]);    // zbase = axpy(beta, z, n)
                zo[v] = dsig == 0.0 ? zb : axpy1(md, axpy1(sigma, to[v], so[v]), zb);
            }
            qo[v] = qn; po[v] = pn;
            xo[v] = axpy1(alpha, pn, R.x[v]);                   // x = axpy(alpha, p, x)
            if constexpr (VAR) wo[v] = sub2(w, alpha, zo[v], dsig, R.r[v]);   // w = _sub2(w, a, z, dsig, r)
            ro[v] = sub2(R.r[v], alpha, so[v], asig, to[v]);    // r = _sub2(r, a, s, asig, t)
            if constexpr (PC == KPL_PC_IDENTITY) uo[v] = ro[v];
            else uo[v] = sub2(uin, alpha, qn, asig, pn);        // u = _sub2(u, a, q, asig, p)
            if constexpr (!VAR) wo[v] = __dsub_rn(w, __dmul_rn(alpha, zo[v]));   // w = w - alpha*z
            const double dv = axpy1(sigma, ro[v], wo[v]);       // axpy(sigma, r, w)
            accp(acc, 0, v, sk, k, __dmul_rn(ro[v], uo[v]));
            accp(acc, 1, v, sk, k, __dmul_rn(dv, uo[v]));
            accp(acc, 2, v, sk, k, __dmul_rn(ro[v], ro[v]));
            if (want_xi) accp(acc, 3, v, sk, k, __dmul_rn(xo[v], xo[v]));
        }
        st_cs<V>(x, k, xo);
        st_cs<V>(r, k, ro);
        st_cs<V>(z, k, zo);
        st_cs<V>(s, k, so);
        st_cs<V>(t, k, to);
        st_cs<V>(wout, k, wo);
        if constexpr (PC != KPL_PC_IDENTITY) {
            st_cs<V>(u, k, uo);
            st_cs<V>(q, k, qo);
            st_cs<V>(p, k, po);
        }
        if constexpr (PC == KPL_PC_JACOBI_VEC) {
            if (mout) {
                double mo[V];
#pragma unroll
                for (int v = 0; v < V; ++v) mo[v] = __dmul_rn(wo[v], R.d[v]);   // precond.py:89
                st_cs<V>(mout, k, mo);
            }
        }
    }
};

// bodies a deferred peer fold may precede (kpl_sweep_peer, KPL_SW_ITER)
template <class B> struct is_pcg_iter : std::false_type {};
template <int PC, bool VAR> struct is_pcg_iter<BodyPcgIter<PC, VAR>> : std::true_type {};

// track_gaps record sweeps (solvers.py:142-167, gap_vectors / measure_gaps):
//   F: input x;  t = b - A x -> (t,t), (t - r, t - r)
//   G: input p;  axpy(-sigma_prev, t, A p) - s
//   H: input u;  axpy(-sigma_prev, r, A u) - w
//   J: input q;  A q - z
// sigma_prev is the record's shift (schedule[i] for pcg_var_sh).
enum GapMode : int { GAP_F = 0, GAP_G = 1, GAP_H = 2, GAP_J = 3 };

template <int MODE>
struct BodyGap {
    static constexpr int NQ = MODE == GAP_F ? 2 : 1;
    static constexpr bool kStencil = true;
    Sink sk;              // reference-order product sink
    const double *b, *r, *t, *s, *z, *w0, *w1;
    const double *schedule;
    double sig;
    const double *w;
    template <int V> struct Regs { double a[V], c[V]; };
    __device__ void setup(const Ws &ws) {
        sk.set(ws);
        w = pick(ws.head, SEL_ITER, w0, w1);
        if (schedule) sig = schedule[ws.head->iter];
    }
    template <int V> __device__ void load(long long k, Regs<V> &R) const {
        if constexpr (MODE == GAP_F) { ld_cs<V>(b, k, R.a); ld_cs<V>(r, k, R.c); }
        if constexpr (MODE == GAP_G) { ld_cs<V>(t, k, R.a); ld_cs<V>(s, k, R.c); }
        if constexpr (MODE == GAP_H) { ld_cs<V>(r, k, R.a); ld_cs<V>(w, k, R.c); }
        if constexpr (MODE == GAP_J) { ld_cs<V>(z, k, R.c); }
    }
    template <int V>
    __device__ void compute(long long k, const Regs<V> &R, const double (&n)[V], const double (&)[V],
                            double (&acc)[NQ][V]) const {
#pragma unroll
        for (int v = 0; v < V; ++v) {
            if constexpr (MODE == GAP_F) {
                const double tr = __dsub_rn(R.a[v], n[v]);
                const double f = __dsub_rn(tr, R.c[v]);
                accp(acc, 0, v, sk, k, __dmul_rn(tr, tr));
                accp(acc, 1, v, sk, k, __dmul_rn(f, f));
            } else {
                double g;
                if constexpr (MODE == GAP_J) g = __dsub_rn(n[v], R.c[v]);
                else g = __dsub_rn(axpy1(-sig, R.a[v], n[v]), R.c[v]);
                accp(acc, 0, v, sk, k, __dmul_rn(g, g));
            }
        }
    }
};

// Classic CG pass 1 (solvers.py:269-271): p = axpy(beta, p, u) (evaluated by
// InCgP, incl. at neighbours), s = A p, partial delta = (s, p).
struct BodyCgP {
    static constexpr int NQ = 1;
    static constexpr bool kStencil = true;
    Sink sk;              // reference-order product sink
    double *p0, *p1, *s;
    double *pout;
    template <int V> struct Regs { double d; };
    __device__ void setup(const Ws &ws) {
        sk.set(ws);
        pout = const_cast<double *>(pick(ws.head, SEL_ITER1, p0, p1));
    }
    template <int V> __device__ void load(long long, Regs<V> &) const {}
    template <int V>
    __device__ void compute(long long k, const Regs<V> &, const double (&n)[V], const double (&pn)[V],
                            double (&acc)[1][V]) const {
#pragma unroll
        for (int v = 0; v < V; ++v) accp(acc, 0, v, sk, k, __dmul_rn(n[v], pn[v]));
        st_cs<V>(pout, k, pn);
        st_cs<V>(s, k, n);
    }
};

// Classic CG pass 2 (solvers.py:290-292): x = axpy(alpha, p, x); r = r - alpha*s;
// u = M r; partials (r,u), (r,r) of the next head (:258-259).
template <int PC>
struct BodyCgX {
    static constexpr int NQ = 2;
    static constexpr bool kStencil = false;
    Sink sk;              // reference-order product sink
    double *x, *r, *u, *p0, *p1;
    const double *s, *dinv;
    double c, alpha;
    const double *p;
    template <int V> struct Regs { double x[V], r[V], s[V], p[V], d[V]; };
    __device__ void setup(const Ws &ws) {
        sk.set(ws);
        alpha = ws.head->cg_alpha;
        p = pick(ws.head, SEL_ITER1, p0, p1);
    }
    template <int V> __device__ void load(long long k, Regs<V> &R) const {
        ld_cs<V>(x, k, R.x);
        ld_cs<V>(r, k, R.r);
        ld_cs<V>(s, k, R.s);
        ld_cs<V>(p, k, R.p);
        if constexpr (PC == KPL_PC_JACOBI_VEC) ld_cs<V>(dinv, k, R.d);
    }
    template <int V>
    __device__ void compute(long long k, const Regs<V> &R, const double (&)[V], const double (&)[V],
                            double (&acc)[NQ][V]) const {
        double xo[V], ro[V], uo[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            xo[v] = axpy1(alpha, R.p[v], R.x[v]);
            ro[v] = __dsub_rn(R.r[v], __dmul_rn(alpha, R.s[v]));
            if constexpr (PC == KPL_PC_IDENTITY) uo[v] = ro[v];
            else if constexpr (PC == KPL_PC_JACOBI_CONST) uo[v] = __dmul_rn(ro[v], c);
            else if constexpr (PC == KPL_PC_JACOBI_VEC) uo[v] = __dmul_rn(ro[v], R.d[v]);
            else uo[v] = 0.0;                 // IC(0): u after the substitution sweeps
            accp(acc, 0, v, sk, k, __dmul_rn(ro[v], uo[v]));
            accp(acc, 1, v, sk, k, __dmul_rn(ro[v], ro[v]));
        }
        st_cs<V>(x, k, xo);
        st_cs<V>(r, k, ro);
        if constexpr (PC != KPL_PC_IDENTITY && PC != KPL_PC_IC0) st_cs<V>(u, k, uo);
    }
};

// pcg_rr explicit recomputation (solvers.py:600-605), second and third sweeps:
//   mode 0: w = A u (into the buffer the next update reads)
//   mode 1: s = A p, q = M s
template <int PC>
struct BodyRepl {
    static constexpr int NQ = 0;
    static constexpr bool kStencil = true;
    int mode;
    double *w0, *w1, *s, *q;
    const double *dinv;
    double c;
    double *wout;
    double *mout;          // mode 0, CSR + vector Jacobi: m = w * inv_diag
    template <int V> struct Regs { double d[V]; };
    __device__ void setup(const Ws &ws) { wout = const_cast<double *>(pick(ws.head, SEL_ITER1, w0, w1)); }
    template <int V> __device__ void load(long long k, Regs<V> &R) const {
        if constexpr (PC == KPL_PC_JACOBI_VEC) { if (mode == 1 || mout) ld_cs<V>(dinv, k, R.d); }
    }
    template <int V>
    __device__ void compute(long long k, const Regs<V> &R, const double (&n)[V], const double (&)[V],
                            double (&)[1][V]) const {
        if (mode == 0) {
            st_cs<V>(wout, k, n);
            if constexpr (PC == KPL_PC_JACOBI_VEC) {
                if (mout) {
                    double mm[V];
#pragma unroll
                    for (int v = 0; v < V; ++v) mm[v] = __dmul_rn(n[v], R.d[v]);
                    st_cs<V>(mout, k, mm);
                }
            }
            return;
        }
        st_cs<V>(s, k, n);
        if constexpr (PC != KPL_PC_IDENTITY && PC != KPL_PC_IC0) {
            double qq[V];
#pragma unroll
            for (int v = 0; v < V; ++v) {
                if constexpr (PC == KPL_PC_JACOBI_CONST) qq[v] = __dmul_rn(n[v], c);
                else qq[v] = __dmul_rn(n[v], R.d[v]);
            }
            st_cs<V>(q, k, qq);
        }
    }
};

// pcg_rr last replacement sweep: z = A q, then the next record's reductions
// gamma=(r,u), delta=(w,u), rho=(r,r) over the replaced vectors.
struct BodyReplZ {
    static constexpr int NQ = 3;
    static constexpr bool kStencil = true;
    Sink sk;              // reference-order product sink
    double *z;
    const double *r, *u, *w0, *w1;
    int ident;
    const double *w;
    template <int V> struct Regs { double r[V], u[V], w[V]; };
    __device__ void setup(const Ws &ws) { sk.set(ws); w = pick(ws.head, SEL_ITER1, w0, w1); }
    template <int V> __device__ void load(long long k, Regs<V> &R) const {
        ld_cs<V>(r, k, R.r);
        ld_cs<V>(w, k, R.w);
        if (!ident) ld_cs<V>(u, k, R.u);
    }
    template <int V>
    __device__ void compute(long long k, const Regs<V> &R, const double (&n)[V], const double (&)[V],
                            double (&acc)[NQ][V]) const {
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const double uu = ident ? R.r[v] : R.u[v];
            accp(acc, 0, v, sk, k, __dmul_rn(R.r[v], uu));
            accp(acc, 1, v, sk, k, __dmul_rn(R.w[v], uu));
            accp(acc, 2, v, sk, k, __dmul_rn(R.r[v], R.r[v]));
        }
        st_cs<V>(z, k, n);
    }
};

// Products of vector pairs: acc[q] += a[q][k] * b[q][k].  IC(0) runs the
// reductions that the fused bodies cannot (u = M r is produced by the
// substitution sweeps after them) as this separate pass, with the same
// per-element products, so the reduction tree and values are unchanged.
template <int Q>
struct BodyPairs {
    static constexpr int NQ = Q;
    static constexpr bool kStencil = false;
    Sink sk;
    const double *a[Q], *b[Q];
    template <int V> struct Regs { double a[Q][V], b[Q][V]; };
    __device__ void setup(const Ws &ws) { sk.set(ws); }
    template <int V> __device__ void load(long long k, Regs<V> &R) const {
#pragma unroll
        for (int q = 0; q < Q; ++q) { ld_cs<V>(a[q], k, R.a[q]); ld_cs<V>(b[q], k, R.b[q]); }
    }
    template <int V>
    __device__ void compute(long long k, const Regs<V> &R, const double (&)[V], const double (&)[V],
                            double (&acc)[NQ][V]) const {
#pragma unroll
        for (int v = 0; v < V; ++v)
#pragma unroll
            for (int q = 0; q < Q; ++q) accp(acc, q, v, sk, k, __dmul_rn(R.a[q][v], R.b[q][v]));
    }
};

}  // namespace kpl
