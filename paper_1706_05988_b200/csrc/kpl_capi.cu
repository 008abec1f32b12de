// kpl_capi.cu -- extern "C" entry points of libkpl_b200.so (include/kpl_b200.h).
//
// Host side: layout selection, workspace carving, template dispatch on
// (operator kind, vector width, preconditioner), and the per-iteration
// launch sequences of the four solvers.  No allocation, no synchronisation
// except kpl_read_status.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <atomic>
#include <type_traits>
#include <algorithm>

#include <cudaTypedefs.h>
#include <cstdlib>
#include <mutex>

#include "kpl_bodies.cuh"
#include "kpl_sweep.cuh"
#include "kpl_tma.cuh"
#include "kpl_ic0.cuh"
#include "kpl_peer.cuh"
#include "kpl_spmv_band.cuh"

using namespace kpl;

namespace {

thread_local std::string g_err;
std::atomic<long long> g_launches{0};   // kernels this library has launched (bench evidence)
// limit of every device-side peer wait (kpl_set_peer_timeout; KPL_PEER_TIMEOUT_S at load)
std::atomic<unsigned long long> g_peer_timeout_ns{[] {
    const char *e = std::getenv("KPL_PEER_TIMEOUT_S");
    const double s = e ? std::atof(e) : 20.0;
    return (unsigned long long)((s > 0.0 ? s : 20.0) * 1e9);
}()};

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

int cuda_check(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(KPL_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return KPL_OK;
}

long long cdiv(long long a, long long b) { return (a + b - 1) / b; }
long long align256(long long v) { return (v + 255) & ~255LL; }

constexpr int kSMs = 148;

// ring slots of the window SpMV that fit next to the running sums and the two windows
// (device.py:band_ring_slots computes the same)
BandRing band_ring(const kpl_op *op) {
    BandRing r{0, 0};
    r.cap = (op->bd_round_max + 63) / 64 * 64;
    const long long room = 227LL * 1024 - 8LL * op->bd_rows - 16LL * op->bd_w - 128;
    r.ns = (int)std::max<long long>(0, std::min<long long>(12, room / (long long)r.slot()));
    return r;
}

int make_layout(const kpl_op *op, Layout &L) {
    if (!op) return fail(KPL_EINVAL, "null operator");
    std::memset(&L, 0, sizeof(L));
    if (op->order != KPL_ORDER_TREE && op->order != KPL_ORDER_BLOCKED8) return fail(KPL_EINVAL, "unknown order");
    if (op->order == KPL_ORDER_BLOCKED8 && op->chunks_global > 0)
        return fail(KPL_EUNSUPPORTED, "reference (blocked) order is single-GPU only");
    if (op->precond == KPL_PC_IC0 && (op->kind != KPL_OP_CSR || op->chunks_global > 0))
        return fail(KPL_EUNSUPPORTED, "IC(0) runs with single-GPU CSR operators");
    if (op->kind == KPL_OP_STENCIL) {
        if (op->nx < 1 || op->ny < 1 || op->nz < 1) return fail(KPL_EINVAL, "grid dimensions must be >= 1");
        if (op->n != op->nx * op->ny * op->nz) return fail(KPL_EINVAL, "n != nx*ny*nz");
        int vx = op->vx ? op->vx : ((op->nx % 2 == 0) ? 2 : 1);
        if (vx != 1 && vx != 2) return fail(KPL_EINVAL, "vx must be 1 or 2");
        if (vx == 2 && (op->nx % 2)) return fail(KPL_EINVAL, "vx=2 needs an even nx");
        L.vx = vx;
        if (op->ny == 1) { L.wx = NWARP; L.wy = 1; } else { L.wx = 1; L.wy = NWARP; }
        const long long TX = 32LL * vx * L.wx, TY = L.wy;
        L.ntx = (int)cdiv(op->nx, TX);
        L.nty = (int)cdiv(op->ny, TY);
        L.T = L.ntx * L.nty;
        int zc = op->zc;
        if (zc <= 0) {
            zc = 16;   // shrink until the grid has >= 4 CTAs per SM
            while (zc > 1 && (long long)L.T * cdiv(op->nz, zc) < 4LL * kSMs) zc >>= 1;
        }
        L.zc = zc;
        L.nch = cdiv(op->nz, zc);
        L.items = L.nch * L.T;
        return KPL_OK;
    }
    if (op->kind == KPL_OP_CSR) {
        if (op->n < 1) return fail(KPL_EINVAL, "matrix dimension must be >= 1");
        // row_ptr == NULL describes a plain vector (dot / axpy layout, no SpMV)
        if (op->row_ptr && ((!op->col_idx && op->nnz) || (!op->values && op->nnz)))
            return fail(KPL_EINVAL, "CSR arrays missing");
        const long long blocks = cdiv(op->n, RB);
        const int cb = op->chunk_blocks > 0 ? op->chunk_blocks : 8;
        if (cb > 64) return fail(KPL_EINVAL, "chunk_blocks must be <= 64");
        if (op->sp_col && (!op->sp_val || !op->sp_dest || op->sp_rows < 1 || op->sp_max < 1 ||
                           op->sp_max > 65535 || 8LL * op->sp_max > 227 * 1024))
            return fail(KPL_EINVAL, "bad column-sorted SpMV layout");
        if (op->bd_stream && (!op->bd_roff || !op->bd_sb || !op->bd_win ||
                           op->bd_rows < 32 || op->bd_rows % 32 || op->bd_rows > 4608 || op->bd_w < 2 ||
                           (op->bd_w & 1) || op->bd_w > 65536 || op->bd_round_max < 0 || band_ring(op).ns < 2))
            return fail(KPL_EINVAL, "bad window SpMV layout");
        L.vx = 1; L.wx = NWARP; L.wy = 1; L.zc = cb;
        L.T = cb;
        L.items = blocks;
        L.nch = cdiv(blocks, cb);
        return KPL_OK;
    }
    return fail(KPL_EINVAL, "unknown operator kind");
}

struct Offsets { long long items, chunks, cnt, hist, reps, nbuf, mbuf, prod, ic0, pheads, total; };

// Persistent redundant-epilogue kernel (small single-GPU stencils): one head +
// scratch history row per CTA beyond the first (CTA 0 uses the real head).
constexpr long long kPersistMaxCtas = 2LL * kSMs;
constexpr long long kPheadBytes = 1024 + 256;
bool has_pheads(const kpl_op *op) { return op->kind == KPL_OP_STENCIL && op->chunks_global <= 0; }

bool is_ic0(const kpl_op *op) { return op->precond == KPL_PC_IC0; }

bool ordered(const kpl_op *op) { return op->order == KPL_ORDER_BLOCKED8; }

// CSR with a vector Jacobi on one GPU keeps m = w * inv_diag next to w, so the
// SpMV gathers one vector per nonzero instead of two (w and inv_diag).
bool use_mbuf(const kpl_op *op) {
    return op->kind == KPL_OP_CSR && op->row_ptr && op->chunks_global <= 0 &&
           (op->precond == KPL_PC_JACOBI_VEC || op->precond == KPL_PC_IC0);
}

Offsets offsets(const kpl_op *op, const Layout &L, long long max_iters) {
    Offsets o;
    const long long cg = op->chunks_global > 0 ? op->chunks_global : L.nch;
    o.items = 1024;                    // two item buffers (the persistent kernel alternates them)
    o.chunks = o.items + 2 * align256(8LL * NQ * L.items);
    o.cnt = o.chunks + align256(8LL * NQ * cg);
    o.hist = o.cnt + align256(4LL * L.nch);
    o.reps = o.hist + align256(8LL * HC * (max_iters + 1));
    o.nbuf = o.reps + align256(8LL * (max_iters + 1));
    o.mbuf = o.nbuf + (op->kind == KPL_OP_CSR && op->row_ptr ? align256(8LL * op->n) : 0);
    o.prod = o.mbuf + (use_mbuf(op) ? align256(8LL * op->n) : 0);
    o.ic0 = o.prod + (ordered(op) ? align256(8LL * NQ * op->n) : 0);
    // IC(0): y = L^-1 v, two tickets
    o.pheads = o.ic0 + (is_ic0(op) ? align256(8LL * op->n) + 256 : 0);
    o.total = o.pheads + (has_pheads(op) ? kPersistMaxCtas * kPheadBytes : 0);
    return o;
}

Ws make_ws(const kpl_op *op, const Layout &L, long long max_iters, void *workspace) {
    const Offsets o = offsets(op, L, max_iters);
    char *base = static_cast<char *>(workspace);
    Ws ws;
    ws.head = reinterpret_cast<WsHead *>(base);
    ws.items = reinterpret_cast<double *>(base + o.items);
    ws.chunks = reinterpret_cast<double *>(base + o.chunks);
    ws.chunk_cnt = reinterpret_cast<unsigned int *>(base + o.cnt);
    ws.hist = reinterpret_cast<double *>(base + o.hist);
    ws.reps = reinterpret_cast<long long *>(base + o.reps);
    ws.nbuf = reinterpret_cast<double *>(base + o.nbuf);
    ws.mbuf = use_mbuf(op) ? reinterpret_cast<double *>(base + o.mbuf) : nullptr;
    ws.chunk_offset = op->chunks_global > 0 ? op->chunk_offset : 0;
    ws.chunks_global = op->chunks_global > 0 ? op->chunks_global : L.nch;
    ws.inline_final = op->chunks_global > 0 || ordered(op) ? 0 : 1;
    ws.prod = ordered(op) ? reinterpret_cast<double *>(base + o.prod) : nullptr;
    ws.nprod = op->n;
    ws.hist_scratch = 0;
    ws.px = nullptr;
    ws.epoch = 0;
    ws.tpar = ws.push = ws.wpar = 0;
    ws.wait_epoch = 0;
    ws.wait_tpar = 0;
    ws.timeout_ns = g_peer_timeout_ns.load(std::memory_order_relaxed);
    ws.final_cnt = &ws.head->final_cnt;
    return ws;
}

Ic0Ws make_ic0_ws(const kpl_op *op, const Layout &L, long long max_iters, void *workspace) {
    Ic0Ws s{};
    if (!is_ic0(op)) return s;
    const Offsets o = offsets(op, L, max_iters);
    char *base = static_cast<char *>(workspace) + o.ic0;
    s.y = reinterpret_cast<double *>(base);
    s.tickets = reinterpret_cast<unsigned int *>(base + align256(8LL * op->n));
    return s;
}

Tri ic0_lower(const kpl_op *op) {
    return Tri{op->ic_l_row_ptr, op->ic_l_col_idx, op->ic_l_values, op->ic_l_order};
}
Tri ic0_upper(const kpl_op *op) {
    return Tri{op->ic_u_row_ptr, op->ic_u_col_idx, op->ic_u_values, op->ic_u_order};
}

// out = U^-1 L^-1 pick(v0, v1): the two sync-free substitution sweeps
int ic0_apply(const kpl_op *op, const Ic0Ws &s, const WsHead *head, const double *v0, const double *v1,
              int sel, double *out, int pred, long long row, cudaStream_t st) {
    if (!op->ic_l_row_ptr || !op->ic_u_row_ptr) return fail(KPL_EINVAL, "IC(0) factor arrays missing");
    const unsigned grid = (unsigned)cdiv(op->n, NT);
    g_launches.fetch_add(2, std::memory_order_relaxed);
    ic0_lower_kernel<<<grid, NT, 0, st>>>(op->n, ic0_lower(op), v0, v1, sel, out, s, head, pred, row);
    ic0_upper_kernel<<<grid, NT, 0, st>>>(op->n, ic0_upper(op), out, s, head, pred, row);
    return cuda_check("IC(0) apply");
}

// y := empty, tickets := 0 (before the first apply on a workspace)
int ic0_reset(const kpl_op *op, const Ic0Ws &s, cudaStream_t st) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    ic0_empty_kernel<<<(unsigned)std::min<long long>(cdiv(op->n, 256), 148LL * 8), 256, 0, st>>>(op->n, s.y);
    cudaMemsetAsync(s.tickets, 0, 2 * sizeof(unsigned int), st);
    return cuda_check("IC(0) reset");
}

Cfg make_cfg(const kpl_cfg *c) {
    Cfg k;
    k.method = c ? c->method : KPL_M_PCG_SH;
    k.track_gaps = c ? c->track_gaps : 0;
    k.schedule = c ? c->shift_schedule : nullptr;
    k.shift = c ? c->shift : 0.0;
    k.rtol = c ? c->rtol : 0.0;
    k.tau = c ? c->rr_threshold : 0.0;
    k.coef = c ? c->rr_coef : 0.0;
    k.max_iters = c ? c->max_iters : 0;
    return k;
}

// ------------------------------------------------------------ dispatch
struct NoSpmvIn {};

// Launch with programmatic stream serialisation (PDL): the kernel's CTAs may be
// scheduled while the previous kernel drains; the kernel itself starts with
// griddepcontrol.wait.  KPL_PDL=0 launches normally.
template <class Kern, class... Args>
void launch_pdl(Kern kern, unsigned grid, unsigned block, size_t smem, cudaStream_t st, Args... args) {
    static const bool off = [] { const char *e = std::getenv("KPL_PDL"); return e && e[0] == '0'; }();
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(block);
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = off ? 0 : 1;
    cudaLaunchKernelEx(&lc, kern, args...);
}

// Column-sorted SpMV launch (kpl_op.sp_*): dynamic shared memory of the
// largest block's products; KPL_SORTED_NT picks the CTA size (tuning knob).
template <class SIn, int NTS, int PER>
void launch_sorted_nt(const CGeo &g, const SGather &sg, const SIn &in, double *out, const Ws &ws, int pred,
                      long long row, unsigned grid, size_t smem, cudaStream_t st) {
    auto kern = csr_sorted_spmv<SIn, NTS, PER>;
    if (smem > 48 * 1024)    // per device and cheap: set before every launch
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_pdl(kern, grid, NTS, smem, st, g, sg, in, out, ws, pred, row);
}
template <class SIn>
void launch_sorted(const kpl_op *op, const CGeo &g, const SIn &in, double *out, const Ws &ws, int pred,
                   long long row, cudaStream_t st) {
    static const int nts = [] { const char *e = std::getenv("KPL_SORTED_NT"); return e ? std::atoi(e) : 512; }();
    static const int per = [] { const char *e = std::getenv("KPL_SORTED_PER"); return e ? std::atoi(e) : 4; }();
    const SGather sg{op->sp_col, op->sp_val, reinterpret_cast<const unsigned short *>(op->sp_dest), op->sp_rows};
    const long long nblk = cdiv(op->n, op->sp_rows);
    // (a bulk-TMA-fed variant of this kernel was removed in r2: tools/stress_spmv.py found it returning
    // wrong rows in ~2 % of the launches under concurrent load)
    const size_t smem = 8 * (size_t)op->sp_max;
    // persistent: one CTA per SM (two when the products fit twice), striding over the
    // blocks so the next block's first stream loads overlap this block's row sums
    const long long per_sm = smem > 110 * 1024 ? 1 : 2;
    const unsigned grid = (unsigned)std::min(nblk, pred == PRED_FIRE ? 2LL * kSMs : per_sm * kSMs);
    if (nts == 1024) {
        if (per == 8) launch_sorted_nt<SIn, 1024, 8>(g, sg, in, out, ws, pred, row, grid, smem, st);
        else launch_sorted_nt<SIn, 1024, 4>(g, sg, in, out, ws, pred, row, grid, smem, st);
    } else {
        if (per == 8) launch_sorted_nt<SIn, 512, 8>(g, sg, in, out, ws, pred, row, grid, smem, st);
        else launch_sorted_nt<SIn, 512, 4>(g, sg, in, out, ws, pred, row, grid, smem, st);
    }
}

// Shared-memory-window SpMV (kpl_op.bd_*): one CTA per super-block of bd_rows rows.
// Taken for plain vector inputs whose storage allows 16-byte bulk copies; anything
// else (a Jacobi diagonal gathered per column, multi-GPU row blocks) keeps the
// CSR-order kernels.
template <class SIn> struct band_capable : std::false_type {};
template <> struct band_capable<InVec<KPL_PC_IDENTITY, 0>> : std::true_type {};

template <class SIn>
bool band_ok(const kpl_op *op, const SIn &in) {
    if constexpr (band_capable<SIn>::value) {
        return op->bd_stream && op->chunks_global <= 0 && !((reinterpret_cast<uintptr_t>(in.a0) | reinterpret_cast<uintptr_t>(in.a1)) & 15);
    } else {
        return false;
    }
}

template <class SIn>
void launch_band(const kpl_op *op, const SIn &in, double *out, const Ws &ws, int pred, long long row,
                 cudaStream_t st) {
    if constexpr (band_capable<SIn>::value) {
        const BandGeo bg{op->bd_stream, op->bd_roff, reinterpret_cast<const int4 *>(op->bd_sb), op->bd_win,
                         op->bd_w, op->bd_rows};
        const BandRing ring = band_ring(op);
        auto kern = csr_band_ring_spmv<SIn>;
        const size_t smem = ring.bytes(op->bd_rows, op->bd_w);
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const unsigned grid = (unsigned)cdiv(op->n, (long long)op->bd_rows);
        launch_pdl(kern, grid, BAND_CW * 32 + 32, smem, st, (long long)op->n, bg, ring, in, out, ws, pred, row);
    }
}

// CSR-order SpMV: KPL_SPMV=plain keeps the one-window-at-a-time kernel for A/B
// runs; the default pipelines the next window's loads under the row sums.
template <class SIn>
void launch_csr_spmv(bool long_rows, unsigned grid, cudaStream_t st, const CGeo &g, const SIn &in, double *out,
                     const Ws &ws, int pred, long long row) {
    static const bool plain = [] { const char *e = std::getenv("KPL_SPMV"); return e && !std::strcmp(e, "plain"); }();
    if (plain) {
        if (long_rows) launch_pdl(csr_spmv_kernel<SIn, 512>, grid, NT, 0, st, g, in, out, ws, pred, row);
        else launch_pdl(csr_spmv_kernel<SIn, CSR_WIN, true>, grid, NT, 0, st, g, in, out, ws, pred, row);
        return;
    }
    // long scattered rows: the pipelined kernel (config 5: 0.301 -> 0.287 ms/iteration); short rows keep
    // the one-window kernel at 8 CTAs/SM (pipelined at 6 CTAs/SM: config 4 0.786 -> 0.825, 2-CSR 0.200 -> 0.211)
    if (long_rows) launch_pdl(csr_spmv_pipe<SIn, 512, false, 8>, grid, NT, 0, st, g, in, out, ws, pred, row);
    else launch_pdl(csr_spmv_kernel<SIn, CSR_WIN, true>, grid, NT, 0, st, g, in, out, ws, pred, row);
}

// `spin`: input of the CSR SpMV when it differs from the body's stencil input
// (m = w * inv_diag materialised in the workspace); NoSpmvIn = use `in`.
template <class In, class Body, class SpIn = NoSpmvIn>
int launch(const kpl_op *op, const Layout &L, In in, Body body, const Ws &ws, const Cfg &cfg,
           int phase, int pred, long long row, cudaStream_t st, SpIn spin = SpIn()) {
    if (L.items <= 0) return KPL_OK;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    // the replacement sweeps are predicated on a rare device trigger: a small
    // grid striding over the items keeps their idle cost at a few CTAs
    const long long cap = pred == PRED_FIRE ? 2LL * kSMs : (1LL << 31) - 1;
    if (op->kind == KPL_OP_STENCIL) {
        SGeo g{op->nx, op->ny, op->nz, op->diag, op->halo_lo, op->halo_hi, op->zhalo};
        const unsigned grid = (unsigned)std::min(L.items, cap);
        const bool fold = ws.px && ws.wait_epoch;          // deferred peer fold (kpl_sweep_peer)
        if constexpr (is_pcg_iter<Body>::value) {
            if (fold) {
                if (L.vx == 2)
                    launch_pdl(stencil_sweep<2, In, Body, true>, grid, NT, 0, st, g, L, in, body, ws, cfg, phase,
                               pred, row);
                else
                    launch_pdl(stencil_sweep<1, In, Body, true>, grid, NT, 0, st, g, L, in, body, ws, cfg, phase,
                               pred, row);
                return cuda_check("sweep launch");
            }
        } else if (fold) {
            return fail(KPL_EUNSUPPORTED, "deferred fold: iteration sweeps only");
        }
        if (L.vx == 2)
            launch_pdl(stencil_sweep<2, In, Body>, grid, NT, 0, st, g, L, in, body, ws, cfg, phase, pred, row);
        else
            launch_pdl(stencil_sweep<1, In, Body>, grid, NT, 0, st, g, L, in, body, ws, cfg, phase, pred, row);
    } else {
        // split CSR: high-occupancy SpMV into the workspace, then the chunk sweep
        CGeo g{op->n, op->row_ptr, op->col_idx, op->values};
        if constexpr (Body::kStencil) {
            g_launches.fetch_add(1, std::memory_order_relaxed);
            const unsigned sgrid = (unsigned)std::min(L.items, cap);
            // long rows with scattered columns (> 16 nonzeros per row on average): shorter
            // windows, more resident warps for the gathers (config 5: 0.303 -> 0.296 ms)
            // short rows (structured matrices): gathers L2-direct (configs 2-CSR, 4: -4 %); long
            // scattered rows keep the read-only path (ld.global.nc is 3 % faster on config 5)
            const bool long_rows = op->nnz > 16 * op->n;
            bool band = false;
            if constexpr (std::is_same<SpIn, NoSpmvIn>::value) band = band_ok(op, in);
            else band = band_ok(op, spin);
            if (band) {
                // scattered band: input windows in shared memory, one CTA per super-block
                if constexpr (std::is_same<SpIn, NoSpmvIn>::value) launch_band(op, in, ws.nbuf, ws, pred, row, st);
                else launch_band(op, spin, ws.nbuf, ws, pred, row, st);
            } else if (op->sp_col) {
                // column-sorted gathers (scattered matrices): one CTA per block of sp_rows rows
                if constexpr (std::is_same<SpIn, NoSpmvIn>::value) launch_sorted(op, g, in, ws.nbuf, ws, pred, row, st);
                else launch_sorted(op, g, spin, ws.nbuf, ws, pred, row, st);
            } else if constexpr (std::is_same<SpIn, NoSpmvIn>::value) {
                launch_csr_spmv(long_rows, sgrid, st, g, in, ws.nbuf, ws, pred, row);
            } else {
                launch_csr_spmv(long_rows, sgrid, st, g, spin, ws.nbuf, ws, pred, row);
            }
        }
        launch_pdl(csr_chunk_sweep<In, Body, true>, (unsigned)std::min(L.nch, cap), NT, 0, st, g, L, in, body,
                   (const double *)ws.nbuf, ws, cfg, phase, pred, row);
    }
    if (ws.prod && phase != PH_NONE && Body::NQ > 0) {
        g_launches.fetch_add(1, std::memory_order_relaxed);
        // large even n: the chain fed from a shared-memory ring of bulk copies (same chain, ~8x faster)
        if (ws.nprod >= (1 << 16) && ws.nprod % 2 == 0) {
            cudaFuncSetAttribute(blocked_final_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BF_SMEM);
            blocked_final_tma_kernel<<<1, 64, BF_SMEM, st>>>(ws, cfg, phase, pred, row, Body::NQ);
        } else {
            blocked_final_kernel<<<1, 32, 0, st>>>(ws, cfg, phase, pred, row, Body::NQ);
        }
    }
    return cuda_check("sweep launch");
}

template <int PC, int COH = 0>
InVec<PC, COH> in_vec(const kpl_op *op, const double *a0, const double *a1, int sel) {
    InVec<PC, COH> in;
    in.a0 = a0; in.a1 = a1; in.sel = sel; in.c = op->pc_const; in.dinv = op->inv_diag; in.a = a0;
    return in;
}

// Calls f(std::integral_constant<int, PC>) for the operator's preconditioner.
template <class F>
int with_pc(const kpl_op *op, F &&f) {
    if (op->kind == KPL_OP_STENCIL) {
        if (op->precond == KPL_PC_IDENTITY) return f(std::integral_constant<int, KPL_PC_IDENTITY>());
        if (op->precond == KPL_PC_JACOBI_CONST) return f(std::integral_constant<int, KPL_PC_JACOBI_CONST>());
        return fail(KPL_EUNSUPPORTED, "stencil operators take identity or constant-diagonal Jacobi");
    }
    if (op->precond == KPL_PC_IDENTITY) return f(std::integral_constant<int, KPL_PC_IDENTITY>());
    if (op->precond == KPL_PC_JACOBI_VEC) {
        if (!op->inv_diag) return fail(KPL_EINVAL, "Jacobi needs inv_diag");
        return f(std::integral_constant<int, KPL_PC_JACOBI_VEC>());
    }
    if (op->precond == KPL_PC_IC0) return f(std::integral_constant<int, KPL_PC_IC0>());
    return fail(KPL_EUNSUPPORTED, "CSR operators take identity, vector Jacobi or IC(0)");
}

// ------------------------------------------------------------ TMA path
#ifndef KPL_TMA_DEPTH
#define KPL_TMA_DEPTH 2
#endif
#ifndef KPL_TMA_DEPTH8_2D
#define KPL_TMA_DEPTH8_2D 2
#endif
constexpr int kTmaDepth = KPL_TMA_DEPTH;

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

// ring depth: 2 planes ahead for <= 5 streams (89 KB, 2 CTAs/SM); 1 ahead for
// the 8-stream Jacobi update (86 KB, 2 CTAs/SM)
template <class Body>
constexpr int tma_depth() { return Body::kTmaStreams > 5 ? 1 : kTmaDepth; }
template <class Body, bool TWO_D>
constexpr int tma_depth2() { return (TWO_D && Body::kTmaStreams > 5) ? KPL_TMA_DEPTH8_2D : tma_depth<Body>(); }

template <class Body, int PCIN = 0>
void tma_prepare() {
    cudaFuncSetAttribute(tma_sweep<Body, tma_depth2<Body, false>(), PCIN, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)TmaRing<tma_depth2<Body, false>(), Body::kTmaStreams, false>::bytes());
    cudaFuncSetAttribute(tma_sweep<Body, tma_depth2<Body, true>(), PCIN, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)TmaRing<tma_depth2<Body, true>(), Body::kTmaStreams, true>::bytes());
    if constexpr (is_pcg_iter<Body>::value) {        // the deferred-fold variants (multi-GPU)
        cudaFuncSetAttribute(tma_sweep<Body, tma_depth2<Body, false>(), PCIN, false, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)TmaRing<tma_depth2<Body, false>(), Body::kTmaStreams, false>::bytes());
        cudaFuncSetAttribute(tma_sweep<Body, tma_depth2<Body, true>(), PCIN, true, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)TmaRing<tma_depth2<Body, true>(), Body::kTmaStreams, true>::bytes());
    }
    cudaGetLastError();
}

bool tma_available() {
    std::call_once(g_encode_once, [] {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
        cudaGetLastError();
        if (g_encode) {
            tma_prepare<BodyPcgIter<KPL_PC_IDENTITY>>();
            tma_prepare<BodyPcgIter<KPL_PC_JACOBI_CONST>, 1>();
            tma_prepare<BodyTrue>();
            tma_prepare<BodyInitR<KPL_PC_IDENTITY>>();
            tma_prepare<BodyInitR<KPL_PC_JACOBI_CONST>>();
            tma_prepare<BodyInitW>();
        }
    });
    const char *env = std::getenv("KPL_NO_TMA");
    return g_encode != nullptr && !(env && env[0] == '1');
}

bool encode_box(CUtensorMap *m, const double *base, const kpl_op *op, unsigned bx, unsigned by, int zext = 0) {
    // zext = 1: the map starts one plane before `base` and spans nz + 2 planes (z halos)
    base -= zext * op->nx * op->ny;
    const cuuint64_t dims[3] = {(cuuint64_t)op->nx, (cuuint64_t)op->ny, (cuuint64_t)(op->nz + 2 * zext)};
    const cuuint64_t strides[2] = {(cuuint64_t)op->nx * 8, (cuuint64_t)op->nx * op->ny * 8};
    const cuuint32_t box[3] = {bx, by, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    return g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double *>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// TMA sweeps cover the 3D identity-preconditioned stencil sweeps (config 3's
// hot kernel and its cadence/init sweeps); everything else uses the register
// sweep of kpl_sweep.cuh.
bool tma_eligible(const kpl_op *op, const Layout &L) {
    const bool shape3d = L.wx == 1 && L.wy == NWARP;             // 64 x 8 tiles
    const bool shape2d = L.wx == NWARP && L.wy == 1 && op->ny == 1;  // 512 x 1 tiles (2D grids)
    return op->kind == KPL_OP_STENCIL && op->precond != KPL_PC_JACOBI_VEC && L.vx == 2 && !ordered(op) &&
           (shape3d || shape2d) && !op->halo_lo && !op->halo_hi && op->nx % 2 == 0 && tma_available();
    // (op->zhalo is supported: the stencil-input maps then cover planes -1..nz)
}

// in0/in1: stencil input (ping-pong pair or twice the same vector, wsel 0/1);
// streams: the body's kTmaStreams plane-wise operands.
template <class Body, int PCIN = 0>
int launch_tma(const kpl_op *op, const Layout &L, const double *in0, const double *in1, int wsel,
               const double *const *streams, const Body &body, const Ws &ws, const Cfg &cfg, int phase,
               int pred, long long row, cudaStream_t st) {
    constexpr int NSTR = Body::kTmaStreams;
    constexpr int DEPTH = tma_depth2<Body, false>(), DEPTH2 = tma_depth2<Body, true>();
    TmaMaps maps;
    std::memset(&maps, 0, sizeof(maps));
    const int zext = op->zhalo ? 1 : 0;
    const bool two_d = L.wy == 1;
    const unsigned wbx = two_d ? TmaShape<true>::WBX : TmaShape<false>::WBX;
    const unsigned wby = two_d ? TmaShape<true>::WBY : TmaShape<false>::WBY;
    const unsigned sbx = two_d ? TmaShape<true>::SBX : TmaShape<false>::SBX;
    const unsigned sby = two_d ? TmaShape<true>::SBY : TmaShape<false>::SBY;
    bool ok = encode_box(&maps.w[0], in0, op, wbx, wby, zext) && encode_box(&maps.w[1], in1, op, wbx, wby, zext);
    for (int s = 0; s < NSTR && ok; ++s) ok = encode_box(&maps.s[s], streams[s], op, sbx, sby);
    if (!ok) return fail(KPL_ECUDA, "cuTensorMapEncodeTiled failed");
    SGeo g{op->nx, op->ny, op->nz, op->diag, nullptr, nullptr, op->zhalo};
    g_launches.fetch_add(1, std::memory_order_relaxed);
    const bool fold = ws.px && ws.wait_epoch;
    if constexpr (is_pcg_iter<Body>::value) {
        if (fold) {
            if (two_d)
                launch_pdl(tma_sweep<Body, DEPTH2, PCIN, true, true>, (unsigned)L.items, NT + 32,
                           TmaRing<DEPTH2, NSTR, true>::bytes(), st, maps, g, L, body, ws, cfg, phase, pred, row,
                           wsel, zext, op->pc_const);
            else
                launch_pdl(tma_sweep<Body, DEPTH, PCIN, false, true>, (unsigned)L.items, NT + 32,
                           TmaRing<DEPTH, NSTR, false>::bytes(), st, maps, g, L, body, ws, cfg, phase, pred, row,
                           wsel, zext, op->pc_const);
            return cuda_check("tma sweep launch");
        }
    } else if (fold) {
        return fail(KPL_EUNSUPPORTED, "deferred fold: iteration sweeps only");
    }
    if (two_d)
        launch_pdl(tma_sweep<Body, DEPTH2, PCIN, true>, (unsigned)L.items, NT + 32,
                   TmaRing<DEPTH2, NSTR, true>::bytes(), st, maps, g, L, body, ws, cfg, phase, pred, row, wsel, zext,
                   op->pc_const);
    else
        launch_pdl(tma_sweep<Body, DEPTH, PCIN, false>, (unsigned)L.items, NT + 32,
                   TmaRing<DEPTH, NSTR, false>::bytes(), st, maps, g, L, body, ws, cfg, phase, pred, row, wsel,
                   zext, op->pc_const);
    return cuda_check("tma sweep launch");
}

__global__ void head_init_kernel(WsHead *h, double *hist, long long nrows, unsigned int *cnt, long long ncnt) {
    const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (tid == 0) {
        h->state = KPL_ST_RUNNING;
        h->iter = -1;
        h->converged = 0;
        h->bd_iter = -1;
        h->bd_code = 0;
        h->n_rep = 0;
        h->fire = 0;
        h->alpha = 0.0;
        h->beta = 0.0;
        h->gamma_prev = 0.0;    // solvers.py:382
        h->alpha_prev = 1.0;    // solvers.py:383
        h->final_cnt = 0u;
        h->bar_cnt = 0u;
        h->bar_gen = 0u;
        h->bar_arrive = 0ull;
        h->fold_cnt = 0u;
        h->fold_fail = 0u;
        h->cg_gamma = 0.0;
    }
    const double nan = __longlong_as_double(0x7ff8000000000000LL);
    for (long long k = tid; k < nrows * HC; k += gridDim.x * (long long)blockDim.x) hist[k] = nan;
    for (long long k = tid; k < ncnt; k += gridDim.x * (long long)blockDim.x) cnt[k] = 0u;
}

__global__ void gather_kernel(long long n, const int *__restrict__ idx, const double *__restrict__ src,
                              double *__restrict__ dst) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += gridDim.x * (long long)blockDim.x)
        dst[k] = __ldg(src + idx[k]);
}

// precond.py:88-89: v * inv_diag (one rounding); `d` NULL -> the constant c
__global__ void jacobi_kernel(long long n, const double *__restrict__ d, double c, const double *__restrict__ v,
                              double *__restrict__ out) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += gridDim.x * (long long)blockDim.x)
        out[k] = __dmul_rn(v[k], d ? d[k] : c);
}

__global__ void axpy_kernel(long long n, double a, const double *__restrict__ x, const double *__restrict__ y,
                            double *__restrict__ out) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += gridDim.x * (long long)blockDim.x)
        out[k] = axpy1(a, x[k], y[k]);
}

}  // namespace

// =====================================================================
extern "C" {

int kpl_version(void) { return 1; }

int64_t kpl_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

const char *kpl_last_error(void) { return g_err.c_str(); }

const char *kpl_breakdown_message(int64_t code) {
    switch (code) {
    case BD_NONPOS_RU: return "nonpositive (r, u)";
    case BD_NONPOS_WU: return "nonpositive curvature (w, u)";
    case BD_VANISH_RU: return "vanishing (r, u)";
    case BD_VANISH_DEN: return "vanishing alpha denominator";
    case BD_NONFINITE: return "non-finite coefficients";
    case BD_NONPOS_SP: return "nonpositive curvature (s, p)";
    case BD_PEER_TIMEOUT: return "peer exchange timeout";
    case BD_BARRIER_TIMEOUT: return "device barrier timeout";
    case BD_PEER_FAILED: return "peer rank failed";
    default: return "";
    }
}

int64_t kpl_workspace_bytes(const kpl_op *op, int64_t max_iters) {
    Layout L;
    if (make_layout(op, L) != KPL_OK) return KPL_EINVAL;
    return offsets(op, L, max_iters < 0 ? 0 : max_iters).total;
}

int64_t kpl_history_offset(const kpl_op *op) {
    Layout L;
    if (make_layout(op, L) != KPL_OK) return KPL_EINVAL;
    return offsets(op, L, 0).hist;
}

int64_t kpl_replacements_offset(const kpl_op *op, int64_t max_iters) {
    Layout L;
    if (make_layout(op, L) != KPL_OK) return KPL_EINVAL;
    return offsets(op, L, max_iters).reps;
}

int kpl_reduction_layout(const kpl_op *op, int64_t *out8) {
    Layout L;
    int rc = make_layout(op, L);
    if (rc != KPL_OK) return rc;
    if (op->kind == KPL_OP_STENCIL) {
        const int64_t v[8] = {L.vx, L.wx, L.wy, L.zc, L.ntx, L.nty, L.nch, L.T};
        std::memcpy(out8, v, sizeof(v));
    } else {
        const int64_t v[8] = {1, RB, 1, L.zc, 0, 0, L.nch, L.T};
        std::memcpy(out8, v, sizeof(v));
    }
    return KPL_OK;
}

static int need_matrix(const kpl_op *op) {
    if (op->kind == KPL_OP_CSR && !op->row_ptr) return fail(KPL_EINVAL, "CSR arrays missing");
    return KPL_OK;
}

int kpl_spmv(const kpl_op *op, const double *v, double *out, void *stream) {
    Layout L;
    int rc = make_layout(op, L);
    if (rc != KPL_OK) return rc;
    if ((rc = need_matrix(op)) != KPL_OK) return rc;
    Ws ws{};
    Cfg cfg{};
    BodySpmv body;
    body.out = out;
    InVec<KPL_PC_IDENTITY> in = in_vec<KPL_PC_IDENTITY>(op, v, v, SEL_FIXED);
    if (op->kind == KPL_OP_CSR) {
        CGeo g{op->n, op->row_ptr, op->col_idx, op->values};
        g_launches.fetch_add(1, std::memory_order_relaxed);
        if (band_ok(op, in) && !(reinterpret_cast<uintptr_t>(v) & 15))
            launch_band(op, in, out, ws, PRED_ALWAYS, 0, (cudaStream_t)stream);
        else if (op->sp_col)
            launch_sorted(op, g, in, out, ws, PRED_ALWAYS, 0, (cudaStream_t)stream);
        else
            csr_spmv_kernel<InVec<KPL_PC_IDENTITY>><<<(unsigned)L.items, NT, 0, (cudaStream_t)stream>>>(
                g, in, out, ws, PRED_ALWAYS, 0);
        return cuda_check("spmv launch");
    }
    return launch(op, L, in, body, ws, cfg, PH_NONE, PRED_ALWAYS, 0, (cudaStream_t)stream);
}

int kpl_dot(const kpl_op *op, const double *u, const double *v, double *result, void *workspace,
            void *stream) {
    Layout L;
    int rc = make_layout(op, L);
    if (rc != KPL_OK) return rc;
    if (!workspace) return fail(KPL_EINVAL, "workspace required");
    cudaStream_t st = (cudaStream_t)stream;
    Ws ws = make_ws(op, L, 0, workspace);
    Cfg cfg{};
    g_launches.fetch_add(1, std::memory_order_relaxed);
    head_init_kernel<<<1, 256, 0, st>>>(ws.head, ws.hist, 0, ws.chunk_cnt, L.nch);
    BodyDot body;
    body.a = u; body.b = v;
    rc = launch(op, L, InNone(), body, ws, cfg, PH_DOT, PRED_ALWAYS, 0, st);
    if (rc != KPL_OK) return rc;
    if (result) {
        cudaMemcpyAsync(result, &ws.head->dot_result, sizeof(double), cudaMemcpyDeviceToDevice, st);
        return cuda_check("dot result copy");
    }
    return KPL_OK;
}

int kpl_axpy(int64_t n, double alpha, const double *x, const double *y, double *out, void *stream) {
    if (n < 0) return fail(KPL_EINVAL, "negative length");
    if (n == 0) return KPL_OK;
    const long long blocks = std::min<long long>(cdiv(n, 256), 148LL * 16);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    axpy_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(n, alpha, x, y, out);
    return cuda_check("axpy");
}

int kpl_gather(int64_t n, const int32_t *idx, const double *src, double *dst, void *stream) {
    if (n < 0) return fail(KPL_EINVAL, "negative length");
    if (n == 0) return KPL_OK;
    const long long blocks = std::min<long long>(cdiv(n, 256), 148LL * 8);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    gather_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(n, idx, src, dst);
    return cuda_check("gather");
}

int kpl_read_status(const void *workspace, kpl_status *out, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    cudaMemcpyAsync(out, workspace, sizeof(kpl_status), cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail(KPL_ECUDA, std::string("status read: ") + cudaGetErrorString(e));
    return KPL_OK;
}

}  // extern "C"

namespace {

struct Ctx {
    const kpl_op *op;
    Layout L;
    Cfg cfg;
    Ws ws;
    const kpl_vecs *v;
    cudaStream_t st;
    bool ident;
    bool ic0;              // IC(0): M^-1 by the substitution sweeps between fused sweeps
    Ic0Ws ic;
    double sigma;
};

int make_ctx(const kpl_op *op, const kpl_cfg *cfgp, const kpl_vecs *v, void *workspace, void *stream, Ctx &c) {
    int rc = make_layout(op, c.L);
    if (rc != KPL_OK) return rc;
    if (!cfgp || !v || !workspace) return fail(KPL_EINVAL, "null argument");
    if ((rc = need_matrix(op)) != KPL_OK) return rc;
    c.op = op;
    c.cfg = make_cfg(cfgp);
    c.ws = make_ws(op, c.L, c.cfg.max_iters, workspace);
    c.v = v;
    c.st = (cudaStream_t)stream;
    c.ident = op->precond == KPL_PC_IDENTITY;
    c.ic0 = is_ic0(op);
    c.ic = make_ic0_ws(op, c.L, c.cfg.max_iters, workspace);
    if (c.ic0 && (!op->ic_l_row_ptr || !op->ic_u_row_ptr)) return fail(KPL_EINVAL, "IC(0) factor arrays missing");
    // sigma of the fixed-shift recurrences; pcg_var_sh passes schedule[0] here
    // (used by the init sweep) and reads the rest of the schedule on the device
    c.sigma = (c.cfg.method == KPL_M_PCG_SH || c.cfg.method == KPL_M_PCG_VAR_SH) ? c.cfg.shift : 0.0;
    if (c.cfg.method == KPL_M_PCG_VAR_SH && !c.cfg.schedule) return fail(KPL_EINVAL, "pcg_var_sh needs a schedule");
    return KPL_OK;
}

// (phase, predicate) of each sweep kind
int kind_phase(int kind, int &phase, int &pred) {
    switch (kind) {
    case KPL_SW_BNORM: phase = PH_BNORM; pred = PRED_ALWAYS; return KPL_OK;
    case KPL_SW_INIT_R: phase = PH_INITR; pred = PRED_ALWAYS; return KPL_OK;
    case KPL_SW_INIT_W: phase = PH_PIPE; pred = PRED_ALWAYS; return KPL_OK;
    // an iteration never runs over a pending residual replacement (p-CG-rr with the
    // replacement issued by the host on demand: kpl_solver_iterate2 + kpl_solver_replace)
    case KPL_SW_ITER: phase = PH_PIPE; pred = PRED_NOFIRE; return KPL_OK;
    case KPL_SW_TRUE: phase = PH_TRUE; pred = PRED_ROW; return KPL_OK;
    case KPL_SW_CG_P: phase = PH_CGDELTA; pred = PRED_RUNNING; return KPL_OK;
    case KPL_SW_CG_X: phase = PH_CGHEAD; pred = PRED_RUNNING; return KPL_OK;
    case KPL_SW_RR_R: phase = PH_NONE; pred = PRED_FIRE; return KPL_OK;
    case KPL_SW_RR_W: phase = PH_NONE; pred = PRED_FIRE; return KPL_OK;
    case KPL_SW_RR_S: phase = PH_NONE; pred = PRED_FIRE; return KPL_OK;
    case KPL_SW_RR_Z: phase = PH_RRFINAL; pred = PRED_FIRE; return KPL_OK;
    case KPL_SW_GAP_F: phase = PH_GAPF; pred = PRED_ROW; return KPL_OK;
    case KPL_SW_GAP_G: phase = PH_GAPG; pred = PRED_ROW; return KPL_OK;
    case KPL_SW_GAP_H: phase = PH_GAPH; pred = PRED_ROW; return KPL_OK;
    case KPL_SW_GAP_J: phase = PH_GAPJ; pred = PRED_ROW; return KPL_OK;
    default: return fail(KPL_EINVAL, "unknown sweep kind");
    }
}

// One sweep of the given kind (the building block of every solver sequence).
// Input vectors of stencil sweeps are read raw at neighbours; with op->zhalo
// they carry one halo plane on each side (multi-GPU z-slabs).
int do_sweep(const Ctx &c, int kind, long long row) {
    const kpl_op *op = c.op;
    const Layout &L = c.L;
    const kpl_vecs *v = c.v;
    int phase, pred;
    int rc = kind_phase(kind, phase, pred);
    if (rc != KPL_OK) return rc;
    // only p-CG-rr ever raises `fire`: the other methods skip the second head load every CTA
    // would make before it starts (a serial L2 round trip per CTA: config 4 0.875 -> 0.78 ms/iteration)
    if (pred == PRED_NOFIRE && c.cfg.method != KPL_M_PCG_RR) pred = PRED_RUNNING;
    const bool tma = tma_eligible(op, L);
    const double *u = c.ident ? v->r : v->u;
    switch (kind) {
    case KPL_SW_BNORM: {                 // norm2(b)  (solvers.py:372)
        BodyDot body;
        body.a = v->b; body.b = v->b;
        return launch(op, L, InNone(), body, c.ws, c.cfg, phase, pred, row, c.st);
    }
    case KPL_SW_INIT_R:                  // r = b - A x; u = M r  (solvers.py:374-375)
    case KPL_SW_RR_R: {                  // replacement r = b - A x, u = M r (:600-601)
        const int ph = c.ic0 ? PH_NONE : phase;
        rc = with_pc(op, [&](auto pc) -> int {
            constexpr int PC = decltype(pc)::value;
            BodyInitR<PC> body;
            body.b = v->b; body.x = v->x; body.r = v->r; body.u = v->u;
            body.dinv = op->inv_diag; body.c = op->pc_const; body.copy_x = 0;
            if constexpr (PC != KPL_PC_JACOBI_VEC && PC != KPL_PC_IC0) {
                if (tma) {
                    const double *streams[1] = {v->b};
                    return launch_tma(op, L, v->x, v->x, 0, streams, body, c.ws, c.cfg, ph, pred, row, c.st);
                }
            }
            return launch(op, L, in_vec<KPL_PC_IDENTITY>(op, v->x, v->x, SEL_FIXED), body, c.ws, c.cfg, ph,
                          pred, row, c.st);
        });
        if (rc != KPL_OK || !c.ic0) return rc;
        // IC(0): u = M r, then the reductions (x,x), (r,r), (r,u) of BodyInitR
        if ((rc = ic0_apply(op, c.ic, c.ws.head, v->r, v->r, SEL_FIXED, v->u, pred, row, c.st)) != KPL_OK)
            return rc;
        if (phase == PH_NONE) return KPL_OK;
        BodyPairs<3> red;
        red.a[0] = v->x; red.b[0] = v->x; red.a[1] = v->r; red.b[1] = v->r; red.a[2] = v->r; red.b[2] = v->u;
        return launch(op, L, InNone(), red, c.ws, c.cfg, phase, pred, row, c.st);
    }
    case KPL_SW_INIT_W: {                // w = axpy(-sigma, r, A u) + first reductions (:376, :388-390)
        BodyInitW body;
        body.r = v->r; body.u = u; body.w = v->w0; body.sigma = c.sigma; body.ident = c.ident;
        body.dinv = op->inv_diag; body.mout = op->precond == KPL_PC_JACOBI_VEC ? c.ws.mbuf : nullptr;
        if (tma) {
            const double *streams[1] = {v->r};
            return launch_tma(op, L, u, u, 0, streams, body, c.ws, c.cfg, phase, pred, row, c.st);
        }
        rc = launch(op, L, in_vec<KPL_PC_IDENTITY>(op, u, u, SEL_FIXED), body, c.ws, c.cfg, phase, pred, row,
                    c.st);
        if (rc != KPL_OK || !c.ic0) return rc;
        return ic0_apply(op, c.ic, c.ws.head, v->w0, v->w0, SEL_FIXED, c.ws.mbuf, pred, row, c.st);  // m = M w
    }
    case KPL_SW_TRUE: {                  // ||b - A x|| (:233-234, :401-402)
        BodyTrue body;
        body.b = v->b;
        if (tma) {
            const double *streams[1] = {v->b};
            return launch_tma(op, L, v->x, v->x, 0, streams, body, c.ws, c.cfg, phase, pred, row, c.st);
        }
        return launch(op, L, in_vec<KPL_PC_IDENTITY>(op, v->x, v->x, SEL_FIXED), body, c.ws, c.cfg, phase, pred,
                      row, c.st);
    }
    case KPL_SW_ITER: {                  // the fused pipelined iteration (:408-421 + :388-390)
        if (c.cfg.method == KPL_M_PCG_VAR_SH)
            rc = with_pc(op, [&](auto pc) -> int {
                constexpr int PC = decltype(pc)::value;
                BodyPcgIter<PC, true> body;
                body.x = v->x; body.r = v->r; body.u = v->u; body.z = v->z; body.q = v->q;
                body.s = v->s; body.t = v->t; body.p = v->p; body.w0 = v->w0; body.w1 = v->w1;
                body.dinv = op->inv_diag; body.c = op->pc_const; body.sigma = 0.0; body.dsig = 0.0;
                body.schedule = c.cfg.schedule; body.want_xi = 0;
                body.alpha = 0.0; body.beta = 0.0; body.asig = 0.0; body.wout = v->w1;
                body.mout = c.ws.mbuf; body.mld = c.ws.mbuf;
                if constexpr (PC == KPL_PC_JACOBI_VEC || PC == KPL_PC_IC0) {
                    if (c.ws.mbuf)
                        return launch(op, L, in_vec<PC>(op, v->w0, v->w1, SEL_ITER), body, c.ws, c.cfg, phase, pred,
                                      row, c.st, in_vec<KPL_PC_IDENTITY>(op, c.ws.mbuf, c.ws.mbuf, SEL_FIXED));
                }
                return launch(op, L, in_vec<PC>(op, v->w0, v->w1, SEL_ITER), body, c.ws, c.cfg, phase, pred, row,
                              c.st);
            });
        else rc = with_pc(op, [&](auto pc) -> int {
            constexpr int PC = decltype(pc)::value;
            BodyPcgIter<PC> body;
            body.schedule = nullptr; body.dsig = 0.0; body.mout = c.ws.mbuf; body.mld = c.ws.mbuf;
            body.x = v->x; body.r = v->r; body.u = v->u; body.z = v->z; body.q = v->q;
            body.s = v->s; body.t = v->t; body.p = v->p; body.w0 = v->w0; body.w1 = v->w1;
            body.dinv = op->inv_diag; body.c = op->pc_const; body.sigma = c.sigma;
            body.want_xi = c.cfg.method == KPL_M_PCG_RR;
            body.alpha = 0.0; body.beta = 0.0; body.asig = 0.0; body.wout = v->w1;
            if constexpr (PC == KPL_PC_IDENTITY) {
                if (tma) {
                    const double *streams[5] = {v->x, v->r, v->z, v->s, v->t};
                    return launch_tma(op, L, v->w0, v->w1, 1, streams, body, c.ws, c.cfg, phase, pred, row, c.st);
                }
            } else if constexpr (PC == KPL_PC_JACOBI_CONST) {
                if (tma) {
                    const double *streams[8] = {v->x, v->r, v->z, v->s, v->t, v->u, v->q, v->p};
                    return launch_tma<BodyPcgIter<PC>, 1>(op, L, v->w0, v->w1, 1, streams, body, c.ws, c.cfg, phase,
                                                          pred, row, c.st);
                }
            }
            if constexpr (PC == KPL_PC_JACOBI_VEC || PC == KPL_PC_IC0) {
                if (c.ws.mbuf)      // SpMV on the materialised m (one gather per nonzero)
                    return launch(op, L, in_vec<PC>(op, v->w0, v->w1, SEL_ITER), body, c.ws, c.cfg, phase, pred,
                                  row, c.st, in_vec<KPL_PC_IDENTITY>(op, c.ws.mbuf, c.ws.mbuf, SEL_FIXED));
            }
            return launch(op, L, in_vec<PC>(op, v->w0, v->w1, SEL_ITER), body, c.ws, c.cfg, phase, pred, row,
                          c.st);
        });
        if (rc != KPL_OK || !c.ic0) return rc;
        // IC(0): m = M^-1 w of the w just written (the current w once the epilogue advanced iter)
        return ic0_apply(op, c.ic, c.ws.head, v->w0, v->w1, SEL_ITER, c.ws.mbuf, pred, row, c.st);
    }
    case KPL_SW_CG_P: {                  // p = axpy(beta, p, u); s = A p; delta = (s, p) (:269-271)
        InCgP in;
        in.p0 = v->p; in.p1 = v->p1; in.u = u; in.p = v->p; in.beta = 0.0;
        BodyCgP bp;
        bp.p0 = v->p; bp.p1 = v->p1; bp.s = v->s; bp.pout = v->p1;
        {
            // window SpMV: materialise p_new first so the SpMV gathers one plain vector from shared memory
            const InVec<KPL_PC_IDENTITY> pn = in_vec<KPL_PC_IDENTITY>(op, v->p, v->p1, SEL_ITER1);
            if (op->kind == KPL_OP_CSR && band_ok(op, pn)) {
                g_launches.fetch_add(1, std::memory_order_relaxed);
                const unsigned grid = (unsigned)std::min<long long>(cdiv(op->n, 256), 8LL * kSMs);
                launch_pdl(cg_p_materialise_kernel, grid, 256, 0, c.st, (long long)op->n, in, v->p, v->p1, c.ws, pred,
                           row);
                return launch(op, L, in, bp, c.ws, c.cfg, phase, pred, row, c.st, pn);
            }
        }
        return launch(op, L, in, bp, c.ws, c.cfg, phase, pred, row, c.st);
    }
    case KPL_SW_CG_X: {                  // x, r, u updates + next head (:290-292, :258-259)
        const int ph = c.ic0 ? PH_NONE : phase;
        rc = with_pc(op, [&](auto pc) -> int {
            constexpr int PC = decltype(pc)::value;
            BodyCgX<PC> bx;
            bx.x = v->x; bx.r = v->r; bx.u = v->u; bx.p0 = v->p; bx.p1 = v->p1; bx.s = v->s;
            bx.dinv = op->inv_diag; bx.c = op->pc_const; bx.alpha = 0.0; bx.p = v->p;
            return launch(op, L, InNone(), bx, c.ws, c.cfg, ph, pred, row, c.st);
        });
        if (rc != KPL_OK || !c.ic0) return rc;
        // IC(0): u = M r, then the head's reductions (r,u), (r,r)
        if ((rc = ic0_apply(op, c.ic, c.ws.head, v->r, v->r, SEL_FIXED, v->u, pred, row, c.st)) != KPL_OK)
            return rc;
        BodyPairs<2> red;
        red.a[0] = v->r; red.b[0] = v->u; red.a[1] = v->r; red.b[1] = v->r;
        return launch(op, L, InNone(), red, c.ws, c.cfg, phase, pred, row, c.st);
    }
    case KPL_SW_RR_W:                    // replacement w = A u (:602)
    case KPL_SW_RR_S:                    // replacement s = A p, q = M s (:603-604)
        rc = with_pc(op, [&](auto pc) -> int {
            constexpr int PC = decltype(pc)::value;
            BodyRepl<PC> rw;
            rw.mode = kind == KPL_SW_RR_W ? 0 : 1;
            rw.w0 = v->w0; rw.w1 = v->w1; rw.s = v->s; rw.q = v->q; rw.dinv = op->inv_diag;
            rw.c = op->pc_const; rw.wout = v->w1;
            rw.mout = kind == KPL_SW_RR_W && op->precond == KPL_PC_JACOBI_VEC ? c.ws.mbuf : nullptr;
            const double *in = kind == KPL_SW_RR_W ? u : (c.ident ? v->t : v->p);
            return launch(op, L, in_vec<KPL_PC_IDENTITY>(op, in, in, SEL_FIXED), rw, c.ws, c.cfg, phase, pred,
                          row, c.st);
        });
        if (rc != KPL_OK || !c.ic0) return rc;
        if (kind == KPL_SW_RR_W)         // m = M w of the replaced w
            return ic0_apply(op, c.ic, c.ws.head, v->w0, v->w1, SEL_ITER1, c.ws.mbuf, pred, row, c.st);
        return ic0_apply(op, c.ic, c.ws.head, v->s, v->s, SEL_FIXED, v->q, pred, row, c.st);   // q = M s
    case KPL_SW_RR_Z: {                  // replacement z = A q + the next record's reductions (:605)
        BodyReplZ rz;
        rz.z = v->z; rz.r = v->r; rz.u = u; rz.w0 = v->w0; rz.w1 = v->w1; rz.ident = c.ident; rz.w = v->w0;
        const double *qq = c.ident ? v->s : v->q;
        return launch(op, L, in_vec<KPL_PC_IDENTITY>(op, qq, qq, SEL_FIXED), rz, c.ws, c.cfg, phase, pred, row,
                      c.st);
    }
    case KPL_SW_GAP_F: case KPL_SW_GAP_G: case KPL_SW_GAP_H: case KPL_SW_GAP_J: {
        auto go = [&](auto body, const double *in) -> int {
            body.b = v->b; body.r = v->r; body.t = v->t; body.s = v->s; body.z = v->z;
            body.w0 = v->w0; body.w1 = v->w1; body.w = v->w0; body.sig = c.sigma;
            body.schedule = c.cfg.method == KPL_M_PCG_VAR_SH ? c.cfg.schedule : nullptr;
            return launch(op, L, in_vec<KPL_PC_IDENTITY>(op, in, in, SEL_FIXED), body, c.ws, c.cfg, phase, pred,
                          row, c.st);
        };
        if (kind == KPL_SW_GAP_F) return go(BodyGap<GAP_F>(), v->x);
        if (kind == KPL_SW_GAP_G) return go(BodyGap<GAP_G>(), c.ident ? v->t : v->p);
        if (kind == KPL_SW_GAP_H) return go(BodyGap<GAP_H>(), u);
        return go(BodyGap<GAP_J>(), c.ident ? v->s : v->q);
    }
    default:
        return fail(KPL_EINVAL, "unknown sweep kind");
    }
}

// The record-point sweeps of row j: all gap norms with track_gaps, otherwise
// the true residual on the cadence (solvers.py:398-402, :233-234).
int record_sweeps(const Ctx &c, long long j, bool cadence_only) {
    int rc;
    if (c.cfg.track_gaps) {
        if ((rc = do_sweep(c, KPL_SW_GAP_F, j)) != KPL_OK) return rc;
        if (c.cfg.method == KPL_M_CG) return KPL_OK;
        for (int k : {KPL_SW_GAP_G, KPL_SW_GAP_H, KPL_SW_GAP_J})
            if ((rc = do_sweep(c, k, j)) != KPL_OK) return rc;
        return KPL_OK;
    }
    if (cadence_only && j % 10 != 0) return KPL_OK;
    return do_sweep(c, KPL_SW_TRUE, j);
}

int head_init(const Ctx &c) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    head_init_kernel<<<64, 256, 0, c.st>>>(c.ws.head, c.ws.hist, c.cfg.max_iters + 1, c.ws.chunk_cnt, c.L.nch);
    return cuda_check("head init");
}

// zero the interior of a state vector (halo planes, if any, are the caller's)
void zero_vec(const Ctx &c, double *p) { cudaMemsetAsync(p, 0, sizeof(double) * c.op->n, c.st); }

}  // namespace

extern "C" {

int kpl_solver_prepare(const kpl_op *op, const kpl_cfg *cfgp, const kpl_vecs *v, void *workspace, void *stream) {
    Ctx c;
    int rc = make_ctx(op, cfgp, v, workspace, stream, c);
    if (rc != KPL_OK) return rc;
    if ((rc = head_init(c)) != KPL_OK) return rc;
    // state vectors that start at zero (solvers.py:252, :377-381)
    if (c.cfg.method == KPL_M_CG) {
        zero_vec(c, v->p);
    } else {
        zero_vec(c, v->z);
        zero_vec(c, v->s);
        zero_vec(c, v->t);
        if (!c.ident) { zero_vec(c, v->q); zero_vec(c, v->p); }
    }
    if (c.ic0) {                         // substitution sweeps start from an empty y, fresh tickets
        const int rc2 = ic0_reset(op, c.ic, c.st);
        if (rc2 != KPL_OK) return rc2;
    }
    return cuda_check("prepare");
}

int kpl_sweep(const kpl_op *op, const kpl_cfg *cfgp, const kpl_vecs *v, int32_t kind, int64_t row,
              void *workspace, void *stream) {
    Ctx c;
    int rc = make_ctx(op, cfgp, v, workspace, stream, c);
    if (rc != KPL_OK) return rc;
    return do_sweep(c, kind, row);
}

int kpl_sweep_peer(const kpl_op *op, const kpl_cfg *cfgp, const kpl_vecs *v, int32_t kind, int64_t row,
                   void *workspace, const kpl_peer_sweep *px, uint64_t epoch, int32_t table_parity, int32_t push,
                   int32_t wpar, uint64_t wait_epoch, int32_t wait_parity, void *stream) {
    Ctx c;
    int rc = make_ctx(op, cfgp, v, workspace, stream, c);
    if (rc != KPL_OK) return rc;
    if (!px) return fail(KPL_EINVAL, "null peer descriptor");
    if (op->kind != KPL_OP_STENCIL || kind != KPL_SW_ITER || op->chunks_global <= 0)
        return fail(KPL_EUNSUPPORTED, "fused peer exchange: multi-GPU stencil iteration sweeps only");
    if (table_parity < 0 || table_parity > 1 || wpar < 0 || wpar > 1 || (push & ~(KPL_PUSH_W | KPL_PUSH_X)) ||
        wait_parity < 0 || wait_parity > 1)
        return fail(KPL_EINVAL, "bad parity / push mask");
    if (wait_epoch && (c.cfg.method == KPL_M_PCG_RR || c.cfg.track_gaps))
        return fail(KPL_EUNSUPPORTED, "deferred fold: p-CG / p-CG-sh / p-CG-var-sh without gaps only");
    c.ws.px = px;
    c.ws.wait_epoch = (unsigned long long)wait_epoch;
    c.ws.wait_tpar = wait_parity;
    c.ws.epoch = (unsigned long long)epoch;
    c.ws.tpar = table_parity;
    c.ws.push = push;
    c.ws.wpar = wpar;
    return do_sweep(c, kind, row);
}

int kpl_set_peer_timeout(double seconds) {
    if (!(seconds > 0.0) || seconds > 1e6) return fail(KPL_EINVAL, "peer timeout must be in (0, 1e6] s");
    g_peer_timeout_ns.store((unsigned long long)(seconds * 1e9), std::memory_order_relaxed);
    return KPL_OK;
}

int kpl_sweep_phase(int32_t kind) {
    int phase, pred;
    if (kind_phase(kind, phase, pred) != KPL_OK) return KPL_EINVAL;
    return phase;
}

int kpl_solver_init(const kpl_op *op, const kpl_cfg *cfgp, const kpl_vecs *v, const double *x0,
                    void *workspace, void *stream) {
    Ctx c;
    int rc = make_ctx(op, cfgp, v, workspace, stream, c);
    if (rc != KPL_OK) return rc;
    if (op->chunks_global > 0) return fail(KPL_EINVAL, "multi-GPU operators are driven sweep by sweep");
    if ((rc = kpl_solver_prepare(op, cfgp, v, workspace, stream)) != KPL_OK) return rc;
    if ((rc = do_sweep(c, KPL_SW_BNORM, 0)) != KPL_OK) return rc;
    // x = x0.copy() (solvers.py:373); x0 = None -> zeros
    if (!x0) cudaMemsetAsync(v->x, 0, sizeof(double) * op->n, c.st);
    else if (x0 != v->x) cudaMemcpyAsync(v->x, x0, sizeof(double) * op->n, cudaMemcpyDeviceToDevice, c.st);
    if ((rc = do_sweep(c, KPL_SW_INIT_R, 0)) != KPL_OK) return rc;
    if (c.cfg.method == KPL_M_CG) return KPL_OK;           // head of row 0 done by INIT_R's epilogue
    return do_sweep(c, KPL_SW_INIT_W, 0);
}

int kpl_solver_iterate(const kpl_op *op, const kpl_cfg *cfgp, const kpl_vecs *v, int64_t first,
                       int64_t count, void *workspace, void *stream) {
    return kpl_solver_iterate2(op, cfgp, v, first, count, 0, workspace, stream);
}

int kpl_solver_replace(const kpl_op *op, const kpl_cfg *cfgp, const kpl_vecs *v, void *workspace, void *stream) {
    Ctx c;
    int rc = make_ctx(op, cfgp, v, workspace, stream, c);
    if (rc != KPL_OK) return rc;
    if (c.cfg.method != KPL_M_PCG_RR) return fail(KPL_EINVAL, "replacement is a p-CG-rr step");
    for (int k : {KPL_SW_RR_R, KPL_SW_RR_W, KPL_SW_RR_S, KPL_SW_RR_Z})
        if ((rc = do_sweep(c, k, 0)) != KPL_OK) return rc;
    return KPL_OK;
}

int kpl_solver_iterate2(const kpl_op *op, const kpl_cfg *cfgp, const kpl_vecs *v, int64_t first,
                        int64_t count, int32_t flags, void *workspace, void *stream) {
    Ctx c;
    int rc = make_ctx(op, cfgp, v, workspace, stream, c);
    if (rc != KPL_OK) return rc;
    if (op->chunks_global > 0) return fail(KPL_EINVAL, "multi-GPU operators are driven sweep by sweep");
    if (flags & ~KPL_ITER_LAZY_REPLACE) return fail(KPL_EINVAL, "unknown iterate flags");
    const bool lazy = (flags & KPL_ITER_LAZY_REPLACE) != 0;
    for (int64_t j = first; j < first + count; ++j) {
        if ((rc = record_sweeps(c, j, true)) != KPL_OK) return rc;
        if (c.cfg.method == KPL_M_CG) {
            if ((rc = do_sweep(c, KPL_SW_CG_P, 0)) != KPL_OK) return rc;
            if ((rc = do_sweep(c, KPL_SW_CG_X, 0)) != KPL_OK) return rc;
            continue;
        }
        if ((rc = do_sweep(c, KPL_SW_ITER, 0)) != KPL_OK) return rc;
        if (c.cfg.method == KPL_M_PCG_RR && !lazy) {
            // explicit replacement, predicated on the device trigger (solvers.py:599-607)
            for (int k : {KPL_SW_RR_R, KPL_SW_RR_W, KPL_SW_RR_S, KPL_SW_RR_Z})
                if ((rc = do_sweep(c, k, 0)) != KPL_OK) return rc;
        }
    }
    return KPL_OK;
}

// Persistent cooperative solve of `count` iterations (small stencil problems,
// pipelined methods without gaps/replacement): see persistent_pipelined.
int kpl_solver_iterate_persistent(const kpl_op *op, const kpl_cfg *cfgp, const kpl_vecs *v, int64_t first,
                                  int64_t count, void *workspace, void *stream) {
    Ctx c;
    int rc = make_ctx(op, cfgp, v, workspace, stream, c);
    if (rc != KPL_OK) return rc;
    const int m = c.cfg.method;
    if (op->kind != KPL_OP_STENCIL || op->chunks_global > 0 || ordered(op) || c.cfg.track_gaps ||
        !(m == KPL_M_PCG || m == KPL_M_PCG_SH || m == KPL_M_PCG_VAR_SH))
        return fail(KPL_EUNSUPPORTED, "persistent solve: single-GPU stencil p-CG / p-CG-sh / var-sh only");
    if (count <= 0) return KPL_OK;
    const Layout &L = c.L;
    SGeo g{op->nx, op->ny, op->nz, op->diag, op->halo_lo, op->halo_hi, op->zhalo};
    BodyTrue tb;
    tb.b = v->b;
    auto in_x = in_vec<KPL_PC_IDENTITY, 1>(op, v->x, v->x, SEL_FIXED);   // L2-direct: written in-kernel
    return with_pc(op, [&](auto pc) -> int {
        constexpr int PC = decltype(pc)::value;
        auto go = [&](auto body) -> int {
            using B = decltype(body);
            auto in_w = in_vec<PC, 1>(op, v->w0, v->w1, SEL_ITER);
            body.x = v->x; body.r = v->r; body.u = v->u; body.z = v->z; body.q = v->q;
            body.s = v->s; body.t = v->t; body.p = v->p; body.w0 = v->w0; body.w1 = v->w1;
            body.dinv = op->inv_diag; body.c = op->pc_const; body.sigma = c.sigma; body.dsig = 0.0;
            body.schedule = c.cfg.schedule; body.want_xi = 0; body.mout = nullptr;
            body.alpha = 0.0; body.beta = 0.0; body.asig = 0.0; body.wout = v->w1;
            void *args[] = {&g, const_cast<Layout *>(&L), &in_w, &body, &in_x, &tb,
                            const_cast<Ws *>(&c.ws), const_cast<Cfg *>(&c.cfg), &first, &count, nullptr};
            int nb = 0, dev = 0;
            cudaGetDevice(&dev);
            int sms = kSMs;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            // redundant epilogue (one barrier per pass) when chunks are <= 32 items
            // and the chunk table fits in shared memory; KPL_PERSIST_INLINE=1 forces
            // the inline (counter-based) epilogue
            const char *env = std::getenv("KPL_PERSIST_INLINE");
            const size_t dsm = sizeof(double) * NQ * (size_t)(L.items + L.nch);   // item + chunk tables
            if (L.T <= 32 && dsm <= 64 * 1024 && !(env && env[0] == '1')) {
                char *ph = static_cast<char *>(workspace) + offsets(op, L, c.cfg.max_iters).pheads;
                args[10] = &ph;
                auto launch_red = [&](auto kern) -> int {
                    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, NT, dsm);
                    const long long cap = std::min((long long)nb * sms, kPersistMaxCtas);
                    const unsigned grid = (unsigned)std::max(1LL, std::min(L.items, cap));
                    g_launches.fetch_add(1, std::memory_order_relaxed);
                    cudaLaunchCooperativeKernel((void *)kern, grid, NT, args, dsm, c.st);
                    return cuda_check("persistent launch");
                };
                if (L.vx == 2) return launch_red(persistent_redundant<2, decltype(in_w), B, decltype(in_x)>);
                return launch_red(persistent_redundant<1, decltype(in_w), B, decltype(in_x)>);
            }
            if (L.vx == 2) {
                auto kern = persistent_pipelined<2, decltype(in_w), B, decltype(in_x)>;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, NT, 0);
                const unsigned grid = (unsigned)std::max(1LL, std::min(L.items, (long long)nb * sms));
                g_launches.fetch_add(1, std::memory_order_relaxed);
                cudaLaunchCooperativeKernel((void *)kern, grid, NT, args, 0, c.st);
            } else {
                auto kern = persistent_pipelined<1, decltype(in_w), B, decltype(in_x)>;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, NT, 0);
                const unsigned grid = (unsigned)std::max(1LL, std::min(L.items, (long long)nb * sms));
                g_launches.fetch_add(1, std::memory_order_relaxed);
                cudaLaunchCooperativeKernel((void *)kern, grid, NT, args, 0, c.st);
            }
            return cuda_check("persistent launch");
        };
        if (m == KPL_M_PCG_VAR_SH) return go(BodyPcgIter<PC, true>());
        return go(BodyPcgIter<PC, false>());
    });
}

int kpl_solver_cg_pass(const kpl_op *op, const kpl_cfg *cfgp, const kpl_vecs *v, int64_t j, int32_t pass,
                       void *workspace, void *stream) {
    Ctx c;
    int rc = make_ctx(op, cfgp, v, workspace, stream, c);
    if (rc != KPL_OK) return rc;
    if (c.cfg.method != KPL_M_CG) return fail(KPL_EINVAL, "cg_pass is for classic CG");
    if (pass == 1) {
        if ((rc = record_sweeps(c, j, true)) != KPL_OK) return rc;
        return do_sweep(c, KPL_SW_CG_P, 0);
    }
    return do_sweep(c, KPL_SW_CG_X, 0);
}

int kpl_solver_finish(const kpl_op *op, const kpl_cfg *cfgp, const kpl_vecs *v, void *workspace,
                      void *stream) {
    Ctx c;
    int rc = make_ctx(op, cfgp, v, workspace, stream, c);
    if (rc != KPL_OK) return rc;
    kpl_status s;
    if ((rc = kpl_read_status(workspace, &s, stream)) != KPL_OK) return rc;
    if (s.state != KPL_ST_DONE) return KPL_OK;
    // the final record always carries ||b - A x|| (solvers.py:233-234, `last`);
    // the cadence produced it already iff its slot is no longer NaN
    double have = 0.0;
    cudaMemcpyAsync(&have, c.ws.hist + HC * s.iter + 5, sizeof(double), cudaMemcpyDeviceToHost, c.st);
    if (cudaStreamSynchronize(c.st) != cudaSuccess) return cuda_check("finish");
    if (!std::isnan(have)) return KPL_OK;
    return record_sweeps(c, s.iter, false);
}

int kpl_finalize_global(const kpl_op *op, const kpl_cfg *cfgp, int32_t kind, int64_t row, void *workspace,
                        void *stream) {
    Layout L;
    int rc = make_layout(op, L);
    if (rc != KPL_OK) return rc;
    if (!cfgp || !workspace) return fail(KPL_EINVAL, "null argument");
    int phase, pred;
    if ((rc = kind_phase(kind, phase, pred)) != KPL_OK) return rc;
    if (phase == PH_NONE) return KPL_OK;
    const Cfg cfg = make_cfg(cfgp);
    if (pred == PRED_NOFIRE && cfg.method != KPL_M_PCG_RR) pred = PRED_RUNNING;
    const Ws ws = make_ws(op, L, cfg.max_iters, workspace);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    finalize_kernel<<<1, NT, 0, (cudaStream_t)stream>>>(ws, cfg, phase, pred, row);
    return cuda_check("finalize");
}

int64_t kpl_ic0_scratch_bytes(int64_t n) {
    if (n < 1) return fail(KPL_EINVAL, "matrix dimension must be >= 1");
    return align256(4LL * n) + 256;
}

int kpl_ic0_levels(int64_t n, const int32_t *row_ptr, const int32_t *col_idx, int32_t upper, int32_t *level,
                   void *scratch, void *stream) {
    if (n < 1 || !row_ptr || !col_idx || !level || !scratch) return fail(KPL_EINVAL, "null argument");
    cudaStream_t st = (cudaStream_t)stream;
    char *base = static_cast<char *>(scratch);
    int *flag = reinterpret_cast<int *>(base);
    unsigned int *ticket = reinterpret_cast<unsigned int *>(base + align256(4LL * n));
    cudaMemsetAsync(flag, 0, sizeof(int) * n, st);
    cudaMemsetAsync(ticket, 0, sizeof(unsigned int), st);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    ic0_levels_kernel<<<(unsigned)cdiv(n, NT), NT, 0, st>>>(n, Tri{row_ptr, col_idx, nullptr, nullptr},
                                                           upper ? 1 : 0, level, flag, ticket);
    return cuda_check("IC(0) levels");
}

int kpl_ic0_factor(int64_t n, const int32_t *row_ptr, const int32_t *col_idx, const int32_t *order,
                   const double *a_values, double diag_scale, double *l_values, void *scratch, int64_t *bad_row,
                   void *stream) {
    if (n < 1 || !row_ptr || !col_idx || !a_values || !l_values || !scratch || !bad_row)
        return fail(KPL_EINVAL, "null argument");
    cudaStream_t st = (cudaStream_t)stream;
    char *base = static_cast<char *>(scratch);
    int *flag = reinterpret_cast<int *>(base);
    unsigned int *ticket = reinterpret_cast<unsigned int *>(base + align256(4LL * n));
    unsigned long long *bad = reinterpret_cast<unsigned long long *>(base + align256(4LL * n) + 8);
    const unsigned long long none = ~0ULL;
    cudaMemsetAsync(flag, 0, sizeof(int) * n, st);
    cudaMemsetAsync(ticket, 0, sizeof(unsigned int), st);
    cudaMemcpyAsync(bad, &none, sizeof(none), cudaMemcpyHostToDevice, st);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    ic0_factor_kernel<<<(unsigned)cdiv(n, NT), NT, 0, st>>>(n, Tri{row_ptr, col_idx, nullptr, order}, a_values, diag_scale,
                                                           l_values, flag, ticket, bad);
    int rc = cuda_check("IC(0) factor");
    if (rc != KPL_OK) return rc;
    unsigned long long b = none;
    cudaMemcpyAsync(&b, bad, sizeof(b), cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail(KPL_ECUDA, std::string("IC(0) factor: ") + cudaGetErrorString(e));
    *bad_row = b == none ? -1 : (int64_t)b;
    return KPL_OK;
}

int kpl_precond_apply(const kpl_op *op, const double *v, double *out, void *workspace, void *stream) {
    Layout L;
    int rc = make_layout(op, L);
    if (rc != KPL_OK) return rc;
    if (!v || !out) return fail(KPL_EINVAL, "null argument");
    cudaStream_t st = (cudaStream_t)stream;
    switch (op->precond) {
    case KPL_PC_IDENTITY:
        if (out != v) cudaMemcpyAsync(out, v, sizeof(double) * op->n, cudaMemcpyDeviceToDevice, st);
        return cuda_check("identity apply");
    case KPL_PC_JACOBI_CONST: case KPL_PC_JACOBI_VEC: {
        const long long blocks = std::min<long long>(cdiv(op->n, 256), 148LL * 16);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        jacobi_kernel<<<(unsigned)blocks, 256, 0, st>>>(op->n, op->precond == KPL_PC_JACOBI_VEC ? op->inv_diag
                                                                                               : nullptr,
                                                        op->pc_const, v, out);
        return cuda_check("Jacobi apply");
    }
    case KPL_PC_IC0: {
        if (!workspace) return fail(KPL_EINVAL, "workspace required");
        const Ic0Ws s = make_ic0_ws(op, L, 0, workspace);
        if ((rc = ic0_reset(op, s, st)) != KPL_OK) return rc;
        return ic0_apply(op, s, nullptr, v, v, SEL_FIXED, out, PRED_ALWAYS, 0, st);
    }
    default:
        return fail(KPL_EINVAL, "unknown preconditioner");
    }
}

int kpl_peer_post(const kpl_post *post, uint64_t epoch, void *stream) {
    if (!post || !post->counter) return fail(KPL_EINVAL, "null post / counter");
    if (post->ncopies < 0 || post->ncopies > KPL_PEER_MAX_COPIES) return fail(KPL_EINVAL, "too many copies");
    if (post->nsignals < 0 || post->nsignals > KPL_PEER_MAX_RANKS) return fail(KPL_EINVAL, "too many signals");
    long long most = 0;
    for (int c = 0; c < post->ncopies; ++c) {
        const kpl_copy &cp = post->copies[c];
        if (cp.count < 0 || (cp.count && (!cp.src || !cp.dst))) return fail(KPL_EINVAL, "bad copy");
        most = std::max(most, (long long)cp.count);
    }
    const unsigned grid = (unsigned)std::max(1LL, std::min(cdiv(most, NT), 2LL * kSMs));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    peer_post_kernel<<<grid, NT, 0, (cudaStream_t)stream>>>(*post, (unsigned long long)epoch);
    return cuda_check("peer post");
}

int kpl_peer_finalize(const kpl_op *op, const kpl_cfg *cfgp, int32_t kind, int64_t row, void *workspace,
                      const double *table, const uint64_t *flags, int32_t nranks, uint64_t epoch, void *stream) {
    Layout L;
    int rc = make_layout(op, L);
    if (rc != KPL_OK) return rc;
    if (!cfgp || !workspace || !flags) return fail(KPL_EINVAL, "null argument");
    if (nranks < 1 || nranks > KPL_PEER_MAX_RANKS) return fail(KPL_EINVAL, "bad rank count");
    int phase = PH_NONE, pred = PRED_ALWAYS;
    if (kind != 0 && (rc = kind_phase(kind, phase, pred)) != KPL_OK) return rc;
    if (phase != PH_NONE && !table) return fail(KPL_EINVAL, "reducing sweep needs the exchange table");
    const Cfg cfg = make_cfg(cfgp);
    if (pred == PRED_NOFIRE && cfg.method != KPL_M_PCG_RR) pred = PRED_RUNNING;
    Ws ws = make_ws(op, L, cfg.max_iters, workspace);
    if (table) ws.chunks = const_cast<double *>(table);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    peer_finalize_kernel<<<1, NT, 0, (cudaStream_t)stream>>>(ws, cfg, phase, pred, row,
                                                             reinterpret_cast<const unsigned long long *>(flags),
                                                             nranks, (unsigned long long)epoch);
    return cuda_check("peer finalize");
}

int kpl_ipc_alloc(int64_t bytes, void **ptr, void *handle64) {
    if (bytes <= 0 || !ptr || !handle64) return fail(KPL_EINVAL, "bad argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    void *p = nullptr;
    if (cudaMalloc(&p, (size_t)bytes) != cudaSuccess) return cuda_check("IPC region cudaMalloc");
    if (cudaMemset(p, 0, (size_t)bytes) != cudaSuccess) { cudaFree(p); return cuda_check("IPC region memset"); }
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, p) != cudaSuccess) { cudaFree(p); return cuda_check("cudaIpcGetMemHandle"); }
    std::memcpy(handle64, &h, sizeof(h));
    *ptr = p;
    return KPL_OK;
}

int kpl_ipc_open(const void *handle64, void **ptr) {
    if (!handle64 || !ptr) return fail(KPL_EINVAL, "bad argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof(h));
    if (cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
        return cuda_check("cudaIpcOpenMemHandle");
    return KPL_OK;
}

int kpl_ipc_close(void *ptr) {
    if (cudaIpcCloseMemHandle(ptr) != cudaSuccess) return cuda_check("cudaIpcCloseMemHandle");
    return KPL_OK;
}

int kpl_ipc_free(void *ptr) {
    if (cudaFree(ptr) != cudaSuccess) return cuda_check("IPC region cudaFree");
    return KPL_OK;
}

int kpl_chunk_table(const kpl_op *op, void *workspace, void **local, void **global, int64_t *local_bytes) {
    Layout L;
    int rc = make_layout(op, L);
    if (rc != KPL_OK) return rc;
    Ws ws = make_ws(op, L, 0, workspace);
    if (global) *global = ws.chunks;
    if (local) *local = ws.chunks + ws.chunk_offset * NQ;
    if (local_bytes) *local_bytes = 8LL * NQ * L.nch;
    return KPL_OK;
}

}  // extern "C"
