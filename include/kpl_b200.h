/*
 * kpl_b200.h -- C ABI of the B200-native shifted pipelined CG (p-CG-sh) path.
 *
 * Drop-in boundary for the reference package `kpl` (arXiv 1706.05988 lab).
 * The reference's "FFI" for this path is its numba layer plus the solver
 * loop that drives it; each entry point below names the reference interface
 * it replaces (file:line into pkg/src/kpl/).
 *
 * Conventions
 *  - Every pointer is a DEVICE pointer unless stated otherwise; sizes are
 *    element counts; `stream` is a cudaStream_t passed as void*.
 *  - The library never allocates or frees device memory, except the
 *    peer-shareable regions of kpl_ipc_alloc (multi-GPU).  Scratch space is
 *    a caller buffer of kpl_workspace_bytes() bytes (256-byte aligned).
 *  - Return value: 0 = ok, < 0 = error (see KPL_E*); kpl_last_error()
 *    returns a static message for the most recent error on the calling thread.
 *  - All launches are asynchronous on `stream`; nothing synchronises except
 *    kpl_read_status() (one 128-byte device->host copy).
 *  - Floating-point: fp64 everywhere, compiled with --fmad=false, so every
 *    elementwise operation rounds exactly like the reference's numpy ufuncs.
 *  - Reductions use the deterministic tile/chunk tree order documented in
 *    DESIGN.md ("Reduction order"); kpl_reduction_layout() reports the
 *    parameters so a CPU emulation can reproduce it bit for bit.
 */
#ifndef KPL_B200_H
#define KPL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes ------------------------------------------------------- */
#define KPL_OK              0
#define KPL_EINVAL         -1   /* invalid argument (reference: ValueError)      */
#define KPL_ECUDA          -2   /* CUDA runtime error                            */
#define KPL_EUNSUPPORTED   -3   /* combination not built                          */

/* ---- operator description --------------------------------------------- */
#define KPL_OP_STENCIL   1   /* unscaled Dirichlet Laplacian, matrix-free         */
#define KPL_OP_CSR       2   /* CSR, int32 row_ptr/col_idx, fp64 values           */

#define KPL_PC_IDENTITY     0   /* precond.py:84-85  apply returns v              */
#define KPL_PC_JACOBI_CONST 1   /* precond.py:88-89  v * inv_diag, inv_diag == c  */
#define KPL_PC_JACOBI_VEC   2   /* precond.py:88-89  v * inv_diag[k]              */
#define KPL_PC_IC0          3   /* precond.py:90-94  L^-T L^-1 v (CSR, 1 GPU)     */

typedef struct kpl_op {
    int32_t kind;            /* KPL_OP_*                                         */
    int32_t precond;         /* KPL_PC_*                                         */
    int64_t n;               /* local rows (this rank)                           */
    /* stencil: grid (nx, ny, nz), id = x + nx*(y + ny*z); a 2D nx-by-ny grid
       is (nx, 1, ny).  Off-diagonals are -1, the diagonal is `diag`.        */
    int64_t nx, ny, nz;      /* local grid (nz = planes owned by this rank)      */
    double  diag;
    int32_t zc;              /* planes per reduction chunk (0 = library default) */
    int32_t vx;              /* 0 = auto, 1 or 2 elements per thread along x     */
    /* z-slab halos of the stencil input (multi-GPU; NULL = Dirichlet ghost).
       Each holds one plane of nx*ny raw input values.                      */
    const double *halo_lo;   /* plane z = -1 of the current stencil input        */
    const double *halo_hi;   /* plane z = nz                                     */
    /* csr                                                                   */
    const int32_t *row_ptr;  /* n+1 local offsets                                */
    const int32_t *col_idx;  /* global column ids (single GPU: local)           */
    const double  *values;
    int64_t nnz;
    int32_t chunk_blocks;    /* 256-row blocks per reduction chunk (0 = default) */
    int32_t zhalo;           /* stencil: 1 = every stencil-input vector carries one
                                halo plane before plane 0 and after plane nz-1
                                (z-slab multi-GPU; filled by the caller)       */
    /* preconditioner                                                        */
    double  pc_const;        /* KPL_PC_JACOBI_CONST                              */
    const double *inv_diag;  /* KPL_PC_JACOBI_VEC, length n (gathered via col)   */
    /* multi-GPU reduction: this rank's first global chunk, total chunks
       (0 = single GPU: the last CTA finalises inline)                       */
    int64_t chunk_offset;
    int64_t chunks_global;
    /* reduction order of every dot product / norm (single GPU):
       KPL_ORDER_TREE     the fixed tile/chunk tree (default, bandwidth-bound)
       KPL_ORDER_BLOCKED8 the reference's blocked_dot order exactly
                          (_kernels.py:16-41: 8 sequential lanes over k mod 8,
                          lanes folded pairwise, tail added last): results are
                          bit-identical to the reference's solvers, at the cost
                          of a sequential n/8-long fold after each sweep      */
    int32_t order;
    int32_t _reserved;
    /* KPL_PC_IC0: the factor L (lower CSR, diagonal last in each row) and its
       transpose U = L^T (diagonal first), as built by make_ic0
       (precond.py:134-154, factor from kpl_ic0_factor)                      */
    const int32_t *ic_l_row_ptr;
    const int32_t *ic_l_col_idx;
    const double  *ic_l_values;
    const int32_t *ic_u_row_ptr;
    const int32_t *ic_u_col_idx;
    const double  *ic_u_values;
    /* row processing orders of the two substitution sweeps: any topological
       order (from kpl_ic0_levels, rows sorted by level); NULL = natural     */
    const int32_t *ic_l_order;
    const int32_t *ic_u_order;
    /* CSR, optional column-sorted gather layout of the SpMV (NULL = gather in
       CSR order).  Rows are grouped in blocks of sp_rows; block b's nonzeros
       (row_ptr[b*sp_rows] .. row_ptr[min((b+1)*sp_rows, n)]) are stored sorted
       by column: sp_col[k] and sp_val[k] are col_idx/values of the entry whose
       position inside the block, in CSR order, is sp_dest[k].  The SpMV gathers
       its input in column order (a warp's lanes share cache lines) into shared
       memory at sp_dest and sums every row left to right from there, so the
       result is bit-identical to csr_matvec (_kernels.py:44-52).  sp_max = the
       largest block's nonzero count (<= 65535; shared memory 8*sp_max bytes). */
    const int32_t  *sp_col;
    const double   *sp_val;
    const uint16_t *sp_dest;
    int32_t sp_rows;
    int32_t sp_max;
    /* CSR, optional shared-memory-window layout of the SpMV for scattered
       banded matrices (NULL = not used; takes precedence over sp_*).  Rows are
       grouped in super-blocks of bd_rows rows, one CTA each.  Super-block s
       walks the bd_sb[4s+1] windows of bd_w columns in which its rows have
       nonzeros, in ascending column order; its j-th window is "pass"
       p = bd_sb[4s] + j and starts at column bd_win[p] (even).  The CTA keeps
       the window's slice of the input vector in shared memory (bulk copies,
       double-buffered), so the gathers are shared-memory loads, and the
       running sum of every row of the super-block in shared memory as well.
       A pass has RBP = 1024*ceil(bd_rows/1024) slots, one per local row (the
       tail slots are empty), ordered so that the 32 slots of a group hold rows
       with (nearly) the same number of nonzeros inside the window, longest
       first; the groups of a pass are dealt to its RBP/1024 rounds of 32
       groups in turn.  The matrix is stored as one byte stream of round
       records, one bulk copy each; round r (counted over all passes) is
       bytes 16*bd_roff[r] .. 16*bd_roff[r+1] of bd_stream:
           int32  grp[36]    first entry of each of the 32 groups, then the end
                             (absolute entry numbers; 3 unused), 16 bytes pad
           uint8  len[1024]  nonzeros of the slot's row inside the window (<= 255)
           uint16 row[1024]  the slot's local row
           uint16 col[cnt]   entry columns relative to the window start
           double val[cnt]   entry values            (cnt = grp[32] - grp[0])
       A group stores L full steps of 32 entries (L = its longest row; entry
       32k+l is the k-th nonzero of slot l's row, zero-filled past the row's
       end).  A lane adds its row's products to the row's running sum left to
       right, pass after pass, i.e. in ascending column order from +0.0: the
       csr_matvec order (_kernels.py:44-52), bit for bit.
       bd_round_max = most entries in one round.                              */
    const uint8_t  *bd_stream;
    const int32_t  *bd_roff;
    const int32_t  *bd_sb;
    const int32_t  *bd_win;  /* first column of every pass                        */
    int32_t bd_rows;         /* rows per super-block (multiple of 32, <= 4608)    */
    int32_t bd_w;            /* window length in columns (even, <= 65536)         */
    int32_t bd_round_max;
    int32_t _reserved2;
} kpl_op;

#define KPL_ORDER_TREE      0
#define KPL_ORDER_BLOCKED8  1

/* ---- solver configuration (mirror of SolverConfig, solvers.py:60-86) ---- */
#define KPL_M_CG         0
#define KPL_M_PCG        1
#define KPL_M_PCG_SH     2
#define KPL_M_PCG_VAR_SH 3
#define KPL_M_PCG_RR     4

typedef struct kpl_cfg {
    int32_t method;          /* KPL_M_*                                          */
    int32_t track_gaps;      /* 1: gap norms + true residual at every record      */
    double  shift;           /* sigma (pcg_sh)                                    */
    int64_t max_iters;
    double  rtol;
    double  rr_threshold;    /* tau (pcg_rr)                                      */
    double  rr_coef;         /* (mu*sqrt(n)+1)*norm_inf(A)  (solvers.py:514)      */
    const double *shift_schedule;  /* DEVICE, max_iters+1 values (pcg_var_sh)     */
} kpl_cfg;

/* Solver vectors (device, length n).  With KPL_PC_IDENTITY the reference's
   u, q, p are bitwise copies of r, s, t (precond.py:84-85 returns the same
   object), so pass u=r, q=s, p=t and the kernels skip them.  `w0`/`w1` are
   the ping-pong buffers of w (the stencil input is read at neighbours while
   the next w is written); `p0`/`p1` likewise for classic CG's direction.  */
typedef struct kpl_vecs {
    double *x, *r, *u, *w0, *w1, *z, *q, *s, *t, *p, *p1;
    const double *b;
} kpl_vecs;

/* Device status, copied to the host by kpl_read_status (16 x 8 bytes). */
#define KPL_ST_RUNNING    0
#define KPL_ST_DONE       1
#define KPL_ST_BREAKDOWN  2

typedef struct kpl_status {
    int64_t state;           /* KPL_ST_*                                         */
    int64_t iter;            /* index of the latest history row                  */
    int64_t converged;
    int64_t bd_iter;         /* BreakdownError.iteration                         */
    int64_t bd_code;         /* index into kpl_breakdown_message()               */
    int64_t n_replacements;  /* pcg_rr                                           */
    int64_t fire;            /* pcg_rr: replacement pending                      */
    int64_t _pad[9];
} kpl_status;

/* History row layout (fp64, 10 columns, row i = record i; NaN = None):
   alpha, beta, gamma, delta, rnorm_recursive, rnorm_true, gap_f, gap_g,
   gap_h, gap_j  (IterationRecord, solvers.py:89-101).                       */
#define KPL_HIST_COLS 10

/* ---- sizing / introspection -------------------------------------------- */
int64_t kpl_workspace_bytes(const kpl_op *op, int64_t max_iters);
/* byte offsets of the history table / replacement list inside the workspace */
int64_t kpl_history_offset(const kpl_op *op);
int64_t kpl_replacements_offset(const kpl_op *op, int64_t max_iters);
/* Reduction layout: out[0..7] = {vx, wx, wy, zc, tiles_x, tiles_y, chunks,
   items_per_chunk} for stencils; {1, 256, 1, chunk_blocks, 0, 0, chunks,
   chunk_blocks} for CSR.                                                  */
int kpl_reduction_layout(const kpl_op *op, int64_t *out8);
const char *kpl_last_error(void);
const char *kpl_breakdown_message(int64_t code);
int kpl_version(void);
/* Number of kernels this library has launched in the process (bench evidence). */
int64_t kpl_launch_count(void);

/* ---- level-1/2 kernels (reference: sparse.py / _kernels.py) ------------ */
/* out = A v                    -- sparse.py:153-160 -> _kernels.py:44-52     */
int kpl_spmv(const kpl_op *op, const double *v, double *out, void *stream);
/* *result = (u, v), deterministic tree order -- sparse.py:163-169 ->
   _kernels.py:15-41.  `result` is a device double.                          */
int kpl_dot(const kpl_op *op, const double *u, const double *v, double *result,
            void *workspace, void *stream);
/* out = alpha*x + y, alpha == 0 -> exact copy of y -- sparse.py:172-180      */
int kpl_axpy(int64_t n, double alpha, const double *x, const double *y, double *out,
             void *stream);

/* ---- solver (reference: solvers.py solve_* loop bodies) ---------------- */
/* Initialise workspace + vectors: bnorm = ||b||, x = x0 (NULL -> 0),
   r = b - A x, u = M r, w = A u - sigma r, z=q=s=t=p=0, history row 0 and
   (alpha_0, beta_0).  Reference: solvers.py:369-393 (pcg_sh), :306-329
   (pcg), :246-285 (cg), :545-571 (pcg_rr).                                 */
int kpl_solver_init(const kpl_op *op, const kpl_cfg *cfg, const kpl_vecs *v,
                    const double *x0, void *workspace, void *stream);
/* Enqueue `count` iterations starting at nominal index `first`
   (host's count of updates issued).  Each is a predicated no-op once the
   device status leaves RUNNING.  Reference: one pass of the loop body
   solvers.py:387-421 (pcg_sh) -- n = A M^-1 w, the nine recurrences and the
   next (gamma, delta, ||r||) fused into one sweep -- plus the true-residual
   cadence of solvers.py:233-234 before every update whose index is a
   multiple of 10.                                                          */
int kpl_solver_iterate(const kpl_op *op, const kpl_cfg *cfg, const kpl_vecs *v,
                       int64_t first, int64_t count, void *workspace, void *stream);
/* kpl_solver_iterate with flags.  KPL_ITER_LAZY_REPLACE (p-CG-rr): do not
   enqueue the four residual-replacement sweeps (solvers.py:599-607) after
   every iteration; when the device trigger fires, the following iterations
   are predicated off (the status shows fire = 1 at row iter) until the host
   calls kpl_solver_replace and re-issues from index iter + 1.  The executed
   operations -- and so every bit of the result -- are the same as with the
   eager sequence; the idle replacement launches disappear.               */
#define KPL_ITER_LAZY_REPLACE 1
int kpl_solver_iterate2(const kpl_op *op, const kpl_cfg *cfg, const kpl_vecs *v,
                        int64_t first, int64_t count, int32_t flags, void *workspace, void *stream);
/* Enqueue the residual replacement r = b - A x, u = M r, w = A u, s = A p,
   q = M s, z = A q + the record of the replaced row (solvers.py:600-607),
   predicated on the device trigger.                                       */
int kpl_solver_replace(const kpl_op *op, const kpl_cfg *cfg, const kpl_vecs *v, void *workspace,
                       void *stream);
/* Same as kpl_solver_iterate, as ONE cooperative (persistent) launch with a
   grid barrier between passes -- for small problems where per-iteration
   launch latency dominates.  Single-GPU stencil p-CG / p-CG-sh / p-CG-var-sh
   without track_gaps (KPL_EUNSUPPORTED otherwise).  Bit-identical results.  */
int kpl_solver_iterate_persistent(const kpl_op *op, const kpl_cfg *cfg, const kpl_vecs *v,
                                  int64_t first, int64_t count, void *workspace, void *stream);
/* Classic CG in two halves so a host callback can observe the record
   point (solvers.py:286-287): pass 1 = true-residual cadence + p, s = A p,
   delta, record; pass 2 = x, r, u updates and the next head.               */
int kpl_solver_cg_pass(const kpl_op *op, const kpl_cfg *cfg, const kpl_vecs *v, int64_t j,
                       int32_t pass, void *workspace, void *stream);
/* After the device reports DONE: ||b - A x|| for the final record if the
   cadence did not already produce it (solvers.py:401-402, `last`).          */
int kpl_solver_finish(const kpl_op *op, const kpl_cfg *cfg, const kpl_vecs *v,
                      void *workspace, void *stream);
/* Synchronous copy of the device status to host memory `out`.               */
int kpl_read_status(const void *workspace, kpl_status *out, void *stream);

/* ---- sweep-level interface (multi-GPU drivers, custom schedules) ------- */
#define KPL_SW_BNORM   1   /* ||b|| (solvers.py:372)                              */
#define KPL_SW_INIT_R  2   /* r = b - A x, u = M r (input x) (:374-375)           */
#define KPL_SW_INIT_W  3   /* w = A u - sigma r + row-0 reductions (:376, :388)   */
#define KPL_SW_ITER    4   /* fused pipelined iteration (:408-421 + :388-390)      */
#define KPL_SW_TRUE    5   /* ||b - A x|| into history row `row` (:233-234)       */
#define KPL_SW_CG_P    6   /* classic CG p, s = A p, delta (:269-289)             */
#define KPL_SW_CG_X    7   /* classic CG x, r, u + next head (:290-292, :258)     */
#define KPL_SW_RR_R    8   /* replacement r = b - A x, u = M r (:600-601)         */
#define KPL_SW_RR_W    9   /* replacement w = A u (:602)                          */
#define KPL_SW_RR_S   10   /* replacement s = A p, q = M s (:603-604)             */
#define KPL_SW_RR_Z   11   /* replacement z = A q + next reductions (:605)        */
#define KPL_SW_GAP_F  12   /* track_gaps: ||b-Ax||, ||f|| at row `row` (:148-149) */
#define KPL_SW_GAP_G  13   /* ||axpy(-sigma, t, A p) - s|| (:153)                 */
#define KPL_SW_GAP_H  14   /* ||axpy(-sigma, r, A u) - w|| (:152)                 */
#define KPL_SW_GAP_J  15   /* ||A q - z|| (:154)                                  */
/* Reset the workspace head/history and zero the state vectors that start at 0. */
int kpl_solver_prepare(const kpl_op *op, const kpl_cfg *cfg, const kpl_vecs *v, void *workspace,
                       void *stream);
/* Launch one sweep.  Single GPU (chunks_global == 0): its last CTA folds the
   reduction and runs the scalar epilogue.  Multi-GPU: it only writes this
   rank's chunk partials; gather the chunk table, then kpl_finalize_global. */
int kpl_sweep(const kpl_op *op, const kpl_cfg *cfg, const kpl_vecs *v, int32_t kind, int64_t row,
              void *workspace, void *stream);
/* Reduction phase of a sweep kind (0 = no reduction / nothing to finalize). */
int kpl_sweep_phase(int32_t kind);

/* ---- IC(0) preconditioner (reference: precond.py:134-154, _kernels.py:55-115)
   The factor and both substitutions run as sync-free row sweeps on the
   device, bit-identical to the reference's sequential loops.              */
/* Scratch bytes kpl_ic0_factor / kpl_ic0_levels need for n rows.          */
int64_t kpl_ic0_scratch_bytes(int64_t n);
/* level[i] = 1 + max level of the rows row i depends on (0 if none): upper
   = 0 for L (columns < i, diagonal last), 1 for L^T (columns > i, diagonal
   first).  Sorting rows by level gives the processing order the sweeps
   use (kpl_op.ic_*_order); it does not change any value computed.         */
int kpl_ic0_levels(int64_t n, const int32_t *row_ptr, const int32_t *col_idx, int32_t upper, int32_t *level,
                   void *scratch, void *stream);
/* l_values = IC(0) factor of the lower pattern (row_ptr, col_idx; diagonal
   last; rows processed in `order`, NULL = natural) whose values are a_values
   (A's lower triangle); each diagonal entry
   is multiplied by diag_scale = 1 + eta first (precond.py:41-42; x * 1.0 is
   exact, so eta = 0 needs no special case).  *bad_row (host) = -1, or the
   first row whose pivot is not positive (_kernels.py:112-113 ->
   PreconditionerBreakdown).  Blocks until the factor is done.              */
int kpl_ic0_factor(int64_t n, const int32_t *row_ptr, const int32_t *col_idx, const int32_t *order,
                   const double *a_values, double diag_scale, double *l_values, void *scratch, int64_t *bad_row,
                   void *stream);
/* out = M^-1 v for the operator's preconditioner (identity: copy; Jacobi:
   v * inv_diag; IC(0): upper_solve(lower_solve(v))) -- precond.py:82-94.
   `workspace`: kpl_workspace_bytes(op, 0) bytes.                           */
int kpl_precond_apply(const kpl_op *op, const double *v, double *out, void *workspace, void *stream);

/* ---- multi-GPU hooks (one process per GPU; host drives NCCL) ----------- */
/* dst[k] = src[idx[k]] for k < n: packs the rows a neighbour needs (the
   general halo gather of row-block CSR partitions).                        */
int kpl_gather(int64_t n, const int32_t *idx, const double *src, double *dst, void *stream);
/* Level-4 fold of the gathered chunk table + the scalar epilogue of sweep
   `kind` (same predicate as the sweep).  Every rank runs it on identical
   data, so every rank holds identical scalars and history.                */
int kpl_finalize_global(const kpl_op *op, const kpl_cfg *cfg, int32_t kind, int64_t row,
                        void *workspace, void *stream);
/* Device pointer + byte size of this rank's slice of the chunk table and of
   the whole table (for ncclAllGather).                                      */
int kpl_chunk_table(const kpl_op *op, void *workspace, void **local, void **global,
                    int64_t *local_bytes);

/* ---- device-initiated exchange over peer memory (NVLink P2P) ----------
   Replaces the host-driven NCCL halo send/recv + chunk-table all-gather of
   the multi-GPU sweep sequence (the reference has no parallel layer; the
   paper's runs used PETSc/MPI, PAPER.md:625-630 -- the communication the
   p-CG-sh recurrences exist to hide).  Peer pointers come from
   kpl_ipc_open (one process per GPU) or are plain device pointers when
   several ranks share a device.  After each sweep, kpl_peer_post stores the
   halo planes / ghost rows of the next sweep's stencil inputs and this
   rank's chunk partials straight into the peers' memory and then publishes
   `epoch` into every rank's flag word for this rank; kpl_peer_finalize waits
   for every rank's flag and folds the gathered table (same tree as one GPU,
   so results are bit-identical to the single-GPU solve).                 */
#define KPL_PEER_MAX_COPIES 40
#define KPL_PEER_MAX_RANKS  16

typedef struct kpl_copy {
    const double  *src;      /* local device vector                             */
    const int32_t *idx;      /* NULL: dst[k] = src[k]; else dst[k] = src[idx[k]] */
    double        *dst;      /* peer (or local) device pointer                  */
    int64_t        count;
} kpl_copy;

typedef struct kpl_post {
    int32_t   ncopies;                          /* <= KPL_PEER_MAX_COPIES          */
    int32_t   nsignals;                         /* <= KPL_PEER_MAX_RANKS           */
    kpl_copy  copies[KPL_PEER_MAX_COPIES];
    uint64_t *signal[KPL_PEER_MAX_RANKS];       /* flag word of THIS rank in every
                                                   rank's flag array (incl. own)  */
    unsigned int *counter;                      /* local device word, initially 0,
                                                   self-resetting                 */
    const void *status;                         /* this rank's workspace (its head):
                                                   once its exchange has failed the
                                                   post signals epoch | 2^63 (poison)
                                                   so every peer fails fast; NULL =
                                                   never poison                   */
} kpl_post;

/* Fused form for the hot sweep (stencil z-slabs, KPL_SW_ITER): the sweep
   itself stores its tile of the slab's boundary planes of the pushed outputs
   into the neighbours' halos (read back from what each thread just wrote),
   every chunk-completing CTA stores its chunk partial into every rank's
   exchange-table slot `table_parity`, and the rank's last chunk signals
   `epoch` -- so the exchange overlaps the sweep and no post kernel runs.
   `px` is a DEVICE copy of this struct.  Follow with kpl_peer_finalize.   */
#define KPL_PUSH_W 1     /* the ping-pong output w[wpar] (next sweep's input) */
#define KPL_PUSH_X 2     /* x (next record's true-residual cadence input)      */

typedef struct kpl_peer_sweep {
    int32_t   nranks, rank;
    double   *table[2][KPL_PEER_MAX_RANKS];     /* every rank's table slot, by parity */
    uint64_t *signal[KPL_PEER_MAX_RANKS];       /* as kpl_post.signal                 */
    const double *w_src[2];                     /* local interiors of w0, w1          */
    double   *w_lo[2], *w_hi[2];                /* neighbour halo planes (NULL at the
                                                   global boundary)                  */
    const double *x_src;
    double   *x_lo, *x_hi;
    const uint64_t *flags;                      /* THIS rank's flag array (one word per
                                                   rank; for the deferred fold)     */
} kpl_peer_sweep;

/* wait_epoch != 0: deferred fold.  The previous sweep was a fused iteration
   sweep of the same solve whose exchange (epoch wait_epoch, table slot
   wait_parity) has NOT been finalised: instead of a kpl_peer_finalize launch
   in between, every CTA of this sweep waits for the flags, folds the slot and
   runs the scalar epilogue itself (the paper's reduction overlap,
   PAPER.md:43-45); results are bit-identical to sweep + finalize.          */
int kpl_sweep_peer(const kpl_op *op, const kpl_cfg *cfg, const kpl_vecs *v, int32_t kind, int64_t row,
                   void *workspace, const kpl_peer_sweep *px, uint64_t epoch, int32_t table_parity,
                   int32_t push, int32_t wpar, uint64_t wait_epoch, int32_t wait_parity, void *stream);
/* Limit of every device-side peer wait (default 20 s; KPL_PEER_TIMEOUT_S is
   read at load time).  A wait that times out turns the device status into
   BREAKDOWN "peer exchange timeout"; a rank that sees a peer's poison,
   "peer rank failed".                                                       */
int kpl_set_peer_timeout(double seconds);
/* Enqueue the copies of `post`, then (after a system-scope fence) store
   `epoch` into every signal word.  Host-side `post` is passed by value.    */
int kpl_peer_post(const kpl_post *post, uint64_t epoch, void *stream);
/* Wait until flags[0..nranks) >= epoch (acquire, system scope; the peer
   timeout turns the device status into BREAKDOWN with bd_code 7, "peer
   exchange timeout", a peer's poison into bd_code 9, "peer rank failed"), then, for a reducing sweep `kind` (0 = wait only),
   fold `table` (chunks_global x 4 doubles) and run the sweep's scalar
   epilogue, as kpl_finalize_global does.                                  */
int kpl_peer_finalize(const kpl_op *op, const kpl_cfg *cfg, int32_t kind, int64_t row, void *workspace,
                      const double *table, const uint64_t *flags, int32_t nranks, uint64_t epoch,
                      void *stream);
/* Peer-shareable device memory (the one allocation the library makes):
   cudaMalloc + zero fill + cudaIpcGetMemHandle; `handle64` receives the 64-byte
   handle to send to the other ranks.  kpl_ipc_open maps a peer's handle
   (cudaIpcMemLazyEnablePeerAccess).                                       */
int kpl_ipc_alloc(int64_t bytes, void **ptr, void *handle64);
int kpl_ipc_open(const void *handle64, void **ptr);
int kpl_ipc_close(void *ptr);
int kpl_ipc_free(void *ptr);

#ifdef __cplusplus
}
#endif
#endif /* KPL_B200_H */
