/*
 * plss.h -- C ABI of libplss, the B200 (sm_100a) hot path of PLSS with residual sketches
 * (arXiv 2207.07615, "PLSS: A Projected Linear Systems Solver").
 *
 * What is computed: Algorithm 1 with WI = I for a consistent system
 * A x = b, b in range(A) (eq:axb, L25-29), A in R^{m x n} sparse, square or rectangular:
 *
 *   init  : r = b - A x0; rho = r^T r; y = A^T r; phi = y^T y; p = (rho/phi) y;
 *           theta = p^T p; x = x0 + p                                        (L784-797)
 *   loop  : r <- r - A p  (eq:recRes L663-666)      rho = r^T r              (L801, L804)
 *           stop if sqrt(rho)/||b|| <= tol                                   (L828-831, L977)
 *           y = A^T r; phi = y^T y; psi = y^T p_{k-1} (diagnostic, L671-672) (L802, L806)
 *           tau = sqrt(theta phi)/rho; beta = 1/((tau-1)(tau+1));
 *           gamma = (theta/rho) beta                                         (L807-809)
 *           p <- beta p + gamma y (Thm 4.1 eq:pkShort L628-712); theta = p^T p; x <- x + p
 *                                                                            (L811-813)
 * Readings where the paper is silent or misprinted are listed in DESIGN.md ("Readings"):
 * gamma follows Algorithm 1 (L809), not the misprinted theorem statement (L639-643).
 *
 * Conventions
 *  - Every call returns plss_status (0 = OK); no call aborts or exits the process.
 *  - Matrix arrays must be 16-byte aligned with 16-byte padded allocations (TMA bulk copies read
 *    the 16-byte superset of a range); plss_create checks the alignment.
 *  - Index arrays are int32, values fp64 (binary64, round-to-nearest-even).
 *  - CSR: row_ptr[m+1] (row_ptr[0] = 0, nondecreasing, row_ptr[m] = nnz), col_idx[nnz] strictly
 *    ascending within each row, val[nnz]. CSC copy of the SAME matrix: col_ptr[n+1],
 *    row_idx[nnz] strictly ascending within each column, val_t[nnz] (SPEC.md L29-35 invariants).
 *  - "dev" pointers must be CUDA device memory of the ctx's device. Pointers marked
 *    "host or dev" may be either; the library detects the kind with cudaPointerGetAttributes
 *    and copies host data through the ctx stream.
 *  - All work is enqueued on the ctx stream (the caller's, e.g. torch's current stream).
 */
#ifndef PLSS_H
#define PLSS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PLSS_REC 8  /* doubles per iteration record, see plss_solve / plss_finish `diag` */

typedef struct plss_ctx plss_ctx; /* opaque; one per matrix (per rank) and stream */

typedef enum {
  PLSS_OK = 0,
  PLSS_E_INVALID = 1, /* bad argument value (tol < 0, maxit < 1 or > maxit_cap, NULL ctx, ...)  */
  PLSS_E_DIM = 2,     /* inconsistent dimensions / sizes / workspace too small                  */
  PLSS_E_FORMAT = 3,  /* CSR/CSC invariant violated (validate = 1)                              */
  PLSS_E_CUDA = 4,    /* a CUDA runtime call failed; see plss_last_error                        */
  PLSS_E_NCCL = 5,    /* an NCCL call failed; see plss_last_error                               */
  PLSS_E_NOMEM = 6,   /* host allocation failed                                                 */
  PLSS_E_STATE = 7    /* call out of order (plss_step / plss_finish without plss_start)         */
} plss_status;

typedef enum {
  PLSS_CONVERGED = 0,            /* sqrt(rho_k)/||b|| <= tol (relative) or sqrt(rho_k) <= tol */
  PLSS_MAXIT = 1,                /* iteration cap reached                                      */
  PLSS_BREAKDOWN_Y_VANISHED = 2, /* phi <= 1e-300 while rho above tol (b not in range(A))      */
  PLSS_BREAKDOWN_STAGNATION = 3, /* tau - 1 <= 1e-14 (Cauchy-Schwarz equality)   */
  PLSS_RUNNING = -1
} plss_outcome;

/* The matrix, as two borrowed DEVICE copies. The arrays must outlive the ctx and must not be
 * mutated while it exists. They may be shared by several ctxs (e.g. one per stream). On a rank
 * of a distributed solve, m and the arrays describe the LOCAL row block (rows rebased to 0) and
 * n is the global column count. */
typedef struct {
  int64_t m, n, nnz;
  const int32_t *row_ptr, *col_idx; /* CSR */
  const double *val;
  const int32_t *col_ptr, *row_idx; /* CSC copy of the same matrix */
  const double *val_t;
  int32_t validate; /* 1: O(nnz) device check of every invariant above, incl. CSR == CSC^T */
} plss_matrix;

typedef struct {
  int32_t slabs;       /* row slabs that tile the gather of A^T r into L2 (0 = auto, 1 = off).
                          With S > 1 the library keeps a slab-major CSC copy in the workspace. */
  int32_t graph_chunk; /* iterations per CUDA-graph launch (0 = auto)                        */
  int32_t maxit_cap;   /* largest maxit a solve on this ctx may request (sizes the history)  */
  int32_t flags;       /* bit0: disable the SELL-32 format (saves its ~2 x 1.15 nnz x 12 B of
                          workspace); bit1: disable the shared-memory windows of the gathered
                          vector (SELL segments then gather every entry from global memory);
                          bit2 (distributed ctx only): the reduce-scatter step -- y is
                          reduce-scattered to column shards of n / nranks, phi / psi and K3 run
                          on the shard, one all-reduce carries {rho, phi, psi, theta}, p is
                          all-gathered; x is gathered by plss_finish (then collective);
                          bit3 (distributed ctx only, <= 8 ranks, not with bit2): the
                          peer-memory step (SURVEY 8(e) improvement 3) -- instead of
                          ncclAllReduce, the library's own kernels sum y | rho over the ranks
                          through NVLink peer memory: per K2 column chunk each rank sums its
                          column shard of every rank's partial in rank order 0..G-1 and stores
                          the sum into every rank's y, overlapped with the next chunk's K2.
                          The ctx then also cudaMallocs 2 x 8(n+2) B + 1 KB of device memory
                          (CUDA IPC needs an allocation base), and every rank's region is
                          mapped by CUDA IPC at create (all ranks on one node);
                          other bits must be 0                                             */
} plss_options;

/* Bytes of DEVICE workspace a ctx needs (vectors r, y, p, x, reduction partials, control block,
 * history of (maxit_cap+1)*PLSS_REC doubles, tile maps, the optional slab-major CSC copy, the
 * SELL-32 copies of A (unless opt->flags bit0) and the (n+1)-double AllReduce buffer). opt may be NULL (defaults).
 * The caller allocates it (e.g. a torch uint8 tensor), 256-byte aligned, and keeps it alive
 * for the ctx's lifetime. Returns 0 on invalid input. */
size_t plss_workspace_bytes(const plss_matrix *A, const plss_options *opt);

/* Create a single-device ctx. A: device arrays (see plss_matrix). workspace: dev, >= ws_bytes =
 * plss_workspace_bytes(A, opt). cuda_stream: cudaStream_t (NULL = legacy default stream).
 * Synchronizes the stream once (setup). Errors: E_INVALID, E_DIM, E_FORMAT, E_CUDA. */
plss_status plss_create(const plss_matrix *A, const plss_options *opt, void *workspace,
                        size_t ws_bytes, void *cuda_stream, plss_ctx **out);

/* Distributed row-block ctx: this rank owns rows [row_offset, row_offset + A->m)
 * of a global m_global x n matrix; x, p, y are replicated. Each iteration does local A p and
 * A^T r and an ncclAllReduce(sum, fp64) of n+1 values (partial y and the local rho). When the last
 * K2 segment is SELL-32 with a sigma perm, A^T r runs as column chunks (PLSS_DIST_CHUNKS, default 4)
 * and each chunk is all-reduced on a second stream while the next one computes.
 * id: 128 bytes from plss_get_unique_id on rank 0, broadcast by the caller (e.g. through
 * torch.distributed). Collective: every rank must call it. Errors: as plss_create + E_NCCL. */
plss_status plss_get_unique_id(uint8_t id[128]);
plss_status plss_create_dist(const plss_matrix *A_local, int64_t row_offset, int64_t m_global,
                             const uint8_t id[128], int32_t rank, int32_t nranks,
                             const plss_options *opt, void *workspace, size_t ws_bytes,
                             void *cuda_stream, plss_ctx **out);

/* Distributed column-block ctx ("column-block alternative", for m < n): this rank owns
 * columns [col_offset, col_offset + A_local->n) of a global m x n_global matrix. A_local is that
 * column block as an m x n_local matrix: CSR over LOCAL column indices (global column - col_offset)
 * and the CSC of its columns (row indices global, 0..m-1). r (m) is replicated; x, p, y are this
 * rank's column shards. Per iteration: K1 computes u <- u - A_g p_g (u = r on rank 0, u = 0 on the
 * others), one ncclAllReduce of m+1 values (u and the previous K3's theta partial) gives every
 * rank r = r - A p; rho = r^T r, the stop test and the rho tail run replicated; K2 forms y_g =
 * A_g^T r over the local columns; phi, psi partials go through an ncclAllReduce of 2 values; K3
 * updates the shard. Messages are m+1 and 2 doubles instead of n+1 (C4: 2M vs 8M).
 * In this mode: plss_start / plss_solve take the full b (m, the same on every rank) and x0 / x as
 * this rank's shard (n_local); plss_column_norms gives the local columns' norms (whole columns, no
 * collective); plss_set_wi takes the local shard; plss_spmv / plss_spmvT are the local products
 * A_g x_g and A_g^T u; plss_true_residual takes the full b and the local x shard (collective).
 * options.flags bit2 / bit3 are rejected (E_INVALID). Collective. Errors: as plss_create_dist. */
plss_status plss_create_dist_cols(const plss_matrix *A_local, int64_t col_offset, int64_t n_global,
                                  const uint8_t id[128], int32_t rank, int32_t nranks,
                                  const plss_options *opt, void *workspace, size_t ws_bytes,
                                  void *cuda_stream, plss_ctx **out);

/* Full solve = plss_start + plss_step until done + plss_finish.
 *  b      : host or dev, m (local rows on a rank) doubles.
 *  x0     : host or dev, n doubles, or NULL for x0 = 0.
 *  tol    : >= 0. tol_mode 0: stop when sqrt(rho)/||b|| <= tol (||b|| = 0 -> denominator 1);
 *           1: stop when sqrt(rho) <= tol.
 *  maxit  : 1 <= maxit <= maxit_cap; caps the number of updates x <- x + p.
 *  flags  : bit0 = freeze mode (fixed-iteration timing): never stop early; once
 *           sqrt(rho)/||b|| <= 64 eps, tol is met, or a breakdown guard fires, beta = gamma = 0
 *           so x stays fixed while every kernel still runs with the same memory traffic.
 *  x      : host or dev, n doubles, out (may alias x0).
 *  iters  : host, out: updates applied.  outcome: host, out.
 *  hist   : host, nullable, maxit+1 doubles: hist[k] = sqrt(rho_k)/||b|| (or sqrt(rho_k)).
 *  diag   : host, nullable, (maxit+1)*PLSS_REC doubles; record k = {hist_k, rho_k, phi, psi,
 *           theta, tau, beta, gamma} of loop step k (k = 0: initialization).
 * Returns after the stream is synchronized. */
plss_status plss_solve(plss_ctx *ctx, const double *b, const double *x0, double tol,
                       int32_t tol_mode, int32_t maxit, int32_t flags, double *x, int32_t *iters,
                       double *hist, double *diag, plss_outcome *outcome);

/* Asynchronous pieces of plss_solve (same argument meaning), for timing and pipelining:
 * plss_start copies b / x0 in and resets the device state; plss_step enqueues k more loop steps
 * (CUDA graphs; steps after the stop condition are no-ops); plss_finish synchronizes and copies
 * out x, iters, hist, diag, outcome. Between plss_step and plss_finish the device copy of x may lag
 * the last update p_k by one (the row-slab steps update x every other step, R25);
 * plss_finish applies it, and stepping may continue after plss_finish. */
plss_status plss_start(plss_ctx *ctx, const double *b, const double *x0, double tol,
                       int32_t tol_mode, int32_t maxit, int32_t flags);
plss_status plss_step(plss_ctx *ctx, int32_t k);
plss_status plss_finish(plss_ctx *ctx, double *x, int32_t *iters, double *hist, double *diag,
                        plss_outcome *outcome);

/* PLSS W (Algorithm 1's optional B^T B, L777-783): wi (host or dev, n doubles,
 * finite and > 0) is the diagonal of WI = B^T B = W^{-1}; later solves on this ctx use
 * WIy = y ./ wi, phi = y^T WIy, p = beta p + gamma WIy, theta = p^T (WI p). wi = NULL restores
 * WI = I. Copies wi into the workspace; synchronizes. Errors: E_INVALID (bad entries).
 * On a distributed ctx every rank passes the same (global) wi. */
plss_status plss_set_wi(plss_ctx *ctx, const double *wi);

/* c_j = ||A_{:,j}|| (sum of squares in ascending row order, then sqrt; zero columns 1, SPEC.md
 * L137) into c (host or dev, n doubles): the paper's PLSS W weights, WI = diag(c) i.e.
 * W = diag(1/||A_{:,j}||) (L761-764, L977-979). On a distributed ctx the per-rank sums are
 * all-reduced (collective). Synchronizes. */
plss_status plss_column_norms(plss_ctx *ctx, double *c);

/* Test entry points. y = A x (x: dev n, y: dev m); v = A^T u (u: dev m,
 * v: dev n). Sums are sequential in ascending index order per output element. Synchronous. */
plss_status plss_spmv(plss_ctx *ctx, const double *x, double *y);
plss_status plss_spmvT(plss_ctx *ctx, const double *u, double *v);

/* Test entry point of the peer-memory step (options.flags bit3): one step of its all-reduce over
 * G <= 8 VIRTUAL ranks on the current device, the reduce kernels launched cooperatively with one
 * grid row per virtual rank (their CTAs wait on one another). part[h], red[h]: device buffers of
 * virtual rank h (its partial and its reduced vector, >= bounds[nch] doubles, 16-byte aligned);
 * flags[h]: rank h's 256-word flag block (device, zeroed before the first call, then left to the
 * library: it carries the step epoch across calls). Chunks c = [bounds[c], bounds[c+1]),
 * 1 <= nch <= 8 (host array of nch + 1 non-decreasing offsets). After the call red[h][j] =
 * ((part[0][j] + part[1][j]) + ...) + part[G-1][j] (binary64, rank order) for every h and every j
 * in [bounds[0], bounds[nch]); nothing else is written. Synchronizes `cuda_stream`. */
plss_status plss_peer_reduce_emulate(int32_t G, double *const *part, double *const *red, uint32_t *const *flags,
                                     int32_t nch, const int64_t *bounds, void *cuda_stream);

/* The true residual of an iterate (the solve stops on the recursive residual of
 * Algorithm 1; report the true one once at exit): out[0] = ||b - A x||_2, out[1] = ||b||_2 (host,
 * 2 doubles). b: host or dev, m (local) doubles; x: host or dev, n doubles. One SpMV (the sequential
 * row sums of plss_spmv) and a fixed-order reduction; on a distributed ctx the sums of squares are
 * all-reduced (collective: every rank calls it). Synchronizes. */
plss_status plss_true_residual(plss_ctx *ctx, const double *b, const double *x, double *out);

/* Per-kernel device time of k loop steps launched one kernel at a time (not graphs), with CUDA
 * events on the ctx stream around each launch; call after plss_start. ms (host, 5 doubles)
 * receives the average per step of: K1 (all slabs), K2 (all slabs), the NCCL all-reduce,
 * the distributed dots/tail kernel, K3. Synchronizes. */
plss_status plss_profile(plss_ctx *ctx, int32_t k, double *ms);

/* Introspection (bench / ncu): kernel launches per loop step, number of row slabs, CSR-tile nnz
 * window, grid sizes of the first K1 / K2 launch, how many of the 2*slabs SpMV segments use
 * the SELL-32 format (the rest use TMA-staged CSR tiles) and how many of those gather through a
 * shared-memory window of the gathered vector. Any pointer may be NULL. */
plss_status plss_query(const plss_ctx *ctx, int32_t *launches_per_step, int32_t *slabs,
                       int32_t *tile_nnz, int32_t *grid_k1, int32_t *grid_k2,
                       int32_t *sell_segments, int32_t *window_segments);

/* The format a ctx chose for K1 (which = 1) or K2 (which = 2) of row slab `slab`:
 * info[0] fmt (0 CSR tiles, 1 SELL-32 grid-stride, 2 SELL-32 + shared-memory window, 3 SELL-32 over
 * per-SM ranges, 5 a thread per short row), info[1] the sigma window of a sigma-permuted SELL segment
 * (512 or 1024; 0 otherwise), info[2] 1 if globally length-sorted, info[3] SELL slices, info[4] long
 * rows (run by k_longchunks, or by k_longrows when info[8] = 0), info[5] static stepping (1, or 2
 * with 6 entries in flight), info[6] the grid, info[7] the segment's rows, info[8] the long rows'
 * chunks of LCH entries (k_longchunks; 0 without long rows or with PLSS_LCHUNK=0), info[9] 1 if the
 * segment (K2's finalizing one, one device) leaves psi = y^T p_{k-1} to K3 and reads no p, info[10]
 * 1 if the ctx's K3 updates x every other step (one device; plss_finish applies a pending update)
 * (R25), info[11] / info[12] the first one-step slice / the first empty slice of a globally
 * sorted segment, whose tail k_sell runs in batches of one-step slices (-1: no batched tail),
 * info[13] 1 if k_sell runs the segment's long-row chunks itself (no k_longchunks launch).
 * PLSS_E_INVALID for a bad ctx / which / slab. */
plss_status plss_query_segment(const plss_ctx *ctx, int32_t which, int32_t slab, int32_t info[14]);

/* Diagnostics (not part of the method): per-CTA record of the last launch of K1 (which = 1) or K2
 * (which = 2) of row slab `slab`, for ctxs created with the environment variable PLSS_DBG_CTA=1:
 * out (host, 4 * grid uint64) = {start ns, end ns (%globaltimer), stored entries, units} per CTA
 * of the persistent grid; *grid receives the grid size. PLSS_E_STATE without PLSS_DBG_CTA. */
plss_status plss_debug_cta_times(plss_ctx *ctx, int32_t which, int32_t slab, uint64_t *out, int32_t *grid);

/* ---- Randomized projection ("Rand. Proj.", the paper's comparison method) ----
 * eq:pkLong with W = I and a fresh random sketch S_k in R^{m x r} each
 * iteration (L171-176; Experiment I L985-991: standard normal, r = 10; Experiment III L1164-1170:
 * sparse normal; Fig. 2):
 *   Y = A^T S_k; M = Y^T Y; v = S_k^T r_{k-1}; z = M^+ v (pivoted Cholesky at the numerical rank,
 *   DESIGN.md reading R18); p_k = Y z; x_k = x_{k-1} + p_k; r_k = r_{k-1} - A p_k (K1: rho, stop test
 *   sqrt(rho_k)/||b|| <= tol or sqrt(rho_k) <= tol, as plss_solve).
 * S_k comes from the counter-based generator of DESIGN.md reading R17, keyed by (seed, k, row,
 * column): entry (i, c) does not depend on m. density = 1: standard normal; density < 1: each
 * entry is kept with that probability (sparse normal).
 * Runs on a single-device ctx (E_INVALID on a distributed one) and uses the ctx's r, p, x,
 * control block and history: a PLSS solve in progress on the same ctx is invalidated (and an
 * RP solve by plss_start). r: 1..64. workspace: dev, 256-byte aligned, >= ws_bytes =
 * plss_rp_workspace_bytes(ctx, r) (S: m r, Y: n r doubles + partials); the caller keeps it
 * alive until plss_rp_finish. maxit <= the ctx's maxit_cap. S_k is kept in binary32 (m x
 * 8 ceil(r/8) floats); every product and sum of the projection is fp64.
 * record k of `diag` = {hist_k, rho_k, numerical rank of Y_k^T Y_k, 0...}. */
size_t plss_rp_workspace_bytes(const plss_ctx *ctx, int32_t r); /* 0 on invalid input */
plss_status plss_rp_solve(plss_ctx *ctx, int32_t r, uint64_t seed, double density, void *workspace,
                          size_t ws_bytes, const double *b, const double *x0, double tol,
                          int32_t tol_mode, int32_t maxit, double *x, int32_t *iters, double *hist,
                          double *diag, plss_outcome *outcome);
/* Asynchronous pieces of plss_rp_solve (as plss_start / plss_step / plss_finish). */
plss_status plss_rp_start(plss_ctx *ctx, int32_t r, uint64_t seed, double density, void *workspace,
                          size_t ws_bytes, const double *b, const double *x0, double tol,
                          int32_t tol_mode, int32_t maxit);
plss_status plss_rp_step(plss_ctx *ctx, int32_t k);
plss_status plss_rp_finish(plss_ctx *ctx, double *x, int32_t *iters, double *hist, double *diag,
                           plss_outcome *outcome);
/* Per-kernel device time of k randomized-projection steps launched one kernel at a time (CUDA
 * events on the ctx stream), after plss_rp_start; ms (host, 6 doubles) receives the average per
 * step of: sketch + S^T r, A^T S, Gram, r x r solve, p/x update, K1 (all slabs). Synchronizes. */
plss_status plss_rp_profile(plss_ctx *ctx, int32_t k, double *ms);
/* Test entry points. plss_rp_sketch writes S_k of iteration k >= 1 as binary32 (reading R17)
 * into S (dev, m x ld row-major floats; ld even, r <= ld <= 512; columns r..ld-1 are written 0).
 * plss_spmmT: Y = A^T S (S: dev binary32 m x ld row-major, ld >= r; Y: dev fp64 n x r
 * row-major); Y[j, c] is the sequential ascending-row fp64 sum of val * (double)S[row, c] -- the
 * kernel the solves use (they keep S with ld = 8 ceil(r/8)). Synchronous. */
plss_status plss_rp_sketch(plss_ctx *ctx, int32_t r, uint64_t seed, double density, int32_t k,
                           int32_t ld, float *S);
plss_status plss_spmmT(plss_ctx *ctx, int32_t r, int32_t ld, const float *S, double *Y);

/* ---- PLSS Kaczmarz (section 7) ----
 * Identity-column sketches S_k = [e_{i_1} .. e_{i_k}] in the caller's row order `rows`, with the
 * history-corrected row action eq:pkKacz (L952-956):
 *   d = Theta^{-1/2} P^T a_i (P^T a_i read from the stored [A p_1 .. A p_{k-1}], L961-966),
 *   gamma = r_{k-1}[i] / ((||a_i|| - ||d||)(||a_i|| + ||d||)), p_k = gamma (a_i - P Theta^{-1} P^T a_i),
 *   x_k = x_{k-1} + p_k, r_k = r_{k-1} - A p_k; stop test as plss_solve.
 * A row with ||a_i||^2 - ||d||^2 <= 1e-14 ||a_i||^2 (already in the span of the history, or empty)
 * or r_{k-1}[i] = 0 (already satisfied) is skipped: p_k = 0, nothing is appended, the step still
 * counts (reading R20). After kmax stored updates
 * the history P, A P, Theta is cleared and later updates start a new one at the current x (R21).
 * Single-device ctx (E_INVALID on a distributed one); shares the ctx's r, p, x, control block and
 * history like randomized projection. rows: host or dev, maxit int32 row indices in [0, m)
 * (E_INVALID otherwise). workspace: dev, 256-byte aligned, >= plss_kz_workspace_bytes(ctx, kmax)
 * = 8 (n + m) kmax bytes for P and A P + O(m + n + kmax); alive until plss_kz_finish.
 * record k of `diag` = {hist_k, rho_k, skipped (0/1), gamma, theta_k, history size after step}. */
size_t plss_kz_workspace_bytes(const plss_ctx *ctx, int32_t kmax); /* 0 on invalid input */
plss_status plss_kz_solve(plss_ctx *ctx, int32_t kmax, void *workspace, size_t ws_bytes,
                          const int32_t *rows, const double *b, const double *x0, double tol,
                          int32_t tol_mode, int32_t maxit, double *x, int32_t *iters, double *hist,
                          double *diag, plss_outcome *outcome);
plss_status plss_kz_start(plss_ctx *ctx, int32_t kmax, void *workspace, size_t ws_bytes,
                          const int32_t *rows, const double *b, const double *x0, double tol,
                          int32_t tol_mode, int32_t maxit);
plss_status plss_kz_step(plss_ctx *ctx, int32_t k);
plss_status plss_kz_finish(plss_ctx *ctx, double *x, int32_t *iters, double *hist, double *diag,
                           plss_outcome *outcome);
/* Per-kernel device ms per step (CUDA events, one kernel at a time) after plss_kz_start; ms (host,
 * 4 doubles): 0 (the row preparation runs inside the residual kernel), the P GEMV + update,
 * A p_k (SpMV), residual + record + next row preparation. */
plss_status plss_kz_profile(plss_ctx *ctx, int32_t k, double *ms);

/* ---- Growing-sketch engine, triangular factorization (section 2.4, Thm 2.1 / Cor 2.2,
 * L284-441) ----
 * For a sketch column s_k per step -- sketch 0: residual s_k = r_{k-1} (eq:S; Thm 4.1: PLSS's
 * updates); 1: identity s_k = e_{rows[k-1]} (section 7: PLSS Kaczmarz's updates); 2: Gaussian
 * s_k = column 0 of randomized projection's binary32 generator (reading R17) keyed by seed --
 * with y_k = A^T s_k and the stored Y (n x hk), R = [t_1 .. t_hk], D = diag(1/delta_j):
 *   g = Y^T y_k; t_hat = R D R^T g; delta = y_k^T y_k - g^T t_hat;
 *   p_k = (s_k^T r_{k-1} / delta) (y_k - Y t_hat)   (eq:compute-pk-alpha1, no solves);
 *   append y_k, t_hat, 1/delta; x_k = x_{k-1} + p_k; r_k = r_{k-1} - A p_k; stop test as plss_solve.
 * A step with delta <= 1e-14 y^T y, y = 0 or s^T r = 0 is skipped (p = 0, nothing appended;
 * reading R22); after kmax stored columns the history is cleared (R21). rows: host or dev,
 * maxit indices in [0, m) (identity sketch only; may be NULL otherwise). Single-device ctx;
 * shares the ctx's r, y, p, x, control block and history. workspace: dev, 256-byte aligned,
 * >= plss_eg_workspace_bytes(ctx, kmax) = 8 n kmax + 8 kmax^2 bytes + O(m + n).
 * factor 0: the triangular factorization above; factor 1: the QR variant (section 2.3, eq:pkQR,
 * L247-282): Y_k = Q_k T_k kept as Householder reflectors in compact WY form Q = I - V T V^T
 * (V in the Y store, T in the R store), p_k = (s_k^T r_{k-1} / r_kk) q_k with q_k = Q_k e_k;
 * delta_k = r_kk^2 (four passes over the store per step instead of two).
 * record k of `diag` = {hist_k, rho_k, delta_k, skipped (0/1), s_k^T r_{k-1}, history size}. */
size_t plss_eg_workspace_bytes(const plss_ctx *ctx, int32_t kmax); /* 0 on invalid input */
plss_status plss_eg_solve(plss_ctx *ctx, int32_t sketch, int32_t factor, int32_t kmax,
                          void *workspace, size_t ws_bytes, const int32_t *rows, uint64_t seed,
                          const double *b, const double *x0, double tol, int32_t tol_mode,
                          int32_t maxit, double *x, int32_t *iters, double *hist, double *diag,
                          plss_outcome *outcome);
plss_status plss_eg_start(plss_ctx *ctx, int32_t sketch, int32_t factor, int32_t kmax,
                          void *workspace, size_t ws_bytes, const int32_t *rows, uint64_t seed,
                          const double *b, const double *x0, double tol, int32_t tol_mode,
                          int32_t maxit);
plss_status plss_eg_step(plss_ctx *ctx, int32_t k);
plss_status plss_eg_finish(plss_ctx *ctx, double *x, int32_t *iters, double *hist, double *diag,
                           plss_outcome *outcome);
/* Per-kernel device ms per step (CUDA events, one kernel at a time) after plss_eg_start; ms
 * (host, 5 doubles): sketch + y = A^T s, Y^T y (partials + their reduction), triangular update,
 * p = coef (y - Y t_hat),
 * K1 (r <- r - A p). */
plss_status plss_eg_profile(plss_ctx *ctx, int32_t k, double *ms);

void plss_destroy(plss_ctx *ctx);
const char *plss_status_str(plss_status s);
const char *plss_last_error(const plss_ctx *ctx); /* NULL ctx: last error of create calls */

#ifdef __cplusplus
}
#endif
#endif /* PLSS_H */
