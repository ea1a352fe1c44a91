/*
 * sdpc.h - C ABI of libsdpc, the B200-native Schur-complement (SCM) engine for the
 * matrix-completion primal-dual interior-point method (MC-PDIPM) of
 * Yamashita & Nakata, arXiv 1310.6919 (PAPER.md, cited as P:<line>).
 *
 * One PDIPM iteration's hot path is three calls:
 *   sdpc_factor_xinv   (a1)  Algorithm 1: X-hat^{-1} = L D L^T from the partial X-bar on E
 *                            (Alg. 1; L-hat = L D^{1/2}).
 *   sdpc_scm_build     (a2)  Y = L_Y D_Y L_Y^T on E (type (v)),
 *                      (b)   x_p = X-hat e_p, y_q = Y^{-1} e_q by multi-RHS supernodal solves
 *                            (P:686-688 Eq. newSCM2, Alg. 2 Step 3-3),
 *                      (c)   B_kl = sum_{(p,q) in A_l} [A_l]_pq x_p^T A_k y_q  for k >= l
 *                            (P:380 Eq. SCM; lower triangle only).
 *   sdpc_scm_cholesky  (d)   dense B = R R^T in FP64 (type (i)).
 *   sdpc_iteration           (a1)..(d) in one call, (a1) || (a2) on two streams, one sync.
 *   sdpc_scm_solve           the SCE B dz = g with R.
 *   nranks > 1: sdpc_scm_build writes the rank's 2D block-cyclic tiles; sdpc_potrf_tile,
 *   sdpc_trsm_panel, sdpc_update_tiles are the tile kernels of the distributed Cholesky (row (e)).
 *
 * Conventions for every entry point:
 *   - 0-based indices.  "E" is the extended sparsity pattern as a lower CSC
 *     in ELIMINATION order: column j holds row j first, then struct(L_{*j}) ascending.
 *   - Host arrays passed in are COPIED; the caller keeps ownership.  Device pointers
 *     (xbar_E, y_E, B, L_E, D, ...) are owned by the caller (e.g. torch tensors) and
 *     must stay valid until the call returns.  The handle owns its factors,
 *     structure and workspaces and frees them in sdpc_destroy.
 *   - Calls enqueue on `stream` (a cudaStream_t passed as void*; NULL = legacy default)
 *     and RETURN AFTER THE STREAM WORK COMPLETED, so status and info are exact.
 *   - No exceptions or exit() cross the ABI.  Errors are status codes; the index
 *     of a failing pivot / clique is available through sdpc_last_info().
 *   - One handle per rank (GPU); calls on one handle must be serialised by the caller.
 *   - There is no CPU fallback: without a usable sm_100 device sdpc_create fails
 *     with SDPC_ERR_CUDA.
 */
#ifndef SDPC_H
#define SDPC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SDPC_OK = 0,
  SDPC_ERR_INVALID_ARG = 1,  /* bad size/pointer/pattern (e.g. perm not a permutation)           */
  SDPC_ERR_NOT_PD = 2,       /* a clique block, Y, or B is not positive definite; see last_info  */
  SDPC_ERR_OOM = 3,          /* device or host allocation failed                                 */
  SDPC_ERR_CUDA = 4,         /* CUDA runtime error, or no sm_100 device                          */
  SDPC_ERR_NCCL = 5,         /* NCCL failure (multi-GPU)                                         */
  SDPC_ERR_STATE = 6         /* call order violated (e.g. scm_build before factor_xinv)          */
} sdpc_status;

typedef struct sdpc_ctx* sdpc_handle;

/* Host views into the handle's symbolic structure (valid until sdpc_destroy). */
typedef struct {
  int32_t n;             /* order of X and Y                                                   */
  int32_t m;             /* number of constraints A_1..A_m                                      */
  int64_t nnzE;          /* |E| lower incl. diagonal                                            */
  const int32_t* perm;   /* [n] perm[new] = old (elimination order)                            */
  const int32_t* parent; /* [n] elimination-tree parent (new ids), -1 at roots                 */
  const int64_t* colptr; /* [n+1] CSC column pointers of E                                     */
  const int32_t* rowind; /* [nnzE] row indices, ascending, diagonal first in each column        */
  int32_t nsuper;        /* number of fundamental supernodes = cliques C_r of Algorithm 1      */
  const int32_t* super_ptr; /* [nsuper+1] first column of each supernode (S_r = [sp[r], sp[r+1])) */
} sdpc_structure;

/* 2D block-cyclic layout of B on this rank (1x1 grid when nranks == 1). */
typedef struct {
  int32_t nb;            /* tile size                                                          */
  int32_t Pr, Pc;        /* process grid                                                       */
  int32_t myrow, mycol;  /* this rank's grid coordinates                                       */
  int64_t mloc, nloc;    /* local rows / columns of B held by this rank                        */
  int64_t lld;           /* required minimum leading dimension of the local buffer             */
} sdpc_layout;

/*
 * sdpc_create - set up the problem (P): min A_0.X s.t. A_k.X = b_k (k = 1..m), X >= 0
 * (P:83-106), and run the one-time symbolic analysis:
 * aggregate pattern, elimination order, E, elimination tree,
 * fundamental supernodes used as the cliques C_r / S_r, solve schedules.
 *
 *   n, m        : order and number of constraints (n >= 1, m >= 1).
 *   a_ptr[m+2]  : entries of A_k are [a_ptr[k], a_ptr[k+1]) for k = 0..m (A_0 = objective).
 *   a_row, a_col, a_val : lower triplets, ORIGINAL ids, row >= col; [A_k]_ij = [A_k]_ji = val.
 *                 Duplicates within one A_k are summed.
 *   b[m]        : right-hand side; validated finite, does not enter B.
 *   perm[n]     : elimination order, perm[new] = old; NULL => built-in exact minimum degree
 *                 (ties -> smallest original id).
 *   device      : CUDA device ordinal this handle runs on.
 *   nranks, rank : multi-GPU world.  B is distributed 2D block-cyclically
 *                 in kScmNB = 256 tiles over a Pr x Pc grid (Pr = largest divisor of nranks
 *                 <= sqrt(nranks); rank = myrow * Pc + mycol; see sdpc_get_scm_layout).  Each
 *                 rank builds exactly its own tiles of B (columns l with (l/256) mod Pc == mycol
 *                 need the RHS x_p, y_q of A_l only, Eq. newSCM2: columns of B are
 *                 independent); (a1)/(a2) are replicated.  The library holds no
 *                 communicator unless created with an NCCL id (see nccl_id).
 *   nccl_id     : NULL, or the 128-byte NCCL unique id from sdpc_get_unique_id on one rank, shipped to
 *                 every rank by the caller (e.g. a torch.distributed broadcast).  With an id, the
 *                 nranks callers create collectively an NCCL world communicator plus process-row and
 *                 process-column communicators owned by the handle, and sdpc_scm_cholesky factors the
 *                 distributed B collectively.  Without one (nranks > 1), the caller drives the tile
 *                 entries below, or sdpc_scm_cholesky_virtual on one device.
 * Host arrays are copied.  Errors: INVALID_ARG (sizes, out-of-range ids, row < col,
 * perm not a permutation, rank outside [0, nranks)), OOM, CUDA (no device / not sm_100),
 * NCCL (communicator creation failed; message in sdpc_last_error_message).
 */
sdpc_status sdpc_create(sdpc_handle* out, int32_t n, int32_t m,
                        const int64_t* a_ptr, const int32_t* a_row, const int32_t* a_col,
                        const double* a_val, const double* b, const int32_t* perm,
                        int32_t device, int32_t nranks, int32_t rank, const void* nccl_id);

/* The 128-byte NCCL unique id for sdpc_create's nccl_id (call on one rank, broadcast to all).  NCCL is
 * loaded at run time (libnccl.so.2, or the path in SDPC_NCCL_LIB).  Errors: NCCL. */
sdpc_status sdpc_get_unique_id(void* id_out);

sdpc_status sdpc_get_structure(sdpc_handle h, sdpc_structure* out);
sdpc_status sdpc_get_scm_layout(sdpc_handle h, sdpc_layout* out);

/*
 * sdpc_factor_xinv - (a1) Algorithm 1: for every clique r, reverse-permute
 * X-bar_{C_r C_r} (Step 2-1), Cholesky it (Step 2-2), form L_r = P_r M_r^{-T} P_r (Step 2-3)
 * and keep its first |S_r| columns (Step 3).  Kept on device in the handle as unit-lower
 * L and diagonal D with L-hat = L D^{1/2}, X-hat^{-1} = L D L^T (SURVEY §8(c) reading #1).
 *   xbar_E : DEVICE [nnzE] fp64, X-bar on E in E's CSC order (sdpc_get_structure).
 * Errors: NOT_PD with sdpc_last_info() = clique index r (0-based) whose block failed.
 */
sdpc_status sdpc_factor_xinv(sdpc_handle h, const double* xbar_E, void* stream);

/* Copy the (a1) factor out: L_E DEVICE [nnzE] (unit diagonal stored), D DEVICE [n]. */
sdpc_status sdpc_get_xinv_factor(sdpc_handle h, double* L_E, double* D, void* stream);

/*
 * sdpc_scm_build - (a2)+(b)+(c).  Factors Y = L_Y D_Y L_Y^T on E (NOT_PD: last_info =
 * elimination column j), evaluates x_p = X-hat e_p and y_q = Y^{-1} e_q for the needed
 * columns, and writes B_kl = (X-hat A_k Y^{-1}) . A_l for k >= l into the lower triangle of
 * the column-major B (constraint order as given; k, l = 0..m-1 <-> A_1..A_m).
 * The strict upper triangle of B is not referenced.
 *   y_E : DEVICE [nnzE] fp64, Y on E in E's CSC order.
 *   B   : DEVICE, m x m column-major with leading dimension ldb >= m (nranks == 1), or this
 *         rank's local 2D block-cyclic array (mloc x nloc, ldb >= lld; sdpc_get_scm_layout)
 *         when nranks > 1: only the rank's own tiles are written, at local addresses.
 * Requires a successful sdpc_factor_xinv on this handle (else STATE).
 */
sdpc_status sdpc_scm_build(sdpc_handle h, const double* y_E, double* B, int64_t ldb, void* stream);

/* Copy the (a2) factor out: L_Y DEVICE [nnzE], D_Y DEVICE [n] (after sdpc_scm_build). */
sdpc_status sdpc_get_y_factor(sdpc_handle h, double* LY_E, double* DY, void* stream);

/*
 * Truncated backward sweep (default on).  For a max-cut SCM on one rank (B = X-hat o Y^{-1}),
 * the multi-RHS backward solve for the RHS panel starting at column p stops at row p: the entry
 * {k, l} of B is taken from the panel of the smaller elimination index (SURVEY §8(a) notes).
 * Off (0): every column is solved in full (needed for sdpc_get_inverse_columns).
 */
sdpc_status sdpc_set_truncation(sdpc_handle h, int32_t on);

/*
 * Schedule of the one-GPU SCM Cholesky (d).  1 (default): one persistent kernel over the
 * tile task graph (128-tiles; POTRF / TRSM / trailing-update tasks popped from device ready queues as
 * their inputs complete); used when B is 16-byte aligned with an even ldb, else 0 is used.  0: the
 * multi-launch blocked schedule with depth-2 lookahead on two streams.  Same result up to rounding.
 */
sdpc_status sdpc_set_cholesky_schedule(sdpc_handle h, int32_t task_graph);

/*
 * Diagnostics of the task-graph Cholesky: with cap > 0 every later factorisation records up to cap
 * tasks as {task word, start ns, end ns, smid | cta << 32} (GPU global timer; task word = type << 60 |
 * half << 56 | k << 32 | i << 16 | j, type 1 POTRF, 2 TRSM, 3 UPD); cap = 0 turns it off.
 * sdpc_get_cholesky_trace copies the trace buffer (HOST out [4 cap]) and the record count; when
 * cap >= 1 + 4T (T = ceil(m / 128)) its last 16T words hold per-POTRF phase stamps [T][16] (start, tile
 * loaded, 4 x panel factored, L stored, end, inverse computed, 6 x inverse block done).
 */
sdpc_status sdpc_set_cholesky_trace(sdpc_handle h, int64_t cap);
sdpc_status sdpc_get_cholesky_trace(sdpc_handle h, uint64_t* out, int64_t cap, int64_t* n);

/*
 * Copy selected columns of X-hat and Y^{-1} computed by the last sdpc_scm_build ((b) output,
 * for verification; STATE if that build used the truncated sweep).  cols: HOST [ncols] ORIGINAL vertex ids.  X_out, Y_out: DEVICE
 * n x ncols column-major (ld = n), rows in ORIGINAL order.
 */
sdpc_status sdpc_get_inverse_columns(sdpc_handle h, const int32_t* cols, int32_t ncols,
                                     double* X_out, double* Y_out, void* stream);

/*
 * sdpc_scm_cholesky - (d) in place: lower(B) <- R with B = R R^T (LAPACK potrf 'L' rule).
 *   info (HOST): 0 on success; k > 0 if the leading minor of order k is not positive
 *   definite (pivot <= 0 or NaN), in which case status = NOT_PD and last_info = k.
 * Handle created with an NCCL id: B is this rank's local 2D block-cyclic array (mloc x nloc, ldb >= lld)
 *   and the call is collective over the nranks processes: right-looking 256-tile steps (tile potrf on
 *   the owner, broadcast down the process column, panel trsm, the live panel slice broadcast along process
 *   rows and all-gathered in process columns, local DMMA trailing updates with depth-1 lookahead; row (e),
 *   SURVEY §8(e)).  info is the smallest failing global column, identical on every rank.
 * nranks > 1 without a communicator: STATE.
 */
sdpc_status sdpc_scm_cholesky(sdpc_handle h, double* B, int64_t ldb, int32_t* info, void* stream);

/*
 * sdpc_scm_cholesky_virtual - the same distributed factorisation with every rank of the grid in this
 * process on one device (test transport: hs[r] = the handle of rank r, created with nranks and no NCCL
 * id; B[r] its local array): the host runs each rank's part of every step in turn on `stream` and the
 * collectives are device copies between the ranks' buffers (no rank waits on another inside a kernel).
 * info and status as for sdpc_scm_cholesky (set on every handle).
 */
sdpc_status sdpc_scm_cholesky_virtual(const sdpc_handle* hs, int32_t nranks, double* const* B, int64_t ldb,
                                      int32_t* info, void* stream);

/*
 * sdpc_scm_solve - the Schur complement equation (SCE) of the search direction, B dz = g
 * (SURVEY §8(f) NEXT row 2), with the factor of sdpc_scm_cholesky: (R R^T) X = G.
 *   R : DEVICE m x m column-major (ldr >= m), lower triangle = R (as left in B by the Cholesky).
 *   G : DEVICE m x nrhs column-major (ldg >= m), overwritten with X.
 * Blocked forward / backward substitution (128-row blocks); nranks == 1.  The inverses of R's diagonal
 * 128-tiles are formed first, one CTA per tile in parallel, so the serial step of each block is a
 * 128 x 128 matrix-vector product; each sweep is one cooperative launch that reads R once (an R that is
 * not 16-byte aligned with an even ldr solves the diagonal triangles serially instead).
 */
sdpc_status sdpc_scm_solve(sdpc_handle h, const double* R, int64_t ldr, double* G, int64_t ldg,
                           int32_t nrhs, void* stream);

/*
 * Tile entries of the distributed (nranks > 1) SCM Cholesky, a 2D block-cyclic right-looking
 * blocked Cholesky (P:711-713 type (i), P:1012 SDPARA-C's distributed variant).
 * Per step k (tile column k of size kb <= 256, global rows from k1 = 256 k):
 *   owner of tile (k, k):  sdpc_potrf_tile   (factor the tile, 128-block inverses out)
 *   process column k:      sdpc_trsm_panel   (its panel tiles <- A L_kk^{-T})
 *   every rank:            sdpc_update_tiles (its trailing tiles -= panel panel^T)
 * with the caller broadcasting the factored tile down the process column and gathering the panel
 * to every rank between the calls.  All three are ASYNCHRONOUS: enqueued on `stream`, they return
 * without synchronising (unlike the rest of this ABI).  Matrices are column-major DEVICE arrays.
 *
 * sdpc_potrf_tile: A (n x n, lda >= n, n <= 256) <- its lower Cholesky factor in place (upper
 *   part untouched); inv (DEVICE, 2 x 128 x 128, column-major) <- inverses of the factor's two
 *   128-diagonal blocks (input of sdpc_trsm_panel); info_dev (DEVICE int32) <- 0x7f7f7f7f if PD,
 *   else the 1-based local column of the first non-positive pivot (LAPACK rule).
 */
sdpc_status sdpc_potrf_tile(sdpc_handle h, double* A, int32_t n, int64_t lda, double* inv,
                            int32_t* info_dev, void* stream);

/* sdpc_trsm_panel: A (rows x kb, lda >= rows) <- A L^{-T}, L = the kb x kb factored tile
 * (ldl >= kb) and inv its block inverses from sdpc_potrf_tile (a failed tile factorisation is
 * reported by its info; the later tile calls still run, on meaningless values). */
sdpc_status sdpc_trsm_panel(sdpc_handle h, double* A, int64_t rows, int64_t lda, const double* L,
                            int64_t ldl, const double* inv, int32_t kb, void* stream);

/* sdpc_update_tiles: for every local tile (I, J) of this rank with I >= J, 256 J >= k1 and
 * jlo <= J < jhi (global tile columns; jhi <= 0: no upper bound): C_IJ -= P_I P_J^T (lower part
 * only when I == J).  C = local array (mloc x nloc, ldc >= mloc); P = the gathered panel: row r is
 * global row k1 + r (r < m - k1), K columns, ldp >= m - k1.  The column range lets the caller
 * update the next panel's tile column first (lookahead) and the rest on another stream. */
sdpc_status sdpc_update_tiles(sdpc_handle h, double* C, int64_t ldc, const double* P, int64_t ldp,
                              int64_t k1, int32_t K, int64_t jlo, int64_t jhi, void* stream);

/*
 * sdpc_iteration - the whole hot path on DEVICE buffers in one call (what bench.py times):
 * (a1) sdpc_factor_xinv and (a2) the factorisation of Y run concurrently on two streams (they are
 * independent), then (b), (c) and (d) as in sdpc_scm_build + sdpc_scm_cholesky, with a single
 * synchronisation at the end.  Arguments as for those calls (B: m x m column-major, ldb >= m).
 * Errors: NOT_PD with sdpc_last_info() = the index of the first failing phase in the order (a1)
 * clique r, (a2) column j, (d) leading minor k; *info = k only for (d) (else 0).  nranks == 1 only.
 */
sdpc_status sdpc_iteration(sdpc_handle h, const double* xbar_E, const double* y_E, double* B,
                           int64_t ldb, int32_t* info, void* stream);

/*
 * sdpc_iteration_host - the whole hot path from HOST buffers (what a host-side PDIPM driver
 * calls once per iteration): copies xbar_E and y_E (HOST [nnzE]) to the device, runs
 * sdpc_iteration into a handle-owned B, and copies back
 * rdiag (HOST [m], the diagonal of R; NULL allowed) and info (HOST).
 */
sdpc_status sdpc_iteration_host(sdpc_handle h, const double* xbar_E, const double* y_E,
                                double* rdiag, int32_t* info, void* stream);

/* Per-phase device times (ms) of the last calls, from CUDA events on the call's stream:
 * t[0]=(a1) t[1]=(a2) t[2]=(b) t[3]=(c) t[4]=(d) t[5]=(d) trailing-update kernels only,
 * t[6]=number of (d) trailing-update launches, t[7]=their total algorithmic flops.
 * After sdpc_iteration, where (a1), (a2) and (b) overlap, t[0], t[1], t[2] are the times from the
 * start of the iteration to the end of (a1), (a2) and (b) respectively. */
sdpc_status sdpc_get_phase_times(sdpc_handle h, double* t /* [8] */);

/* Kernel windows (ms) of the last sdpc_iteration, CUDA events on the launching streams: t[0] = the X-hat
 * solve launch ((b), factor 1), t[1] = the Y^{-1} solve launch ((b), factor 2; runs concurrently with
 * t[0]'s tail), t[2] = the accumulate (c), t[3] = the SCM Cholesky kernel(s) (d), t[4] = start -> (a1)
 * done, t[5] = start -> (a2) done, t[6], t[7] reserved (0).  Used for the per-phase roofline fractions. */
sdpc_status sdpc_get_kernel_times(sdpc_handle h, double* t /* [8] */);

/* Enable (1) / disable (0) per-phase event timing (default on; costs a few events per call). */
sdpc_status sdpc_set_timing(sdpc_handle h, int32_t on);

/* Number of kernel launches the handle issued since creation (evidence for gpu_launches). */
int64_t sdpc_launch_count(sdpc_handle h);

/*
 * sdpc_search_direction - the HKM search direction of the iteration,
 * after sdpc_scm_build (or sdpc_iteration) and sdpc_scm_cholesky on the same handle, as printed in
 * PAPER.md §2.2:
 *   g_k  = A_k . (beta_mu Y^{-1} - X-hat - X-hat G Y^{-1})   (k = 1..m; A_k . X-hat = A_k . X-bar on E)
 *   B dz = g            (forward / backward substitution with R, the factor left in B by the Cholesky)
 *   dY   = G - sum_k A_k dz_k                                on E
 *   dX   = (dX-hat + dX-hat^T) / 2 on E, column k of dX-hat = beta_mu Y^{-1} e_k - X-hat e_k
 *          - X-hat dY Y^{-1} e_k   (P-MATRIX, Eq. newdX2; only entries on E are kept)
 *   xbar_E, G_E : DEVICE [nnzE] X-bar and the residual matrix G on E (E's CSC order).  G is taken as
 *                 given (the paper prints G = A_0 - sum A_k z_k).
 *   beta_mu     : beta * mu, mu = X . Y / n.
 *   R, ldr      : DEVICE, the SCM factor (lower triangle of the B passed to sdpc_scm_cholesky).
 *   g, dz       : DEVICE [m] out;  dY_E, dX_E : DEVICE [nnzE] out.
 * Uses the handle's X-hat / Y^{-1} columns (re-solved in full when the build used the truncated max-cut
 * sweep) and an extra dense panel buffer (the size of one of them).  Synchronous.  Errors: STATE
 * (nranks > 1, no build, or some vertex in no constraint: every vertex must be a solve RHS), OOM.
 */
sdpc_status sdpc_search_direction(sdpc_handle h, const double* xbar_E, const double* G_E, double beta_mu,
                                  const double* R, int64_t ldr, double* g, double* dz, double* dY_E,
                                  double* dX_E, void* stream);

/*
 * sdpc_step_lengths - Step 3 of the PDIPM with the completion (Eq. primal_length2):
 *   alpha_p = min_r max{alpha in (0,1] : X-bar_{C_rC_r} + alpha dX_{C_rC_r} >= 0}  (cliques = supernodes)
 *   alpha_d = max{alpha in (0,1] : Y + alpha dY >= 0}
 * by bisection with attempted Cholesky factorisations: per clique block for alpha_p (one CTA per clique,
 * 40 steps, the returned value is feasible and within 2^-40 of the boundary), the sparse LDL^T of
 * Y + alpha dY on E for alpha_d (30 steps, within 2^-30).  All inputs DEVICE [nnzE] on E; alpha_p and
 * alpha_d HOST out.  The handle's Y factor is overwritten (a later sdpc_scm_build refactors Y).
 */
sdpc_status sdpc_step_lengths(sdpc_handle h, const double* xbar_E, const double* dX_E, const double* y_E,
                              const double* dY_E, double* alpha_p, double* alpha_d, void* stream);

/*
 * FP64 roof microbenchmarks (N10): sustained DMMA (mma.sync m8n8k4 f64 -> DMMA.8x8x4) and
 * DFMA throughput over all SMs for about `ms` milliseconds each.  Outputs TFLOP/s.
 */
sdpc_status sdpc_fp64_peak(int32_t device, double ms, double* dmma_tflops, double* dfma_tflops);

sdpc_status sdpc_destroy(sdpc_handle h);
const char* sdpc_status_string(sdpc_status s);
int64_t sdpc_last_info(sdpc_handle h);
/* Human-readable detail of the last CUDA/NCCL error seen by the handle ("" if none). */
const char* sdpc_last_error_message(sdpc_handle h);

#ifdef __cplusplus
}
#endif
#endif /* SDPC_H */
