// Internal handle state of libsdpc and the kernel launchers' interfaces.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "common.cuh"
#include "symbolic.hpp"

namespace sdpc {

// Device mirror of the symbolic structure (all arrays owned by the handle).
struct DevSym {
  int32_t n = 0, m = 0, nsuper = 0;
  int64_t nnzE = 0;
  int64_t* colptr = nullptr;
  int32_t* rowind = nullptr;
  int32_t* super_ptr = nullptr;
  int32_t* snc = nullptr;
  int32_t* sns = nullptr;
  int32_t* sparent = nullptr;
  int64_t* panel_off = nullptr;
  int32_t* e2p = nullptr;
  int64_t* umap_off = nullptr;
  int32_t* umap = nullptr;
  int64_t* relind_off = nullptr;
  int32_t* relind = nullptr;
  int64_t* upd_off = nullptr;
  int32_t* child_ptr = nullptr;
  int32_t* child_list = nullptr;
  int32_t* hlev_sn = nullptr;   // supernodes sorted by height
  int32_t* dlev_ptr = nullptr;  // depth level pointers (device copy)
  int32_t* dlev_sn = nullptr;
  int32_t* preorder = nullptr;
  int32_t* border = nullptr;
  int32_t* sub_ptr = nullptr;
  int32_t* perm = nullptr;
  int32_t* iperm = nullptr;
  int32_t* reach_ptr = nullptr;  // per RHS panel: supernodes on the union of etree paths
  int32_t* reach_sn = nullptr;
  int32_t npanels = 0;
  // RHS slots: the solves compute X-hat e_v and Y^{-1} e_v for v = rhs[s] (elimination id, -1 =
  // padding), s = 32 P + lane; slot_of[v] = s or -1.  rhs = every vertex that is a column p of some
  // A_l with l a column of B held by this rank (all touched vertices when nranks == 1).
  int32_t* rhs = nullptr;
  int32_t* slot_of = nullptr;
  int32_t nrhs = 0;
  int32_t* all_sn = nullptr;     // 0 .. nsuper-1 (full forward sweep of a dense RHS panel)
  // search direction (k_direction.cu): symmetric CSR of E (row i: columns j with (i, j) or (j, i) in E,
  // sym_pos = offset of that entry in E's CSC value order); per E entry the constraint entries on it
  int32_t* sym_ptr = nullptr;
  int32_t* sym_col = nullptr;
  int32_t* sym_pos = nullptr;
  int32_t* ecs_ptr = nullptr;    // [nnzE + 1]
  int32_t* ecs_k = nullptr;      // constraint (0-based)
  double* ecs_val = nullptr;     // value of its entry (lower triplet, duplicates listed separately)
  int32_t* cons_epos = nullptr;  // per symmetric-expanded constraint entry (DevCons order): E offset
};

// Size classes of the batched per-clique kernels ((a1) and (a2)).
struct CliqueClass {
  int threads = 64;
  size_t smem = 0;          // dynamic shared memory bytes (0 => global workspace)
  std::vector<int32_t> sn;  // supernodes in this class
  int32_t* d_sn = nullptr;
};

// Constraint data in elimination ids, symmetric-expanded (for (c)).
struct DevCons {
  bool maxcut = false;
  int32_t m = 0;
  int64_t* ptr = nullptr;  // [m+1]
  int32_t* ei = nullptr;   // entry row (new id)
  int32_t* ej = nullptr;   // entry col (new id)
  double* ev = nullptr;
  int32_t* large = nullptr;     // list of constraint ids with many entries
  int32_t nlarge = 0;
  uint8_t* is_large = nullptr;  // [m]
  // max-cut fast path
  int32_t* vrow = nullptr;      // [m] elimination row of constraint k's vertex
  double* aval = nullptr;       // [m] value a_k
  int32_t* col_cons = nullptr;  // [n] constraint index whose vertex is elimination column j, or -1
  // staged-rows accumulation (one rank, identity slots): see k_scm.cu
  bool rows_mode = false;
  int32_t nvmax = 0, ndiag = 0;
  int32_t* vptr = nullptr;      // [m+1] distinct vertices V_l of small constraint l
  int32_t* vlist = nullptr;
  int32_t* eloc = nullptr;      // [2 * entries] positions of p (= ej) and q (= ei) in V_l
  uint8_t* diag_large = nullptr;  // [m] large constraint with diagonal entries only
  double* wdiag = nullptr;      // [ndiag][n] their weights
  int32_t* dlist = nullptr;     // [ndiag] their constraint ids
};
constexpr size_t kRowsSmemCap = 200 * 1024;

}  // namespace sdpc

struct sdpc_ctx {
  int device = 0;
  int nranks = 1, rank = 0;
  sdpc::Grid grid;                 // 2D block-cyclic process grid of B
  std::vector<int32_t> slot_of_host;  // host copy of DevSym::slot_of
  std::vector<int32_t> diag_ids;      // host copy of DevCons::dlist
  double* pair_ws = nullptr;          // partial sums of the diagonal-large pair reductions
  double* sce_ws = nullptr;           // scratch of sdpc_scm_solve (nrhs x 128)
  double* sce_linv = nullptr;         // inverses of R's diagonal 128-tiles (sdpc_scm_solve)
  int64_t sce_linv_cap = 0;
  int64_t sce_cap = 0;
  int64_t mloc = 0, nloc = 0;      // local rows / columns of B on this rank
  sdpc::Symbolic S;
  sdpc::DevSym d;
  sdpc::DevCons cons;
  std::vector<sdpc::CliqueClass> a1cls, a2cls;  // per-level classes for (a2) are rebuilt per level
  std::vector<std::vector<sdpc::CliqueClass>> a2lev;
  double* ws = nullptr;          // global workspace for large cliques of (a1)
  double* ws2 = nullptr;         // ... and of (a2) (separate: the two may run concurrently)
  int64_t* d_ws_off = nullptr;   // per supernode offset into ws (doubles), -1 if smem class
  // (a2) pre-pass extend-add for global fronts with many children (per height level)
  uint8_t* d_pre = nullptr;
  int32_t* d_pre_child = nullptr;
  int32_t* d_pre_parent = nullptr;
  int32_t* d_zero_list = nullptr;
  std::vector<int32_t> pre_ptr, zero_ptr;
  // (a2) big fronts (global workspace) per etree height: list offsets, max Schur tiles, panel smem
  std::vector<int32_t> big_ptr, big_tiles;
  std::vector<uint8_t> big_thin, big_wide;  // level has big fronts with |S| <= 32 / > 32
  // (a1) big cliques (a1cls[3], decreasing c): workspace offsets / dims / error slots, L^{-1} buffers
  int32_t nbig1 = 0;
  std::vector<int32_t> big1_c;
  int64_t* big1_off = nullptr;
  int32_t* big1_dim = nullptr;
  int32_t* big1_err = nullptr;
  double* big1_ws = nullptr;
  double* big1_linv = nullptr;
  int32_t* d_big_list = nullptr;
  size_t big_smem = 0;
  double* Lx = nullptr;          // X factor panels
  double* Dx = nullptr;
  double* Ly = nullptr;          // Y factor panels
  double* Dy = nullptr;
  double* upd = nullptr;         // multifrontal update matrices
  double* Xh = nullptr;          // dense X-hat, panel-major [npanels][n][32]
  double* Yh = nullptr;          // dense Y^{-1}
  double* Uh = nullptr;          // search direction: dense panels G Y^{-1} / dY Y^{-1}, then X-hat times them
  double* dir_ws = nullptr;      // search direction scratch (m doubles + flags)
  std::vector<int64_t> step_off; // primal step length: per clique offset of its 3 c x c blocks
  int64_t* d_step_off = nullptr;
  double* step_ws = nullptr;
  unsigned long long* d_amin = nullptr;
  double* ytmp = nullptr;        // dual step length: Y + alpha dY on E
  int32_t* d_err = nullptr;
  int32_t* d_ok = nullptr;       // constant kNoError flag (distributed tile kernels)
  double* Bown = nullptr;        // handle-owned B for sdpc_iteration_host
  double* xin = nullptr;         // device staging for sdpc_iteration_host
  double* yin = nullptr;
  double* pinned_in = nullptr;   // pinned host staging (2*nnzE)
  double* pinned_out = nullptr;  // pinned host staging (m)
  double* potrf_ws = nullptr;    // inverses of the diagonal blocks (2 x nb x nb, double-buffered)
  // persistent task-graph Cholesky (k_chol_dag.cu): zeroed control/counters/queues, L_kk^{-1} tiles
  void* dag_ws = nullptr;
  double* dag_linv = nullptr;
  int64_t* dag_koff = nullptr;
  int dag_T = -1, dag_dev = -1, dag_grid = 0;
  bool use_dag = true;           // sdpc_set_cholesky_schedule: 1 = task graph, 0 = round-1 multi-launch
  size_t dag_zero_bytes = 0;
  unsigned long long* dag_trace = nullptr;  // optional per-task trace (sdpc_set_cholesky_trace)
  int64_t dag_trace_cap = 0;
  cudaStream_t st2 = nullptr;    // lookahead stream of the SCM Cholesky
  void* nccl_world = nullptr;    // ncclComm_t (sdpc_create with an NCCL id): world, process row, process column
  void* nccl_row = nullptr;
  void* nccl_col = nullptr;
  cudaStream_t dist_side = nullptr;  // side stream of the distributed Cholesky's bulk updates
  cudaStream_t side[4] = {nullptr, nullptr, nullptr, nullptr};  // = sides[0]: (a1) size classes
  cudaEvent_t side_ev[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaStream_t sides[2][4] = {};   // [0]: (a1) / (a2) size classes, [1]: (a2) inside sdpc_iteration
  cudaEvent_t sides_ev[2][4] = {};
  cudaEvent_t fork_ev = nullptr, fork_ev2 = nullptr;
  cudaStream_t st3 = nullptr;      // (a2) stream of sdpc_iteration (concurrent with (a1))
  cudaEvent_t it_fork = nullptr, it_join = nullptr;
  cudaEvent_t evA = nullptr, evB = nullptr;
  bool have_x = false, have_y = false;
  bool truncate = true;          // allow the truncated backward sweep (max-cut, one rank)
  bool trunc_active = false;     // the last sdpc_scm_build used it
  int64_t last_info = 0;
  bool timing = true;
  double times[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  double ktimes[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // sdpc_get_kernel_times
  int64_t launches = 0;
  cudaEvent_t ev[16];
  std::vector<cudaEvent_t> upd_ev;  // per trailing-update launch (pairs)
  std::string err;
};

namespace sdpc {
// Launchers (each returns number of kernels launched; errors via cudaGetLastError).
int launch_alg1(sdpc_ctx* h, const double* xbar, cudaStream_t st);
int launch_ldl_y(sdpc_ctx* h, const double* y, cudaStream_t st, int32_t* err = nullptr, int set = 0);
int launch_inverse_panels(sdpc_ctx* h, cudaStream_t st, int fac0 = 0, int nfac = 2, int max_ctas = 0);
int launch_apply_inverse(sdpc_ctx* h, cudaStream_t st, int fac, const double* in, double* out);
bool solve_smem_fits(int64_t nsuper);
int launch_scm(sdpc_ctx* h, double* B, int64_t ldb, cudaStream_t st);
int launch_panels_to_E(sdpc_ctx* h, const double* panels, double* E, cudaStream_t st);
int launch_gather_columns(sdpc_ctx* h, const int32_t* d_cols_new, int32_t ncols, double* Xo, double* Yo,
                          cudaStream_t st);
// Dense FP64 Cholesky of the lower triangle of B (m x m, ld).  Returns launches; info via d_err
// (1-based failing column, kNoError if ok).  If upd_times, records an event pair per trailing update.
int potrf_lower(sdpc_ctx* h, double* B, int64_t m, int64_t ld, int32_t* d_err, cudaStream_t st, double* flops_upd,
                int* n_upd, double* linv_ws);
// The same factorisation as one persistent kernel over the tile task graph (k_chol_dag.cu); needs B
// 16-byte aligned with an even ld (potrf_dag_usable).  Returns launches (-1: workspace allocation failed).
bool potrf_dag_usable(const double* B, int64_t ld);
int tile_inverses(const double* R, int64_t ldr, int64_t m, double* out, cudaStream_t st);
int potrf_dag(sdpc_ctx* h, double* B, int64_t m, int64_t ld, int32_t* d_err, cudaStream_t st);
// Batched right-looking Cholesky (k_chol_dag.cu), step q over the first nact matrices (sorted by
// decreasing dim; maxdim = dim of the first).  Matrix b: base + off[b], ld = dim + (dim & 1), 16-byte
// aligned.  err_slot[b] (kNoError-initialised) records its failure, err_id[b] is reported into *err.
struct BatchDesc {
  double* base;
  const int64_t* off;
  const int32_t* dim;
  int32_t* err_slot;
  const int32_t* err_id;
  int32_t* err;
  double* linv;  // [nbatch][128 * 128]
};
int batched_chol_step(const BatchDesc& d, int q, int nact, int maxdim, cudaStream_t st);
// Search direction and step lengths (k_direction.cu); each returns launches or -1.
int direction_g(sdpc_ctx* h, const double* xbar_E, const double* G_E, double bmu, double* g, cudaStream_t st);
int direction_dY_dX(sdpc_ctx* h, const double* xbar_E, const double* G_E, double bmu, const double* dz, double* dY_E,
                    double* dX_E, cudaStream_t st);
int primal_step(sdpc_ctx* h, const double* xbar_E, const double* dX_E, double* alpha_p, cudaStream_t st);
int dual_step(sdpc_ctx* h, const double* y_E, const double* dY_E, double* alpha_d, int steps, cudaStream_t st);
// NCCL (dist_chol.cu, loaded with dlopen) and the distributed SCM Cholesky behind sdpc_scm_cholesky.
int nccl_unique_id(void* out, std::string* why);
int nccl_init(sdpc_ctx* h, const void* id, std::string* why);
void nccl_destroy(sdpc_ctx* h);
int dist_cholesky_handles(sdpc_ctx* const* hs, double* const* B, int64_t ld, int nloc_ranks, bool virt,
                          cudaStream_t st, int64_t* info, std::string* why);
// Distributed-Cholesky tile kernels; see sdpc.h.
int trsm_panel(double* A, int64_t rows, int64_t lda, const double* Lt, int64_t ldl, const double* inv, int kb,
               const int32_t* d_err, cudaStream_t st);
int update_tiles(double* C, int64_t ldc, const double* P, int64_t ldp, int64_t k1, int K, const Grid& g, int64_t m,
                 int64_t mloc, int64_t nloc, const int32_t* d_err, cudaStream_t st, int64_t jlo, int64_t jhi);
int launch_diag_copy(double* B, int64_t m, int64_t ld, double* out, cudaStream_t st);
// (R R^T) X = G in place, R lower (m x m, ldr); S: nrhs x 128 doubles of scratch
int scm_solve(const double* R, int64_t ldr, int64_t m, double* G, int64_t ldg, int nrhs, double* S, cudaStream_t st,
              const double* Linv = nullptr);
cudaError_t fp64_peak(int device, double ms, double* dmma, double* dfma);
}  // namespace sdpc
