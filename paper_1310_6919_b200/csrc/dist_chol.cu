// Row (e): the distributed SCM Cholesky of a 2D block-cyclic B behind sdpc_scm_cholesky (
// PAPER.md P:711-713 type (i), P:1012 SDPARA-C's distributed variant).
//
// Right-looking, 256-tiles over a Pr x Pc grid (ScaLAPACK convention, include/sdpc.h).  Per step k:
//   1. the owner of tile (k, k) factors it (tile potrf, also returning the two 128-block inverses);
//   2. tile + inverses are broadcast down process column k mod Pc;
//   3. that process column solves its panel tiles (trsm with the explicit inverses);
//   4. the panel reaches every rank: broadcast along each process row from column k mod Pc (only the
//      live kb x (rows) slice), then all-gathered within each process column and laid out by global
//      tile row (assemble_panel_kernel);
//   5. every rank updates its trailing tiles: tile column k+1 first, the rest on a side stream while
//      panel k+1 is factored and communicated (depth-1 lookahead).
// info = the smallest failing global column over all ranks (LAPACK potrf rule), identical everywhere.
//
// Transports.  NCCL (one process per GPU): a world communicator from the caller's 128-byte id plus
// process-row / process-column communicators (ncclCommSplit); NCCL is loaded with dlopen, so the
// library links against no particular NCCL and shares the one already loaded by the process.
// Virtual ranks (test transport, one device): the host drives every rank's part of each step in turn
// on one stream and implements the collectives as device copies between the ranks' buffers - no rank
// ever waits on another inside a kernel.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "ctx.hpp"

namespace sdpc {

// ---------------------------------------------------------------- NCCL by dlopen
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
};

static NcclApi load_nccl() {
  NcclApi a;
  const char* env = getenv("SDPC_NCCL_LIB");
  void* lib = nullptr;
  for (const char* name : {env, "libnccl.so.2", "libnccl.so"}) {
    if (!name) continue;
    lib = dlopen(name, RTLD_NOW | RTLD_LOCAL);
    if (lib) break;
  }
  if (!lib) {
    a.why = "libnccl.so.2 not found (set SDPC_NCCL_LIB)";
    return a;
  }
#define SYM(field, name)                                                     \
  a.field = reinterpret_cast<decltype(a.field)>(dlsym(lib, name));           \
  if (!a.field) {                                                            \
    a.why = std::string("NCCL symbol missing: ") + name;                     \
    return a;                                                                \
  }
  SYM(getUniqueId, "ncclGetUniqueId");
  SYM(commInitRank, "ncclCommInitRank");
  SYM(commSplit, "ncclCommSplit");
  SYM(commDestroy, "ncclCommDestroy");
  SYM(broadcast, "ncclBroadcast");
  SYM(allGather, "ncclAllGather");
  SYM(allReduce, "ncclAllReduce");
  SYM(errorString, "ncclGetErrorString");
#undef SYM
  a.ok = true;
  return a;
}

static NcclApi& nccl() {
  static NcclApi a = load_nccl();
  return a;
}

int nccl_unique_id(void* out, std::string* why) {
  NcclApi& n = nccl();
  if (!n.ok) {
    *why = n.why;
    return -1;
  }
  ncclUniqueId id;
  const ncclResult_t r = n.getUniqueId(&id);
  if (r != ncclSuccess) {
    *why = n.errorString(r);
    return -1;
  }
  std::memcpy(out, &id, sizeof(id));
  return 0;
}

int nccl_init(sdpc_ctx* h, const void* id, std::string* why) {
  NcclApi& n = nccl();
  if (!n.ok) {
    *why = n.why;
    return -1;
  }
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t w = nullptr, row = nullptr, col = nullptr;
  ncclResult_t r = n.commInitRank(&w, h->nranks, uid, h->rank);
  if (r == ncclSuccess) r = n.commSplit(w, h->grid.pr, h->grid.pc, &row, nullptr);  // same process row
  if (r == ncclSuccess) r = n.commSplit(w, h->grid.pc, h->grid.pr, &col, nullptr);  // same process column
  if (r != ncclSuccess) {
    *why = n.errorString(r);
    return -1;
  }
  h->nccl_world = w;
  h->nccl_row = row;
  h->nccl_col = col;
  return 0;
}

void nccl_destroy(sdpc_ctx* h) {
  if (!nccl().ok) return;
  for (void* c : {h->nccl_col, h->nccl_row, h->nccl_world})
    if (c) nccl().commDestroy(static_cast<ncclComm_t>(c));
  h->nccl_world = h->nccl_row = h->nccl_col = nullptr;
}

// ---------------------------------------------------------------- schedule
constexpr int NB = kScmNB;
constexpr int kInv = 2 * 128 * 128;

// P[c * ldp + (t_glob - (k + 1)) * NB + e] = src_pr[c * ldg + t * NB + e] for the tiles of process row
// pr: t_glob = first_pr + t Pr (the all-gathered panel laid out by global tile row)
__global__ void assemble_panel_kernel(double* P, int64_t ldp, const double* G, int64_t ldg, int64_t stride_pr,
                                      int kb, int Pr, int k, int nt) {
  const int pr = blockIdx.y;
  const int first = k + 1 + (((pr - (k + 1)) % Pr) + Pr) % Pr;
  const int cnt = first < nt ? (nt - first + Pr - 1) / Pr : 0;
  const double* src = G + (int64_t)pr * stride_pr;
  const int64_t tot = (int64_t)kb * cnt * NB;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < tot; x += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(x / ((int64_t)cnt * NB));
    const int64_t rem = x % ((int64_t)cnt * NB);
    const int t = (int)(rem / NB), e = (int)(rem % NB);
    P[(int64_t)c * ldp + (int64_t)(first + t * Pr - (k + 1)) * NB + e] = src[(int64_t)c * ldg + (int64_t)t * NB + e];
  }
}

struct DRank {
  sdpc_ctx* h = nullptr;
  double* B = nullptr;
  int64_t ld = 0;
  cudaStream_t main = nullptr, side = nullptr;
  cudaEvent_t ev = nullptr;
  double* diag = nullptr;      // NB x NB tile (ld NB) + the two 128-block inverses
  double* piece[2] = {nullptr, nullptr};
  double* gathered[2] = {nullptr, nullptr};
  double* pfull[2] = {nullptr, nullptr};
  int32_t* infos = nullptr;    // [nt] 1-based failing column in tile k or kNoError
  double* cur_piece = nullptr;  // piece / gathered / pfull of the current step
  double* cur_gath = nullptr;
  double* cur_full = nullptr;
  std::vector<void*> owned;
};

struct Geo {
  int m, nt, Pr, Pc;
  int first(int k, int pr) const { return k + 1 + (((pr - (k + 1)) % Pr) + Pr) % Pr; }
  int count(int k, int pr) const {
    const int f = first(k, pr);
    return f < nt ? (nt - f + Pr - 1) / Pr : 0;
  }
  int gmax(int k) const {
    int g = 0;
    for (int pr = 0; pr < Pr; ++pr) g = std::max(g, count(k, pr));
    return g;
  }
  int64_t lrow(int I) const { return (int64_t)(I / Pr) * NB; }
  int64_t lcol(int J) const { return (int64_t)(J / Pc) * NB; }
};

enum class Mode { kNccl, kVirtual };

static cudaError_t alloc_rank(DRank& R, const Geo& g) {
  auto al = [&](void** p, size_t bytes) {
    cudaError_t e = cudaMalloc(p, std::max<size_t>(bytes, 16));
    if (e == cudaSuccess) R.owned.push_back(*p);
    return e;
  };
  const size_t pc = (size_t)NB * std::max(1, (g.nt + g.Pr - 1) / g.Pr) * NB;
  cudaError_t e = al((void**)&R.diag, sizeof(double) * (NB * NB + kInv));
  for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
    e = al((void**)&R.piece[b], sizeof(double) * pc);
    if (e == cudaSuccess && g.Pr > 1) e = al((void**)&R.gathered[b], sizeof(double) * pc * g.Pr);
    if (e == cudaSuccess && g.Pr > 1) e = al((void**)&R.pfull[b], sizeof(double) * (size_t)NB * g.nt * NB);
  }
  if (e == cudaSuccess) e = al((void**)&R.infos, sizeof(int32_t) * std::max(1, g.nt));
  if (e == cudaSuccess) e = cudaMemsetAsync(R.infos, 0x7f, sizeof(int32_t) * std::max(1, g.nt), R.main);
  return e;
}

static void free_rank(DRank& R) {
  for (void* p : R.owned) cudaFree(p);
  R.owned.clear();
}

// collectives: NCCL on the handle's communicators (one local rank), or device copies between the
// virtual ranks of one process (all ranks listed in R, one stream)
struct Coll {
  Mode mode;
  std::vector<DRank>* R;
  const Geo* g;
  std::string err;
  bool fail = false;
  void check(ncclResult_t r) {
    if (r != ncclSuccess && !fail) {
      fail = true;
      err = nccl().errorString(r);
    }
  }
  DRank& at(int pr, int pc) { return (*R)[pr * g->Pc + pc]; }
  // double* DRank::*buf, count doubles, root = process row src_row, in process column col
  void bcast_col(double* DRank::*buf, size_t count, int src_row, int col) {
    if (mode == Mode::kNccl) {
      DRank& r = (*R)[0];
      if (r.h->grid.pc != col) return;
      check(nccl().broadcast(r.*buf, r.*buf, count, ncclDouble, src_row, (ncclComm_t)r.h->nccl_col, r.main));
      return;
    }
    DRank& s = at(src_row, col);
    for (int pr = 0; pr < g->Pr; ++pr)
      if (pr != src_row) cudaMemcpyAsync(at(pr, col).*buf, s.*buf, count * sizeof(double), cudaMemcpyDeviceToDevice, s.main);
  }
  void bcast_row(double* DRank::*buf, size_t count, int src_col) {
    if (mode == Mode::kNccl) {
      DRank& r = (*R)[0];
      check(nccl().broadcast(r.*buf, r.*buf, count, ncclDouble, src_col, (ncclComm_t)r.h->nccl_row, r.main));
      return;
    }
    for (int pr = 0; pr < g->Pr; ++pr) {
      DRank& s = at(pr, src_col);
      for (int pc = 0; pc < g->Pc; ++pc)
        if (pc != src_col) cudaMemcpyAsync(at(pr, pc).*buf, s.*buf, count * sizeof(double), cudaMemcpyDeviceToDevice, s.main);
    }
  }
  void allgather_col(double* DRank::*send, double* DRank::*recv, size_t count) {
    if (mode == Mode::kNccl) {
      DRank& r = (*R)[0];
      check(nccl().allGather(r.*send, r.*recv, count, ncclDouble, (ncclComm_t)r.h->nccl_col, r.main));
      return;
    }
    for (int pc = 0; pc < g->Pc; ++pc)
      for (int pr = 0; pr < g->Pr; ++pr)
        for (int q = 0; q < g->Pr; ++q)
          cudaMemcpyAsync(at(pr, pc).*recv + (size_t)q * count, at(q, pc).*send, count * sizeof(double),
                          cudaMemcpyDeviceToDevice, at(pr, pc).main);
  }
};

// Factor the distributed B (every rank of `R` local to this process).  Returns 0 and *info on success
// (info identical on every rank), -1 on a CUDA / NCCL error (message in *why).
int dist_cholesky(std::vector<DRank>& R, Mode mode, int m, int64_t* info, std::string* why) {
  sdpc_ctx* h0 = R[0].h;
  Geo g{m, (m + NB - 1) / NB, h0->grid.Pr, h0->grid.Pc};
  Coll coll{mode, &R, &g};
  for (DRank& r : R)
    if (alloc_rank(r, g) != cudaSuccess) {
      *why = "allocation of the distributed Cholesky buffers failed";
      for (DRank& q : R) free_rank(q);
      return -1;
    }
  struct Panel {
    bool some = false;
    double* DRank::*buf = nullptr;
    int64_t ldp = 0, k1 = 0;
    int kb = 0;
  };
  auto panel = [&](int k) -> Panel {
    Panel out;
    const int buf = k & 1;
    const int64_t k0 = (int64_t)k * NB;
    const int kb = (int)std::min<int64_t>(NB, m - k0);
    const int prk = k % g.Pr, pck = k % g.Pc;
    const int64_t k1 = k0 + kb;
    for (DRank& r : R) {  // 1. tile potrf on the owner of (k, k)
      if (r.h->grid.pc != pck || r.h->grid.pr != prk) continue;
      double* A = r.B + g.lrow(k) + g.lcol(k) * r.ld;
      cudaMemsetAsync(r.h->d_err, 0x7f, sizeof(int32_t), r.main);
      r.h->launches += potrf_lower(r.h, A, kb, r.ld, r.h->d_err, r.main, nullptr, nullptr, r.diag + NB * NB);
      cudaMemcpyAsync(r.infos + k, r.h->d_err, sizeof(int32_t), cudaMemcpyDeviceToDevice, r.main);
      cudaMemcpy2DAsync(r.diag, NB * sizeof(double), A, r.ld * sizeof(double), kb * sizeof(double), kb,
                        cudaMemcpyDeviceToDevice, r.main);
    }
    coll.bcast_col(&DRank::diag, (size_t)NB * NB + kInv, prk, pck);  // 2.
    for (DRank& r : R) {                                                // 3. panel solve
      if (r.h->grid.pc != pck) continue;
      const int cnt = g.count(k, r.h->grid.pr);
      const int64_t r0 = cnt ? g.lrow(g.first(k, r.h->grid.pr)) : r.h->mloc;
      const int64_t rows = r.h->mloc - r0;
      if (rows > 0)
        r.h->launches += trsm_panel(r.B + r0 + g.lcol(k) * r.ld, rows, r.ld, r.diag, NB, r.diag + NB * NB, kb,
                                    r.h->d_ok, r.main);
    }
    if (k1 >= m) return out;
    // 4. panel slice (kb columns, ld = gmax tiles) from process column pck to every rank
    const int gm = std::max(1, g.gmax(k));
    const int64_t ldg = (int64_t)gm * NB;
    for (DRank& r : R) {
      if (r.h->grid.pc != pck) continue;
      const int cnt = g.count(k, r.h->grid.pr);
      if (!cnt) continue;
      const int64_t r0 = g.lrow(g.first(k, r.h->grid.pr));
      cudaMemcpy2DAsync(r.piece[buf], ldg * sizeof(double), r.B + r0 + g.lcol(k) * r.ld, r.ld * sizeof(double),
                        (r.h->mloc - r0) * sizeof(double), kb, cudaMemcpyDeviceToDevice, r.main);
    }
    out.some = true;
    out.kb = kb;
    out.k1 = k1;
    // the collectives address the current (double-buffered) arrays through these members
    for (DRank& r : R) {
      r.cur_piece = r.piece[buf];
      r.cur_gath = r.gathered[buf];
      r.cur_full = r.pfull[buf];
    }
    coll.bcast_row(&DRank::cur_piece, (size_t)kb * ldg, pck);
    if (g.Pr == 1) {
      out.buf = &DRank::cur_piece;
      out.ldp = ldg;
      return out;
    }
    coll.allgather_col(&DRank::cur_piece, &DRank::cur_gath, (size_t)kb * ldg);
    const int ntr = g.nt - (k + 1);
    for (DRank& r : R) {
      const dim3 gr(std::max(1, std::min(1024, (int)((int64_t)kb * gm * NB / 256 + 1))), g.Pr);
      assemble_panel_kernel<<<gr, 256, 0, r.main>>>(r.cur_full, (int64_t)ntr * NB, r.cur_gath, ldg,
                                                     (int64_t)kb * ldg, kb, g.Pr, k, g.nt);
      ++r.h->launches;
    }
    out.buf = &DRank::cur_full;
    out.ldp = (int64_t)ntr * NB;
    return out;
  };
  auto update = [&](const Panel& p, int64_t jlo, int64_t jhi, bool side) {
    for (DRank& r : R) {
      cudaStream_t s = side ? r.side : r.main;
      if (side) {
        cudaEventRecord(r.ev, r.main);
        cudaStreamWaitEvent(r.side, r.ev, 0);
      }
      r.h->launches += update_tiles(r.B, r.ld, r.*(p.buf), p.ldp, p.k1, p.kb, r.h->grid, m, r.h->mloc, r.h->nloc,
                                    r.h->d_ok, s, jlo, jhi);
    }
  };
  Panel cur = panel(0);
  for (int k = 0; k < g.nt && cur.some; ++k) {
    // 5a. tile column k+1 first (it holds panel k+1), after the previous step's bulk update
    for (DRank& r : R) {
      cudaEventRecord(r.ev, r.side);
      cudaStreamWaitEvent(r.main, r.ev, 0);
    }
    update(cur, k + 1, k + 2, false);
    // 5b. the rest on the side stream, overlapping panel k + 1 (the buffers of panel k are not
    // overwritten before step k + 2, and step k + 2's panel waits for this update through 5a)
    update(cur, k + 2, 0, true);
    cur = panel(k + 1);
  }
  for (DRank& r : R) {
    cudaEventRecord(r.ev, r.side);
    cudaStreamWaitEvent(r.main, r.ev, 0);
  }
  // info: smallest failing global column over all ranks
  int64_t best = INT64_MAX;
  std::vector<int32_t> hinf(g.nt);
  for (DRank& r : R) {
    cudaMemcpyAsync(hinf.data(), r.infos, sizeof(int32_t) * g.nt, cudaMemcpyDeviceToHost, r.main);
    if (cudaStreamSynchronize(r.main) != cudaSuccess) {
      *why = cudaGetErrorString(cudaGetLastError());
      for (DRank& q : R) free_rank(q);
      return -1;
    }
    for (int k = 0; k < g.nt; ++k)
      if (hinf[k] != kNoError) {
        best = std::min<int64_t>(best, (int64_t)k * NB + hinf[k]);
        break;
      }
  }
  if (mode == Mode::kNccl && !coll.fail) {
    DRank& r = R[0];
    int64_t* d = reinterpret_cast<int64_t*>(r.diag);
    cudaMemcpyAsync(d, &best, sizeof(int64_t), cudaMemcpyHostToDevice, r.main);
    coll.check(nccl().allReduce(d, d, 1, ncclInt64, ncclMin, (ncclComm_t)r.h->nccl_world, r.main));
    cudaMemcpyAsync(&best, d, sizeof(int64_t), cudaMemcpyDeviceToHost, r.main);
    cudaStreamSynchronize(r.main);
  }
  for (DRank& q : R) free_rank(q);
  if (coll.fail) {
    *why = coll.err;
    return -1;
  }
  *info = best == INT64_MAX ? 0 : best;
  return 0;
}

// Entry for sdpc_scm_cholesky (NCCL: the handle's own rank) and sdpc_scm_cholesky_virtual (every rank of
// the grid as a handle in this process, one device, one stream).
int dist_cholesky_handles(sdpc_ctx* const* hs, double* const* B, int64_t ld, int nloc_ranks, bool virt,
                          cudaStream_t st, int64_t* info, std::string* why) {
  std::vector<DRank> R(nloc_ranks);
  for (int i = 0; i < nloc_ranks; ++i) {
    R[i].h = hs[i];
    R[i].B = B[i];
    R[i].ld = ld;
    R[i].main = st;
    if (virt) {
      R[i].side = st;
    } else {
      if (!hs[i]->dist_side) cudaStreamCreateWithFlags(&hs[i]->dist_side, cudaStreamNonBlocking);
      R[i].side = hs[i]->dist_side;
    }
    cudaEventCreateWithFlags(&R[i].ev, cudaEventDisableTiming);
  }
  const int rc = dist_cholesky(R, virt ? Mode::kVirtual : Mode::kNccl, hs[0]->S.m, info, why);
  for (DRank& r : R) cudaEventDestroy(r.ev);
  return rc;
}

}  // namespace sdpc
