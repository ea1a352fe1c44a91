// libsdpc C ABI (include/sdpc.h): handle lifetime, host preprocessing, phase drivers.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "common.cuh"
#include "ctx.hpp"
#include "sdpc.h"

using namespace sdpc;

namespace {

template <class T>
cudaError_t upload(T** dst, const std::vector<T>& v) {
  *dst = nullptr;
  size_t bytes = std::max<size_t>(1, v.size()) * sizeof(T);
  cudaError_t e = cudaMalloc(dst, bytes);
  if (e != cudaSuccess) return e;
  if (!v.empty()) e = cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
  return e;
}

template <class T>
cudaError_t dalloc(T** dst, size_t count) {
  *dst = nullptr;
  return cudaMalloc(dst, std::max<size_t>(1, count) * sizeof(T));
}

sdpc_status map_cuda(sdpc_ctx* h, cudaError_t e) {
  if (e == cudaSuccess) return SDPC_OK;
  if (h) h->err = cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? SDPC_ERR_OOM : SDPC_ERR_CUDA;
}

#define CK(expr)                                  \
  do {                                            \
    cudaError_t _e = (expr);                      \
    if (_e != cudaSuccess) return map_cuda(h, _e); \
  } while (0)

constexpr size_t kSmemCap = 200 * 1024;   // dynamic smem per clique CTA (static ~8.5 KB on top)
constexpr int kSolveCtasDuringA2 = 192;   // ~96 of 148 SMs at 2 solve CTAs per SM
constexpr size_t kPanelCap = 200 * 1024;  // shared-memory panel of a global-workspace clique

// size classes for the per-clique kernels
int class_of(size_t bytes) {
  if (bytes <= 12 * 1024) return 0;
  if (bytes <= 48 * 1024) return 1;
  if (bytes <= kSmemCap) return 2;
  return 3;
}
const int kClassThreads[4] = {64, 128, 256, 256};

cudaError_t build_classes(std::vector<CliqueClass>& cls, const std::vector<int32_t>& members,
                          const std::vector<size_t>& bytes, const std::vector<int64_t>& ws_off,
                          const std::vector<size_t>& panel_bytes) {
  cls.assign(4, CliqueClass{});
  for (int q = 0; q < 4; ++q) cls[q].threads = kClassThreads[q];
  for (int32_t r : members) {
    int q = ws_off[r] >= 0 ? 3 : class_of(bytes[r]);
    cls[q].sn.push_back(r);
    if (q < 3) cls[q].smem = std::max(cls[q].smem, bytes[r]);
    else cls[q].smem = std::max(cls[q].smem, std::min(kPanelCap, panel_bytes[r]));
  }
  // biggest cliques first so the long CTAs start early
  for (auto& k : cls) {
    if (k.sn.empty()) continue;
    cudaError_t e = upload(&k.d_sn, k.sn);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

void free_classes(std::vector<CliqueClass>& cls) {
  for (auto& k : cls)
    if (k.d_sn) cudaFree(k.d_sn);
  cls.clear();
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float t = 0;
  if (cudaEventElapsedTime(&t, a, b) != cudaSuccess) return 0;
  return t;
}

sdpc_status check_err(sdpc_ctx* h, cudaStream_t st, int32_t* out) {
  int32_t v = kNoError;
  CK(cudaMemcpyAsync(&v, h->d_err, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  CK(cudaGetLastError());
  *out = v;
  return SDPC_OK;
}

}  // namespace

extern "C" {

const char* sdpc_status_string(sdpc_status s) {
  switch (s) {
    case SDPC_OK: return "ok";
    case SDPC_ERR_INVALID_ARG: return "invalid argument";
    case SDPC_ERR_NOT_PD: return "not positive definite";
    case SDPC_ERR_OOM: return "out of memory";
    case SDPC_ERR_CUDA: return "CUDA error";
    case SDPC_ERR_NCCL: return "NCCL error";
    case SDPC_ERR_STATE: return "invalid call order";
  }
  return "unknown status";
}

int64_t sdpc_last_info(sdpc_handle h) { return h ? h->last_info : 0; }
int64_t sdpc_launch_count(sdpc_handle h) { return h ? h->launches : 0; }

const char* sdpc_last_error_message(sdpc_handle h) { return h ? h->err.c_str() : ""; }

sdpc_status sdpc_create(sdpc_handle* out, int32_t n, int32_t m, const int64_t* a_ptr, const int32_t* a_row,
                        const int32_t* a_col, const double* a_val, const double* b, const int32_t* perm,
                        int32_t device, int32_t nranks, int32_t rank, const void* nccl_id) {
  if (!out) return SDPC_ERR_INVALID_ARG;
  *out = nullptr;
  if (n < 1 || m < 1 || !a_ptr || !a_val || !b) return SDPC_ERR_INVALID_ARG;
  if (a_ptr[0] != 0) return SDPC_ERR_INVALID_ARG;
  for (int32_t k = 0; k <= m; ++k)
    if (a_ptr[k + 1] < a_ptr[k]) return SDPC_ERR_INVALID_ARG;
  if (a_ptr[m + 1] > 0 && (!a_row || !a_col)) return SDPC_ERR_INVALID_ARG;
  for (int32_t k = 0; k < m; ++k)
    if (!std::isfinite(b[k])) return SDPC_ERR_INVALID_ARG;
  for (int64_t e = 0; e < a_ptr[m + 1]; ++e)
    if (!std::isfinite(a_val[e])) return SDPC_ERR_INVALID_ARG;
  if (nranks < 1 || rank < 0 || rank >= nranks) return SDPC_ERR_INVALID_ARG;

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) return SDPC_ERR_CUDA;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major != 10) return SDPC_ERR_CUDA;
  if (cudaSetDevice(device) != cudaSuccess) return SDPC_ERR_CUDA;

  sdpc_ctx* h = new (std::nothrow) sdpc_ctx();
  if (!h) return SDPC_ERR_OOM;
  h->device = device;
  h->nranks = nranks;
  h->rank = rank;
  // process grid Pr x Pc = nranks with Pr the largest divisor <= sqrt(nranks) (1x2, 2x2, 2x4, ...)
  int Pr = 1;
  for (int d0 = 1; (int64_t)d0 * d0 <= nranks; ++d0)
    if (nranks % d0 == 0) Pr = d0;
  h->grid.Pr = Pr;
  h->grid.Pc = nranks / Pr;
  h->grid.pr = rank / h->grid.Pc;
  h->grid.pc = rank % h->grid.Pc;
  auto numroc = [](int64_t m0, int64_t p, int64_t P) {  // ScaLAPACK numroc with tile kScmNB
    const int64_t nt = (m0 + kScmNB - 1) / kScmNB;
    int64_t cnt = 0;
    for (int64_t t = p; t < nt; t += P) cnt += std::min<int64_t>(kScmNB, m0 - t * kScmNB);
    return cnt;
  };
  h->mloc = numroc(m, h->grid.pr, h->grid.Pr);
  h->nloc = numroc(m, h->grid.pc, h->grid.Pc);
  Symbolic& S = h->S;
  std::string msg = analyse(S, n, m, a_ptr, a_row, a_col, perm);
  if (!msg.empty()) {
    delete h;
    return SDPC_ERR_INVALID_ARG;
  }
  const int32_t ns = S.nsuper;
  auto fail = [&](sdpc_status s) {
    sdpc_destroy(h);
    return s;
  };

  // ---- per-clique size classes and global workspace
  std::vector<size_t> b1(ns), b2(ns), pb(ns);
  std::vector<int64_t> ws_off(ns, -1);
  int64_t ws_total = 0;
  for (int32_t r = 0; r < ns; ++r) {
    const size_t c = S.snc[r], s = S.sns[r];
    b1[r] = (c * c + c * s) * sizeof(double);
    b2[r] = c * c * sizeof(double);
    pb[r] = c * 32 * sizeof(double);
    if (b1[r] > kSmemCap) {
      ws_off[r] = ws_total;
      ws_total += (int64_t)(c * c + c * s + c * 32);  // A, W, and a panel fallback if c*32 > kPanelCap
    }
  }
  std::vector<int32_t> all(ns);
  for (int32_t r = 0; r < ns; ++r) all[r] = r;
  std::stable_sort(all.begin(), all.end(), [&](int32_t x, int32_t y) { return S.snc[x] > S.snc[y]; });
  if (build_classes(h->a1cls, all, b1, ws_off, pb) != cudaSuccess) return fail(SDPC_ERR_OOM);
  const int nh = (int)S.hlev_ptr.size() - 1;
  h->a2lev.resize(nh);
  // (a2) fronts in the global workspace with many children: their extend-add runs beforehand as a
  // grid-wide kernel (CTAs own column ranges of the front, children added in a fixed order: no atomics)
  // instead of inside the front's own CTA
  std::vector<uint8_t> pre(ns, 0);
  std::vector<int32_t> pre_ptr(nh + 1, 0), pre_child, pre_parent, zero_ptr(nh + 1, 0), zero_list;
  for (int lv = 0; lv < nh; ++lv) {
    for (int32_t q = S.hlev_ptr[lv]; q < S.hlev_ptr[lv + 1]; ++q) {
      const int32_t r = S.hlev_sn[q];
      const int32_t nch = S.child_ptr[r + 1] - S.child_ptr[r];
      if (ws_off[r] >= 0) {  // every global front: the pre-pass assembles it (big-front path)
        pre[r] = 1;
        zero_list.push_back(r);
        for (int32_t cq = S.child_ptr[r]; cq < S.child_ptr[r + 1]; ++cq) {
          pre_child.push_back(S.child_list[cq]);
          pre_parent.push_back(r);
        }
      }
    }
    pre_ptr[lv + 1] = (int32_t)pre_child.size();
    zero_ptr[lv + 1] = (int32_t)zero_list.size();
  }
  h->pre_ptr = pre_ptr;
  h->zero_ptr = zero_ptr;
  // global-workspace fronts take the big-front path (front_panel_kernel + front_schur_kernel), the rest
  // the per-front class kernels
  std::vector<int32_t> big_list;
  h->big_ptr.assign(nh + 1, 0);
  h->big_tiles.assign(nh, 0);
  h->big_thin.assign(nh, 0);
  h->big_wide.assign(nh, 0);
  for (int lv = 0; lv < nh; ++lv) {
    std::vector<int32_t> mem;
    for (int32_t q = S.hlev_ptr[lv]; q < S.hlev_ptr[lv + 1]; ++q) {
      const int32_t r = S.hlev_sn[q];
      if (ws_off[r] >= 0) {
        big_list.push_back(r);
        const int64_t u = S.snc[r] - S.sns[r], t64 = (u + 63) / 64;
        h->big_tiles[lv] = std::max<int32_t>(h->big_tiles[lv], (int32_t)(t64 * (t64 + 1) / 2));
        (S.sns[r] <= 32 ? h->big_thin : h->big_wide)[lv] = 1;  // (kThinS in k_clique.cu)
        h->big_smem = std::max(h->big_smem, std::min(kPanelCap, pb[r]));
      } else {
        mem.push_back(r);
      }
    }
    h->big_ptr[lv + 1] = (int32_t)big_list.size();
    std::stable_sort(mem.begin(), mem.end(), [&](int32_t x, int32_t y) { return S.snc[x] > S.snc[y]; });
    if (build_classes(h->a2lev[lv], mem, b2, ws_off, pb) != cudaSuccess) return fail(SDPC_ERR_OOM);
  }

  // ---- constraints in elimination ids, symmetric expansion, duplicates summed
  std::vector<int64_t> cptr(m + 1, 0);
  std::vector<int32_t> ci, cj;
  std::vector<double> cv;
  std::vector<uint8_t> cmirror;  // 1 for the mirrored copy of an off-diagonal entry
  bool maxcut = true;
  std::vector<int32_t> vrow(m), col_cons(n, -1);
  std::vector<double> aval(m);
  std::vector<uint8_t> is_large(m, 0);
  std::vector<int32_t> large;
  for (int32_t k = 0; k < m; ++k) {
    const int64_t lo = a_ptr[k + 1], hi = a_ptr[k + 2];
    std::vector<std::pair<std::pair<int32_t, int32_t>, double>> ent;
    for (int64_t e = lo; e < hi; ++e) ent.push_back({{a_row[e], a_col[e]}, a_val[e]});
    std::sort(ent.begin(), ent.end(), [](auto& x, auto& y) { return x.first < y.first; });
    std::vector<std::pair<std::pair<int32_t, int32_t>, double>> merged;
    for (auto& x : ent) {
      if (!merged.empty() && merged.back().first == x.first) merged.back().second += x.second;
      else merged.push_back(x);
    }
    for (auto& x : merged) {
      const int32_t r = S.iperm[x.first.first], c = S.iperm[x.first.second];
      ci.push_back(r);
      cj.push_back(c);
      cv.push_back(x.second);
      cmirror.push_back(0);
      if (r != c) {
        ci.push_back(c);
        cj.push_back(r);
        cv.push_back(x.second);
        cmirror.push_back(1);
      }
    }
    cptr[k + 1] = (int64_t)ci.size();
    const int64_t cnt = cptr[k + 1] - cptr[k];
    if (cnt > 64) {
      is_large[k] = 1;
      large.push_back(k);
    }
    if (merged.size() != 1 || merged[0].first.first != merged[0].first.second) {
      maxcut = false;
    } else {
      const int32_t v = S.iperm[merged[0].first.first];
      if (col_cons[v] >= 0) maxcut = false;
      else {
        col_cons[v] = k;
        vrow[k] = v;
        aval[k] = merged[0].second;
      }
    }
  }

  // ---- RHS slots: every vertex p that is a column of some A_l with l a column of B on this rank
  // (Eq. newSCM2 needs x_p, v_p only for the nonzero columns p of A_l), ascending
  // elimination ids so that a 32-slot panel shares most of its etree paths
  std::vector<int32_t> rhs, slot_of(n, -1);
  {
    std::vector<uint8_t> need(n, 0);
    for (int32_t l = 0; l < m; ++l) {
      if (!h->grid.own_col(l)) continue;
      for (int64_t e = cptr[l]; e < cptr[l + 1]; ++e) need[ci[e]] = 1;
    }
    for (int32_t v = 0; v < n; ++v)
      if (need[v]) {
        slot_of[v] = (int32_t)rhs.size();
        rhs.push_back(v);
      }
  }
  const int32_t nrhs = (int32_t)rhs.size();
  const int32_t npanels = (nrhs + kPanelW - 1) / kPanelW;
  rhs.resize((size_t)npanels * kPanelW, -1);
  // per RHS panel: union of the etree paths of its vertices (supernode granularity)
  std::vector<int32_t> reach_ptr(npanels + 1, 0), reach_sn, stamp(ns, -1), tmp;
  for (int32_t P = 0; P < npanels; ++P) {
    tmp.clear();
    for (int32_t t = 0; t < kPanelW; ++t) {
      const int32_t p = rhs[(size_t)P * kPanelW + t];
      if (p < 0) continue;
      for (int32_t r = S.sn_of_col[p]; r >= 0 && stamp[r] != P; r = S.sparent[r]) {
        stamp[r] = P;
        tmp.push_back(r);
      }
    }
    std::sort(tmp.begin(), tmp.end());
    reach_sn.insert(reach_sn.end(), tmp.begin(), tmp.end());
    reach_ptr[P + 1] = (int32_t)reach_sn.size();
  }

  // ---- search direction tables (k_direction.cu): all supernodes; symmetric CSR of E with the E offset
  // of each entry; per E entry the constraint entries on it (dY = G - sum_k A_k dz_k); per
  // expanded constraint entry its E offset (X-bar values in g_k)
  auto epos = [&](int32_t a, int32_t b) -> int32_t {  // offset of (max, min) in E's CSC, -1 if absent
    const int32_t hi = std::max(a, b), lo = std::min(a, b);
    const int32_t* beg = S.rowind.data() + S.colptr[lo];
    const int32_t* end = S.rowind.data() + S.colptr[lo + 1];
    const int32_t* it = std::lower_bound(beg, end, hi);
    return (it != end && *it == hi) ? (int32_t)(it - S.rowind.data()) : -1;
  };
  std::vector<int32_t> all_sn(ns);
  for (int32_t r = 0; r < ns; ++r) all_sn[r] = r;
  std::vector<int32_t> sym_ptr(n + 1, 0), sym_col, sym_pos;
  {
    const int64_t nnzE = S.nnzE();
    for (int32_t j = 0; j < n; ++j)
      for (int64_t q = S.colptr[j]; q < S.colptr[j + 1]; ++q) {
        ++sym_ptr[S.rowind[q] + 1];
        if (S.rowind[q] != j) ++sym_ptr[j + 1];
      }
    for (int32_t i = 0; i < n; ++i) sym_ptr[i + 1] += sym_ptr[i];
    sym_col.resize(sym_ptr[n]);
    sym_pos.resize(sym_ptr[n]);
    std::vector<int32_t> fill(sym_ptr.begin(), sym_ptr.end() - 1);
    for (int32_t j = 0; j < n; ++j)
      for (int64_t q = S.colptr[j]; q < S.colptr[j + 1]; ++q) {
        const int32_t i = S.rowind[q];
        sym_col[fill[i]] = j;
        sym_pos[fill[i]++] = (int32_t)q;
        if (i != j) {
          sym_col[fill[j]] = i;
          sym_pos[fill[j]++] = (int32_t)q;
        }
      }
    (void)nnzE;
  }
  std::vector<int32_t> ecs_ptr(S.nnzE() + 1, 0), ecs_k, cons_epos(ci.size(), -1);
  std::vector<double> ecs_val;
  {
    std::vector<std::pair<int32_t, std::pair<int32_t, double>>> lst;  // (E offset, (k, value))
    for (int32_t k = 0; k < m; ++k)
      for (int64_t e2 = cptr[k]; e2 < cptr[k + 1]; ++e2) {
        const int32_t q = epos(ci[e2], cj[e2]);
        cons_epos[e2] = q;
        if (q >= 0 && !cmirror[e2]) lst.push_back({q, {k, cv[e2]}});
      }
    std::stable_sort(lst.begin(), lst.end(), [](auto& x, auto& y) { return x.first < y.first; });
    for (auto& x : lst) {
      ++ecs_ptr[x.first + 1];
      ecs_k.push_back(x.second.first);
      ecs_val.push_back(x.second.second);
    }
    for (int64_t q = 0; q < S.nnzE(); ++q) ecs_ptr[q + 1] += ecs_ptr[q];
  }

  // ---- staged-rows accumulation (one rank, every vertex a RHS slot in order): per small constraint
  // the distinct vertices V_l of its entries and, per entry, the positions of p and q in V_l;
  // large constraints whose entries are all diagonal ("diag-large", e.g. A_1 = I) as dense weights
  std::vector<int32_t> vptr(m + 1, 0), vlist, eloc(ci.size() * 2, 0);
  std::vector<uint8_t> diag_large(m, 0);
  std::vector<double> wdiag;
  std::vector<int32_t> dlist;
  int nvmax = 0;
  for (int32_t l = 0; l < m; ++l) {
    if (is_large[l]) {
      bool diag = true;
      for (int64_t e2 = cptr[l]; e2 < cptr[l + 1]; ++e2) diag = diag && ci[e2] == cj[e2];
      if (diag) {
        diag_large[l] = 1;
        dlist.push_back(l);
        const size_t o = wdiag.size();
        wdiag.resize(o + n, 0.0);
        for (int64_t e2 = cptr[l]; e2 < cptr[l + 1]; ++e2) wdiag[o + ci[e2]] += cv[e2];
      }
      vptr[l + 1] = (int32_t)vlist.size();
      continue;
    }
    std::vector<int32_t> vs;
    for (int64_t e2 = cptr[l]; e2 < cptr[l + 1]; ++e2) vs.push_back(ci[e2]);
    std::sort(vs.begin(), vs.end());
    vs.erase(std::unique(vs.begin(), vs.end()), vs.end());
    for (int64_t e2 = cptr[l]; e2 < cptr[l + 1]; ++e2) {
      eloc[2 * e2] = (int32_t)(std::lower_bound(vs.begin(), vs.end(), cj[e2]) - vs.begin());      // p = ej
      eloc[2 * e2 + 1] = (int32_t)(std::lower_bound(vs.begin(), vs.end(), ci[e2]) - vs.begin());  // q = ei
    }
    nvmax = std::max<int>(nvmax, (int)vs.size());
    vlist.insert(vlist.end(), vs.begin(), vs.end());
    vptr[l + 1] = (int32_t)vlist.size();
  }
  const size_t rows_smem = (size_t)2 * nvmax * n * sizeof(double);
  h->cons.rows_mode = !maxcut && nranks == 1 && nrhs == n && nvmax > 0 && rows_smem <= kRowsSmemCap;
  h->cons.nvmax = nvmax;
  h->cons.ndiag = (int32_t)dlist.size();

  if (!solve_smem_fits(ns)) {
    // the solve kernel keeps a reach bitmap of the supernodes in shared memory (see k_solve.cu)
    h->err = "too many supernodes for the solve kernel's shared-memory reach bitmap";
    return fail(SDPC_ERR_INVALID_ARG);
  }
  // ---- upload
  DevSym& d = h->d;
  d.n = n;
  d.m = m;
  d.nsuper = ns;
  d.nnzE = S.nnzE();
  d.npanels = npanels;
  d.nrhs = nrhs;
  cudaError_t e = cudaSuccess;
#define UP(dst, v)                                    \
  if ((e = upload(&(dst), (v))) != cudaSuccess) { \
    h->err = cudaGetErrorString(e);                 \
    return fail(SDPC_ERR_OOM);                      \
  }
  UP(d.colptr, S.colptr);
  UP(d.rowind, S.rowind);
  UP(d.super_ptr, S.super_ptr);
  UP(d.snc, S.snc);
  UP(d.sns, S.sns);
  UP(d.sparent, S.sparent);
  UP(d.panel_off, S.panel_off);
  UP(d.e2p, S.e2p);
  UP(d.umap_off, S.umap_off);
  UP(d.umap, S.umap);
  UP(d.relind_off, S.relind_off);
  UP(d.relind, S.relind);
  UP(d.upd_off, S.upd_off);
  UP(d.child_ptr, S.child_ptr);
  UP(d.child_list, S.child_list);
  UP(d.hlev_sn, S.hlev_sn);
  UP(d.dlev_ptr, S.dlev_ptr);
  UP(d.dlev_sn, S.dlev_sn);
  UP(d.preorder, S.preorder);
  UP(d.border, S.border);
  UP(d.sub_ptr, S.sub_ptr);
  UP(d.perm, S.perm);
  UP(d.iperm, S.iperm);
  UP(d.reach_ptr, reach_ptr);
  UP(d.reach_sn, reach_sn);
  UP(d.rhs, rhs);
  UP(d.slot_of, slot_of);
  UP(d.all_sn, all_sn);
  UP(d.sym_ptr, sym_ptr);
  UP(d.sym_col, sym_col);
  UP(d.sym_pos, sym_pos);
  UP(d.ecs_ptr, ecs_ptr);
  UP(d.ecs_k, ecs_k);
  UP(d.ecs_val, ecs_val);
  UP(d.cons_epos, cons_epos);
  h->slot_of_host = slot_of;
  UP(h->d_ws_off, ws_off);
  UP(h->d_pre, pre);
  UP(h->d_pre_child, pre_child);
  UP(h->d_pre_parent, pre_parent);
  UP(h->d_zero_list, zero_list);
  UP(h->d_big_list, big_list);
  DevCons& cs = h->cons;
  cs.maxcut = maxcut;
  cs.m = m;
  UP(cs.ptr, cptr);
  UP(cs.ei, ci);
  UP(cs.ej, cj);
  UP(cs.ev, cv);
  UP(cs.is_large, is_large);
  UP(cs.large, large);
  cs.nlarge = (int32_t)large.size();
  UP(cs.vrow, vrow);
  UP(cs.aval, aval);
  UP(cs.col_cons, col_cons);
  UP(cs.vptr, vptr);
  UP(cs.vlist, vlist);
  UP(cs.eloc, eloc);
  UP(cs.diag_large, diag_large);
  UP(cs.wdiag, wdiag);
  UP(cs.dlist, dlist);
  h->diag_ids = dlist;
#undef UP
#define AL(dst, cnt)                                    \
  if ((e = dalloc(&(dst), (cnt))) != cudaSuccess) { \
    h->err = cudaGetErrorString(e);                   \
    return fail(SDPC_ERR_OOM);                        \
  }
  // (a1): the global-workspace cliques (a1cls[3]) take the big-clique pipeline with its own workspace
  // (A with an even leading dimension for the task kernels' 16-byte staging, then W); h->ws is unused
  {
    const auto& big = h->a1cls[3].sn;
    h->nbig1 = (int32_t)big.size();
    std::vector<int64_t> boff(big.size());
    std::vector<int32_t> bdim(big.size());
    int64_t tot = 0;
    h->big1_c.resize(big.size());
    for (size_t b = 0; b < big.size(); ++b) {
      const int64_t c = S.snc[big[b]], sc = S.sns[big[b]];
      boff[b] = tot;
      bdim[b] = (int32_t)c;
      h->big1_c[b] = (int32_t)c;
      tot += c * (c + (c & 1)) + c * sc;
      tot += tot & 1;
    }
    if (!big.empty()) {
      if ((e = upload(&h->big1_off, boff)) != cudaSuccess || (e = upload(&h->big1_dim, bdim)) != cudaSuccess) {
        h->err = cudaGetErrorString(e);
        return fail(SDPC_ERR_OOM);
      }
      AL(h->big1_ws, (size_t)tot);
      AL(h->big1_linv, big.size() * 128 * 128);
      AL(h->big1_err, big.size());
    }
  }
  AL(h->ws, 1);
  AL(h->ws2, (size_t)ws_total);
  AL(h->Lx, (size_t)S.panel_total);
  AL(h->Ly, (size_t)S.panel_total);
  AL(h->Dx, (size_t)n);
  AL(h->Dy, (size_t)n);
  AL(h->upd, (size_t)S.upd_total);
  AL(h->d_err, 4);  // [0] default / (a1), [1] (a2), [2] (d) in sdpc_iteration
  AL(h->d_ok, 1);
  AL(h->pair_ws, (size_t)std::max(1, npanels) * ((n + 1023) / 1024));
  AL(h->potrf_ws, 2 * 128 * 128);
#undef AL
  for (auto& ev : h->ev) cudaEventCreate(&ev);
  // error flags start at "no error" (kNoError = bytes 0x7f); d_ok never changes: the distributed
  // tile kernels run unconditionally (a failed tile factorisation is reported through info)
  if (cudaMemset(h->d_err, 0x7f, sizeof(int32_t)) != cudaSuccess ||
      cudaMemset(h->d_ok, 0x7f, sizeof(int32_t)) != cudaSuccess)
    return fail(SDPC_ERR_CUDA);
  if (cudaGetLastError() != cudaSuccess) return fail(SDPC_ERR_CUDA);
  if (nccl_id) {
    // NCCL world + process-row / process-column communicators (collective over the nranks callers)
    std::string why;
    if (nccl_init(h, nccl_id, &why) != 0) {
      h->err = why;
      return fail(SDPC_ERR_NCCL);
    }
  }
  *out = h;
  return SDPC_OK;
}

sdpc_status sdpc_get_unique_id(void* id_out) {
  if (!id_out) return SDPC_ERR_INVALID_ARG;
  std::string why;
  return nccl_unique_id(id_out, &why) == 0 ? SDPC_OK : SDPC_ERR_NCCL;
}

sdpc_status sdpc_destroy(sdpc_handle h) {
  if (!h) return SDPC_OK;
  cudaSetDevice(h->device);
  nccl_destroy(h);
  if (h->dist_side) cudaStreamDestroy(h->dist_side);
  DevSym& d = h->d;
  void* ptrs[] = {d.colptr, d.rowind, d.super_ptr, d.snc, d.sns, d.sparent, d.panel_off, d.e2p, d.umap_off,
                  d.umap, d.relind_off, d.relind, d.upd_off, d.child_ptr, d.child_list, d.hlev_sn,
                  d.dlev_ptr, d.dlev_sn, d.preorder, d.border, d.sub_ptr, d.perm, d.iperm, d.reach_ptr, d.reach_sn, d.rhs, d.slot_of, d.all_sn, d.sym_ptr, d.sym_col, d.sym_pos, d.ecs_ptr, d.ecs_k,
                  d.ecs_val, d.cons_epos, h->Uh, h->dir_ws, h->d_step_off, h->step_ws, h->d_amin, h->ytmp, h->d_ws_off, h->d_pre, h->d_pre_child,
                  h->d_pre_parent, h->d_zero_list, h->d_big_list,
                  h->cons.ptr, h->cons.ei, h->cons.ej, h->cons.ev, h->cons.is_large, h->cons.large,
                  h->cons.vrow, h->cons.aval, h->cons.col_cons, h->cons.vptr, h->cons.vlist, h->cons.eloc,
                  h->cons.diag_large, h->cons.wdiag, h->cons.dlist, h->ws, h->ws2, h->Lx, h->Ly, h->Dx, h->Dy, h->upd,
                  h->d_err, h->d_ok, h->pair_ws, h->sce_ws, h->sce_linv, h->potrf_ws, h->Xh, h->Yh, h->Bown, h->xin, h->yin,
                  h->dag_ws, h->dag_linv, h->dag_koff, h->dag_trace, h->big1_off, h->big1_dim, h->big1_err,
                  h->big1_ws, h->big1_linv};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (h->pinned_in) cudaFreeHost(h->pinned_in);
  if (h->pinned_out) cudaFreeHost(h->pinned_out);
  free_classes(h->a1cls);
  for (auto& lv : h->a2lev) free_classes(lv);
  for (auto& ev : h->ev)
    if (ev) cudaEventDestroy(ev);
  for (auto& ev : h->upd_ev) cudaEventDestroy(ev);
  if (h->evA) cudaEventDestroy(h->evA);
  if (h->evB) cudaEventDestroy(h->evB);
  if (h->st2) cudaStreamDestroy(h->st2);
  for (int q = 0; q < 2; ++q)
    for (int i = 0; i < 4; ++i) {
      if (h->sides[q][i]) cudaStreamDestroy(h->sides[q][i]);
      if (h->sides_ev[q][i]) cudaEventDestroy(h->sides_ev[q][i]);
    }
  if (h->fork_ev) cudaEventDestroy(h->fork_ev);
  if (h->fork_ev2) cudaEventDestroy(h->fork_ev2);
  if (h->st3) cudaStreamDestroy(h->st3);
  if (h->it_fork) cudaEventDestroy(h->it_fork);
  if (h->it_join) cudaEventDestroy(h->it_join);
  delete h;
  return SDPC_OK;
}

sdpc_status sdpc_get_structure(sdpc_handle h, sdpc_structure* out) {
  if (!h || !out) return SDPC_ERR_INVALID_ARG;
  const Symbolic& S = h->S;
  out->n = S.n;
  out->m = S.m;
  out->nnzE = S.nnzE();
  out->perm = S.perm.data();
  out->parent = S.parent.data();
  out->colptr = S.colptr.data();
  out->rowind = S.rowind.data();
  out->nsuper = S.nsuper;
  out->super_ptr = S.super_ptr.data();
  return SDPC_OK;
}

sdpc_status sdpc_get_scm_layout(sdpc_handle h, sdpc_layout* out) {
  if (!h || !out) return SDPC_ERR_INVALID_ARG;
  out->nb = kScmNB;
  out->Pr = h->grid.Pr;
  out->Pc = h->grid.Pc;
  out->myrow = h->grid.pr;
  out->mycol = h->grid.pc;
  out->mloc = h->mloc;
  out->nloc = h->nloc;
  out->lld = std::max<int64_t>(1, h->mloc);
  return SDPC_OK;
}

sdpc_status sdpc_set_truncation(sdpc_handle h, int32_t on) {
  if (!h) return SDPC_ERR_INVALID_ARG;
  h->truncate = on != 0;
  return SDPC_OK;
}

sdpc_status sdpc_set_cholesky_schedule(sdpc_handle h, int32_t task_graph) {
  if (!h) return SDPC_ERR_INVALID_ARG;
  h->use_dag = task_graph != 0;
  return SDPC_OK;
}

sdpc_status sdpc_set_cholesky_trace(sdpc_handle h, int64_t cap) {
  if (!h || cap < 0) return SDPC_ERR_INVALID_ARG;
  CK(cudaSetDevice(h->device));
  if (h->dag_trace) cudaFree(h->dag_trace);
  h->dag_trace = nullptr;
  h->dag_trace_cap = 0;
  if (cap > 0) {
    CK(cudaMalloc(&h->dag_trace, sizeof(unsigned long long) * (4 * cap + 1)));
    h->dag_trace_cap = cap;
  }
  return SDPC_OK;
}

sdpc_status sdpc_get_cholesky_trace(sdpc_handle h, uint64_t* out, int64_t cap, int64_t* n) {
  if (!h || !out || !n || !h->dag_trace) return SDPC_ERR_INVALID_ARG;
  CK(cudaSetDevice(h->device));
  unsigned cnt = 0;
  CK(cudaMemcpy(&cnt, h->dag_trace + 4 * h->dag_trace_cap, sizeof(unsigned), cudaMemcpyDeviceToHost));
  const int64_t c = std::min<int64_t>(cap, h->dag_trace_cap);
  CK(cudaMemcpy(out, h->dag_trace, sizeof(uint64_t) * 4 * c, cudaMemcpyDeviceToHost));
  *n = std::min<int64_t>((int64_t)cnt, c);
  return SDPC_OK;
}

sdpc_status sdpc_set_timing(sdpc_handle h, int32_t on) {
  if (!h) return SDPC_ERR_INVALID_ARG;
  h->timing = on != 0;
  return SDPC_OK;
}

sdpc_status sdpc_get_phase_times(sdpc_handle h, double* t) {
  if (!h || !t) return SDPC_ERR_INVALID_ARG;
  for (int i = 0; i < 8; ++i) t[i] = h->times[i];
  return SDPC_OK;
}

sdpc_status sdpc_get_kernel_times(sdpc_handle h, double* t) {
  if (!h || !t) return SDPC_ERR_INVALID_ARG;
  for (int i = 0; i < 8; ++i) t[i] = h->ktimes[i];
  return SDPC_OK;
}

sdpc_status sdpc_factor_xinv(sdpc_handle h, const double* xbar_E, void* stream) {
  if (!h || !xbar_E) return SDPC_ERR_INVALID_ARG;
  CK(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  h->have_x = false;
  h->have_y = false;
  CK(cudaMemsetAsync(h->d_err, 0x7f, sizeof(int32_t), st));
  if (h->timing) CK(cudaEventRecord(h->ev[0], st));
  h->launches += launch_alg1(h, xbar_E, st);
  if (h->timing) CK(cudaEventRecord(h->ev[1], st));
  int32_t v;
  sdpc_status s = check_err(h, st, &v);
  if (s != SDPC_OK) return s;
  if (h->timing) h->times[0] = elapsed(h->ev[0], h->ev[1]);
  if (v != kNoError) {
    h->last_info = v;
    return SDPC_ERR_NOT_PD;
  }
  h->have_x = true;
  return SDPC_OK;
}

sdpc_status sdpc_get_xinv_factor(sdpc_handle h, double* L_E, double* D, void* stream) {
  if (!h || !L_E || !D) return SDPC_ERR_INVALID_ARG;
  if (!h->have_x) return SDPC_ERR_STATE;
  CK(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  h->launches += launch_panels_to_E(h, h->Lx, L_E, st);
  CK(cudaMemcpyAsync(D, h->Dx, sizeof(double) * h->S.n, cudaMemcpyDeviceToDevice, st));
  CK(cudaStreamSynchronize(st));
  CK(cudaGetLastError());
  return SDPC_OK;
}

sdpc_status sdpc_get_y_factor(sdpc_handle h, double* LY_E, double* DY, void* stream) {
  if (!h || !LY_E || !DY) return SDPC_ERR_INVALID_ARG;
  if (!h->have_y) return SDPC_ERR_STATE;
  CK(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  h->launches += launch_panels_to_E(h, h->Ly, LY_E, st);
  CK(cudaMemcpyAsync(DY, h->Dy, sizeof(double) * h->S.n, cudaMemcpyDeviceToDevice, st));
  CK(cudaStreamSynchronize(st));
  CK(cudaGetLastError());
  return SDPC_OK;
}

sdpc_status sdpc_scm_build(sdpc_handle h, const double* y_E, double* B, int64_t ldb, void* stream) {
  if (!h || !y_E || !B || ldb < std::max<int64_t>(1, h->mloc)) return SDPC_ERR_INVALID_ARG;
  if (!h->have_x) return SDPC_ERR_STATE;
  CK(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  h->have_y = false;
  const size_t dense = std::max<size_t>(1, (size_t)h->d.npanels * h->S.n * kPanelW);
  if (!h->Xh) {
    CK(dalloc(&h->Xh, dense));
    CK(dalloc(&h->Yh, dense));
  }
  CK(cudaMemsetAsync(h->d_err, 0x7f, sizeof(int32_t), st));
  if (h->timing) CK(cudaEventRecord(h->ev[2], st));
  h->launches += launch_ldl_y(h, y_E, st);
  if (h->timing) CK(cudaEventRecord(h->ev[3], st));
  int32_t v;
  sdpc_status s = check_err(h, st, &v);
  if (s != SDPC_OK) return s;
  if (v != kNoError) {
    h->last_info = v;
    return SDPC_ERR_NOT_PD;
  }
  h->have_y = true;
  // the truncated sweep needs every vertex as a RHS (single rank) and B = X-hat o Y^{-1} (max-cut)
  h->trunc_active = h->truncate && h->cons.maxcut && h->nranks == 1 && h->d.nrhs == h->S.n;
  h->launches += launch_inverse_panels(h, st);
  if (h->timing) CK(cudaEventRecord(h->ev[4], st));
  h->launches += launch_scm(h, B, ldb, st);
  if (h->timing) CK(cudaEventRecord(h->ev[5], st));
  CK(cudaStreamSynchronize(st));
  CK(cudaGetLastError());
  if (h->timing) {
    h->times[1] = elapsed(h->ev[2], h->ev[3]);
    h->times[2] = elapsed(h->ev[3], h->ev[4]);
    h->times[3] = elapsed(h->ev[4], h->ev[5]);
  }
  return SDPC_OK;
}

sdpc_status sdpc_get_inverse_columns(sdpc_handle h, const int32_t* cols, int32_t ncols, double* X_out, double* Y_out,
                                     void* stream) {
  if (!h || !cols || ncols < 1 || !X_out || !Y_out) return SDPC_ERR_INVALID_ARG;
  if (!h->have_y || !h->Xh || h->trunc_active) return SDPC_ERR_STATE;
  CK(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<int32_t> cn(ncols);
  for (int32_t c = 0; c < ncols; ++c) {
    if (cols[c] < 0 || cols[c] >= h->S.n) return SDPC_ERR_INVALID_ARG;
    cn[c] = h->S.iperm[cols[c]];
    if (h->slot_of_host[cn[c]] < 0) return SDPC_ERR_INVALID_ARG;  // column not computed on this rank
  }
  int32_t* dc = nullptr;
  CK(upload(&dc, cn));
  h->launches += launch_gather_columns(h, dc, ncols, X_out, Y_out, st);
  cudaError_t e = cudaStreamSynchronize(st);
  cudaFree(dc);
  CK(e);
  CK(cudaGetLastError());
  return SDPC_OK;
}

// (d) on one GPU: the persistent task-graph kernel when B allows 16-byte staging (the normal case),
// else round 1's multi-launch schedule.  With timing on, the update-kernel events bracket the whole
// persistent kernel (one launch, m^3/3 flops) or every trailing-update launch of the fallback.
static cudaError_t run_cholesky(sdpc_handle h, double* B, int64_t ldb, int32_t* d_err, cudaStream_t st, double* fl,
                                int* nu) {
  const int64_t m = h->S.m;
  if (h->use_dag && potrf_dag_usable(B, ldb)) {
    if (h->timing && h->upd_ev.size() < 2) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      h->upd_ev.push_back(e0);
      h->upd_ev.push_back(e1);
    }
    if (h->timing) cudaEventRecord(h->upd_ev[0], st);
    const int l = potrf_dag(h, B, m, ldb, d_err, st);
    if (l < 0) return cudaErrorMemoryAllocation;
    if (h->timing) cudaEventRecord(h->upd_ev[1], st);
    h->launches += l;
    *fl = (double)m * m * m / 3.0;
    *nu = 1;
  } else {
    h->launches += potrf_lower(h, B, m, ldb, d_err, st, fl, nu, h->potrf_ws);
  }
  return cudaGetLastError();
}

static sdpc_status dist_status(sdpc_handle h, int rc, int64_t v, const std::string& why, int32_t* info) {
  if (rc != 0) {
    h->err = why;
    return SDPC_ERR_NCCL;
  }
  *info = (int32_t)v;
  h->last_info = v;
  return v ? SDPC_ERR_NOT_PD : SDPC_OK;
}

sdpc_status sdpc_scm_cholesky(sdpc_handle h, double* B, int64_t ldb, int32_t* info, void* stream) {
  if (!h || !B || !info) return SDPC_ERR_INVALID_ARG;
  if (h->nccl_world) {
    // collective over the handle's NCCL communicator: B is this rank's local 2D block-cyclic array
    if (ldb < std::max<int64_t>(1, h->mloc)) return SDPC_ERR_INVALID_ARG;
    CK(cudaSetDevice(h->device));
    std::string why;
    int64_t v = 0;
    double* Bs[1] = {B};
    sdpc_ctx* hs[1] = {h};
    const int rc = dist_cholesky_handles(hs, Bs, ldb, 1, false, (cudaStream_t)stream, &v, &why);
    return dist_status(h, rc, v, why, info);
  }
  if (h->nranks != 1) return SDPC_ERR_STATE;  // distributed without a communicator: the tile entries
  if (ldb < h->S.m) return SDPC_ERR_INVALID_ARG;
  CK(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaMemsetAsync(h->d_err, 0x7f, sizeof(int32_t), st));
  if (h->timing) CK(cudaEventRecord(h->ev[6], st));
  double fl = 0;
  int nu = 0;
  CK(run_cholesky(h, B, ldb, h->d_err, st, &fl, &nu));
  if (h->timing) CK(cudaEventRecord(h->ev[7], st));
  int32_t v;
  sdpc_status s = check_err(h, st, &v);
  if (s != SDPC_OK) return s;
  if (h->timing) {
    h->times[4] = elapsed(h->ev[6], h->ev[7]);
    double tu = 0;
    for (int i = 0; i < nu; ++i) tu += elapsed(h->upd_ev[2 * i], h->upd_ev[2 * i + 1]);
    h->times[5] = tu;
    h->times[6] = nu;
    h->times[7] = fl;
  }
  if (v != kNoError) {
    *info = v;
    h->last_info = v;
    return SDPC_ERR_NOT_PD;
  }
  *info = 0;
  return SDPC_OK;
}

sdpc_status sdpc_scm_cholesky_virtual(const sdpc_handle* hs, int32_t nranks, double* const* B, int64_t ldb,
                                      int32_t* info, void* stream) {
  if (!hs || !B || !info || nranks < 1) return SDPC_ERR_INVALID_ARG;
  for (int32_t r = 0; r < nranks; ++r) {
    if (!hs[r] || !B[r] || hs[r]->nranks != nranks || hs[r]->rank != r || hs[r]->device != hs[0]->device ||
        hs[r]->S.m != hs[0]->S.m || ldb < std::max<int64_t>(1, hs[r]->mloc))
      return SDPC_ERR_INVALID_ARG;
  }
  sdpc_handle h = hs[0];
  CK(cudaSetDevice(h->device));
  std::string why;
  int64_t v = 0;
  std::vector<sdpc_ctx*> hv(hs, hs + nranks);
  const int rc = dist_cholesky_handles(hv.data(), B, ldb, nranks, true, (cudaStream_t)stream, &v, &why);
  sdpc_status s = SDPC_OK;
  for (int32_t r = 0; r < nranks; ++r) s = dist_status(hs[r], rc, v, why, info);
  return s;
}

sdpc_status sdpc_iteration(sdpc_handle h, const double* xbar_E, const double* y_E, double* B, int64_t ldb,
                           int32_t* info, void* stream) {
  if (!h || !xbar_E || !y_E || !B || !info || ldb < h->S.m) return SDPC_ERR_INVALID_ARG;
  if (h->nranks != 1) return SDPC_ERR_STATE;
  CK(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  const size_t dense = std::max<size_t>(1, (size_t)h->d.npanels * h->S.n * kPanelW);
  if (!h->Xh) {
    CK(dalloc(&h->Xh, dense));
    CK(dalloc(&h->Yh, dense));
  }
  if (!h->st3) {
    // (a2) is the critical path of the first half (a level-by-level tree walk): highest priority,
    // so its few CTAs are scheduled ahead of the X-hat solve CTAs that fill the rest of the GPU
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&h->st3, cudaStreamNonBlocking, hi));
    CK(cudaEventCreateWithFlags(&h->it_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&h->it_join, cudaEventDisableTiming));
  }
  h->have_x = h->have_y = false;
  CK(cudaMemsetAsync(h->d_err, 0x7f, 3 * sizeof(int32_t), st));
  if (h->timing) CK(cudaEventRecord(h->ev[0], st));
  // (a1) on st and (a2) on st3 concurrently: both are latency-bound walks over the cliques / the
  // elimination tree with few CTAs in flight, and they do not depend on each other
  // and each factor's multi-RHS solves start as soon as that factor is ready: the X-hat solves fill
  // the SMs the tree-level (a2) launches leave idle
  h->trunc_active = h->truncate && h->cons.maxcut && h->nranks == 1 && h->d.nrhs == h->S.n;
  CK(cudaEventRecord(h->it_fork, st));
  CK(cudaStreamWaitEvent(h->st3, h->it_fork, 0));
  h->launches += launch_alg1(h, xbar_E, st);
  if (h->timing) CK(cudaEventRecord(h->ev[1], st));
  // deep elimination trees (many (a2) levels, each a latency-bound launch): cap the X-hat solve grid
  // (each CTA walks several panels) so that about a third of the SMs stay free for the (a2) levels
  // on the high-priority stream; shallow trees (block-arrow: 2 levels) keep the whole GPU
  const bool deep = h->a2lev.size() >= 8;
  if (h->timing) CK(cudaEventRecord(h->ev[8], st));
  h->launches += launch_inverse_panels(h, st, 0, 1, deep ? kSolveCtasDuringA2 : 0);
  if (h->timing) CK(cudaEventRecord(h->ev[9], st));
  h->launches += launch_ldl_y(h, y_E, h->st3, h->d_err + 1, 1);
  if (h->timing) CK(cudaEventRecord(h->ev[2], h->st3));
  h->launches += launch_inverse_panels(h, h->st3, 1, 1);
  if (h->timing) CK(cudaEventRecord(h->ev[10], h->st3));
  CK(cudaEventRecord(h->it_join, h->st3));
  CK(cudaStreamWaitEvent(st, h->it_join, 0));
  if (h->timing) CK(cudaEventRecord(h->ev[4], st));
  h->launches += launch_scm(h, B, ldb, st);
  if (h->timing) CK(cudaEventRecord(h->ev[5], st));
  double fl = 0;
  int nu = 0;
  CK(run_cholesky(h, B, ldb, h->d_err + 2, st, &fl, &nu));
  if (h->timing) CK(cudaEventRecord(h->ev[7], st));
  int32_t fl3[3];
  CK(cudaMemcpyAsync(fl3, h->d_err, sizeof(fl3), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  CK(cudaGetLastError());
  if (h->timing) {
    // (a1), (a2) and the two solve launches overlap: t[0] = start -> (a1) done, t[1] = start ->
    // (a2) done, t[2] = start -> both solves done (all measured from the start of the iteration)
    h->times[0] = elapsed(h->ev[0], h->ev[1]);
    h->times[1] = elapsed(h->ev[0], h->ev[2]);
    h->times[2] = elapsed(h->ev[0], h->ev[4]);
    h->times[3] = elapsed(h->ev[4], h->ev[5]);
    h->times[4] = elapsed(h->ev[5], h->ev[7]);
    double tu = 0;
    for (int i = 0; i < nu; ++i) tu += elapsed(h->upd_ev[2 * i], h->upd_ev[2 * i + 1]);
    h->times[5] = tu;
    h->times[6] = nu;
    h->times[7] = fl;
    // kernel windows: X-hat solve launch(es), Y^{-1} solve launch(es), accumulate, Cholesky kernel
    h->ktimes[0] = elapsed(h->ev[8], h->ev[9]);
    h->ktimes[1] = elapsed(h->ev[2], h->ev[10]);
    h->ktimes[2] = h->times[3];
    h->ktimes[3] = tu;
    h->ktimes[4] = h->times[0];
    h->ktimes[5] = h->times[1];
  }
  *info = 0;
  if (fl3[0] != kNoError) {
    h->last_info = fl3[0];
    return SDPC_ERR_NOT_PD;
  }
  if (fl3[1] != kNoError) {
    h->last_info = fl3[1];
    return SDPC_ERR_NOT_PD;
  }
  h->have_x = h->have_y = true;
  if (fl3[2] != kNoError) {
    *info = fl3[2];
    h->last_info = fl3[2];
    return SDPC_ERR_NOT_PD;
  }
  return SDPC_OK;
}

sdpc_status sdpc_iteration_host(sdpc_handle h, const double* xbar_E, const double* y_E, double* rdiag,
                                int32_t* info, void* stream) {
  if (!h || !xbar_E || !y_E || !info) return SDPC_ERR_INVALID_ARG;
  if (h->nranks != 1) return SDPC_ERR_STATE;
  CK(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t nnz = h->S.nnzE(), m = h->S.m;
  const int64_t ldb = m + (m & 1);
  if (!h->Bown) {
    CK(dalloc(&h->Bown, (size_t)ldb * m));
    CK(dalloc(&h->xin, (size_t)std::max(nnz, m)));
    CK(dalloc(&h->yin, (size_t)nnz));
    CK(cudaMallocHost(&h->pinned_in, sizeof(double) * 2 * nnz));
    CK(cudaMallocHost(&h->pinned_out, sizeof(double) * m));
  }
  std::memcpy(h->pinned_in, xbar_E, sizeof(double) * nnz);
  std::memcpy(h->pinned_in + nnz, y_E, sizeof(double) * nnz);
  CK(cudaMemcpyAsync(h->xin, h->pinned_in, sizeof(double) * nnz, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(h->yin, h->pinned_in + nnz, sizeof(double) * nnz, cudaMemcpyHostToDevice, st));
  sdpc_status s = sdpc_iteration(h, h->xin, h->yin, h->Bown, ldb, info, stream);
  if (s != SDPC_OK && !(s == SDPC_ERR_NOT_PD && *info > 0)) return s;
  if (rdiag) {
    h->launches += launch_diag_copy(h->Bown, m, ldb, h->xin, st);
    CK(cudaMemcpyAsync(h->pinned_out, h->xin, sizeof(double) * m, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    std::memcpy(rdiag, h->pinned_out, sizeof(double) * m);
  }
  return s;
}

sdpc_status sdpc_potrf_tile(sdpc_handle h, double* A, int32_t n, int64_t lda, double* inv, int32_t* info_dev,
                            void* stream) {
  if (!h || !A || !inv || !info_dev || n < 1 || n > kScmNB || lda < n) return SDPC_ERR_INVALID_ARG;
  CK(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaMemsetAsync(h->d_err, 0x7f, sizeof(int32_t), st));
  const bool tim = h->timing;
  h->timing = false;
  h->launches += potrf_lower(h, A, n, lda, h->d_err, st, nullptr, nullptr, inv);
  h->timing = tim;
  CK(cudaMemcpyAsync(info_dev, h->d_err, sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  CK(cudaGetLastError());
  return SDPC_OK;
}

sdpc_status sdpc_trsm_panel(sdpc_handle h, double* A, int64_t rows, int64_t lda, const double* L, int64_t ldl,
                            const double* inv, int32_t kb, void* stream) {
  if (!h || rows < 0 || kb < 1 || kb > kScmNB || (rows > 0 && (!A || lda < rows)) || !L || ldl < kb || !inv)
    return SDPC_ERR_INVALID_ARG;
  CK(cudaSetDevice(h->device));
  h->launches += trsm_panel(A, rows, lda, L, ldl, inv, kb, h->d_ok, (cudaStream_t)stream);
  CK(cudaGetLastError());
  return SDPC_OK;
}

sdpc_status sdpc_update_tiles(sdpc_handle h, double* C, int64_t ldc, const double* P, int64_t ldp, int64_t k1,
                              int32_t K, int64_t jlo, int64_t jhi, void* stream) {
  if (!h || k1 < 0 || K < 1 || K > kScmNB || k1 % kScmNB != 0) return SDPC_ERR_INVALID_ARG;
  if (h->mloc > 0 && h->nloc > 0 && k1 < h->S.m && (!C || !P || ldc < h->mloc || ldp < h->S.m - k1))
    return SDPC_ERR_INVALID_ARG;
  CK(cudaSetDevice(h->device));
  h->launches += update_tiles(C, ldc, P, ldp, k1, K, h->grid, h->S.m, h->mloc, h->nloc, h->d_ok,
                              (cudaStream_t)stream, jlo, jhi);
  CK(cudaGetLastError());
  return SDPC_OK;
}

// The inverses of R's diagonal 128-tiles for the SCE sweeps (nullptr: unaligned R, the sweeps then solve the
// diagonal triangles serially).
static const double* sce_tile_inverses(sdpc_handle h, const double* R, int64_t ldr, cudaStream_t st) {
  const int64_t m = h->S.m, T = (m + 127) / 128;
  if (!potrf_dag_usable(R, ldr)) return nullptr;
  if (h->sce_linv_cap < T) {
    if (h->sce_linv) cudaFree(h->sce_linv);
    h->sce_linv = nullptr;
    h->sce_linv_cap = 0;
    if (cudaMalloc(&h->sce_linv, sizeof(double) * 128 * 128 * T) != cudaSuccess) return nullptr;
    h->sce_linv_cap = T;
  }
  const int l = tile_inverses(R, ldr, m, h->sce_linv, st);
  if (l < 0) return nullptr;
  h->launches += l;
  return h->sce_linv;
}

sdpc_status sdpc_scm_solve(sdpc_handle h, const double* R, int64_t ldr, double* G, int64_t ldg, int32_t nrhs,
                           void* stream) {
  if (!h || !R || !G || nrhs < 1 || ldr < h->S.m || ldg < h->S.m) return SDPC_ERR_INVALID_ARG;
  if (h->nranks != 1) return SDPC_ERR_STATE;
  CK(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  // scratch: nrhs x 128 doubles (serial-triangle sweeps) or 2 flags per 128-row block (flag sweeps)
  const int64_t sce_need = std::max<int64_t>((int64_t)nrhs * 128, (h->S.m + 127) / 128 + 8);
  if (h->sce_cap < sce_need) {
    if (h->sce_ws) cudaFree(h->sce_ws);
    h->sce_ws = nullptr;
    CK(dalloc(&h->sce_ws, (size_t)sce_need));
    h->sce_cap = sce_need;
  }
  const double* linv = sce_tile_inverses(h, R, ldr, st);
  const int ls = scm_solve(R, ldr, h->S.m, G, ldg, nrhs, h->sce_ws, st, linv);
  if (ls < 0) {
    h->err = "cooperative launch of the SCE solve failed";
    return SDPC_ERR_CUDA;
  }
  h->launches += ls;
  CK(cudaStreamSynchronize(st));
  CK(cudaGetLastError());
  return SDPC_OK;
}

sdpc_status sdpc_search_direction(sdpc_handle h, const double* xbar_E, const double* G_E, double beta_mu,
                                  const double* R, int64_t ldr, double* g, double* dz, double* dY_E, double* dX_E,
                                  void* stream) {
  if (!h || !xbar_E || !G_E || !R || !g || !dz || !dY_E || !dX_E || ldr < h->S.m) return SDPC_ERR_INVALID_ARG;
  if (h->nranks != 1) return SDPC_ERR_STATE;
  if (!h->have_x || !h->have_y || !h->Xh) return SDPC_ERR_STATE;
  if (h->d.nrhs != h->S.n) {
    h->err = "search direction needs every vertex as a solve RHS (some vertex is in no constraint)";
    return SDPC_ERR_STATE;
  }
  CK(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  if (h->timing) CK(cudaEventRecord(h->ev[12], st));
  int l = direction_g(h, xbar_E, G_E, beta_mu, g, st);
  if (l < 0) return SDPC_ERR_OOM;
  h->launches += l;
  const int m = h->S.m;
  const int64_t sce_need = std::max<int64_t>(128, (m + 127) / 128 + 8);
  if (h->sce_cap < sce_need) {
    if (h->sce_ws) cudaFree(h->sce_ws);
    h->sce_ws = nullptr;
    CK(dalloc(&h->sce_ws, (size_t)sce_need));
    h->sce_cap = sce_need;
  }
  CK(cudaMemcpyAsync(dz, g, sizeof(double) * m, cudaMemcpyDeviceToDevice, st));
  const double* linv = sce_tile_inverses(h, R, ldr, st);
  const int ls = scm_solve(R, ldr, m, dz, m, 1, h->sce_ws, st, linv);  // B dz = g (Eq. SCE)
  if (ls < 0) {
    h->err = "cooperative launch of the SCE solve failed";
    return SDPC_ERR_CUDA;
  }
  h->launches += ls;
  if (h->timing) CK(cudaEventRecord(h->ev[13], st));
  l = direction_dY_dX(h, xbar_E, G_E, beta_mu, dz, dY_E, dX_E, st);
  if (l < 0) return SDPC_ERR_OOM;
  h->launches += l;
  if (h->timing) CK(cudaEventRecord(h->ev[14], st));
  CK(cudaStreamSynchronize(st));
  CK(cudaGetLastError());
  if (h->timing) {
    h->ktimes[6] = elapsed(h->ev[12], h->ev[13]);  // g + SCE solve
    h->ktimes[7] = elapsed(h->ev[13], h->ev[14]);  // dY + P-MATRIX
  }
  return SDPC_OK;
}

sdpc_status sdpc_step_lengths(sdpc_handle h, const double* xbar_E, const double* dX_E, const double* y_E,
                              const double* dY_E, double* alpha_p, double* alpha_d, void* stream) {
  if (!h || !xbar_E || !dX_E || !y_E || !dY_E || !alpha_p || !alpha_d) return SDPC_ERR_INVALID_ARG;
  CK(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  int l = primal_step(h, xbar_E, dX_E, alpha_p, st);
  if (l < 0) return SDPC_ERR_CUDA;
  h->launches += l;
  l = dual_step(h, y_E, dY_E, alpha_d, 30, st);
  if (l < 0) return SDPC_ERR_CUDA;
  h->launches += l;
  CK(cudaGetLastError());
  return SDPC_OK;
}

sdpc_status sdpc_fp64_peak(int32_t device, double ms, double* dmma_tflops, double* dfma_tflops) {
  if (!dmma_tflops || !dfma_tflops) return SDPC_ERR_INVALID_ARG;
  cudaError_t e = fp64_peak(device, ms, dmma_tflops, dfma_tflops);
  return e == cudaSuccess ? SDPC_OK : SDPC_ERR_CUDA;
}

}  // extern "C"
