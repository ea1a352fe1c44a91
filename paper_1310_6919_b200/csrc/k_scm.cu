// (c) SCM accumulation: B_kl = sum_{(p,q) in A_l} [A_l]_pq x_p^T A_k y_q for k >= l
// (PAPER.md P:380 Eq. SCM, P:686-688 Eq. newSCM2, Alg. 2 Step 3-3, lower triangle only
// P:918-919), reading the materialised columns of X-hat and Y^{-1} (panel-major RHS slots,
// elimination order).
//
// Written out per entry pair: B_kl = sum_{(i,j,v) in A_k} sum_{(p,q,w) in A_l} v w X-hat_{jp} Y^{-1}_{iq}.
// Only columns p, q of A_l are read (X-hat e_p, Y^{-1} e_q: the paper's x_p and v = Y^{-1}[A_l]_{*p}),
// so a rank that holds the columns l of B it builds needs only those RHS.
//  * max-cut (every A_k = a_k e_{v_k} e_{v_k}^T, distinct v_k): B_kl = a_k a_l X-hat_{v_k v_l} Y^{-1}_{v_k v_l},
//    i.e. B = X-hat o Y^{-1} (SURVEY §8(c) pins).  Full solves (multi-rank): one thread per
//    row k reads whole 256-byte panel rows of both inverses and writes 32 columns of B; truncated
//    solves (one rank): one warp per 32 rows x one panel, coalesced row reads, transposed through
//    shared memory (scm_maxcut_trunc_kernel).
//  * general: one thread per (k, l); A_l's entries staged in shared memory.
//  * "large" constraints (many entries, e.g. A_1 = I of the theta SDP): one CTA per (K, l) pair
//    with a block reduction over the entry-pair product (SURVEY: warp-shuffle reductions).
// Entries are written only where this rank holds B's tile (Grid::own_row / own_col), at the local
// 2D block-cyclic address (Pr = Pc = 1: the plain column-major B).
#include <cuda_runtime.h>

#include "common.cuh"
#include "ctx.hpp"

namespace sdpc {

// column c of a panel-major dense matrix, through its RHS slot
__device__ __forceinline__ double pm(const double* __restrict__ M, const int32_t* __restrict__ slot_of, int n,
                                     int row, int col) {
  const int s = slot_of[col];
  return M[((size_t)(s >> 5) * n + row) * kPanelW + (s & 31)];
}

__global__ void __launch_bounds__(256) scm_maxcut_kernel(int n, int m, const double* __restrict__ Xh,
                                                         const double* __restrict__ Yh,
                                                         const int32_t* __restrict__ rhs,
                                                         const int32_t* __restrict__ vrow,
                                                         const double* __restrict__ aval,
                                                         const int32_t* __restrict__ col_cons, double* B,
                                                         int64_t ldb, Grid g) {
  __shared__ int32_t lcol[kPanelW];
  __shared__ double lval[kPanelW];
  const int P = blockIdx.y;
  if (threadIdx.x < kPanelW) {
    const int v = rhs[P * kPanelW + threadIdx.x];
    const int l = v >= 0 ? col_cons[v] : -1;
    lcol[threadIdx.x] = l;
    lval[threadIdx.x] = l >= 0 ? aval[l] : 0.0;
  }
  __syncthreads();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m || !g.own_row(k)) return;
  const int i = vrow[k];
  const double ak = aval[k];
  double* Bk = B + g.lrow(k);
  const double2* xr = reinterpret_cast<const double2*>(Xh + ((size_t)P * n + i) * kPanelW);
  const double2* yr = reinterpret_cast<const double2*>(Yh + ((size_t)P * n + i) * kPanelW);
#pragma unroll 4
  for (int h = 0; h < kPanelW / 2; ++h) {
    const double2 x = xr[h], y = yr[h];
    const int l0 = lcol[2 * h], l1 = lcol[2 * h + 1];
    if (l0 >= 0 && k >= l0) Bk[g.lcol(l0) * ldb] = ak * lval[2 * h] * x.x * y.x;
    if (l1 >= 0 && k >= l1) Bk[g.lcol(l1) * ldb] = ak * lval[2 * h + 1] * x.y * y.y;
  }
}

// Max-cut with truncated solves (one rank): column v of the panel is valid at rows i >= v only; the pair
// {k, l} is taken from the panel of the smaller elimination index and written to the lower triangle of B.
// One warp per 32 consecutive constraints k and one panel: the 32 panel rows vrow[k] of X-hat and Y^{-1}
// are read as whole 256-byte rows (lane = panel column, two L1 wavefronts per load instead of the 32 of a
// thread-per-row double2 walk), the products go through a padded per-warp shared square and are written
// with lane = k, so the k >= l stores are 256-byte runs of a column of B.
constexpr int kTruncWarps = 4;
__global__ void __launch_bounds__(kTruncWarps * 32) scm_maxcut_trunc_kernel(
    int n, int m, const double* __restrict__ Xh, const double* __restrict__ Yh, const int32_t* __restrict__ rhs,
    const int32_t* __restrict__ vrow, const double* __restrict__ aval, const int32_t* __restrict__ col_cons,
    double* B, int64_t ldb) {
  __shared__ int32_t lcol[kPanelW], lvtx[kPanelW];
  __shared__ double lval[kPanelW];
  __shared__ double tile[kTruncWarps][kPanelW][kPanelW + 1];
  const int P = blockIdx.y;
  if (threadIdx.x < kPanelW) {
    const int v = rhs[P * kPanelW + threadIdx.x];
    const int l = v >= 0 ? col_cons[v] : -1;
    lcol[threadIdx.x] = l;
    lvtx[threadIdx.x] = v;
    lval[threadIdx.x] = l >= 0 ? aval[l] : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int k = (blockIdx.x * kTruncWarps + wid) * 32 + lane;
  const int v0 = lvtx[0];
  if (v0 < 0) return;
  const int i = k < m ? vrow[k] : -1;
  const double ak = k < m ? aval[k] : 0.0;
  if (!__any_sync(0xffffffffu, i >= v0)) return;
  const double lv = lval[lane];
  const double* xp = Xh + (size_t)P * n * kPanelW + lane;
  const double* yp = Yh + (size_t)P * n * kPanelW + lane;
  double(*T)[kPanelW + 1] = tile[wid];
#pragma unroll 8
  for (int r = 0; r < 32; ++r) {
    const int ir = __shfl_sync(0xffffffffu, i, r);
    const double ar = __shfl_sync(0xffffffffu, ak, r);
    if (ir >= v0) T[r][lane] = ar * lv * __ldg(xp + (size_t)ir * kPanelW) * __ldg(yp + (size_t)ir * kPanelW);
  }
  __syncwarp();
  if (i < v0) return;
#pragma unroll 4
  for (int c = 0; c < kPanelW; ++c) {
    const int l = lcol[c];
    if (l >= 0 && i >= lvtx[c]) {
      const double v = T[lane][c];
      if (k >= l) B[k + (size_t)l * ldb] = v;
      else B[l + (size_t)k * ldb] = v;
    }
  }
}

constexpr int kMaxSmall = 64;  // entries of a "small" constraint held in shared memory

__global__ void __launch_bounds__(256) scm_general_kernel(int n, int m, const double* __restrict__ Xh,
                                                          const double* __restrict__ Yh,
                                                          const int32_t* __restrict__ slot_of,
                                                          const int64_t* __restrict__ ptr,
                                                          const int32_t* __restrict__ ei,
                                                          const int32_t* __restrict__ ej,
                                                          const double* __restrict__ ev,
                                                          const uint8_t* __restrict__ is_large, double* B,
                                                          int64_t ldb, Grid g) {
  __shared__ int32_t sp[kMaxSmall], sq[kMaxSmall];
  __shared__ double sw[kMaxSmall];
  const int l = blockIdx.x;
  if (is_large[l] || !g.own_col(l)) return;
  const int64_t lb = ptr[l];
  const int nl = (int)(ptr[l + 1] - lb);
  // the RHS slots of A_l's columns are looked up once per CTA (sp / sq hold the element offset of the
  // slot's panel column, so a gather is one dependent load, not two)
  for (int t = threadIdx.x; t < nl; t += blockDim.x) {
    const int s0 = slot_of[ei[lb + t]], s1 = slot_of[ej[lb + t]];
    sp[t] = s0;
    sq[t] = s1;
    sw[t] = ev[lb + t];
  }
  __syncthreads();
  double* Bl = B + g.lcol(l) * ldb;
  for (int k = l + threadIdx.x; k < m; k += blockDim.x) {
    if (is_large[k] || !g.own_row(k)) continue;
    double sum = 0.0;
    for (int64_t e = ptr[k]; e < ptr[k + 1]; ++e) {
      const int i = ei[e], j = ej[e];
      const double v = ev[e];
      for (int t = 0; t < nl; ++t) {
        const int s0 = sp[t], s1 = sq[t];
        sum += v * sw[t] * Xh[((size_t)(s0 >> 5) * n + j) * kPanelW + (s0 & 31)] *
               Yh[((size_t)(s1 >> 5) * n + i) * kPanelW + (s1 & 31)];
      }
    }
    Bl[g.lrow(k)] = sum;
  }
}

// Staged-rows accumulation (one rank, RHS slot = vertex): by symmetry X-hat_{jp} = row p of X-hat at
// column j, and row p of the panel-major array is npanels contiguous 256-byte pieces.  The CTA of
// column l stages the rows of X-hat and Y^{-1} of the distinct vertices V_l of A_l in shared memory
// (coalesced), then every B_kl, k >= l, is sum_e v_e sum_f w_f Xr[p_f][j_e] Yr[q_f][i_e] with
// shared-memory reads only; the entries (K, l) with K a diagonal-only large constraint (A_1 = I of
// the theta SDP) are the block reductions sum_f w_f sum_t wK[t] Xr[p_f][t] Yr[q_f][t].
__global__ void __launch_bounds__(1024) scm_rows_kernel(int n, int m, const double* __restrict__ Xh,
                                                       const double* __restrict__ Yh,
                                                       const int64_t* __restrict__ ptr,
                                                       const int32_t* __restrict__ ei,
                                                       const int32_t* __restrict__ ej,
                                                       const double* __restrict__ ev,
                                                       const uint8_t* __restrict__ is_large,
                                                       const int32_t* __restrict__ vptr,
                                                       const int32_t* __restrict__ vlist,
                                                       const int32_t* __restrict__ eloc,
                                                       const double* __restrict__ wdiag,
                                                       const int32_t* __restrict__ dlist, int ndiag, double* B,
                                                       int64_t ldb) {
  extern __shared__ double rows_sm[];
  __shared__ int32_t sp[kMaxSmall], sq[kMaxSmall];
  __shared__ double sw[kMaxSmall];
  __shared__ double red[32];
  const int l = blockIdx.x;
  if (is_large[l]) return;
  const int nv = vptr[l + 1] - vptr[l];
  double* Xr = rows_sm;             // [nv][n]
  double* Yr = rows_sm + (size_t)nv * n;
  const int tid = threadIdx.x;
  // rows are staged by cp.async (no register round trip: every thread has all its copies in flight);
  // 16-byte copies when n is even (row starts in shared memory stay 16-byte aligned)
  for (int a = 0; a < nv; ++a) {
    const int v = vlist[vptr[l] + a];
    if ((n & 1) == 0) {
      for (int t = 2 * tid; t < n; t += 2 * blockDim.x) {
        const size_t o = ((size_t)(t >> 5) * n + v) * kPanelW + (t & 31);
        cp_async16(Xr + (size_t)a * n + t, Xh + o, true);
        cp_async16(Yr + (size_t)a * n + t, Yh + o, true);
      }
    } else {
      for (int t = tid; t < n; t += blockDim.x) {
        const size_t o = ((size_t)(t >> 5) * n + v) * kPanelW + (t & 31);
        cp_async8(Xr + (size_t)a * n + t, Xh + o, true);
        cp_async8(Yr + (size_t)a * n + t, Yh + o, true);
      }
    }
  }
  cp_async_commit();
  const int64_t lb = ptr[l];
  const int nl = (int)(ptr[l + 1] - lb);
  for (int t = tid; t < nl; t += blockDim.x) {
    sp[t] = eloc[2 * (lb + t)];
    sq[t] = eloc[2 * (lb + t) + 1];
    sw[t] = ev[lb + t];
  }
  cp_async_wait<0>();
  __syncthreads();
  for (int k = l + tid; k < m; k += blockDim.x) {
    if (is_large[k]) continue;
    double sum = 0.0;
    for (int64_t e = ptr[k]; e < ptr[k + 1]; ++e) {
      const int i = ei[e], j = ej[e];
      const double v = ev[e];
      double inner = 0.0;
      for (int t = 0; t < nl; ++t) inner += sw[t] * Xr[(size_t)sp[t] * n + j] * Yr[(size_t)sq[t] * n + i];
      sum += v * inner;
    }
    B[k + (size_t)l * ldb] = sum;
  }
  // pairs with the diagonal-only large constraints
  for (int dq = 0; dq < ndiag; ++dq) {
    const int K = dlist[dq];
    const double* wk = wdiag + (size_t)dq * n;
    double acc = 0.0;
    for (int t = tid; t < n; t += blockDim.x) {
      double inner = 0.0;
      for (int f = 0; f < nl; ++f) inner += sw[f] * Xr[(size_t)sp[f] * n + t] * Yr[(size_t)sq[f] * n + t];
      acc += wk[t] * inner;
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((tid & 31) == 0) red[tid >> 5] = acc;
    __syncthreads();
    if (tid == 0) {
      double sacc = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) sacc += red[w];
      const int hi = K > l ? K : l, lo = K > l ? l : K;
      B[hi + (size_t)lo * ldb] = sacc;
    }
    __syncthreads();
  }
}

// Pairs (K large, l any): the entry lands in column c = min(K, l), row r = max(K, l); the sum runs
// over A_r's entries (k role) and A_c's entries (l role), reading only the RHS of column c.
__global__ void __launch_bounds__(512) scm_large_kernel(int n, int m, const double* __restrict__ Xh,
                                                        const double* __restrict__ Yh,
                                                        const int32_t* __restrict__ slot_of,
                                                        const int64_t* __restrict__ ptr,
                                                        const int32_t* __restrict__ ei,
                                                        const int32_t* __restrict__ ej,
                                                        const double* __restrict__ ev,
                                                        const int32_t* __restrict__ large,
                                                        const uint8_t* __restrict__ is_large,
                                                        const uint8_t* __restrict__ diag_large, bool rows_mode,
                                                        double* B, int64_t ldb, Grid g) {
  __shared__ double red[32];
  const int l = blockIdx.x;
  const int K = large[blockIdx.y];
  if (is_large[l] && l > K) return;  // large x large pairs computed once (l <= K)
  if (rows_mode && diag_large[K] && (!is_large[l] || diag_large[l])) return;  // rows / pair kernels
  const int r = K > l ? K : l, c = K > l ? l : K;
  if (!g.own_row(r) || !g.own_col(c)) return;
  const int64_t rb = ptr[r], nr = ptr[r + 1] - rb;
  const int64_t cb = ptr[c], nc = ptr[c + 1] - cb;
  double sum = 0.0;
  for (int64_t idx = threadIdx.x; idx < nr * nc; idx += blockDim.x) {
    const int64_t a = idx / nc, b = idx % nc;
    const int i = ei[rb + a], j = ej[rb + a];
    const int p = ei[cb + b], q = ej[cb + b];
    sum += ev[rb + a] * ev[cb + b] * pm(Xh, slot_of, n, j, p) * pm(Yh, slot_of, n, i, q);
  }
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) red[wid] = sum;
  __syncthreads();
  if (wid == 0) {
    sum = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) B[g.lrow(r) + g.lcol(c) * ldb] = sum;
  }
}

// Pairs of diagonal-only large constraints (K, K'): B = sum_{t,s} wK[t] wK'[s] X-hat_ts Y^{-1}_ts, a
// reduction over all n^2 entries of X-hat o Y^{-1} (e.g. B_11 = trace(X-hat Y^{-1}) for A_1 = I).
// Grid (panels, row chunks), one partial sum per block, summed in a fixed order by the second kernel.
constexpr int kPairRows = 1024;
__global__ void __launch_bounds__(256) scm_diag_pair_partial(int n, const double* __restrict__ Xh,
                                                             const double* __restrict__ Yh,
                                                             const int32_t* __restrict__ rhs,
                                                             const double* __restrict__ wa,
                                                             const double* __restrict__ wb, double* partial) {
  __shared__ double red[8];
  const int P = blockIdx.x, r0 = blockIdx.y * kPairRows;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int v = rhs[P * kPanelW + lane];
  const double wv = v >= 0 ? wb[v] : 0.0;
  double acc = 0.0;
  for (int i = r0 + wid; i < min(n, r0 + kPairRows); i += 8) {
    const size_t o = ((size_t)P * n + i) * kPanelW + lane;
    acc += wa[i] * Xh[o] * Yh[o];
  }
  acc *= wv;
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) red[wid] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += red[w];
    partial[blockIdx.y * gridDim.x + blockIdx.x] = s;
  }
}

__global__ void scm_diag_pair_finish(const double* __restrict__ partial, int np, double* dst) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) acc += partial[i];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    *dst = s;
  }
}

int launch_scm(sdpc_ctx* h, double* B, int64_t ldb, cudaStream_t st) {
  const int n = h->S.n, m = h->S.m;
  const DevCons& c = h->cons;
  const Grid g = h->grid;
  if (c.maxcut) {
    if (h->d.npanels == 0) return 0;
    dim3 grid((m + 255) / 256, h->d.npanels);
    if (h->trunc_active)
      scm_maxcut_trunc_kernel<<<dim3((m + kTruncWarps * 32 - 1) / (kTruncWarps * 32), h->d.npanels),
                                kTruncWarps * 32, 0, st>>>(n, m, h->Xh, h->Yh, h->d.rhs, c.vrow, c.aval, c.col_cons, B,
                                                           ldb);
    else
      scm_maxcut_kernel<<<grid, 256, 0, st>>>(n, m, h->Xh, h->Yh, h->d.rhs, c.vrow, c.aval, c.col_cons, B,
                                                      ldb, g);
    return 1;
  }
  int nl = 0;
  if (c.rows_mode) {
    const size_t smem = (size_t)2 * c.nvmax * n * sizeof(double);
    static std::atomic<uint64_t> attr{0};
    if (once_per_device(attr))
      cudaFuncSetAttribute(scm_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRowsSmemCap);
    // one or two CTAs fit an SM when the staged rows are big: more warps per CTA hide the gather latency
    scm_rows_kernel<<<m, smem > 48 * 1024 ? 1024 : 256, smem, st>>>(n, m, h->Xh, h->Yh, c.ptr, c.ei, c.ej, c.ev, c.is_large, c.vptr, c.vlist,
                                          c.eloc, c.wdiag, c.dlist, c.ndiag, B, ldb);
  } else {
    scm_general_kernel<<<m, 256, 0, st>>>(n, m, h->Xh, h->Yh, h->d.slot_of, c.ptr, c.ei, c.ej, c.ev, c.is_large, B,
                                          ldb, g);
  }
  ++nl;
  if (c.nlarge > 0) {
    dim3 grid(m, c.nlarge);
    scm_large_kernel<<<grid, 512, 0, st>>>(n, m, h->Xh, h->Yh, h->d.slot_of, c.ptr, c.ei, c.ej, c.ev, c.large,
                                           c.is_large, c.diag_large, c.rows_mode, B, ldb, g);
    ++nl;
  }
  if (c.rows_mode && c.ndiag > 0) {
    const int np = h->d.npanels, nchunk = (n + kPairRows - 1) / kPairRows;
    for (int a = 0; a < c.ndiag; ++a)
      for (int b = a; b < c.ndiag; ++b) {
        const int K = h->diag_ids[a], K2 = h->diag_ids[b];
        const int hi = K > K2 ? K : K2, lo = K > K2 ? K2 : K;
        scm_diag_pair_partial<<<dim3(np, nchunk), 256, 0, st>>>(n, h->Xh, h->Yh, h->d.rhs, c.wdiag + (size_t)a * n,
                                                                 c.wdiag + (size_t)b * n, h->pair_ws);
        scm_diag_pair_finish<<<1, 256, 0, st>>>(h->pair_ws, np * nchunk, B + hi + (size_t)lo * ldb);
        nl += 2;
      }
  }
  return nl;
}

}  // namespace sdpc
