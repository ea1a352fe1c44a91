// (c) SCM accumulation: B_kl = sum_{(p,q) in A_l} [A_l]_pq x_p^T A_k y_q for k >= l
// (PAPER.md P:380 Eq. SCM, P:686-688 Eq. newSCM2, Alg. 2 Step 3-3, lower triangle only
// P:918-919), reading the materialised X-hat and Y^{-1} (panel-major, elimination order).
//
// Written out per entry pair: B_kl = sum_{(i,j,v) in A_k} sum_{(p,q,w) in A_l} v w X-hat_{jp} Y^{-1}_{qi}.
//  * max-cut (every A_k = a_k e_{v_k} e_{v_k}^T, distinct v_k): B_kl = a_k a_l X-hat_{v_k v_l} Y^{-1}_{v_k v_l},
//    i.e. B = X-hat o Y^{-1} (SURVEY §8(c) pins).  One thread per row k reads whole
//    256-byte panel rows of both inverses and writes 32 columns of B with coalesced stores.
//  * general: one thread per (k, l); A_l's entries staged in shared memory.
//  * "large" constraints (many entries, e.g. A_1 = I of the theta SDP): one CTA per (K, l) pair
//    with a block reduction over the entry-pair product (SURVEY: warp-shuffle reductions).
#include <cuda_runtime.h>

#include "common.cuh"
#include "ctx.hpp"

namespace sdpc {

__device__ __forceinline__ double pm(const double* __restrict__ M, int n, int row, int col) {
  // panel-major dense matrix: column col lives in panel col/32, lane col%32
  return M[((size_t)(col >> 5) * n + row) * kPanelW + (col & 31)];
}

__global__ void __launch_bounds__(256) scm_maxcut_kernel(int n, int m, const double* __restrict__ Xh,
                                                         const double* __restrict__ Yh,
                                                         const int32_t* __restrict__ vrow,
                                                         const double* __restrict__ aval,
                                                         const int32_t* __restrict__ col_cons, double* B,
                                                         int64_t ldb) {
  __shared__ int32_t lcol[kPanelW];
  __shared__ double lval[kPanelW];
  const int P = blockIdx.y;
  if (threadIdx.x < kPanelW) {
    const int e = P * kPanelW + threadIdx.x;
    const int l = e < n ? col_cons[e] : -1;
    lcol[threadIdx.x] = l;
    lval[threadIdx.x] = l >= 0 ? aval[l] : 0.0;
  }
  __syncthreads();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int i = vrow[k];
  const double ak = aval[k];
  const double2* xr = reinterpret_cast<const double2*>(Xh + ((size_t)P * n + i) * kPanelW);
  const double2* yr = reinterpret_cast<const double2*>(Yh + ((size_t)P * n + i) * kPanelW);
#pragma unroll 4
  for (int h = 0; h < kPanelW / 2; ++h) {
    const double2 x = xr[h], y = yr[h];
    const int l0 = lcol[2 * h], l1 = lcol[2 * h + 1];
    if (l0 >= 0 && k >= l0) B[k + (size_t)l0 * ldb] = ak * lval[2 * h] * x.x * y.x;
    if (l1 >= 0 && k >= l1) B[k + (size_t)l1 * ldb] = ak * lval[2 * h + 1] * x.y * y.y;
  }
}

constexpr int kMaxSmall = 64;  // entries of a "small" constraint held in shared memory

__global__ void __launch_bounds__(256) scm_general_kernel(int n, int m, const double* __restrict__ Xh,
                                                          const double* __restrict__ Yh,
                                                          const int64_t* __restrict__ ptr,
                                                          const int32_t* __restrict__ ei,
                                                          const int32_t* __restrict__ ej,
                                                          const double* __restrict__ ev,
                                                          const uint8_t* __restrict__ is_large, double* B,
                                                          int64_t ldb) {
  __shared__ int32_t sp[kMaxSmall], sq[kMaxSmall];
  __shared__ double sw[kMaxSmall];
  const int l = blockIdx.x;
  if (is_large[l]) return;
  const int64_t lb = ptr[l];
  const int nl = (int)(ptr[l + 1] - lb);
  for (int t = threadIdx.x; t < nl; t += blockDim.x) {
    sp[t] = ei[lb + t];
    sq[t] = ej[lb + t];
    sw[t] = ev[lb + t];
  }
  __syncthreads();
  for (int k = l + threadIdx.x; k < m; k += blockDim.x) {
    if (is_large[k]) continue;
    double sum = 0.0;
    for (int64_t e = ptr[k]; e < ptr[k + 1]; ++e) {
      const int i = ei[e], j = ej[e];
      const double v = ev[e];
      for (int t = 0; t < nl; ++t) sum += v * sw[t] * pm(Xh, n, j, sp[t]) * pm(Yh, n, sq[t], i);
    }
    B[k + (size_t)l * ldb] = sum;
  }
}

__global__ void __launch_bounds__(512) scm_large_kernel(int n, int m, const double* __restrict__ Xh,
                                                        const double* __restrict__ Yh,
                                                        const int64_t* __restrict__ ptr,
                                                        const int32_t* __restrict__ ei,
                                                        const int32_t* __restrict__ ej,
                                                        const double* __restrict__ ev,
                                                        const int32_t* __restrict__ large,
                                                        const uint8_t* __restrict__ is_large, double* B,
                                                        int64_t ldb) {
  __shared__ double red[32];
  const int l = blockIdx.x;
  const int K = large[blockIdx.y];
  if (is_large[l] && l > K) return;  // large x large pairs computed once (l <= K)
  const int64_t kb = ptr[K], nk = ptr[K + 1] - kb;
  const int64_t lb = ptr[l], nl = ptr[l + 1] - lb;
  double sum = 0.0;
  for (int64_t idx = threadIdx.x; idx < nk * nl; idx += blockDim.x) {
    const int64_t a = idx / nl, b = idx % nl;
    const int i = ei[kb + a], j = ej[kb + a];
    const int p = ei[lb + b], q = ej[lb + b];
    sum += ev[kb + a] * ev[lb + b] * pm(Xh, n, j, p) * pm(Yh, n, q, i);
  }
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) red[wid] = sum;
  __syncthreads();
  if (wid == 0) {
    sum = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) {
      const int hi = K > l ? K : l, lo = K > l ? l : K;
      B[hi + (size_t)lo * ldb] = sum;
    }
  }
}

int launch_scm(sdpc_ctx* h, double* B, int64_t ldb, cudaStream_t st) {
  const int n = h->S.n, m = h->S.m;
  const DevCons& c = h->cons;
  if (c.maxcut) {
    dim3 grid((m + 255) / 256, h->d.npanels);
    scm_maxcut_kernel<<<grid, 256, 0, st>>>(n, m, h->Xh, h->Yh, c.vrow, c.aval, c.col_cons, B, ldb);
    return 1;
  }
  int nl = 0;
  scm_general_kernel<<<m, 256, 0, st>>>(n, m, h->Xh, h->Yh, c.ptr, c.ei, c.ej, c.ev, c.is_large, B, ldb);
  ++nl;
  if (c.nlarge > 0) {
    dim3 grid(m, c.nlarge);
    scm_large_kernel<<<grid, 512, 0, st>>>(n, m, h->Xh, h->Yh, c.ptr, c.ei, c.ej, c.ev, c.large, c.is_large, B,
                                           ldb);
    ++nl;
  }
  return nl;
}

}  // namespace sdpc
