// the rest of one MC-PDIPM iteration after the SCM, on the GPU.
//
// Search direction (HKM, §2.2, as printed):
//   g_k  = A_k . (beta mu Y^{-1} - X-hat - X-hat G Y^{-1})
//   B dz = g   (with the factor R of sdpc_scm_cholesky)
//   dY   = G - sum_k A_k dz_k   on E
//   P-MATRIX (Eq. newdX2): column k of dX-hat = beta mu Y^{-1} e_k - X-hat e_k -
//        X-hat dY Y^{-1} e_k, kept on E, dX = (dX-hat + dX-hat^T) / 2.
// X-hat G Y^{-1} and X-hat dY Y^{-1} are formed panel by panel: the symmetric sparse matrix (on E)
// times the materialised Y^{-1} panels (spmm_sym_kernel), then X-hat applied to those dense panels by
// the multi-RHS supernodal solve of (b) with general right-hand sides (launch_apply_inverse).
//
// Step lengths (Step 3 P:351-361, Eq. primal_length2):
//   alpha_p = min_r max{alpha in (0,1] : X-bar_{C_rC_r} + alpha dX_{C_rC_r} >= 0}: one CTA per clique,
//             bisection on alpha with attempted Cholesky factorisations of the clique block;
//   alpha_d = max{alpha in (0,1] : Y + alpha dY >= 0}: bisection with attempted sparse LDL^T of
//             Y + alpha dY (the (a2) multifrontal factorisation as the cone test).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "ctx.hpp"

namespace sdpc {

// out[P][i][:] = sum_{j} S_ij in[P][j][:]  (S symmetric on E: lower values in E's CSC order)
__global__ void __launch_bounds__(256) spmm_sym_kernel(int n, const int32_t* __restrict__ sym_ptr,
                                                       const int32_t* __restrict__ sym_col,
                                                       const int32_t* __restrict__ sym_pos,
                                                       const double* __restrict__ vals,
                                                       const double* __restrict__ in, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (i >= n) return;
  const size_t pb = (size_t)blockIdx.y * n * kPanelW;
  double acc = 0.0;
  for (int t = sym_ptr[i]; t < sym_ptr[i + 1]; ++t)
    acc += vals[sym_pos[t]] * in[pb + (size_t)sym_col[t] * kPanelW + lane];
  out[pb + (size_t)i * kPanelW + lane] = acc;
}

// entry (row i, column j) of a panel-major matrix whose column j sits in RHS slot slot_of[j]
__device__ __forceinline__ double pmat(const double* __restrict__ M, const int32_t* __restrict__ slot_of, int n,
                                       int i, int j) {
  const int s = slot_of[j];
  return M[((size_t)(s >> 5) * n + i) * kPanelW + (s & 31)];
}

// g_k = sum over the (symmetric-expanded) entries (i, j, a) of A_k of a (bmu Yinv_ij - Xbar_ij - W_ij),
// W = X-hat G Y^{-1}; one warp per constraint
__global__ void __launch_bounds__(256) g_kernel(int m, int n, const int64_t* __restrict__ cptr,
                                                const int32_t* __restrict__ ei, const int32_t* __restrict__ ej,
                                                const double* __restrict__ ev, const int32_t* __restrict__ epos,
                                                const int32_t* __restrict__ slot_of, const double* __restrict__ Yh,
                                                const double* __restrict__ Wh, const double* __restrict__ xbar,
                                                double bmu, double* __restrict__ g) {
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (k >= m) return;
  double acc = 0.0;
  for (int64_t e = cptr[k] + lane; e < cptr[k + 1]; e += 32) {
    const int i = ei[e], j = ej[e];
    acc += ev[e] * (bmu * pmat(Yh, slot_of, n, i, j) - xbar[epos[e]] - pmat(Wh, slot_of, n, i, j));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) g[k] = acc;
}

// dY_q = G_q - sum_{(k, a) on E entry q} dz_k a
__global__ void __launch_bounds__(256) dY_kernel(int64_t nnz, const double* __restrict__ G,
                                                 const int32_t* __restrict__ ecs_ptr,
                                                 const int32_t* __restrict__ ecs_k,
                                                 const double* __restrict__ ecs_val, const double* __restrict__ dz,
                                                 double* __restrict__ dY) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nnz) return;
  double v = G[q];
  for (int t = ecs_ptr[q]; t < ecs_ptr[q + 1]; ++t) v -= dz[ecs_k[t]] * ecs_val[t];
  dY[q] = v;
}

// dX on E: entry (i, j), i >= j: bmu Yinv_ij - Xbar_ij - (Z_ij + Z_ji) / 2, Z = X-hat dY Y^{-1}
// (column j of Z is the panel column of slot j); one warp per column j
__global__ void __launch_bounds__(256) dX_kernel(int n, const int64_t* __restrict__ colptr,
                                                 const int32_t* __restrict__ rowind,
                                                 const int32_t* __restrict__ slot_of, const double* __restrict__ Yh,
                                                 const double* __restrict__ Zh, const double* __restrict__ xbar,
                                                 double bmu, double* __restrict__ dX) {
  const int lane = threadIdx.x & 31;
  const int j = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (j >= n) return;
  for (int64_t q = colptr[j] + lane; q < colptr[j + 1]; q += 32) {
    const int i = rowind[q];
    dX[q] = bmu * pmat(Yh, slot_of, n, i, j) - xbar[q] - 0.5 * (pmat(Zh, slot_of, n, i, j) + pmat(Zh, slot_of, n, j, i));
  }
}

__global__ void axpy_kernel(int64_t nnz, const double* __restrict__ y, const double* __restrict__ dy, double alpha,
                            double* __restrict__ out) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < nnz) out[q] = y[q] + alpha * dy[q];
}

// ---------------------------------------------------------------- primal step length, per clique
constexpr int kStepThreads = 256;
constexpr int kBisect = 40;  // bisection steps on alpha in (0, 1): |error| <= 2^-40

// In place lower Cholesky of the c x c matrix M (column-major, ld c); true iff positive definite.
__device__ bool block_potrf(double* M, int c) {
  const int tid = threadIdx.x;
  for (int j = 0; j < c; ++j) {
    const double d = M[j + (size_t)j * c];
    if (!(d > 0.0)) return false;  // uniform: every thread read the same value after the last barrier
    const double rl = rsqrt_nr(d);
    // (only the PD test is needed: the diagonal is left unscaled, so no thread overwrites the pivot
    // another thread may still be reading)
    for (int i = j + 1 + tid; i < c; i += kStepThreads) M[i + (size_t)j * c] *= rl;
    __syncthreads();
    const int w = c - j - 1;
    for (int e = tid; e < w * w; e += kStepThreads) {
      const int r = j + 1 + e % w, cc = j + 1 + e / w;
      if (r >= cc) M[r + (size_t)cc * c] -= M[r + (size_t)j * c] * M[cc + (size_t)j * c];
    }
    __syncthreads();
  }
  return true;
}

__global__ void __launch_bounds__(kStepThreads) primal_step_kernel(
    const int32_t* __restrict__ super_ptr, const int32_t* __restrict__ snc, const int64_t* __restrict__ colptr,
    const int32_t* __restrict__ rowind, const int64_t* __restrict__ blk_off, const double* __restrict__ xbar,
    const double* __restrict__ dX, double* ws, unsigned long long* amin) {
  const int r = blockIdx.x;
  const int f = super_ptr[r], c = snc[r];
  const int32_t* C = rowind + colptr[f];  // clique vertices: S_r then U_r, ascending
  double* Xc = ws + blk_off[r];
  double* dXc = Xc + (size_t)c * c;
  double* M = dXc + (size_t)c * c;
  const int tid = threadIdx.x;
  // gather the lower triangles of X-bar_CC and dX_CC (entry (a, b), a >= b, is E's (C_a, C_b))
  for (int e = tid; e < c * c; e += kStepThreads) {
    const int a = e % c, b = e / c;
    if (a < b) continue;
    const int32_t* beg = rowind + colptr[C[b]];
    const int32_t* end = rowind + colptr[C[b] + 1];
    int lo = 0, hi = (int)(end - beg) - 1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (beg[mid] < C[a]) lo = mid + 1;
      else hi = mid;
    }
    const int64_t q = colptr[C[b]] + lo;
    Xc[a + (size_t)b * c] = xbar[q];
    dXc[a + (size_t)b * c] = dX[q];
  }
  __syncthreads();
  auto pd = [&](double alpha) {
    for (int e = tid; e < c * c; e += kStepThreads) M[e] = Xc[e] + alpha * dXc[e];
    __syncthreads();
    return block_potrf(M, c);
  };
  __shared__ double s_cur;
  double lo = 0.0, hi = 1.0;
  if (!pd(1.0)) {
    for (int it = 0; it < kBisect; ++it) {
      // a clique whose interval lies above the current minimum cannot lower it (read by one thread and
      // broadcast: the decision must be uniform over the CTA)
      if (tid == 0) s_cur = __longlong_as_double((long long)*(volatile unsigned long long*)amin);
      __syncthreads();
      const double cur = s_cur;
      __syncthreads();
      if (lo >= cur) break;
      const double mid = 0.5 * (lo + hi);
      if (pd(mid)) lo = mid;
      else hi = mid;
    }
  } else {
    lo = 1.0;
  }
  if (tid == 0) atomicMin(amin, (unsigned long long)__double_as_longlong(lo));  // positive doubles: ordered bits
}

// ---------------------------------------------------------------- host side
static int64_t ensure_dir(sdpc_ctx* h) {
  const size_t dense = std::max<size_t>(1, (size_t)h->d.npanels * h->S.n * kPanelW);
  if (!h->Uh && cudaMalloc(&h->Uh, dense * sizeof(double)) != cudaSuccess) return -1;
  if (!h->dir_ws && cudaMalloc(&h->dir_ws, sizeof(double) * (2 * (size_t)h->S.m + 64)) != cudaSuccess) return -1;
  return 0;
}

// g (device, m) for the last scm_build's X-hat and Y^{-1}; returns launches or -1 (allocation failed)
int direction_g(sdpc_ctx* h, const double* xbar_E, const double* G_E, double bmu, double* g, cudaStream_t st) {
  const int n = h->S.n, m = h->S.m, np = h->d.npanels;
  if (ensure_dir(h) < 0) return -1;
  int launches = 0;
  if (h->trunc_active) {  // the max-cut build kept only the lower parts of its columns: full solves
    h->trunc_active = false;
    launches += launch_inverse_panels(h, st, 0, 2, 0);
  }
  const dim3 grow((n + 7) / 8, np);
  // W = X-hat (G Y^{-1}), then g
  spmm_sym_kernel<<<grow, 256, 0, st>>>(n, h->d.sym_ptr, h->d.sym_col, h->d.sym_pos, G_E, h->Yh, h->Uh);
  launches += 1 + launch_apply_inverse(h, st, 0, h->Uh, h->Uh);
  g_kernel<<<(m + 7) / 8, 256, 0, st>>>(m, n, h->cons.ptr, h->cons.ei, h->cons.ej, h->cons.ev, h->d.cons_epos,
                                        h->d.slot_of, h->Yh, h->Uh, xbar_E, bmu, g);
  return launches + 1;
}

// dY and the P-MATRIX dX on E from dz
int direction_dY_dX(sdpc_ctx* h, const double* xbar_E, const double* G_E, double bmu, const double* dz, double* dY_E,
                    double* dX_E, cudaStream_t st) {
  const int n = h->S.n, np = h->d.npanels;
  const int64_t nnz = h->S.nnzE();
  int launches = 0;
  dY_kernel<<<(unsigned)((nnz + 255) / 256), 256, 0, st>>>(nnz, G_E, h->d.ecs_ptr, h->d.ecs_k, h->d.ecs_val, dz, dY_E);
  const dim3 grow((n + 7) / 8, np);
  spmm_sym_kernel<<<grow, 256, 0, st>>>(n, h->d.sym_ptr, h->d.sym_col, h->d.sym_pos, dY_E, h->Yh, h->Uh);
  launches += 2 + launch_apply_inverse(h, st, 0, h->Uh, h->Uh);
  dX_kernel<<<(n + 7) / 8, 256, 0, st>>>(n, h->d.colptr, h->d.rowind, h->d.slot_of, h->Yh, h->Uh, xbar_E, bmu, dX_E);
  return launches + 1;
}

int primal_step(sdpc_ctx* h, const double* xbar_E, const double* dX_E, double* alpha_p, cudaStream_t st) {
  const int ns = h->S.nsuper;
  if (h->step_off.empty()) {
    h->step_off.resize(ns + 1, 0);
    for (int r = 0; r < ns; ++r) {
      const int64_t c = h->S.snc[r];
      h->step_off[r + 1] = h->step_off[r] + 3 * c * c;
    }
    if (cudaMalloc(&h->d_step_off, sizeof(int64_t) * (ns + 1)) != cudaSuccess) return -1;
    cudaMemcpy(h->d_step_off, h->step_off.data(), sizeof(int64_t) * (ns + 1), cudaMemcpyHostToDevice);
    if (cudaMalloc(&h->step_ws, sizeof(double) * std::max<int64_t>(1, h->step_off[ns])) != cudaSuccess) return -1;
    if (cudaMalloc(&h->d_amin, sizeof(unsigned long long)) != cudaSuccess) return -1;
  }
  static const double kOne = 1.0;  // (a static host source: the copy may still be pending at return)
  cudaMemcpyAsync(h->d_amin, &kOne, sizeof(kOne), cudaMemcpyHostToDevice, st);
  primal_step_kernel<<<ns, kStepThreads, 0, st>>>(h->d.super_ptr, h->d.snc, h->d.colptr, h->d.rowind, h->d_step_off,
                                                   xbar_E, dX_E, h->step_ws, h->d_amin);
  unsigned long long bits = 0;
  cudaMemcpyAsync(&bits, h->d_amin, sizeof(bits), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return -1;
  double a;
  std::memcpy(&a, &bits, sizeof(a));
  *alpha_p = a;
  return 1;
}

// alpha_d by bisection: PD(Y + alpha dY) tested by the multifrontal LDL^T of (a2) (its NOT_PD flag)
int dual_step(sdpc_ctx* h, const double* y_E, const double* dY_E, double* alpha_d, int steps, cudaStream_t st) {
  const int64_t nnz = h->S.nnzE();
  if (!h->ytmp && cudaMalloc(&h->ytmp, sizeof(double) * nnz) != cudaSuccess) return -1;
  int launches = 0;
  auto pd = [&](double alpha) -> int {
    axpy_kernel<<<(unsigned)((nnz + 255) / 256), 256, 0, st>>>(nnz, y_E, dY_E, alpha, h->ytmp);
    cudaMemsetAsync(h->d_err + 3, 0x7f, sizeof(int32_t), st);
    launches += 1 + launch_ldl_y(h, h->ytmp, st, h->d_err + 3, 0);
    int32_t v = 0;
    cudaMemcpyAsync(&v, h->d_err + 3, sizeof(v), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return -1;
    return v == kNoError ? 1 : 0;
  };
  double lo = 0.0, hi = 1.0;
  int r = pd(1.0);
  if (r < 0) return -1;
  if (r) {
    lo = 1.0;
  } else {
    for (int it = 0; it < steps; ++it) {
      const double mid = 0.5 * (lo + hi);
      r = pd(mid);
      if (r < 0) return -1;
      if (r) lo = mid;
      else hi = mid;
    }
  }
  h->have_y = false;  // the Y factor buffers now hold the last attempted factorisation
  *alpha_d = lo;
  return launches;
}

}  // namespace sdpc
