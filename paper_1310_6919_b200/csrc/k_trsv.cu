// Schur complement equation solve with the SCM Cholesky factor: (R R^T) X = G in place
// (the SCE  B dz = g  of the HKM direction, solved with
// the factor of type (i)).  R is the lower factor left in B by sdpc_scm_cholesky.
//
// Blocked by kTb = 128 rows.  Forward (R Y = G): for each block j, one CTA solves the diagonal
// triangle for all right-hand sides (warp per RHS, lanes over rows of the 32-row sub-blocks), then a
// grid-wide update G[below] -= R[below, j] Y_j (thread per row, coalesced reads of the column panel).
// Backward (R^T X = Y): for each block j from the last, a grid-wide reduction S_j = R[below, j]^T X
// (CTA per column of the block) then the CTA-wide transposed triangle.  The factor is read once per
// sweep: the solve is HBM-bound (m^2/2 doubles per sweep) plus 2 * (m / 128) dependent launches.
#include <cuda_runtime.h>

#include "common.cuh"
#include "ctx.hpp"

#include <algorithm>

namespace sdpc {

constexpr int kTb = 128;

// lower triangle of block j: Y[j0 + i] = (G[j0 + i] - sum_{c < i} R[j0+i, j0+c] Y[j0+c]) / R[j0+i, j0+i]
// one warp per right-hand side, the block's rows in shared memory
__global__ void __launch_bounds__(256) trsv_fwd_diag(const double* __restrict__ R, int64_t ldr, int64_t m, int j0,
                                                     double* G, int64_t ldg, int nrhs) {
  extern __shared__ double trsv_sm[];
  double (*Rs)[kTb + 1] = reinterpret_cast<double (*)[kTb + 1]>(trsv_sm);
  const int nb = (int)(m - j0 < kTb ? m - j0 : kTb);
  for (int idx = threadIdx.x; idx < nb * nb; idx += blockDim.x) {
    const int i = idx % nb, c = idx / nb;
    Rs[i][c] = i >= c ? R[(j0 + i) + (size_t)(j0 + c) * ldr] : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int q = wid; q < nrhs; q += blockDim.x / 32) {
    double* g = G + (size_t)q * ldg + j0;
    // lane l holds rows l, l+32, l+64, l+96 of the block
    double y[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) y[t] = (lane + 32 * t < nb) ? g[lane + 32 * t] : 0.0;
    for (int i = 0; i < nb; ++i) {
      const int ti = i >> 5, li = i & 31;
      double yi = __shfl_sync(0xffffffffu, y[0], li);
      if (ti == 1) yi = __shfl_sync(0xffffffffu, y[1], li);
      if (ti == 2) yi = __shfl_sync(0xffffffffu, y[2], li);
      if (ti == 3) yi = __shfl_sync(0xffffffffu, y[3], li);
      yi /= Rs[i][i];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int r = lane + 32 * t;
        if (r == i) y[t] = yi;
        else if (r > i && r < nb) y[t] -= Rs[r][i] * yi;
      }
    }
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (lane + 32 * t < nb) g[lane + 32 * t] = y[t];
  }
}

// G[r] -= sum_c R[r, j0 + c] Y[j0 + c] for rows r >= j0 + nb (thread per row and RHS)
__global__ void __launch_bounds__(256) trsv_fwd_update(const double* __restrict__ R, int64_t ldr, int64_t m, int j0,
                                                       double* G, int64_t ldg, int nrhs) {
  const int nb = (int)(m - j0 < kTb ? m - j0 : kTb);
  const int64_t r = j0 + nb + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int q = blockIdx.y;
  if (r >= m) return;
  double* g = G + (size_t)q * ldg;
  double acc = 0.0;
#pragma unroll 8
  for (int c = 0; c < nb; ++c) acc += R[r + (size_t)(j0 + c) * ldr] * g[j0 + c];
  g[r] -= acc;
}

// S[q][c] = sum_{r >= j0 + nb} R[r, j0 + c] X[r]  (CTA per column c, all RHS)
__global__ void __launch_bounds__(256) trsv_bwd_dots(const double* __restrict__ R, int64_t ldr, int64_t m, int j0,
                                                     const double* X, int64_t ldx, int nrhs, double* S) {
  __shared__ double red[8];
  const int nb = (int)(m - j0 < kTb ? m - j0 : kTb);
  const int c = blockIdx.x;
  const int q = blockIdx.y;
  const double* col = R + (size_t)(j0 + c) * ldr;
  const double* x = X + (size_t)q * ldx;
  double acc = 0.0;
  for (int64_t r = j0 + nb + threadIdx.x; r < m; r += blockDim.x) acc += col[r] * x[r];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += red[w];
    S[(size_t)q * kTb + c] = s;
  }
}

// transposed triangle of block j: X[j0+i] = (Y[j0+i] - S[i] - sum_{r > i} R[j0+r, j0+i] X[j0+r]) / R_ii
__global__ void __launch_bounds__(256) trsv_bwd_diag(const double* __restrict__ R, int64_t ldr, int64_t m, int j0,
                                                     double* X, int64_t ldx, int nrhs, const double* S) {
  extern __shared__ double trsv_sm[];
  double (*Rs)[kTb + 1] = reinterpret_cast<double (*)[kTb + 1]>(trsv_sm);
  const int nb = (int)(m - j0 < kTb ? m - j0 : kTb);
  for (int idx = threadIdx.x; idx < nb * nb; idx += blockDim.x) {
    const int i = idx % nb, c = idx / nb;
    Rs[i][c] = i >= c ? R[(j0 + i) + (size_t)(j0 + c) * ldr] : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const bool has_s = j0 + nb < m;
  for (int q = wid; q < nrhs; q += blockDim.x / 32) {
    double* x = X + (size_t)q * ldx + j0;
    double v[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int r = lane + 32 * t;
      v[t] = r < nb ? x[r] - (has_s ? S[(size_t)q * kTb + r] : 0.0) : 0.0;
    }
    for (int i = nb - 1; i >= 0; --i) {
      const int ti = i >> 5, li = i & 31;
      double xi = __shfl_sync(0xffffffffu, v[0], li);
      if (ti == 1) xi = __shfl_sync(0xffffffffu, v[1], li);
      if (ti == 2) xi = __shfl_sync(0xffffffffu, v[2], li);
      if (ti == 3) xi = __shfl_sync(0xffffffffu, v[3], li);
      xi /= Rs[i][i];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int r = lane + 32 * t;
        if (r == i) v[t] = xi;
        else if (r < i) v[t] -= Rs[i][r] * xi;
      }
    }
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (lane + 32 * t < nb) x[lane + 32 * t] = v[t];
  }
}

int scm_solve(const double* R, int64_t ldr, int64_t m, double* G, int64_t ldg, int nrhs, double* S,
              cudaStream_t st) {
  const size_t smem = sizeof(double) * kTb * (kTb + 1);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(trsv_fwd_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(trsv_bwd_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  int launches = 0;
  for (int64_t j0 = 0; j0 < m; j0 += kTb) {
    trsv_fwd_diag<<<1, 256, smem, st>>>(R, ldr, m, (int)j0, G, ldg, nrhs);
    ++launches;
    const int64_t rows = m - j0 - kTb;
    if (rows > 0) {
      trsv_fwd_update<<<dim3((unsigned)((rows + 255) / 256), (unsigned)nrhs), 256, 0, st>>>(R, ldr, m, (int)j0, G,
                                                                                           ldg, nrhs);
      ++launches;
    }
  }
  const int64_t nblk = (m + kTb - 1) / kTb;
  for (int64_t jb = nblk - 1; jb >= 0; --jb) {
    const int64_t j0 = jb * kTb;
    const int nb = (int)std::min<int64_t>(kTb, m - j0);
    if (j0 + nb < m) {
      trsv_bwd_dots<<<dim3((unsigned)nb, (unsigned)nrhs), 256, 0, st>>>(R, ldr, m, (int)j0, G, ldg, nrhs, S);
      ++launches;
    }
    trsv_bwd_diag<<<1, 256, smem, st>>>(R, ldr, m, (int)j0, G, ldg, nrhs, S);
    ++launches;
  }
  return launches;
}

}  // namespace sdpc
