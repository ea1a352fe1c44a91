// Schur complement equation solve with the SCM Cholesky factor: (R R^T) X = G in place
// (the SCE  B dz = g  of the HKM direction, solved with
// the factor of type (i)).  R is the lower factor left in B by sdpc_scm_cholesky.
//
// Blocked by kTb = 128 rows, both sweeps right-looking.  Forward (R Y = G): for each block j, one CTA
// solves the diagonal triangle for all right-hand sides (32-row sub-triangles, warp per RHS, lane =
// row), then a grid-wide update G[below] -= R[below, j] Y_j (8 lanes per row split the 128 columns).
// Backward (R^T X = Y): for each block j from the last, the transposed triangle, then a grid-wide
// update X[above] -= R[j, above]^T X_j (8 lanes per row of R^T read contiguous runs of a column of
// R).  The factor is read once per sweep (HBM-bound: m^2/2 doubles per sweep); each sweep is one
// cooperative launch, the next diagonal triangle is prefetched (cp.async) during the update phase.
#include <cuda_runtime.h>

#include "common.cuh"
#include "ctx.hpp"

#include <algorithm>

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace sdpc {

constexpr int kTb = 128;

// One cooperative launch per sweep (the grid waits on itself only, inside one kernel): per 128-row
// block, CTA 0 solves the diagonal triangle while the others wait at a grid barrier, then every CTA
// applies the solved block to its share of the remaining rows (both sweeps right-looking: forward
// G[below] -= R[below, j] Y_j, backward X[above] -= R[j, above]^T X_j).  2 grid barriers per block
// instead of 2 dependent launches.
// Stage the lower triangle of the diagonal block [j0, j0+nb)^2 of R into Rs (upper part zero-filled)
// with cp.async: all loads in flight at once, and issued one block ahead (R is read-only during the
// solve), so the serial triangle solve never waits on DRAM latency.
__device__ __forceinline__ void prefetch_tri(const double* __restrict__ R, int64_t ldr, int64_t m, int64_t j0,
                                             double (*Rs)[kTb + 1]) {
  const int nb = (int)(m - j0 < kTb ? m - j0 : kTb);
  for (int idx = threadIdx.x; idx < nb * nb; idx += blockDim.x) {
    const int i = idx % nb, c = idx / nb;
    cp_async8(&Rs[i][c], i >= c ? R + (j0 + i) + (size_t)(j0 + c) * ldr : R, i >= c);
  }
  cp_async_commit();
}

__device__ __forceinline__ void diag_solve_fwd(const double* __restrict__ R, int64_t ldr, int64_t m, int j0, double* G,
                                               int64_t ldg, int nrhs, double (*Rs)[kTb + 1]) {
  __shared__ double rd[kTb];
  const int nb = (int)(m - j0 < kTb ? m - j0 : kTb);
  cp_async_wait<0>();
  __syncthreads();
  for (int i = threadIdx.x; i < nb; i += blockDim.x) rd[i] = 1.0 / Rs[i][i];  // off the serial chain
  __syncthreads();
  // 32-row sub-blocks: a warp per RHS solves the 32-triangle (lane = row, one shuffle per step),
  // then the CTA applies it to the rows below (thread per (row, RHS)); short serial chains only
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int s0 = 0; s0 < nb; s0 += 32) {
    const int sb = nb - s0 < 32 ? nb - s0 : 32;
    for (int q = wid; q < nrhs; q += nw) {
      double* g = G + (size_t)q * ldg + j0 + s0;
      double y = lane < sb ? g[lane] : 0.0;
      for (int i = 0; i < sb; ++i) {
        const double yi = __shfl_sync(0xffffffffu, y, i) * rd[s0 + i];
        if (lane == i) y = yi;
        else if (lane > i && lane < sb) y -= Rs[s0 + lane][s0 + i] * yi;
      }
      if (lane < sb) g[lane] = y;
    }
    __syncthreads();
    const int rem = nb - s0 - sb;
    for (int idx = threadIdx.x; idx < rem * nrhs; idx += blockDim.x) {
      const int r = s0 + sb + idx % rem, q = idx / rem;
      double* g = G + (size_t)q * ldg + j0;
      double acc = 0.0;
#pragma unroll 8
      for (int c = 0; c < sb; ++c) acc += Rs[r][s0 + c] * g[s0 + c];
      g[r] -= acc;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) trsv_fwd_coop(const double* __restrict__ R, int64_t ldr, int64_t m, double* G,
                                                     int64_t ldg, int nrhs) {
  extern __shared__ double trsv_sm[];
  double (*Rs)[kTb + 1] = reinterpret_cast<double (*)[kTb + 1]>(trsv_sm);
  cg::grid_group grid = cg::this_grid();
  if (blockIdx.x == 0 && m > 0) prefetch_tri(R, ldr, m, 0, Rs);
  for (int64_t j0 = 0; j0 < m; j0 += kTb) {
    const int nb = (int)(m - j0 < kTb ? m - j0 : kTb);
    if (blockIdx.x == 0) {
      diag_solve_fwd(R, ldr, m, (int)j0, G, ldg, nrhs, Rs);
      if (j0 + kTb < m) prefetch_tri(R, ldr, m, j0 + kTb, Rs);  // overlaps the update phase
    }
    grid.sync();
    const int64_t rows = m - j0 - nb;
    // thread = (row, chunk of 16 block columns); the 8 chunks of a row are 8 adjacent lanes
    const int64_t work = rows * nrhs * 8;
    for (int64_t w0 = (int64_t)blockIdx.x * blockDim.x; w0 < work; w0 += (int64_t)gridDim.x * blockDim.x) {
      const int64_t w = w0 + threadIdx.x;
      const int ch = (int)(w & 7);
      const int64_t rw = w >> 3;
      double acc = 0.0;
      int64_t r = 0;
      double* g = G;
      if (w < work) {
        r = j0 + nb + rw % rows;
        g = G + (size_t)(rw / rows) * ldg;
#pragma unroll
        for (int cc = 0; cc < 16; ++cc) {
          const int c = ch * 16 + cc;
          if (c < nb) acc += R[r + (size_t)(j0 + c) * ldr] * g[j0 + c];
        }
      }
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      acc += __shfl_xor_sync(0xffffffffu, acc, 4);
      if (w < work && ch == 0) g[r] -= acc;
    }
    grid.sync();
  }
}

__global__ void __launch_bounds__(256) trsv_bwd_coop(const double* __restrict__ R, int64_t ldr, int64_t m, double* X,
                                                     int64_t ldx, int nrhs) {
  extern __shared__ double trsv_sm[];
  double (*Rs)[kTb + 1] = reinterpret_cast<double (*)[kTb + 1]>(trsv_sm);
  cg::grid_group grid = cg::this_grid();
  const int64_t nblk = (m + kTb - 1) / kTb;
  if (blockIdx.x == 0 && nblk > 0) prefetch_tri(R, ldr, m, (nblk - 1) * kTb, Rs);
  for (int64_t jb = nblk - 1; jb >= 0; --jb) {
    const int64_t j0 = jb * kTb;
    const int nb = (int)(m - j0 < kTb ? m - j0 : kTb);
    if (blockIdx.x == 0) {
      __shared__ double rdb[kTb];
      cp_async_wait<0>();
      __syncthreads();
      for (int i = threadIdx.x; i < nb; i += blockDim.x) rdb[i] = 1.0 / Rs[i][i];
      __syncthreads();
      // 32-row sub-blocks from the last: warp per RHS on the transposed 32-triangle, then the CTA
      // applies it to the rows above
      const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
      for (int s0 = ((nb - 1) / 32) * 32; s0 >= 0; s0 -= 32) {
        const int sb = nb - s0 < 32 ? nb - s0 : 32;
        for (int q = wid; q < nrhs; q += nw) {
          double* x = X + (size_t)q * ldx + j0 + s0;
          double v = lane < sb ? x[lane] : 0.0;
          for (int i = sb - 1; i >= 0; --i) {
            const double xi = __shfl_sync(0xffffffffu, v, i) * rdb[s0 + i];
            if (lane == i) v = xi;
            else if (lane < i) v -= Rs[s0 + i][s0 + lane] * xi;
          }
          if (lane < sb) x[lane] = v;
        }
        __syncthreads();
        for (int idx = threadIdx.x; idx < s0 * nrhs; idx += blockDim.x) {
          const int r = idx % s0, q = idx / s0;
          double* x = X + (size_t)q * ldx + j0;
          double acc = 0.0;
#pragma unroll 8
          for (int c = 0; c < sb; ++c) acc += Rs[s0 + c][r] * x[s0 + c];
          x[r] -= acc;
        }
        __syncthreads();
      }
      if (jb > 0) prefetch_tri(R, ldr, m, (jb - 1) * kTb, Rs);  // overlaps the update phase
    }
    grid.sync();
    // right-looking transposed update of the rows above: X[r] -= sum_c R[j0+c, r] X[j0+c], r < j0.
    // Row j0+c of R restricted to column r is contiguous in c (column-major), so the 8 lanes of a row
    // read interleaved, coalesced 64-B runs of column r
    const int64_t work = j0 * nrhs * 8;
    for (int64_t w0 = (int64_t)blockIdx.x * blockDim.x; w0 < work; w0 += (int64_t)gridDim.x * blockDim.x) {
      const int64_t w = w0 + threadIdx.x;
      const int ch = (int)(w & 7);
      const int64_t rw = w >> 3;
      double acc = 0.0;
      int64_t r = 0;
      double* x = X;
      if (w < work) {
        r = rw % j0;
        x = X + (size_t)(rw / j0) * ldx;
        const double* col = R + (size_t)r * ldr + j0;
#pragma unroll
        for (int cc = 0; cc < 16; ++cc) {
          const int c = ch + 8 * cc;
          if (c < nb) acc += col[c] * x[j0 + c];
        }
      }
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      acc += __shfl_xor_sync(0xffffffffu, acc, 4);
      if (w < work && ch == 0) x[r] -= acc;
    }
    grid.sync();
  }
}

int scm_solve(const double* R, int64_t ldr, int64_t m, double* G, int64_t ldg, int nrhs, double* S,
              cudaStream_t st) {
  const size_t smem = sizeof(double) * kTb * (kTb + 1);
  // cooperative grid: every CTA co-resident, sized per device (SM count and occupancy of that device)
  static int grids[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  int& grid = grids[dev & 63];
  if (!grid) {
    cudaFuncSetAttribute(trsv_fwd_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(trsv_bwd_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int sms = 0, occ = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, trsv_fwd_coop, 256, smem);
    grid = sms * std::max(1, occ);
  }
  void* fa[] = {(void*)&R, (void*)&ldr, (void*)&m, (void*)&G, (void*)&ldg, (void*)&nrhs};
  if (cudaLaunchCooperativeKernel((const void*)trsv_fwd_coop, dim3(grid), dim3(256), fa, smem, st) != cudaSuccess)
    return -1;
  void* ba[] = {(void*)&R, (void*)&ldr, (void*)&m, (void*)&G, (void*)&ldg, (void*)&nrhs};
  (void)S;
  if (cudaLaunchCooperativeKernel((const void*)trsv_bwd_coop, dim3(grid), dim3(256), ba, smem, st) != cudaSuccess)
    return -1;
  return 2;
}

}  // namespace sdpc
