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

// Diagonal step with the block inverse staged in Rs (Rs[i][c] = Linv_jj[i][c], lower): g_j <- Linv_jj g_j
// (forward) or Linv_jj^T g_j (backward), a 128 x 128 GEMV per right-hand side instead of a serial
// triangular solve.
__device__ __forceinline__ void diag_gemv(int nb, double* G, int64_t ldg, int64_t j0, int nrhs, double (*Rs)[kTb + 1],
                                          bool trans) {
  __shared__ double gs[kTb];
  cp_async_wait<0>();
  __syncthreads();
  for (int q = 0; q < nrhs; ++q) {
    double* g = G + (size_t)q * ldg + j0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) gs[i] = g[i];
    __syncthreads();
    for (int i = threadIdx.x; i < nb; i += blockDim.x) {
      double acc = 0.0;
      if (!trans) {
        for (int c = 0; c <= i; ++c) acc += Rs[i][c] * gs[c];
      } else {
        for (int c = i; c < nb; ++c) acc += Rs[c][i] * gs[c];
      }
      g[i] = acc;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) trsv_fwd_coop(const double* __restrict__ R, int64_t ldr, int64_t m, double* G,
                                                     int64_t ldg, int nrhs, const double* __restrict__ Linv) {
  extern __shared__ double trsv_sm[];
  double (*Rs)[kTb + 1] = reinterpret_cast<double (*)[kTb + 1]>(trsv_sm);
  cg::grid_group grid = cg::this_grid();
  // with the block inverses, the staged block is L_jj^{-1} (ld kTb, its own rows and columns 0..nb-1)
  auto stage = [&](int64_t j0) {
    const int nb = (int)(m - j0 < kTb ? m - j0 : kTb);
    if (Linv) prefetch_tri(Linv + (j0 / kTb) * kTb * kTb, kTb, nb, 0, Rs);
    else prefetch_tri(R, ldr, m, j0, Rs);
  };
  if (blockIdx.x == 0 && m > 0) stage(0);
  for (int64_t j0 = 0; j0 < m; j0 += kTb) {
    const int nb = (int)(m - j0 < kTb ? m - j0 : kTb);
    if (blockIdx.x == 0) {
      if (Linv) diag_gemv(nb, G, ldg, j0, nrhs, Rs, false);
      else diag_solve_fwd(R, ldr, m, (int)j0, G, ldg, nrhs, Rs);
      if (j0 + kTb < m) stage(j0 + kTb);  // overlaps the update phase
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
                                                     int64_t ldx, int nrhs, const double* __restrict__ Linv) {
  extern __shared__ double trsv_sm[];
  double (*Rs)[kTb + 1] = reinterpret_cast<double (*)[kTb + 1]>(trsv_sm);
  cg::grid_group grid = cg::this_grid();
  const int64_t nblk = (m + kTb - 1) / kTb;
  auto stage = [&](int64_t j0) {
    const int nb = (int)(m - j0 < kTb ? m - j0 : kTb);
    if (Linv) prefetch_tri(Linv + (j0 / kTb) * kTb * kTb, kTb, nb, 0, Rs);
    else prefetch_tri(R, ldr, m, j0, Rs);
  };
  if (blockIdx.x == 0 && nblk > 0) stage((nblk - 1) * kTb);
  for (int64_t jb = nblk - 1; jb >= 0; --jb) {
    const int64_t j0 = jb * kTb;
    const int nb = (int)(m - j0 < kTb ? m - j0 : kTb);
    if (blockIdx.x == 0 && Linv) {
      diag_gemv(nb, X, ldx, j0, nrhs, Rs, true);
      if (jb > 0) stage((jb - 1) * kTb);
    } else if (blockIdx.x == 0) {
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
      if (jb > 0) stage((jb - 1) * kTb);  // overlaps the update phase
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

// ---------------------------------------------------------------- block-flag sweeps (with the inverses)
// Each CTA owns the 128-row blocks b = blockIdx.x, blockIdx.x + gridDim.x, ... and processes them in
// sweep order.  Forward: y_b = Linv_bb (g_b - sum_{j < b} R_bj y_j); every solved block raises flag[b], and a
// CTA applies block j to its own rows as soon as flag[j] is up (no grid-wide barrier: the serial chain is
// one flag hand-off and one 128 x 128 GEMV per block).  Backward: x_b = Linv_bb^T (y_b - sum_{j > b} R_jb^T
// x_j), blocks in decreasing order.  Deadlock-free with every CTA co-resident (cooperative launch): a CTA
// waits only on smaller (forward) / larger (backward) blocks, whose owners never wait on it.
constexpr int kMaxRhsFlag = 8;  // right-hand sides per pass of the flag sweeps
constexpr size_t kFlagSmem = sizeof(double) * kTb * (kTb + 1);  // the staged block inverse

__device__ __forceinline__ void wait_flag(const int* f) {
  while (*(const volatile int*)f == 0) {
  }
  __threadfence();
}

// Linv_bb (128 x 128, column-major ld kTb) into Ls[c][r] layout Ls[r + c * (kTb + 1)], by cp.async (issued early:
// the CTA then waits for flags while it lands)
__device__ __forceinline__ void stage_linv(const double* __restrict__ Lb, double* Ls) {
  for (int i = threadIdx.x; i < kTb * kTb; i += blockDim.x) {
    const int r = i % kTb, c = i / kTb;
    cp_async8(Ls + r + c * (kTb + 1), Lb + i, r >= c);
  }
  cp_async_commit();
}

__global__ void __launch_bounds__(256) trsv_fwd_flags(const double* __restrict__ R, int64_t ldr, int64_t m, double* G,
                                                      int64_t ldg, int nrhs, const double* __restrict__ Linv,
                                                      int* flags) {
  extern __shared__ double Ls[];  // kTb x (kTb + 1)
  __shared__ double acc[kMaxRhsFlag][kTb];
  __shared__ double ys[kMaxRhsFlag][kTb];
  __shared__ double part[2][kMaxRhsFlag][kTb];
  const int tid = threadIdx.x, r = tid & (kTb - 1), hf = tid >> 7;  // (row, half of the columns)
  const int64_t nblk = (m + kTb - 1) / kTb;
  for (int64_t b = blockIdx.x; b < nblk; b += gridDim.x) {
    const int64_t r0 = b * kTb;
    const int nb = (int)(m - r0 < kTb ? m - r0 : kTb);
    stage_linv(Linv + b * kTb * kTb, Ls);
    for (int q0 = 0; q0 < nrhs; q0 += kMaxRhsFlag) {
      const int nq = nrhs - q0 < kMaxRhsFlag ? nrhs - q0 : kMaxRhsFlag;
      for (int i = tid; i < nq * kTb; i += blockDim.x) {
        const int q = i / kTb, rr = i % kTb;
        acc[q][rr] = rr < nb ? G[(size_t)(q0 + q) * ldg + r0 + rr] : 0.0;
      }
      for (int64_t j = 0; j < b; ++j) {
        if (tid == 0) wait_flag(flags + j);
        __syncthreads();
        for (int i = tid; i < nq * kTb; i += blockDim.x) {
          const int q = i / kTb, c = i % kTb;
          ys[q][c] = __ldcg(G + (size_t)(q0 + q) * ldg + j * kTb + c);
        }
        __syncthreads();
        // acc[:, rows] -= R[rows, j cols] y_j; thread (r, hf) sums 64 columns (coalesced over r)
        double sacc[kMaxRhsFlag];
#pragma unroll
        for (int q = 0; q < kMaxRhsFlag; ++q) sacc[q] = 0.0;
        if (r < nb) {
          const double* Rc = R + (r0 + r) + (size_t)(j * kTb + hf * 64) * ldr;
#pragma unroll 16
          for (int c = 0; c < 64; ++c) {
            const double v = Rc[(size_t)c * ldr];
#pragma unroll
            for (int q = 0; q < kMaxRhsFlag; ++q)
              if (q < nq) sacc[q] += v * ys[q][hf * 64 + c];
          }
        }
#pragma unroll
        for (int q = 0; q < kMaxRhsFlag; ++q) part[hf][q][r] = sacc[q];
        __syncthreads();
        for (int i = tid; i < nq * kTb; i += blockDim.x) {
          const int q = i / kTb, rr = i % kTb;
          acc[q][rr] -= part[0][q][rr] + part[1][q][rr];
        }
      }
      cp_async_wait<0>();
      __syncthreads();
      // y_b = Linv_bb acc
      for (int i = tid; i < nq * kTb; i += blockDim.x) {
        const int q = i / kTb, rr = i % kTb;
        if (rr >= nb) continue;
        double v = 0.0;
        for (int c = 0; c <= rr; ++c) v += Ls[rr + c * (kTb + 1)] * acc[q][c];
        G[(size_t)(q0 + q) * ldg + r0 + rr] = v;
      }
      __syncthreads();
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) atomicExch(flags + b, 1);
  }
}

__global__ void __launch_bounds__(256) trsv_bwd_flags(const double* __restrict__ R, int64_t ldr, int64_t m, double* X,
                                                      int64_t ldx, int nrhs, const double* __restrict__ Linv,
                                                      int* flags) {
  extern __shared__ double Ls[];
  __shared__ double acc[kMaxRhsFlag][kTb];
  __shared__ double xs[kMaxRhsFlag][kTb];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t nblk = (m + kTb - 1) / kTb;
  for (int64_t b = ((nblk - 1) / gridDim.x) * gridDim.x + blockIdx.x; b >= 0; b -= gridDim.x) {
    if (b >= nblk) continue;
    const int64_t r0 = b * kTb;
    const int nb = (int)(m - r0 < kTb ? m - r0 : kTb);
    stage_linv(Linv + b * kTb * kTb, Ls);
    for (int q0 = 0; q0 < nrhs; q0 += kMaxRhsFlag) {
      const int nq = nrhs - q0 < kMaxRhsFlag ? nrhs - q0 : kMaxRhsFlag;
      for (int i = tid; i < nq * kTb; i += blockDim.x) {
        const int q = i / kTb, rr = i % kTb;
        acc[q][rr] = rr < nb ? X[(size_t)(q0 + q) * ldx + r0 + rr] : 0.0;
      }
      for (int64_t j = nblk - 1; j > b; --j) {
        if (tid == 0) wait_flag(flags + j);
        __syncthreads();
        const int64_t c0 = j * kTb;
        const int nc = (int)(m - c0 < kTb ? m - c0 : kTb);
        for (int i = tid; i < nq * kTb; i += blockDim.x) {
          const int q = i / kTb, c = i % kTb;
          xs[q][c] = c < nc ? __ldcg(X + (size_t)(q0 + q) * ldx + c0 + c) : 0.0;
        }
        __syncthreads();
        // acc[rr] -= sum_c R[c0 + c, r0 + rr] x_j[c]: warp per output row, lanes over c (contiguous)
        for (int rr = wid; rr < nb; rr += blockDim.x / 32) {
          const double* Rc = R + c0 + (size_t)(r0 + rr) * ldr;
          double sacc[kMaxRhsFlag];
#pragma unroll
          for (int q = 0; q < kMaxRhsFlag; ++q) sacc[q] = 0.0;
#pragma unroll
          for (int cc = 0; cc < kTb; cc += 32) {
            const int c = cc + lane;
            const double v = c < nc ? Rc[c] : 0.0;
#pragma unroll
            for (int q = 0; q < kMaxRhsFlag; ++q)
              if (q < nq) sacc[q] += v * xs[q][c];
          }
#pragma unroll
          for (int q = 0; q < kMaxRhsFlag; ++q) {
            if (q >= nq) break;
            double v = sacc[q];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) acc[q][rr] -= v;
          }
        }
      }
      cp_async_wait<0>();
      __syncthreads();
      // x_b = Linv_bb^T acc
      for (int i = tid; i < nq * kTb; i += blockDim.x) {
        const int q = i / kTb, rr = i % kTb;
        if (rr >= nb) continue;
        double v = 0.0;
        for (int c = rr; c < nb; ++c) v += Ls[c + rr * (kTb + 1)] * acc[q][c];
        X[(size_t)(q0 + q) * ldx + r0 + rr] = v;
      }
      __syncthreads();
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) atomicExch(flags + b, 1);
  }
}

int scm_solve(const double* R, int64_t ldr, int64_t m, double* G, int64_t ldg, int nrhs, double* S,
              cudaStream_t st, const double* Linv) {
  if (Linv) {
    // block-flag sweeps: one cooperative launch each (co-residency of every CTA), flags zeroed per sweep
    static int grids[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    int& grid = grids[dev & 63];
    if (!grid) {
      int sms = 0, occ = 0;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaFuncSetAttribute(trsv_fwd_flags, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFlagSmem);
      cudaFuncSetAttribute(trsv_bwd_flags, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFlagSmem);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, trsv_fwd_flags, 256, kFlagSmem);
      int occ2 = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, trsv_bwd_flags, 256, kFlagSmem);
      grid = sms * std::max(1, std::min(occ, occ2));
    }
    const int64_t nblk = (m + kTb - 1) / kTb;
    const int g = (int)std::min<int64_t>(grid, std::max<int64_t>(1, nblk));
    int* flags = reinterpret_cast<int*>(S);  // S holds >= 2 nblk ints (sized by the caller)
    if (cudaMemsetAsync(flags, 0, sizeof(int) * 2 * nblk, st) != cudaSuccess) return -1;
    int* f2 = flags + nblk;
    void* fa[] = {(void*)&R, (void*)&ldr, (void*)&m, (void*)&G, (void*)&ldg, (void*)&nrhs, (void*)&Linv, (void*)&flags};
    if (cudaLaunchCooperativeKernel((const void*)trsv_fwd_flags, dim3(g), dim3(256), fa, kFlagSmem, st) != cudaSuccess)
      return -1;
    void* ba[] = {(void*)&R, (void*)&ldr, (void*)&m, (void*)&G, (void*)&ldg, (void*)&nrhs, (void*)&Linv, (void*)&f2};
    if (cudaLaunchCooperativeKernel((const void*)trsv_bwd_flags, dim3(g), dim3(256), ba, kFlagSmem, st) != cudaSuccess)
      return -1;
    return 2;
  }
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
  void* fa[] = {(void*)&R, (void*)&ldr, (void*)&m, (void*)&G, (void*)&ldg, (void*)&nrhs, (void*)&Linv};
  if (cudaLaunchCooperativeKernel((const void*)trsv_fwd_coop, dim3(grid), dim3(256), fa, smem, st) != cudaSuccess)
    return -1;
  void* ba[] = {(void*)&R, (void*)&ldr, (void*)&m, (void*)&G, (void*)&ldg, (void*)&nrhs, (void*)&Linv};
  (void)S;
  if (cudaLaunchCooperativeKernel((const void*)trsv_bwd_coop, dim3(grid), dim3(256), ba, smem, st) != cudaSuccess)
    return -1;
  return 2;
}

}  // namespace sdpc
