// (d) Dense FP64 Cholesky of the SCM, B = R R^T (lower, in place).
// PAPER.md P:711-713 / P:735-736 / P:978-979 (type (i): LAPACK dense Cholesky with multithreaded BLAS).
//
// Blocked right-looking, nb = 128.  Per panel step k0:
//   diag  : one CTA factors the kb x kb diagonal block in shared memory (32-wide sub-panels,
//           warp-level unblocked kernel) and forms its triangular inverse (for the TRSM);
//   trsm  : L21 = A21 L11^{-T} as an FP64 tensor-core GEMM with the explicit inverse;
//   update: A22 -= L21 L21^T over the lower 128 x 128 tiles, FP64 tensor-core GEMM
//           (mma.sync m8n8k4 f64 -> DMMA.8x8x4 on sm_100a; tcgen05 has no f64 kind),
//           operands staged in shared memory by a 3-stage cp.async pipeline.
// Non-PD: the first failing column (1-based, LAPACK potrf rule) is atomicMin'ed into *err and
// every later kernel exits at entry.
#include <cuda_runtime.h>

#include <cmath>
#include <vector>

#include "common.cuh"
#include "ctx.hpp"

namespace sdpc {

constexpr int kNB = 128;       // panel width
constexpr int kTile = 128;     // GEMM tile (BM = BN)
constexpr int kBK = 16;        // k-chunk per pipeline stage
constexpr int kStages = 3;
constexpr int kLdS = kTile + 4;  // smem row stride (doubles): conflict-free fragment loads
constexpr int kGemmThreads = 256;

// ------------------------------------------------------------------ diagonal block
constexpr int kDiagThreads = 256;
constexpr int kLdD = kNB + 1;

__global__ void __launch_bounds__(kDiagThreads) potrf_diag_kernel(double* B, int64_t ld, int k0, int kb,
                                                                  double* Linv, int32_t* err) {
  if (*err != kNoError) return;
  extern __shared__ double A[];  // kb x kb, column-major, ld kLdD
  __shared__ int bad;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double* Bd = B + k0 + (size_t)k0 * ld;
  for (int idx = tid; idx < kb * kb; idx += kDiagThreads) {
    const int i = idx % kb, j = idx / kb;
    A[i + j * kLdD] = i >= j ? Bd[i + (size_t)j * ld] : 0.0;
  }
  if (tid == 0) bad = 0;
  __syncthreads();
  for (int jb = 0; jb < kb; jb += 32) {
    const int jw = min(32, kb - jb);
    if (wid == 0) {  // unblocked Cholesky of the jw x jw sub-block, one warp
      for (int j = jb; j < jb + jw; ++j) {
        const double d = A[j + j * kLdD];
        if (!(d > 0.0)) {
          if (lane == 0) {
            bad = 1;
            report_error(err, k0 + j + 1);
          }
          break;
        }
        const double sq = sqrt(d);
        const int i = jb + lane;
        __syncwarp();
        if (i == j) A[j + j * kLdD] = sq;
        if (i > j && i < jb + jw) A[i + j * kLdD] /= sq;
        __syncwarp();
        for (int jj = j + 1; jj < jb + jw; ++jj)
          if (i >= jj && i < jb + jw) A[i + jj * kLdD] -= A[i + j * kLdD] * A[jj + j * kLdD];
        __syncwarp();
      }
    }
    __syncthreads();
    if (bad) return;
    // rows below the sub-block: forward substitution against the sub-block (row-parallel)
    for (int i = jb + jw + tid; i < kb; i += kDiagThreads) {
      for (int j = jb; j < jb + jw; ++j) {
        double a = A[i + j * kLdD];
        for (int t = jb; t < j; ++t) a -= A[i + t * kLdD] * A[j + t * kLdD];
        A[i + j * kLdD] = a / A[j + j * kLdD];
      }
    }
    __syncthreads();
    // trailing update of the diagonal block
    const int r0 = jb + jw, nr = kb - r0;
    for (int idx = tid; idx < nr * nr; idx += kDiagThreads) {
      const int i = r0 + idx % nr, j = r0 + idx / nr;
      if (i < j) continue;
      double a = A[i + j * kLdD];
      for (int t = jb; t < jb + jw; ++t) a -= A[i + t * kLdD] * A[j + t * kLdD];
      A[i + j * kLdD] = a;
    }
    __syncthreads();
  }
  for (int idx = tid; idx < kb * kb; idx += kDiagThreads) {
    const int i = idx % kb, j = idx / kb;
    if (i >= j) Bd[i + (size_t)j * ld] = A[i + j * kLdD];
  }
  __syncthreads();
  // triangular inverse in place (LAPACK dtrti2 'L' order: columns from the last one)
  __shared__ double tmp[kNB];
  for (int j = kb - 1; j >= 0; --j) {
    const double ajj = 1.0 / A[j + j * kLdD];
    // x = T * A[j+1:, j] with T = already inverted trailing block, then scale by -ajj
    for (int i = j + 1 + tid; i < kb; i += kDiagThreads) {
      double s = 0.0;
      for (int t = j + 1; t <= i; ++t) s += A[i + t * kLdD] * A[t + j * kLdD];
      tmp[i] = -ajj * s;
    }
    __syncthreads();
    for (int i = j + 1 + tid; i < kb; i += kDiagThreads) A[i + j * kLdD] = tmp[i];
    if (tid == 0) A[j + j * kLdD] = ajj;
    __syncthreads();
  }
  for (int idx = tid; idx < kNB * kNB; idx += kDiagThreads) {
    const int i = idx % kNB, j = idx / kNB;
    Linv[idx] = (i < kb && j < kb && i >= j) ? A[i + j * kLdD] : 0.0;
  }
}

// ------------------------------------------------------------------ tensor-core GEMM (C op= A B^T)
struct GemmArgs {
  const double* A;  // element (i, kk) at A[i + kk*lda], i relative to the tile-row base
  int64_t lda;
  const double* Bm;  // element (j, kk) at Bm[j + kk*ldbm]
  int64_t ldbm;
  double* C;  // element (i, j) at C[i + j*ldc]
  int64_t ldc;
  int rows;   // valid rows of A (and of B for SYRK) from base 0
  int cols;   // valid rows of B (TRSM: kb)
  int K;
  const int32_t* err;
};

template <bool SYRK, bool AL16>
__global__ void __launch_bounds__(kGemmThreads, 1) gemm_nt_kernel(GemmArgs g) {
  if (*g.err != kNoError) return;
  extern __shared__ double sm[];
  double* As = sm;                                  // [kStages][kBK][kLdS]
  double* Bs = sm + kStages * kBK * kLdS;           // [kStages][kBK][kLdS]
  int bi, bj;
  if (SYRK) {
    const int t = blockIdx.x;
    bi = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while (bi * (bi + 1) / 2 > t) --bi;
    while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
    bj = t - bi * (bi + 1) / 2;
  } else {
    bi = blockIdx.x;
    bj = 0;
  }
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int wm = wid >> 2, wn = wid & 3;  // 2 x 4 warps, warp tile 64 x 32
  const int g8 = lane >> 2, t4 = lane & 3;
  const int rowA0 = bi * kTile, rowB0 = bj * kTile;
  const int rowsB = SYRK ? g.rows : g.cols;
  const double* Ab = g.A + rowA0;
  const double* Bb = g.Bm + rowB0;

  auto load_stage = [&](int stage, int k0) {
    double* as = As + stage * kBK * kLdS;
    double* bs = Bs + stage * kBK * kLdS;
    if (AL16) {
#pragma unroll
      for (int q = 0; q < (kBK * kTile / 2) / kGemmThreads; ++q) {  // 16B chunks: 2 rows of one column
        const int cid = tid + q * kGemmThreads;
        const int kk = cid / (kTile / 2), rp = (cid % (kTile / 2)) * 2;
        const bool kv = (k0 + kk) < g.K;
        const bool va = kv && (rowA0 + rp) < g.rows;
        cp_async16(as + kk * kLdS + rp, va ? Ab + rp + (size_t)(k0 + kk) * g.lda : g.A, va);
        const bool vb = kv && (rowB0 + rp) < rowsB;
        cp_async16(bs + kk * kLdS + rp, vb ? Bb + rp + (size_t)(k0 + kk) * g.ldbm : g.Bm, vb);
      }
    } else {
#pragma unroll
      for (int q = 0; q < (kBK * kTile) / kGemmThreads; ++q) {  // 8B elements
        const int cid = tid + q * kGemmThreads;
        const int kk = cid / kTile, rp = cid % kTile;
        const bool kv = (k0 + kk) < g.K;
        const bool va = kv && (rowA0 + rp) < g.rows;
        cp_async8(as + kk * kLdS + rp, va ? Ab + rp + (size_t)(k0 + kk) * g.lda : g.A, va);
        const bool vb = kv && (rowB0 + rp) < rowsB;
        cp_async8(bs + kk * kLdS + rp, vb ? Bb + rp + (size_t)(k0 + kk) * g.ldbm : g.Bm, vb);
      }
    }
  };

  double acc[8][4][2];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  const int nk = (g.K + kBK - 1) / kBK;
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nk) load_stage(s, s * kBK);
    cp_async_commit();
  }
  for (int kc = 0; kc < nk; ++kc) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    const int nxt = kc + kStages - 1;
    if (nxt < nk) load_stage(nxt % kStages, nxt * kBK);
    cp_async_commit();
    const double* as = As + (kc % kStages) * kBK * kLdS;
    const double* bs = Bs + (kc % kStages) * kBK * kLdS;
#pragma unroll
    for (int k4 = 0; k4 < kBK / 4; ++k4) {
      double af[8], bf[4];
#pragma unroll
      for (int a = 0; a < 8; ++a) af[a] = as[(k4 * 4 + t4) * kLdS + wm * 64 + a * 8 + g8];
#pragma unroll
      for (int b = 0; b < 4; ++b) bf[b] = bs[(k4 * 4 + t4) * kLdS + wn * 32 + b * 8 + g8];
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
  }
  cp_async_wait<0>();

  // epilogue
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    const int i = rowA0 + wm * 64 + a * 8 + g8;
    if (i >= g.rows) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = rowB0 + wn * 32 + b * 8 + 2 * t4 + e;
        if (SYRK) {
          if (j < g.rows && i >= j) g.C[i + (size_t)j * g.ldc] -= acc[a][b][e];
        } else {
          if (j < g.cols) g.C[i + (size_t)j * g.ldc] = acc[a][b][e];
        }
      }
    }
  }
}

static size_t gemm_smem() { return (size_t)2 * kStages * kBK * kLdS * sizeof(double); }

int potrf_lower(sdpc_ctx* h, double* B, int64_t m, int64_t ld, int32_t* d_err, cudaStream_t st, double* flops_upd,
                int* n_upd) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(potrf_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(gemm_nt_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gemm_smem());
    cudaFuncSetAttribute(gemm_nt_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gemm_smem());
    cudaFuncSetAttribute(gemm_nt_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gemm_smem());
    cudaFuncSetAttribute(gemm_nt_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gemm_smem());
    attr = true;
  }
  const bool al16 = (ld % 2 == 0) && ((reinterpret_cast<uintptr_t>(B) & 15) == 0);
  int launches = 0;
  double fl = 0.0;
  int nu = 0;
  const bool tim = h && h->timing;
  for (int64_t k0 = 0; k0 < m; k0 += kNB) {
    const int kb = (int)std::min<int64_t>(kNB, m - k0);
    potrf_diag_kernel<<<1, kDiagThreads, (size_t)kb * kLdD * sizeof(double), st>>>(B, ld, (int)k0, kb,
                                                                                 h->potrf_ws, d_err);
    ++launches;
    const int64_t base = k0 + kb;
    const int rows = (int)(m - base);
    if (rows <= 0) break;
    GemmArgs g{};
    g.A = B + base + (size_t)k0 * ld;
    g.lda = ld;
    g.Bm = h->potrf_ws;
    g.ldbm = kNB;
    g.C = B + base + (size_t)k0 * ld;
    g.ldc = ld;
    g.rows = rows;
    g.cols = kb;
    g.K = kb;
    g.err = d_err;
    const int T = (rows + kTile - 1) / kTile;
    if (al16) gemm_nt_kernel<false, true><<<T, kGemmThreads, gemm_smem(), st>>>(g);
    else gemm_nt_kernel<false, false><<<T, kGemmThreads, gemm_smem(), st>>>(g);
    ++launches;
    GemmArgs u = g;
    u.Bm = B + base + (size_t)k0 * ld;
    u.ldbm = ld;
    u.C = B + base + (size_t)base * ld;
    if (tim) {
      if ((int)h->upd_ev.size() < 2 * (nu + 1)) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        h->upd_ev.push_back(e0);
        h->upd_ev.push_back(e1);
      }
      cudaEventRecord(h->upd_ev[2 * nu], st);
    }
    if (al16) gemm_nt_kernel<true, true><<<T * (T + 1) / 2, kGemmThreads, gemm_smem(), st>>>(u);
    else gemm_nt_kernel<true, false><<<T * (T + 1) / 2, kGemmThreads, gemm_smem(), st>>>(u);
    if (tim) cudaEventRecord(h->upd_ev[2 * nu + 1], st);
    ++launches;
    ++nu;
    fl += (double)rows * (double)(rows + 1) * (double)kb;
  }
  if (flops_upd) *flops_upd = fl;
  if (n_upd) *n_upd = nu;
  return launches;
}

}  // namespace sdpc
