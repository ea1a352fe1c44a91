// (d) Dense FP64 Cholesky of the SCM, B = R R^T (lower, in place).
// PAPER.md P:711-713 / P:735-736 / P:978-979 (type (i): LAPACK dense Cholesky with multithreaded BLAS).
//
// Blocked right-looking, nb = 128, with depth-1 lookahead on a second stream.  Per panel step k:
//   diag(k)   : one CTA (512 threads) factors the 128 x 128 diagonal block in shared memory
//               (32-column panels, one barrier per column, register-tiled panel updates) and forms
//               L11^{-1} (blocked by 32) for the TRSM;
//   trsm(k)   : L21 = A21 L11^{-T} as an FP64 tensor-core GEMM with the explicit inverse;
//   ucol(k)   : trailing update of block column k+1 only (one column of 128 x 128 tiles);
//   diag(k+1), trsm(k+1) run on the side stream while
//   urest(k)  : the rest of the trailing update A22 -= L21 L21^T runs on the main stream.
// GEMMs: mma.sync m8n8k4 f64 (DMMA.8x8x4 on sm_100a; tcgen05 has no f64 kind), 128 x 128 CTA tiles,
// 8 warps x (64 x 32), operands staged in shared memory by a 3-stage cp.async pipeline.
// Non-PD: the first failing column (1-based, LAPACK potrf rule) is atomicMin'ed into *err and every
// later kernel exits at entry.
#include <cuda_runtime.h>

#include <cmath>
#include <vector>

#include "common.cuh"
#include "ctx.hpp"

namespace sdpc {

constexpr int kNB = 128;         // panel width
constexpr int kTile = 128;       // GEMM tile (BM = BN)
constexpr int kBK = 16;          // k-chunk per pipeline stage
constexpr int kStages = 3;
constexpr int kLdS = kTile + 4;  // smem row stride (doubles): conflict-free fragment loads
constexpr int kGemmThreads = 256;

// ------------------------------------------------------------------ diagonal block
constexpr int kDiagThreads = 256;
constexpr int kLdD = kNB + 1;  // A[i + j*kLdD]

__global__ void __launch_bounds__(kDiagThreads, 1) potrf_diag_kernel(double* B, int64_t ld, int k0, int kb,
                                                                  double* Linv, int32_t* err) {
  if (*err != kNoError) return;
  extern __shared__ double sm[];
  double* A = sm;                  // 128 x 128 (ld 129): lower = L, upper = L^{-T}
  // current 32-column panel, scaled (P[k][i] = L[i, jb+k]), and scratch for the inverse blocks
  double (*P)[kNB] = reinterpret_cast<double (*)[kNB]>(sm + kNB * kLdD);
  double (*T)[32][33] = reinterpret_cast<double (*)[32][33]>(sm + kNB * kLdD + 32 * kNB);
  __shared__ double dL[kNB];
  const int tid = threadIdx.x;
  double* Bd = B + k0 + (size_t)k0 * ld;
  for (int idx = tid; idx < kNB * kNB; idx += kDiagThreads) {
    const int i = idx % kNB, j = idx / kNB;
    double v = 0.0;
    if (i < kb && j < kb) v = i >= j ? Bd[i + (size_t)j * ld] : 0.0;
    else if (i == j) v = 1.0;  // identity padding beyond kb
    A[i + j * kLdD] = v;
  }
  __syncthreads();
  // 32-column panels.  (1) warp 0 factors the 32 x 32 diagonal sub-block in registers (lane = row,
  // shuffles, rsqrt) and inverts it (lane = column, broadcast reads); (2) all threads form the panel
  // rows below with that inverse; (3) register-tiled trailing update.
  __shared__ double inv32[32][33];
  __shared__ int fail_col;
  const int lane = tid & 31, wid = tid >> 5;
#pragma unroll 1
  for (int jb = 0; jb < kNB; jb += 32) {
    if (wid == 0) {
      // factor the 32 x 32 block in place in shared memory: lane = row jb+lane
      double* Ab = A + jb + jb * kLdD;  // Ab[i + k*kLdD]
      int fail = -1;
      double rdiag = 0.0;
      for (int j = 0; j < 32; ++j) {
        const double d = Ab[j + j * kLdD];
        if (!(d > 0.0)) {  // uniform across the warp
          fail = j;
          break;
        }
        const double r = rsqrt(d);
        const double l = Ab[lane + j * kLdD] * r;
        if (lane == j) rdiag = r;
        __syncwarp();
        if (lane >= j) Ab[lane + j * kLdD] = l;
        __syncwarp();
        if (lane > j) {
#pragma unroll 4
          for (int k = j + 1; k <= lane; ++k) Ab[lane + k * kLdD] -= l * Ab[k + j * kLdD];
        }
        __syncwarp();
      }
      if (lane == 0) fail_col = fail;
      if (fail < 0) {
        // inverse: lane = column c; x_i = (delta_ic - sum_{k<i} L[i][k] x_k) / L[i][i]
        for (int i = 0; i < 32; ++i) {
          double sacc = (i == lane) ? 1.0 : 0.0;
          for (int k = lane; k < i; ++k) sacc -= Ab[i + k * kLdD] * inv32[k][lane];
          inv32[i][lane] = (i >= lane) ? sacc * __shfl_sync(0xffffffffu, rdiag, i) : 0.0;
          __syncwarp();
        }
      }
    }
    __syncthreads();
    if (fail_col >= 0) {
      if (tid == 0) report_error(err, k0 + jb + fail_col + 1);
      return;
    }
    const int r0 = jb + 32, nr = kNB - r0;
    if (nr > 0) {
      // panel rows below: L[i, jb+c] = sum_{k>=c} A[i, jb+k] Linv[c][k]... (L21 = A21 L11^{-T})
      for (int idx = tid; idx < nr * 32; idx += kDiagThreads) {
        const int i = r0 + (idx & 31) + (idx >> 10) * 32, c = (idx >> 5) & 31;
        double acc = 0.0;
#pragma unroll 8
        for (int k = 0; k <= 31; ++k) acc += A[i + (jb + k) * kLdD] * inv32[c][k];
        P[c][i] = acc;
      }
      __syncthreads();
      for (int idx = tid; idx < nr * 32; idx += kDiagThreads) {
        const int c = idx / nr, i = r0 + idx % nr;
        A[i + (jb + c) * kLdD] = P[c][i];
      }
      // trailing update of rows/cols >= r0 with the panel: 4 x 4 register tiles
      const int nb4 = nr / 4;
      const int ntile = nb4 * (nb4 + 1) / 2;
      for (int t = tid; t < ntile; t += kDiagThreads) {
        int bi = (int)((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
        while (bi * (bi + 1) / 2 > t) --bi;
        while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
        const int bj = t - bi * (bi + 1) / 2;
        const int i0 = r0 + 4 * bi, j0 = r0 + 4 * bj;
        double acc[4][4] = {};
#pragma unroll 8
        for (int k = 0; k < 32; ++k) {
          double pi[4], pj[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            pi[q] = P[k][i0 + q];
            pj[q] = P[k][j0 + q];
          }
#pragma unroll
          for (int a2 = 0; a2 < 4; ++a2)
#pragma unroll
            for (int b2 = 0; b2 < 4; ++b2) acc[a2][b2] += pi[a2] * pj[b2];
        }
#pragma unroll
        for (int a2 = 0; a2 < 4; ++a2)
#pragma unroll
          for (int b2 = 0; b2 < 4; ++b2)
            if (i0 + a2 >= j0 + b2) A[(i0 + a2) + (j0 + b2) * kLdD] -= acc[a2][b2];
      }
    }
    __syncthreads();
  }
  for (int idx = tid; idx < kb * kb; idx += kDiagThreads) {
    const int i = idx % kb, j = idx / kb;
    if (i >= j) Bd[i + (size_t)j * ld] = A[i + j * kLdD];
  }
  // L^{-1}, kept transposed in A's upper triangle: Linv[i][j] at A[j + i*ld] (i >= j).
  // (1) the four 32 x 32 diagonal blocks: thread (I, c) forward-substitutes column c of block I;
  // (2) off-diagonal blocks by distance d = I - J: Linv[I,J] = -Linv[I,I] sum_{K=J}^{I-1} L[I,K] Linv[K,J].
  if (tid < kNB) dL[tid] = A[tid + tid * kLdD];
  __syncthreads();
  if (tid < kNB) {
    const int I = tid >> 5, c = tid & 31, o = I * 32;
    double* xr = A + (o + c);  // Linv[o+i][o+c] at xr[(o+i) * kLdD]
    xr[(o + c) * kLdD] = 1.0 / dL[o + c];
    for (int i = c + 1; i < 32; ++i) {
      double s0 = 0.0, s1 = 0.0;
      int k = c;
      for (; k + 1 < i; k += 2) {
        s0 += A[(o + i) + (o + k) * kLdD] * xr[(o + k) * kLdD];
        s1 += A[(o + i) + (o + k + 1) * kLdD] * xr[(o + k + 1) * kLdD];
      }
      if (k < i) s0 += A[(o + i) + (o + k) * kLdD] * xr[(o + k) * kLdD];
      xr[(o + i) * kLdD] = -(s0 + s1) / dL[o + i];
    }
  }
  __syncthreads();
  for (int d = 1; d < 4; ++d) {
    const int npair = 4 - d;
    for (int idx = tid; idx < npair * 1024; idx += kDiagThreads) {
      const int p = idx >> 10, e = idx & 1023, a = e & 31, b = e >> 5;
      const int J = p, I = p + d;
      double acc0 = 0.0, acc1 = 0.0;
      // K == J: Linv[J,J] is lower, so only k >= b contributes (the rest of that storage is L)
      for (int k = b; k < 32; ++k) acc0 += A[(I * 32 + a) + (J * 32 + k) * kLdD] * A[(J * 32 + b) + (J * 32 + k) * kLdD];
      for (int K = J + 1; K < I; ++K)
#pragma unroll 8
        for (int k = 0; k < 32; k += 2) {
          acc0 += A[(I * 32 + a) + (K * 32 + k) * kLdD] * A[(J * 32 + b) + (K * 32 + k) * kLdD];
          acc1 += A[(I * 32 + a) + (K * 32 + k + 1) * kLdD] * A[(J * 32 + b) + (K * 32 + k + 1) * kLdD];
        }
      T[p][a][b] = acc0 + acc1;
    }
    __syncthreads();
    for (int idx = tid; idx < npair * 1024; idx += kDiagThreads) {
      const int p = idx >> 10, e = idx & 1023, a = e & 31, b = e >> 5;
      const int J = p, I = p + d;
      double acc = 0.0;
      for (int k = 0; k <= a; ++k) acc -= A[(I * 32 + k) + (I * 32 + a) * kLdD] * T[p][k][b];
      A[(J * 32 + b) + (I * 32 + a) * kLdD] = acc;
    }
    __syncthreads();
  }
  for (int idx = tid; idx < kNB * kNB; idx += kDiagThreads) {
    const int i = idx % kNB, j = idx / kNB;
    Linv[idx] = (i < kb && j < kb && i >= j) ? A[j + i * kLdD] : 0.0;
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

enum { kModeTrsm = 0, kModeSyrkAll = 1, kModeSyrkCol = 2, kModeSyrkRest = 3 };

template <int MODE, bool AL16>
__global__ void __launch_bounds__(kGemmThreads, 1) gemm_nt_kernel(GemmArgs g) {
  if (*g.err != kNoError) return;
  extern __shared__ double sm[];
  double* As = sm;                         // [kStages][kBK][kLdS]
  double* Bs = sm + kStages * kBK * kLdS;  // [kStages][kBK][kLdS]
  int bi, bj;
  if (MODE == kModeSyrkAll || MODE == kModeSyrkRest) {
    const int t = blockIdx.x;
    bi = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while (bi * (bi + 1) / 2 > t) --bi;
    while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
    bj = t - bi * (bi + 1) / 2;
    if (MODE == kModeSyrkRest) {
      ++bi;
      ++bj;
    }
  } else {
    bi = blockIdx.x;
    bj = 0;
  }
  constexpr bool SYRK = MODE != kModeTrsm;
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

  // epilogue.  SYRK: C -= acc with all loads of a half-tile issued before any store (the
  // compiler cannot reorder them itself because C's loads and stores may alias).
  if (SYRK) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double cold[4][4][2];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int i = rowA0 + wm * 64 + (h * 4 + a) * 8 + g8;
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int j = rowB0 + wn * 32 + b * 8 + 2 * t4 + e;
            cold[a][b][e] = (i < g.rows && j < g.rows && i >= j) ? g.C[i + (size_t)j * g.ldc] : 0.0;
          }
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int i = rowA0 + wm * 64 + (h * 4 + a) * 8 + g8;
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int j = rowB0 + wn * 32 + b * 8 + 2 * t4 + e;
            if (i < g.rows && j < g.rows && i >= j) g.C[i + (size_t)j * g.ldc] = cold[a][b][e] - acc[h * 4 + a][b][e];
          }
      }
    }
  } else {
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      const int i = rowA0 + wm * 64 + a * 8 + g8;
      if (i >= g.rows) continue;
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int j = rowB0 + wn * 32 + b * 8 + 2 * t4 + e;
          if (j < g.cols) g.C[i + (size_t)j * g.ldc] = acc[a][b][e];
        }
    }
  }
}

static size_t gemm_smem() { return (size_t)2 * kStages * kBK * kLdS * sizeof(double); }
static size_t diag_smem() { return ((size_t)kNB * kLdD + 32 * kNB + 3 * 32 * 33) * sizeof(double); }

template <int MODE>
static void launch_gemm(bool al16, int grid, const GemmArgs& g, cudaStream_t st) {
  if (grid <= 0) return;
  if (al16) gemm_nt_kernel<MODE, true><<<grid, kGemmThreads, gemm_smem(), st>>>(g);
  else gemm_nt_kernel<MODE, false><<<grid, kGemmThreads, gemm_smem(), st>>>(g);
}

template <int MODE>
static void set_gemm_attr() {
  cudaFuncSetAttribute(gemm_nt_kernel<MODE, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gemm_smem());
  cudaFuncSetAttribute(gemm_nt_kernel<MODE, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gemm_smem());
}

int potrf_lower(sdpc_ctx* h, double* B, int64_t m, int64_t ld, int32_t* d_err, cudaStream_t st, double* flops_upd,
                int* n_upd) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(potrf_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)diag_smem());
    set_gemm_attr<kModeTrsm>();
    set_gemm_attr<kModeSyrkAll>();
    set_gemm_attr<kModeSyrkCol>();
    set_gemm_attr<kModeSyrkRest>();
    attr = true;
  }
  if (!h->st2) {
    cudaStreamCreateWithFlags(&h->st2, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&h->evA, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&h->evB, cudaEventDisableTiming);
  }
  cudaStream_t s2 = h->st2;
  const bool al16 = (ld % 2 == 0) && ((reinterpret_cast<uintptr_t>(B) & 15) == 0);
  const bool tim = h->timing;
  int launches = 0;
  double fl = 0.0;
  int nu = 0;
  const int64_t nsteps = (m + kNB - 1) / kNB;
  auto panel = [&](int64_t k, cudaStream_t s) {  // diag(k) + trsm(k)
    const int64_t k0 = k * kNB;
    const int kb = (int)std::min<int64_t>(kNB, m - k0);
    double* Lw = h->potrf_ws + (k & 1) * kNB * kNB;
    potrf_diag_kernel<<<1, kDiagThreads, diag_smem(), s>>>(B, ld, (int)k0, kb, Lw, d_err);
    ++launches;
    const int64_t base = k0 + kb;
    const int rows = (int)(m - base);
    if (rows <= 0) return;
    GemmArgs g{};
    g.A = B + base + (size_t)k0 * ld;
    g.lda = ld;
    g.Bm = Lw;
    g.ldbm = kNB;
    g.C = B + base + (size_t)k0 * ld;
    g.ldc = ld;
    g.rows = rows;
    g.cols = kb;
    g.K = kb;
    g.err = d_err;
    launch_gemm<kModeTrsm>(al16, (rows + kTile - 1) / kTile, g, s);
    ++launches;
  };
  panel(0, st);
  for (int64_t k = 0; k < nsteps; ++k) {
    const int64_t k0 = k * kNB;
    const int kb = (int)std::min<int64_t>(kNB, m - k0);
    const int64_t base = k0 + kb;
    const int rows = (int)(m - base);
    if (rows <= 0) break;
    GemmArgs u{};
    u.A = B + base + (size_t)k0 * ld;
    u.lda = ld;
    u.Bm = u.A;
    u.ldbm = ld;
    u.C = B + base + (size_t)base * ld;
    u.ldc = ld;
    u.rows = rows;
    u.cols = kb;
    u.K = kb;
    u.err = d_err;
    const int T = (rows + kTile - 1) / kTile;
    // block column k+1 first, then hand the next panel to the side stream
    launch_gemm<kModeSyrkCol>(al16, T, u, st);
    ++launches;
    cudaEventRecord(h->evA, st);
    cudaStreamWaitEvent(s2, h->evA, 0);
    panel(k + 1, s2);
    cudaEventRecord(h->evB, s2);
    if (T > 1) {
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
      launch_gemm<kModeSyrkRest>(al16, (T - 1) * T / 2, u, st);
      if (tim) cudaEventRecord(h->upd_ev[2 * nu + 1], st);
      ++launches;
      ++nu;
      const double r2 = (double)(rows - kTile);
      fl += r2 * (r2 + 1.0) * (double)kb;
    }
    cudaStreamWaitEvent(st, h->evB, 0);
  }
  if (flops_upd) *flops_upd = fl;
  if (n_upd) *n_upd = nu;
  return launches;
}

}  // namespace sdpc
