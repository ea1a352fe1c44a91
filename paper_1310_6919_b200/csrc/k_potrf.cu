// (d) Dense FP64 Cholesky of the SCM, B = R R^T (lower, in place): the multi-launch schedule and the tile
// kernels.  PAPER.md P:711-713 / P:735-736 / P:978-979 (type (i): dense Cholesky with multithreaded BLAS).
// The default one-GPU path is the persistent task-graph kernel of k_chol_dag.cu; this file serves
//   * potrf_lower: the fallback when B cannot be staged with 16-byte copies (odd ld or unaligned B), the
//     tile potrf of the distributed schedule (n <= 256, also returning the 128-block inverses), and
//     sdpc_set_cholesky_schedule(h, 0);
//   * trsm_panel / update_tiles: the panel solve and local trailing update of the distributed Cholesky
//     (dist_chol.cu and the sdpc_trsm_panel / sdpc_update_tiles entries).
// potrf_lower: blocked right-looking, outer block 256 (two 128 sub-panels, so the trailing updates run with
// K = 256), depth-2 lookahead: a high-priority stream carries the critical path (update of the next block
// column, then the next panel: diag -> trsm -> sub-panel update -> diag -> trsm) and the main stream the
// bulk trailing update.
//   diag : one CTA (256 threads) factors a 128 x 128 diagonal block in shared memory (32-column warp
//          factorisations, DMMA panel rows / trailing update / off-diagonal blocks of L^{-1});
//   trsm : L21 = A21 L11^{-T} with the explicit inverse, 64-row x 128-column tiles, 8 warps x (32 x 32),
//          2 CTAs/SM, in place;
//   gemm : trailing updates C -= A B^T on 128 x 64 tiles, 8 warps x (32 x 32) DMMA, 2 CTAs/SM, 16-deep
//          k-chunks in a 4-stage cp.async pipeline, accumulators starting from C.
// GEMMs: mma.sync m8n8k4 f64 (DMMA.8x8x4 on sm_100a; tcgen05 has no f64 kind).
// Non-PD: the first failing column (1-based, LAPACK potrf rule) is atomicMin'ed into *err and every
// later kernel exits at entry.
#include <cuda_runtime.h>

#include <cmath>
#include <vector>

#include "common.cuh"
#include "ctx.hpp"

namespace sdpc {

constexpr int kNB = 128;         // panel width
constexpr int kTile = 128;        // GEMM tile rows (BM); also the row/column unit of the tile grids
constexpr int kBN = 64;           // GEMM tile columns (64: 2 CTAs/SM of 8 warps; 128: 1 CTA/SM of 16 warps)
constexpr int kR = kTile / kBN;   // GEMM column tiles per 128-column unit
constexpr int kBK = 16;           // k-chunk per pipeline stage (4 DMMA k-steps per barrier)
constexpr int kStages = 4;
constexpr int kLdA = kTile + 4;   // smem row strides (doubles): conflict-free fragment loads
constexpr int kLdB = kBN + 4;
constexpr int kWM = 32;           // update-GEMM warp tile rows (warp tile kWM x 32; 64 x 32 with 4 warps
                                  // per CTA measured 25.2 vs 26.0 TF/s)
constexpr int kWA = kWM / 8;      // A fragments per warp and k-step
constexpr int kGemmThreads = 32 * (kTile / kWM) * (kBN / 32);  // (128/kWM) x (kBN/32) warps
constexpr int kGemmCtasPerSm = kBN == 64 ? 2 : 1;
constexpr int kTrsmThreads = 256;  // in-place panel solve: 8 warps x (32 x 32)
// (a persistent bulk-update grid leaving 6 SMs free for the lookahead stream was measured slower:
// 19.3 vs 17.5 ms on configs[1]; the update launches one CTA per tile)

__device__ __forceinline__ double neg(double x) {  // sign flip on the integer pipe
  return __hiloint2double(__double2hiint(x) ^ 0x80000000, __double2loint(x));
}

// ------------------------------------------------------------------ diagonal block
constexpr int kDiagThreads = 256;
constexpr int kLdD = kNB + 4;  // A[i + j*kLdD]; +4 makes the m8n8k4 fragment loads conflict-free

// Warp-level Cholesky + inverse of a 32 x 32 SPD block (lane = row, the row in registers, columns
// broadcast by shuffles; every shuffle is executed by all 32 lanes).  In: Ab (shared, ld kLdD),
// lower part.  Out: Ab lower <- L11; Tinv[i][c] (shared, 32 x 33) <- (L11^{-1})[i][c] (zero above).
// Returns the failing local column or -1 (uniform over the warp).
__device__ __noinline__ int warp_chol_inv32(double* Ab, double (*Tinv)[33], int lane) {
  double row[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) row[c] = c <= lane ? Ab[lane + c * kLdD] : 0.0;
  int fail = -1;
  double rinv = 0.0;  // lane j: 1 / L[j][j]
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const double d = __shfl_sync(0xffffffffu, row[j], j);
    if (fail < 0 && !(d > 0.0)) fail = j;
    const double rl = rsqrt_nr(d);  // MUFU seed + Newton: no out-of-line slow path on the chain
    if (lane == j) {
      row[j] = d * rl;
      rinv = rl;
    } else if (lane > j) {
      row[j] *= rl;
    }
#pragma unroll
    for (int k = j + 1; k < 32; ++k) {
      const double lkj = __shfl_sync(0xffffffffu, row[j], k);
      if (lane >= k) row[k] -= row[j] * lkj;
    }
  }
  if (fail >= 0) return fail;
#pragma unroll
  for (int c = 0; c < 32; ++c)
    if (c <= lane) Ab[lane + c * kLdD] = row[c];
  __syncwarp();
  // inverse, lane = column c, right-looking (column-oriented) forward substitution: at step i,
  // x_i is final; it updates every x_k, k > i, independently (ILP across k instead of one serial
  // dot-product chain per row)
  double x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = (i == lane) ? 1.0 : 0.0;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    x[i] *= __shfl_sync(0xffffffffu, rinv, i);
#pragma unroll
    for (int k = i + 1; k < 32; ++k) x[k] -= Ab[k + i * kLdD] * x[i];
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) Tinv[i][lane] = i >= lane ? x[i] : 0.0;
  return -1;
}

// One warp: acc (8 x 8 tile, m8n8k4 accumulator layout) += sum_{kk < K} Aop(r0 + row, kk) Bop(c0 + col, kk)
// with Aop(i, kk) = Ap[i * as_i + kk * as_k], Bop(j, kk) = Bp[j * bs_j + kk * bs_k] (shared memory).
__device__ __forceinline__ void warp_mma8(double& c0, double& c1, const double* Ap, int as_i, int as_k,
                                          const double* Bp, int bs_j, int bs_k, int K, bool negA, int lane) {
  const int g8 = lane >> 2, t4 = lane & 3;
  const double* ap = Ap + g8 * as_i + t4 * as_k;
  const double* bp = Bp + g8 * bs_j + t4 * bs_k;
#pragma unroll 4
  for (int k0 = 0; k0 < K; k0 += 4) {
    const double av = ap[k0 * as_k];
    dmma_8x8x4(c0, c1, negA ? neg(av) : av, bp[k0 * bs_k]);
  }
}

// Factor the 128 x 128 diagonal block B[k0.., k0..] (kb <= 128 valid, identity-padded) in shared
// memory and form L11^{-1} for the panel solve.  32-column panels: warp 0 factors + inverts the
// 32 x 32 diagonal block in registers; the panel rows below (P = A21 L11^{-T}) and the trailing
// update (A22 -= P P^T) run on the FP64 tensor cores (m8n8k4 DMMA, fragments from shared memory),
// as do the off-diagonal blocks of L^{-1}.
__global__ void __launch_bounds__(kDiagThreads, 1) potrf_diag_kernel(double* B, int64_t ld, int k0, int kb,
                                                                  double* Linv, int32_t* err) {
  if (*err != kNoError) return;
  extern __shared__ double sm[];
  double* A = sm;  // 128 x 128 (ld kLdD): lower = L, upper = L^{-T}
  double* P = sm + kNB * kLdD;  // panel scratch, P[c * kLdD + r] = L[r, jb + c] (32 columns)
  double (*T)[32][33] = reinterpret_cast<double (*)[32][33]>(sm + kNB * kLdD + 32 * kLdD);  // [3]
  __shared__ double Dinv[4][32][33];  // inverses of the four 32 x 32 diagonal blocks
  __shared__ int fail_col;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int g8 = lane >> 2, t4 = lane & 3;
  double* Bd = B + k0 + (size_t)k0 * ld;
  // load the lower triangle, 16 independent loads in flight per thread
  for (int base = 0; base < kNB * kNB; base += 16 * kDiagThreads) {
    double v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int idx = base + q * kDiagThreads + tid;
      const int i = idx % kNB, j = idx / kNB;
      v[q] = (i < kb && j < kb && i >= j) ? Bd[i + (size_t)j * ld] : ((i == j && i >= kb) ? 1.0 : 0.0);
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int idx = base + q * kDiagThreads + tid;
      A[idx % kNB + (idx / kNB) * kLdD] = v[q];
    }
  }
  __syncthreads();
#pragma unroll 1
  for (int jb = 0; jb < kNB; jb += 32) {
    if (wid == 0) {
      const int f = warp_chol_inv32(A + jb + jb * kLdD, Dinv[jb >> 5], lane);
      if (lane == 0) fail_col = f;
    }
    __syncthreads();
    if (fail_col >= 0) {
      if (tid == 0) report_error(err, k0 + jb + fail_col + 1);
      return;
    }
    const int r0 = jb + 32, nr = kNB - r0;
    if (nr > 0) {
      // P(r, c) = sum_k A(r, jb+k) Linv11(c, k): (nr/8) x 4 tiles of 8 x 8, K = 32
      const double* Iv = &Dinv[jb >> 5][0][0];
      const int ntile = (nr / 8) * 4;
      for (int t = wid; t < ntile; t += kDiagThreads / 32) {
        const int tr = t >> 2, tc = t & 3;
        double c0 = 0.0, c1 = 0.0;
        warp_mma8(c0, c1, A + (r0 + tr * 8) + jb * kLdD, 1, kLdD, Iv + tc * 8 * 33, 33, 1, 32, false, lane);
        const int r = r0 + tr * 8 + g8, c = tc * 8 + 2 * t4;
        P[c * kLdD + r] = c0;
        P[(c + 1) * kLdD + r] = c1;
      }
      __syncthreads();
      // panel back into A (its columns are not touched by the update) and the trailing update
      for (int idx = tid; idx < nr * 32; idx += kDiagThreads) {
        const int c = idx / nr, r = r0 + idx % nr;
        A[r + (jb + c) * kLdD] = P[c * kLdD + r];
      }
      // A22 -= P P^T on the 8 x 8 tiles (ti >= tj) of rows/cols r0..127 (the strict upper part of
      // the diagonal tiles is scratch: overwritten by L^{-T} below, never read as L)
      const int nb8 = nr / 8, nt2 = nb8 * (nb8 + 1) / 2;
      for (int t = wid; t < nt2; t += kDiagThreads / 32) {
        int ti = (int)((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
        while (ti * (ti + 1) / 2 > t) --ti;
        while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
        const int tj = t - ti * (ti + 1) / 2;
        const int i0 = r0 + ti * 8, j0 = r0 + tj * 8;
        double* Cp = A + (i0 + g8) + (j0 + 2 * t4) * kLdD;
        double c0 = Cp[0], c1 = Cp[kLdD];
        warp_mma8(c0, c1, P + i0, 1, kLdD, P + j0, 1, kLdD, 32, true, lane);
        Cp[0] = c0;
        Cp[kLdD] = c1;
      }
    }
    __syncthreads();
  }
  for (int idx = tid; idx < kb * kb; idx += kDiagThreads) {
    const int i = idx % kb, j = idx / kb;
    if (i >= j) Bd[i + (size_t)j * ld] = A[i + j * kLdD];
  }
  __syncthreads();  // the upper triangle (and diagonal) of A is overwritten below with L^{-T}
  // L^{-1}, kept transposed in A's upper triangle: Linv[i][j] at A[j + i*ld] (i >= j).
  // (1) the diagonal blocks from the warp factorisations; (2) off-diagonal blocks by distance
  // d = I - J: T = sum_{K=J}^{I-1} L[I,K] Linv[K,J]; Linv[I,J] = -Linv[I,I] T (DMMA 8 x 8 tiles).
  for (int idx = tid; idx < 4 * 1024; idx += kDiagThreads) {
    const int I = idx >> 10, e = idx & 1023, r = e & 31, c = e >> 5;
    if (r >= c) A[(I * 32 + c) + (I * 32 + r) * kLdD] = Dinv[I][r][c];
  }
  __syncthreads();
  for (int d = 1; d < 4; ++d) {
    const int npair = 4 - d;
    for (int t = wid; t < npair * 16; t += kDiagThreads / 32) {
      const int pp = t >> 4, tr = (t >> 2) & 3, tc = t & 3;
      const int J = pp, I = pp + d;
      double c0 = 0.0, c1 = 0.0;
      // K = J: Linv[J,J] from Dinv (lower); Bop(b, k) = Dinv[J][k][b]
      warp_mma8(c0, c1, A + (I * 32 + tr * 8) + (J * 32) * kLdD, 1, kLdD, &Dinv[J][0][tc * 8], 1, 33, 32, false,
                lane);
      for (int K = J + 1; K < I; ++K)  // Bop(b, k) = Linv[K32+k][J32+b] = A[(J32+b) + (K32+k) ld]
        warp_mma8(c0, c1, A + (I * 32 + tr * 8) + (K * 32) * kLdD, 1, kLdD, A + (J * 32 + tc * 8) + (K * 32) * kLdD,
                  1, kLdD, 32, false, lane);
      T[pp][tr * 8 + g8][tc * 8 + 2 * t4] = c0;
      T[pp][tr * 8 + g8][tc * 8 + 2 * t4 + 1] = c1;
    }
    __syncthreads();
    for (int t = wid; t < npair * 16; t += kDiagThreads / 32) {
      const int pp = t >> 4, tr = (t >> 2) & 3, tc = t & 3;
      const int J = pp, I = pp + d;
      double c0 = 0.0, c1 = 0.0;
      // Linv[I,J](a, b) = -sum_k Dinv[I][a][k] T[k][b]
      warp_mma8(c0, c1, &Dinv[I][tr * 8][0], 33, 1, &T[pp][0][tc * 8], 1, 33, 32, true, lane);
      const int a = tr * 8 + g8, b = tc * 8 + 2 * t4;
      A[(J * 32 + b) + (I * 32 + a) * kLdD] = c0;
      A[(J * 32 + b + 1) + (I * 32 + a) * kLdD] = c1;
    }
    __syncthreads();
  }
  for (int idx = tid; idx < kNB * kNB; idx += kDiagThreads) {
    const int i = idx % kNB, j = idx / kNB;
    Linv[idx] = (i < kb && j < kb && i >= j) ? A[j + i * kLdD] : 0.0;
  }
}

// ------------------------------------------------------------------ tensor-core GEMM
// C op= A B^T on 128 x 128 tiles.  TRSM: C = A B^T (acc from zero; B = explicit L11^{-1}).
// Updates (UPD*, RECT, DIST): the accumulators start as C (loaded straight into registers, so the HBM
// read of C overlaps the operand pipeline instead of serialising behind the main loop) and the A
// fragments are negated, so acc = C - A B^T; the epilogue only stores.
struct GemmArgs {
  const double* A;  // element (i, kk) at A[i + kk*lda], i relative to the tile-row base
  int64_t lda;
  const double* Bm;  // element (j, kk) at Bm[j + kk*ldbm]
  int64_t ldbm;
  double* C;  // element (i, j) at C[i + j*ldc]
  int64_t ldc;
  int rows;  // valid rows of A and C (UPD: also of B, the block is square)
  int cols;  // TRSM / RECT: valid rows of B = columns of C
  int K;
  int c0, c1;  // UPD: tile columns [c0, c1) (kModeUpdCols) or [c0, T) (kModeUpdTri)
  // DIST: C is this rank's local 2D block-cyclic array (Grid), A = B = the gathered panel whose row 0
  // is global row k1; local 128-row/column sub-tiles (blockIdx.x, blockIdx.y)
  Grid g;
  int64_t k1, m;
  int64_t jlo, jhi;  // DIST: global tile columns [jlo, jhi) only (lookahead split)
  int ntiles;        // number of tiles (x-extent); the grid may be smaller (persistent loop)
  const int32_t* err;
};

enum { kModeTrsm = 0, kModeUpdCols = 1, kModeUpdTri = 2, kModeRect = 3, kModeDist = 4 };


template <int MODE, bool AL16>
__device__ __forceinline__ void gemm_tile(const GemmArgs& g, const int tile, double* sm) {
  double* As = sm;                          // [kStages][kBK][kLdA]
  double* Bs = sm + kStages * kBK * kLdA;   // [kStages][kBK][kLdB]
  constexpr bool UPD = MODE != kModeTrsm;
  // tile (128 rows x 64 columns) -> operand bases, valid extents, diagonal mask (column j of the
  // tile is global column i0 + doff + j when row i is global row i0 + i; keep j + doff <= i)
  const double* Ab;
  const double* Bb;
  double* Cb;
  int na, nbv, doff = 0;
  bool mask;
  if (MODE == kModeTrsm || MODE == kModeRect) {
    const int bi = tile, bj = blockIdx.y;
    Ab = g.A + (size_t)bi * kTile;
    Bb = g.Bm + (size_t)bj * kBN;
    Cb = g.C + (size_t)bi * kTile + (size_t)bj * kBN * g.ldc;
    na = g.rows - bi * kTile;
    nbv = g.cols - bj * kBN;
    mask = false;
  } else if (MODE == kModeDist) {
    const int64_t la = (int64_t)tile * kTile, lb = (int64_t)blockIdx.y * kBN;
    const int64_t gi = ((la / kScmNB) * g.g.Pr + g.g.pr) * kScmNB + la % kScmNB;
    const int64_t gj = ((lb / kScmNB) * g.g.Pc + g.g.pc) * kScmNB + lb % kScmNB;
    if (gj < g.k1 || gi + kTile <= gj || gi >= g.m) return;
    if (gj / kScmNB < g.jlo || gj / kScmNB >= g.jhi) return;
    Ab = g.A + (gi - g.k1);
    Bb = g.A + (gj - g.k1);
    Cb = g.C + la + lb * g.ldc;
    na = (int)(g.m - gi < kTile ? g.m - gi : kTile);
    nbv = (int)(g.m - gj < kBN ? g.m - gj : kBN);
    doff = (int)(gj - gi);
    mask = gj + kBN > gi;
  } else {
    const int T = (g.rows + kTile - 1) / kTile;
    int t = tile, bi, bj;  // bj in 64-column units
    if (MODE == kModeUpdCols) {  // column-major over the 128-columns [c0, c1), two halves each
      int c = g.c0;
      while (t >= kR * (T - c)) {
        t -= kR * (T - c);
        ++c;
      }
      bi = c + t / kR;
      bj = kR * c + t % kR;
    } else {  // row-major over the lower triangle of 128-columns [c0, T): row r has kR (r + 1) tiles
      const int tt = t / kR;
      int r = (int)((sqrt(8.0 * tt + 1.0) - 1.0) * 0.5);
      while (r * (r + 1) / 2 > tt) --r;
      while ((r + 1) * (r + 2) / 2 <= tt) ++r;
      bi = g.c0 + r;
      bj = kR * g.c0 + (t - kR * (r * (r + 1) / 2));
    }
    Ab = g.A + (size_t)bi * kTile;
    Bb = g.Bm + (size_t)bj * kBN;
    Cb = g.C + (size_t)bi * kTile + (size_t)bj * kBN * g.ldc;
    na = g.rows - bi * kTile;
    nbv = g.rows - bj * kBN;
    doff = bj * kBN - bi * kTile;
    mask = doff + kBN > 0;
  }
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int kWarpsM = kTile / kWM;
  const int wm = wid % kWarpsM, wn = wid / kWarpsM;  // warp tile kWM x 32
  const int g8 = lane >> 2, t4 = lane & 3;

  auto load_stage = [&](int stage, int k0) {
    double* as = As + stage * kBK * kLdA;
    double* bs = Bs + stage * kBK * kLdB;
    if (AL16) {
#pragma unroll
      for (int q = 0; q < (kBK * kTile / 2) / kGemmThreads; ++q) {  // 16B chunks: 2 rows of one column
        const int cid = tid + q * kGemmThreads;
        const int kk = cid / (kTile / 2), rp = (cid % (kTile / 2)) * 2;
        const bool va = (k0 + kk) < g.K && rp < na;
        cp_async16(as + kk * kLdA + rp, va ? Ab + rp + (size_t)(k0 + kk) * g.lda : g.A, va);
      }
#pragma unroll
      for (int q = 0; q < (kBK * kBN / 2) / kGemmThreads; ++q) {
        const int cid = tid + q * kGemmThreads;
        const int kk = cid / (kBN / 2), rp = (cid % (kBN / 2)) * 2;
        const bool vb = (k0 + kk) < g.K && rp < nbv;
        cp_async16(bs + kk * kLdB + rp, vb ? Bb + rp + (size_t)(k0 + kk) * g.ldbm : g.A, vb);
      }
    } else {
#pragma unroll
      for (int q = 0; q < (kBK * kTile) / kGemmThreads; ++q) {  // 8B elements
        const int cid = tid + q * kGemmThreads;
        const int kk = cid / kTile, rp = cid % kTile;
        const bool va = (k0 + kk) < g.K && rp < na;
        cp_async8(as + kk * kLdA + rp, va ? Ab + rp + (size_t)(k0 + kk) * g.lda : g.A, va);
      }
#pragma unroll
      for (int q = 0; q < (kBK * kBN) / kGemmThreads; ++q) {
        const int cid = tid + q * kGemmThreads;
        const int kk = cid / kBN, rp = cid % kBN;
        const bool vb = (k0 + kk) < g.K && rp < nbv;
        cp_async8(bs + kk * kLdB + rp, vb ? Bb + rp + (size_t)(k0 + kk) * g.ldbm : g.A, vb);
      }
    }
  };

  const int nk = (g.K + kBK - 1) / kBK;
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nk) load_stage(s, s * kBK);
    cp_async_commit();
  }

  // accumulators: C for tiles off the diagonal (textbook update order); zero for TRSM and for tiles
  // that meet the diagonal, whose O(1) entries get C added once in the epilogue (one rounding per
  // launch instead of one per DMMA: see k_chol_dag.cu), C prefetched into L2 meanwhile
  const bool cadd = UPD && mask;
  if (cadd)
    for (int q = tid; q < (nbv < kBN ? nbv : kBN) * (kTile / 16); q += kGemmThreads) {
      const int c = q / (kTile / 16), r = (q % (kTile / 16)) * 16;
      if (r < na) prefetch_l2(Cb + r + (size_t)c * g.ldc);
    }
  double acc[kWA][4][2];
#pragma unroll
  for (int a = 0; a < kWA; ++a) {
    const int i = wm * kWM + a * 8 + g8;
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = wn * 32 + b * 8 + 2 * t4 + e;
        acc[a][b][e] = (UPD && !mask && i < na && j < nbv) ? Cb[i + (size_t)j * g.ldc] : 0.0;
      }
  }

  for (int kc = 0; kc < nk; ++kc) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    const int nxt = kc + kStages - 1;
    if (nxt < nk) load_stage(nxt % kStages, nxt * kBK);
    cp_async_commit();
    const double* as = As + (kc % kStages) * kBK * kLdA;
    const double* bs = Bs + (kc % kStages) * kBK * kLdB;
#pragma unroll
    for (int k4 = 0; k4 < kBK / 4; ++k4) {
      double af[kWA], bf[4];
#pragma unroll
      for (int a = 0; a < kWA; ++a) {
        const double v = as[(k4 * 4 + t4) * kLdA + wm * kWM + a * 8 + g8];
        af[a] = UPD ? neg(v) : v;  // (measured: faster than negating C once and accumulating -C)
      }
#pragma unroll
      for (int b = 0; b < 4; ++b) bf[b] = bs[(k4 * 4 + t4) * kLdB + wn * 32 + b * 8 + g8];
#pragma unroll
      for (int a = 0; a < kWA; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
  }
  cp_async_wait<0>();

#pragma unroll
  for (int a = 0; a < kWA; ++a) {
    const int i = wm * kWM + a * 8 + g8;
    if (i >= na) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = wn * 32 + b * 8 + 2 * t4 + e;
        if (j < nbv && (!mask || j + doff <= i)) {
          double* cp = Cb + i + (size_t)j * g.ldc;
          *cp = cadd ? *cp + acc[a][b][e] : acc[a][b][e];
        }
      }
  }
}

// Tiles blockIdx.x, blockIdx.x + gridDim.x, ... < g.ntiles (UpdTri may run on a capped, persistent
// grid so that the panel kernels of the lookahead stream always find free SMs).
template <int MODE, bool AL16>
__global__ void __launch_bounds__(kGemmThreads, kGemmCtasPerSm) gemm_nt_kernel(GemmArgs g) {
  if (*g.err != kNoError) return;
  extern __shared__ double sm[];
  for (int t = blockIdx.x; t < g.ntiles; t += gridDim.x) {
    gemm_tile<MODE, AL16>(g, t, sm);
    __syncthreads();  // the next tile's cp.async stages reuse the shared buffers
  }
}

// In-place panel solve C = A B^T (C == A allowed: each CTA reads all K columns of its rows before
// writing any of them, and owns all <= 128 output columns of those rows).  64-row x 128-column tile,
// 8 warps x (32 x 32) DMMA, 2 CTAs per SM (twice the CTAs of a 128-row tile on the critical path).
constexpr int kTrsmBM = 64;
constexpr int kLdT = kTrsmBM + 4;
template <bool AL16>
__global__ void __launch_bounds__(kTrsmThreads, 2) trsm_kernel(GemmArgs g) {
  if (*g.err != kNoError) return;
  extern __shared__ double sm[];
  double* As = sm;                          // [kStages][kBK][kLdT]
  double* Bs = sm + kStages * kBK * kLdT;   // [kStages][kBK][kLdA]
  const int bi = blockIdx.x;
  const double* Ab = g.A + (size_t)bi * kTrsmBM;
  double* Cb = g.C + (size_t)bi * kTrsmBM;
  const int na = g.rows - bi * kTrsmBM, nbv = g.cols;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int wm = wid >> 2, wn = wid & 3;  // 2 x 4 warps, warp tile 32 x 32
  const int g8 = lane >> 2, t4 = lane & 3;
  auto load_stage = [&](int stage, int k0) {
    double* as = As + stage * kBK * kLdT;
    double* bs = Bs + stage * kBK * kLdA;
#pragma unroll
    for (int q = 0; q < (kBK * kTrsmBM) / kTrsmThreads; ++q) {
      const int cid = tid + q * kTrsmThreads;
      const int kk = cid / kTrsmBM, rp = cid % kTrsmBM;
      const bool va = (k0 + kk) < g.K && rp < na;
      cp_async8(as + kk * kLdT + rp, va ? Ab + rp + (size_t)(k0 + kk) * g.lda : g.A, va);
    }
#pragma unroll
    for (int q = 0; q < (kBK * kTile) / kTrsmThreads; ++q) {
      const int cid = tid + q * kTrsmThreads;
      const int kk = cid / kTile, rp = cid % kTile;
      const bool vb = (k0 + kk) < g.K && rp < nbv;
      if (AL16) {
        if ((rp & 1) == 0) cp_async16(bs + kk * kLdA + rp, vb ? g.Bm + rp + (size_t)(k0 + kk) * g.ldbm : g.A, vb);
      } else {
        cp_async8(bs + kk * kLdA + rp, vb ? g.Bm + rp + (size_t)(k0 + kk) * g.ldbm : g.A, vb);
      }
    }
  };
  const int nk = (g.K + kBK - 1) / kBK;
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nk) load_stage(s, s * kBK);
    cp_async_commit();
  }
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  for (int kc = 0; kc < nk; ++kc) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    const int nxt = kc + kStages - 1;
    if (nxt < nk) load_stage(nxt % kStages, nxt * kBK);
    cp_async_commit();
    const double* as = As + (kc % kStages) * kBK * kLdT;
    const double* bs = Bs + (kc % kStages) * kBK * kLdA;
#pragma unroll
    for (int k4 = 0; k4 < kBK / 4; ++k4) {
      double af[4], bf[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) af[a] = as[(k4 * 4 + t4) * kLdT + wm * 32 + a * 8 + g8];
#pragma unroll
      for (int b = 0; b < 4; ++b) bf[b] = bs[(k4 * 4 + t4) * kLdA + wn * 32 + b * 8 + g8];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();  // every warp of this CTA has read its A rows before any is overwritten
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int i = wm * 32 + a * 8 + g8;
    if (i >= na) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = wn * 32 + b * 8 + 2 * t4 + e;
        if (j < nbv) Cb[i + (size_t)j * g.ldc] = acc[a][b][e];
      }
  }
}

static size_t trsm_smem() { return (size_t)kStages * kBK * (kLdT + kLdA) * sizeof(double); }

static size_t gemm_smem() { return (size_t)kStages * kBK * (kLdA + kLdB) * sizeof(double); }
static size_t diag_smem() { return ((size_t)kNB * kLdD + 32 * kLdD + 3 * 32 * 33) * sizeof(double); }  // + 34 KB static

template <int MODE>
static void launch_gemm(bool al16, dim3 grid, const GemmArgs& g0, cudaStream_t st, int cap = 0) {
  if (grid.x == 0 || grid.y == 0) return;
  GemmArgs g = g0;
  g.ntiles = (int)grid.x;
  if (cap > 0 && (int)grid.x > cap) grid.x = cap;
  if constexpr (MODE == kModeTrsm) {  // in place: one CTA owns all (<= 128) columns of its rows
    if (al16) trsm_kernel<true><<<dim3(grid.x), kTrsmThreads, trsm_smem(), st>>>(g);
    else trsm_kernel<false><<<dim3(grid.x), kTrsmThreads, trsm_smem(), st>>>(g);
  } else {
    if (al16) gemm_nt_kernel<MODE, true><<<grid, kGemmThreads, gemm_smem(), st>>>(g);
    else gemm_nt_kernel<MODE, false><<<grid, kGemmThreads, gemm_smem(), st>>>(g);
  }
}

static void set_all_attrs();

template <int MODE>
static void set_gemm_attr() {  // (never for kModeTrsm: that mode launches trsm_kernel)
  cudaFuncSetAttribute(gemm_nt_kernel<MODE, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gemm_smem());
  cudaFuncSetAttribute(gemm_nt_kernel<MODE, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gemm_smem());
}

// Blocked right-looking Cholesky, outer block width kOuter = 2 * kNB: the trailing updates run with
// K = 256 (half the C traffic of K = 128); each outer panel is factored as two 128-wide sub-panels.
constexpr int kOuter = 2 * kNB;

static void set_all_attrs() {
  static std::atomic<uint64_t> attr{0};
  if (!once_per_device(attr)) return;
  cudaFuncSetAttribute(potrf_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)diag_smem());
  cudaFuncSetAttribute(trsm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)trsm_smem());
  cudaFuncSetAttribute(trsm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)trsm_smem());
  set_gemm_attr<kModeUpdCols>();
  set_gemm_attr<kModeUpdTri>();
  set_gemm_attr<kModeRect>();
  set_gemm_attr<kModeDist>();
}

static bool aligned16(const void* p, int64_t ld) {
  return (ld % 2 == 0) && ((reinterpret_cast<uintptr_t>(p) & 15) == 0);
}

int potrf_lower(sdpc_ctx* h, double* B, int64_t m, int64_t ld, int32_t* d_err, cudaStream_t st, double* flops_upd,
                int* n_upd, double* linv_ws) {
  set_all_attrs();
  if (!h->st2) {
    // the lookahead (panel) stream gets the highest priority: its CTAs are scheduled first as the
    // trailing-update CTAs retire, so the critical path does not queue behind the update
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStreamCreateWithPriority(&h->st2, cudaStreamNonBlocking, hi);
    cudaEventCreateWithFlags(&h->evA, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&h->evB, cudaEventDisableTiming);
  }
  cudaStream_t s2 = h->st2;
  const bool al16 = aligned16(B, ld) && aligned16(linv_ws, 2);  // the TRSM stages linv_ws with 16-byte copies
  const bool tim = h->timing;
  int launches = 0;
  double fl = 0.0;
  int nu = 0;
  int sub = 0;  // sub-panel counter (Linv double buffer)
  auto upd = [&](int mode, int64_t kcol, int kw, int64_t base, int c0, int c1, cudaStream_t s) {
    // B[base:, base:] tile columns [c0, c1) (or [c0, T)) -= B[base:, kcol:kcol+kw] B[base:, kcol:kcol+kw]^T
    const int rows = (int)(m - base);
    const int T = (rows + kTile - 1) / kTile;
    GemmArgs u{};
    u.A = B + base + (size_t)kcol * ld;
    u.lda = ld;
    u.Bm = u.A;
    u.ldbm = ld;
    u.C = B + base + (size_t)base * ld;
    u.ldc = ld;
    u.rows = rows;
    u.K = kw;
    u.c0 = c0;
    u.c1 = c1;
    u.err = d_err;
    int grid = 0;
    if (mode == kModeUpdCols) {
      for (int c = c0; c < std::min(c1, T); ++c) grid += kR * (T - c);
      launch_gemm<kModeUpdCols>(al16, dim3(grid), u, s);
    } else {
      const int S = T - c0;
      grid = S > 0 ? kR * S * (S + 1) / 2 : 0;
      launch_gemm<kModeUpdTri>(al16, dim3(grid), u, s);
    }
    if (grid > 0) ++launches;
    return grid;
  };
  auto subpanel = [&](int64_t k0, int kb, cudaStream_t s) {  // diag + trsm of columns [k0, k0+kb)
    double* Lw = linv_ws + (sub++ & 1) * kNB * kNB;
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
    launch_gemm<kModeTrsm>(al16, dim3((rows + kTrsmBM - 1) / kTrsmBM), g, s);
    ++launches;
  };
  auto panel = [&](int64_t k0, cudaStream_t s) {  // outer block column [k0, k0 + w)
    const int w = (int)std::min<int64_t>(kOuter, m - k0);
    subpanel(k0, std::min(kNB, w), s);
    if (w > kNB) {
      upd(kModeUpdCols, k0, kNB, k0 + kNB, 0, 1, s);
      subpanel(k0 + kNB, w - kNB, s);
    }
  };
  // Schedule (depth-2 lookahead).  s2 (high priority) carries the critical path: for every outer
  // step k, ucol(k) = panel k's update of block column k+1, then panel(k+1).  st carries the bulk:
  // urest(k) = panel k's update of block column k+2 first (uA, so ucol(k+1) can start as soon as it
  // is done) and then of everything beyond (uB).  Events: evB = "panel(k+1) done" (st waits before
  // urest(k+1) reads its L21), evA = "uA(k) done" (s2 waits before ucol(k+1)).
  cudaEventRecord(h->evA, st);  // input ready
  cudaStreamWaitEvent(s2, h->evA, 0);
  panel(0, s2);
  cudaEventRecord(h->evB, s2);
  cudaStreamWaitEvent(st, h->evB, 0);
  bool have_uA = false;
  for (int64_t k0 = 0; k0 < m; k0 += kOuter) {
    const int w = (int)std::min<int64_t>(kOuter, m - k0);
    const int64_t base = k0 + w;
    const int rows = (int)(m - base);
    if (rows <= 0) break;
    const int T = (rows + kTile - 1) / kTile;
    const int ncol = std::min<int>(T, kOuter / kTile);           // tile columns of block column k+1
    const int ncol2 = std::min<int>(T - ncol, kOuter / kTile);   // ... of block column k+2
    // critical path on s2: ucol(k) (needs uA(k-1): block column k+1 complete up to step k-1)
    if (have_uA) cudaStreamWaitEvent(s2, h->evA, 0);
    upd(kModeUpdCols, k0, w, base, 0, ncol, s2);
    panel(base, s2);
    cudaEventRecord(h->evB, s2);
    // bulk on st: urest(k) = uA(k) + uB(k)
    have_uA = false;
    if (T > ncol) {
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
      upd(kModeUpdCols, k0, w, base, ncol, ncol + ncol2, st);
      cudaEventRecord(h->evA, st);
      have_uA = true;
      if (T > ncol + ncol2) upd(kModeUpdTri, k0, w, base, ncol + ncol2, 0, st);
      if (tim) cudaEventRecord(h->upd_ev[2 * nu + 1], st);
      ++nu;
      // algorithmic flops of this update: the lower triangle of the trailing block past the next
      // block column (r2 rows), 2 * w flops per entry
      const double r2 = (double)(rows - ncol * kTile);
      fl += r2 * (r2 + 1.0) * (double)w;
    }
    cudaStreamWaitEvent(st, h->evB, 0);  // urest(k+1) reads panel k+1
  }
  if (flops_upd) *flops_upd = fl;
  if (n_upd) *n_upd = nu;
  return launches;
}

// A (rows x kb, in place) <- A L^{-T} for the factored kb x kb tile L (kb <= 256) whose 128-block
// inverses inv[0], inv[1] came from potrf_lower: X1 = A1 L11^{-T}; A2 -= X1 L21^T; X2 = A2 L22^{-T}.
int trsm_panel(double* A, int64_t rows, int64_t lda, const double* Lt, int64_t ldl, const double* inv, int kb,
               const int32_t* d_err, cudaStream_t st) {
  set_all_attrs();
  if (rows <= 0 || kb <= 0) return 0;
  const bool al16 = aligned16(A, lda) && aligned16(Lt, ldl) && aligned16(inv, 2);  // inv: 16-byte TRSM stages
  const dim3 gr((unsigned)((rows + kTile - 1) / kTile));
  int launches = 0;
  GemmArgs g{};
  g.A = A;
  g.lda = lda;
  g.Bm = inv;
  g.ldbm = kNB;
  g.C = A;
  g.ldc = lda;
  g.rows = (int)rows;
  g.cols = std::min(kb, kNB);
  g.K = g.cols;
  g.err = d_err;
  const dim3 gt((unsigned)((rows + kTrsmBM - 1) / kTrsmBM));
  launch_gemm<kModeTrsm>(al16, gt, g, st);
  ++launches;
  if (kb > kNB) {
    GemmArgs r = g;
    r.C = A + (size_t)kNB * lda;
    r.Bm = Lt + kNB;
    r.ldbm = ldl;
    r.cols = kb - kNB;
    r.K = kNB;
    launch_gemm<kModeRect>(al16, dim3(gr.x, (unsigned)((r.cols + kBN - 1) / kBN)), r, st);
    GemmArgs t = g;
    t.C = A + (size_t)kNB * lda;
    t.A = t.C;
    t.Bm = inv + kNB * kNB;
    t.cols = kb - kNB;
    t.K = kb - kNB;
    launch_gemm<kModeTrsm>(al16, gt, t, st);
    launches += 2;
  }
  return launches;
}

// Local trailing update of a 2D block-cyclic Cholesky step: every local tile (I, J) with
// I >= J, J*nb >= k1 gets C_IJ -= P_I P_J^T (lower part of diagonal tiles), P = the gathered panel
// (global rows k1.. m, K columns).
int update_tiles(double* C, int64_t ldc, const double* P, int64_t ldp, int64_t k1, int K, const Grid& gr, int64_t m,
                 int64_t mloc, int64_t nloc, const int32_t* d_err, cudaStream_t st, int64_t jlo, int64_t jhi) {
  set_all_attrs();
  if (mloc <= 0 || nloc <= 0 || K <= 0 || k1 >= m) return 0;
  GemmArgs g{};
  g.A = P;
  g.lda = ldp;
  g.Bm = P;
  g.ldbm = ldp;
  g.C = C;
  g.ldc = ldc;
  g.K = K;
  g.g = gr;
  g.k1 = k1;
  g.m = m;
  g.jlo = jlo;
  g.jhi = jhi > 0 ? jhi : (int64_t)1 << 40;
  g.err = d_err;
  const bool al16 = aligned16(C, ldc) && aligned16(P, ldp);
  launch_gemm<kModeDist>(al16, dim3((unsigned)((mloc + kTile - 1) / kTile), (unsigned)((nloc + kBN - 1) / kBN)), g,
                         st);
  return 1;
}

}  // namespace sdpc
