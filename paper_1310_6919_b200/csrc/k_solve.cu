// (b) Multi-RHS supernodal solves: dense X-hat = (L D L^T)^{-1} and Y^{-1} = (L_Y D_Y L_Y^T)^{-1},
// one RHS panel of 32 identity columns per CTA (lane <-> RHS column).
//
// PAPER.md P:320-330 (forward/backward substitution instead of forming X-hat),
// P:686-688 (Eq. newSCM2: x_p = L-hat^{-T} L-hat^{-1} e_p, v = N^{-T} N^{-1} [A_j]_{*k}),
// P:859-869 (reuse of x_p across a column of B; on B200 the whole X-hat fits in HBM, so the
// columns are materialised once and reused by every column of B, reading #21).
//
// Per panel P (RHS vertices rhs[32P .. 32P+31], ascending elimination ids):
//   forward  L z = E_P  over the union of the etree paths of the panel's columns (ascending
//            supernodes, whole CTA per supernode; rows off the paths are exactly zero); z <- D^{-1} z;
//   backward L^T x = z  the top of the tree (big supernodes) one supernode at a time by the whole CTA,
//            then whole bottom subtrees, one warp each, in preorder (no write conflicts: a supernode
//            writes only its rows S_r and reads its ancestors' rows U_r).
// Both sweeps keep up to 16 columns of a supernode in registers, so every row x[U_q] is read once
// per 16 columns (not once per column).
// Output layout: panel-major, X[P][i][lane] (row i of the panel = 32 contiguous doubles).
#include <cuda_runtime.h>

#include "common.cuh"
#include "ctx.hpp"

#include <algorithm>

namespace sdpc {

struct SolveArgs {
  int32_t n, nsuper;
  const int32_t* super_ptr;
  const int32_t* snc;
  const int32_t* sns;
  const int64_t* colptr;
  const int32_t* rowind;
  const int64_t* panel_off;
  const int32_t* reach_ptr;
  const int32_t* reach_sn;
  const int32_t* rhs;  // [npanels * 32] RHS vertex of each slot (elimination id), -1 = padding
  const int32_t* border;   // backward task order: top supernodes (level order), then subtrees (preorder)
  const int32_t* sub_ptr;  // [nsub+1] offsets of the subtrees in border (starting at ntop)
  int32_t ntop, nsub;
  int32_t trunc;  // max-cut, one rank: the backward sweep stops below the panel's smallest RHS
  int32_t fac0;   // first factor of this launch (0: X-hat from L, D; 1: Y^{-1} from L_Y, D_Y)
  int32_t npanels;
  const double* Lp[2];
  const double* D[2];
  double* out[2];
  // general right-hand sides (P-MATRIX and g, Eq. newdX2): when rhs_in is set, panel P's input
  // is the dense panel rhs_in[P] (same layout as out; in place allowed) instead of the identity columns
  // e_{rhs[..]}; the forward sweep then runs over every supernode (full_sn = 0..nsuper-1)
  const double* rhs_in;
  const int32_t* full_sn;
};

constexpr int kSolveThreads = 256;
constexpr int kOcc3Panels = 592;           // >= two rounds of the 296 two-per-SM slots: use 3 CTAs per SM
constexpr int kSolveSmemCap = 110 * 1024;  // opt-in of inverse_panel_kernel (2 CTAs per SM)

__device__ __forceinline__ double& xrow(double* X, int row, int lane) { return X[(size_t)row * kPanelW + lane]; }

// backward for one supernode, one warp: x[S] = L_SS^{-T} (y[S] - L_US^T x[U]); CH = register chunk
template <int kCh>
__device__ __forceinline__ void bwd_supernode(const double* __restrict__ Lr, int c, int s, int f,
                                              const int32_t* __restrict__ U, double* X, int lane, bool onpath) {
  for (int t1 = s; t1 > 0; t1 -= kCh) {
    const int t0 = t1 > kCh ? t1 - kCh : 0;
    const int w = t1 - t0;
    double acc[kCh];
#pragma unroll
    for (int j = 0; j < kCh; ++j) acc[j] = (j < w && onpath) ? xrow(X, f + t0 + j, lane) : 0.0;
    const double* Lc = Lr + (size_t)t0 * c;  // Lc[i + j*c] = L[i, t0+j]
    // gathered rows t1..c-1 (the rows of S after the chunk, final by now, then U) in blocks of 32:
    // indices and L values loaded coalesced by the warp, broadcast by shuffles; 8 row loads in flight
    for (int q0 = t1; q0 < c; q0 += 32) {
      const int nq = min(32, c - q0);
      const int myrow = lane < nq ? (q0 + lane < s ? f + q0 + lane : U[q0 + lane - s]) : 0;
      double lv[kCh];
#pragma unroll
      for (int j = 0; j < kCh; ++j) lv[j] = (j < w && lane < nq) ? Lc[q0 + lane + (size_t)j * c] : 0.0;
      for (int k0 = 0; k0 < nq; k0 += 8) {
        double xq[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int rr = __shfl_sync(0xffffffffu, myrow, k0 + k);
          xq[k] = (k0 + k < nq) ? xrow(X, rr, lane) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
#pragma unroll
          for (int j = 0; j < kCh; ++j) acc[j] -= __shfl_sync(0xffffffffu, lv[j], k0 + k) * xq[k];
        }
      }
    }
#pragma unroll
    for (int j = kCh - 1; j >= 0; --j) {
      if (j < w) {
        const double xj = acc[j];
        xrow(X, f + t0 + j, lane) = xj;
#pragma unroll
        for (int jj = 0; jj < j; ++jj) acc[jj] -= Lc[(t0 + j) + (size_t)jj * c] * xj;
      }
    }
  }
}

// backward for one supernode with |S_r| > 8, one warp, FP64 tensor cores: per 16-column chunk, the
// gathered-row product acc(j, n) = sum_q L[q][t0 + j] x[row(q)][n] as m8n8k4 DMMA tiles (2 row tiles x
// 4 RHS slices, K = the rows after the chunk), no per-FMA shuffles; the accumulators go through a
// per-warp shared-memory square (Wm, 16 x 33) to the lane = RHS layout of the chunk triangle.
__device__ __forceinline__ void bwd_supernode_mma(const double* __restrict__ Lr, int c, int s, int f,
                                                  const int32_t* __restrict__ U, double* X, int lane, bool onpath,
                                                  double* Wm) {
  constexpr int kCh = 16;
  const int g8 = lane >> 2, t4 = lane & 3;
  for (int t1 = s; t1 > 0; t1 -= kCh) {
    const int t0 = t1 > kCh ? t1 - kCh : 0;
    const int w = t1 - t0;
    const double* Lc = Lr + (size_t)t0 * c;  // Lc[i + j*c] = L[i, t0+j]
    double d[2][4][2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) d[mt][nt][0] = d[mt][nt][1] = 0.0;
    const int K = c - t1;
#pragma unroll 2
    for (int k0 = 0; k0 < K; k0 += 4) {
      const int q = t1 + k0 + t4;
      const bool kv = k0 + t4 < K;
      const int row = kv ? (q < s ? f + q : U[q - s]) : 0;
      double av[2], bv[4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) av[mt] = (kv && 8 * mt + g8 < w) ? Lc[q + (size_t)(8 * mt + g8) * c] : 0.0;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) bv[nt] = kv ? X[(size_t)row * kPanelW + 8 * nt + g8] : 0.0;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma_8x8x4(d[mt][nt][0], d[mt][nt][1], av[mt], bv[nt]);
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        Wm[(8 * mt + g8) * 33 + 8 * nt + 2 * t4] = d[mt][nt][0];
        Wm[(8 * mt + g8) * 33 + 8 * nt + 2 * t4 + 1] = d[mt][nt][1];
      }
    __syncwarp();
    double acc[kCh];
#pragma unroll
    for (int j = 0; j < kCh; ++j)
      acc[j] = j < w ? (onpath ? xrow(X, f + t0 + j, lane) : 0.0) - Wm[j * 33 + lane] : 0.0;
    __syncwarp();
#pragma unroll
    for (int j = kCh - 1; j >= 0; --j) {
      if (j < w) {
        const double xj = acc[j];
        xrow(X, f + t0 + j, lane) = xj;
#pragma unroll
        for (int jj = 0; jj < j; ++jj) acc[jj] -= Lc[(t0 + j) + (size_t)jj * c] * xj;
      }
    }
    __syncwarp();  // this chunk's rows are read (as gathered rows) by the next chunk
  }
}

// ---- big supernodes (|S_r| >= kBigS): whole CTA, FP64 tensor cores (m8n8k4 DMMA) -------------
// The rectangular parts of both sweeps are small GEMMs whose operands come straight from L2:
// A = a block of the supernode panel L_r, B = 8-RHS slices of gathered rows of the panel X, so
// every warp task is one 8 x 8 output tile (8 rows of the supernode x 8 RHS) with K running over
// the panel rows / columns.  The triangular L_SS parts run on 128-row chunks staged in shared
// memory (16-row diagonal blocks in registers of one warp, the rest of the chunk by all warps).
constexpr int kBigS = kTopMinS;  // supernodes with at least this many columns take this path
constexpr int kChunk = 128;   // rows of S per shared-memory chunk
constexpr int kVs = 36;       // chunk row stride (doubles): conflict-free 8-RHS fragment reads

// row of X holding the k-th operand row of a gather: f + k for k < s (rows S), U[k - s] after
__device__ __forceinline__ int op_row(int k, int f, int s, const int32_t* __restrict__ U) {
  return k < s ? f + k : U[k - s];
}

// One warp, one 8 x 8 tile: (c0, c1) += sum_{k < K} A(t, k) X[row(kb0 + k)][n0 + n] with
// A(t, k) = Ab[t * as_t + k * as_k] for t < nt (zero beyond), rows gathered by op_row.
__device__ __forceinline__ void tile_gemm_gather(double& c0, double& c1, const double* __restrict__ Ab, int as_t,
                                                 int as_k, int nt, const double* X, int kb0, int K, int f, int s,
                                                 const int32_t* __restrict__ U, int n0, int lane) {
  const int g8 = lane >> 2, t4 = lane & 3;
  const bool tv = g8 < nt;
  const double* ap = Ab + (size_t)g8 * as_t + (size_t)t4 * as_k;
#pragma unroll 8
  for (int k0 = 0; k0 < K; k0 += 4) {
    const int k = k0 + t4;
    const bool kv = k < K;
    const double av = (tv && kv) ? ap[(size_t)k0 * as_k] : 0.0;
    const double bv = kv ? X[(size_t)op_row(kb0 + k, f, s, U) * kPanelW + n0 + g8] : 0.0;
    dmma_8x8x4(c0, c1, av, bv);
  }
}

// forward, big supernode r: z[S] = L_SS^{-1} z[S] (chunks ascending), then z[U] -= L_US z[S]
constexpr int kLs = 129;  // stride of the staged 16-column strips of L (chunk triangles)
__device__ void big_fwd(const double* __restrict__ Lr, int c, int s, int f, const int32_t* __restrict__ U,
                        double* X, double* Vs, double* Ls, int tid, int lane, int wid, int nw) {
  const int g8 = lane >> 2, t4 = lane & 3;
  for (int t0 = 0; t0 < s; t0 += kChunk) {
    const int w = min(kChunk, s - t0);
    // V = z[S_c] - L[S_c, S_<c] z[S_<c]   (tile tasks: (w/8) x 4)
    const int ntt = (w + 7) >> 3;
    for (int task = wid; task < ntt * 4; task += nw) {
      const int tt = task >> 2, n0 = (task & 3) * 8;
      const int r0 = tt * 8 + g8;
      double c0 = 0.0, c1 = 0.0;
      if (r0 < w) {
        c0 = X[(size_t)(f + t0 + r0) * kPanelW + n0 + 2 * t4];
        c1 = X[(size_t)(f + t0 + r0) * kPanelW + n0 + 2 * t4 + 1];
      }
      if (t0 > 0) {
        // A(t, k) = L[t0 + tt*8 + t][k]: as_t = 1, as_k = c; negated through the B operand sign
        double d0 = 0.0, d1 = 0.0;
        tile_gemm_gather(d0, d1, Lr + t0 + tt * 8, 1, c, min(8, w - tt * 8), X, 0, t0, f, s, U, n0, lane);
        c0 -= d0;
        c1 -= d1;
      }
      if (r0 < w) {
        Vs[r0 * kVs + n0 + 2 * t4] = c0;
        Vs[r0 * kVs + n0 + 2 * t4 + 1] = c1;
      }
    }
    __syncthreads();
    // chunk triangle, 16-row diagonal blocks; the block's 16 columns of L (rows b0 .. w of the chunk) are
    // staged in shared memory first (Ls[j * kLs + t] = L[t0 + t][t0 + b0 + j]), so the per-row updates read
    // L with broadcast LDS instead of dependent L2 round trips
    for (int b0 = 0; b0 < w; b0 += 16) {
      const int bw = min(16, w - b0);
      for (int idx = tid; idx < 16 * (w - b0); idx += nw * 32) {
        const int j = idx / (w - b0), t = b0 + idx % (w - b0);
        Ls[j * kLs + t] = j < bw ? Lr[(t0 + t) + (size_t)(t0 + b0 + j) * c] : 0.0;
      }
      __syncthreads();
      if (wid == 0) {
        double acc[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = j < bw ? Vs[(b0 + j) * kVs + lane] : 0.0;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
#pragma unroll
          for (int jj = j + 1; jj < 16; ++jj)
            if (jj < bw) acc[jj] -= Ls[j * kLs + b0 + jj] * acc[j];
        }
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (j < bw) Vs[(b0 + j) * kVs + lane] = acc[j];
      }
      __syncthreads();
      for (int t = b0 + bw + wid; t < w; t += nw) {
        double v = Vs[t * kVs + lane];
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (j < bw) v -= Ls[j * kLs + t] * Vs[(b0 + j) * kVs + lane];
        Vs[t * kVs + lane] = v;
      }
      __syncthreads();
    }
    for (int t = wid; t < w; t += nw) X[(size_t)(f + t0 + t) * kPanelW + lane] = Vs[t * kVs + lane];
    __syncthreads();
  }
  // z[U] -= L_US z[S]: tile tasks (u/8) x 4, C = gathered rows of X (read-modify-write)
  const int u = c - s;
  const int nqt = (u + 7) >> 3;
  for (int task = wid; task < nqt * 4; task += nw) {
    const int qt = task >> 2, n0 = (task & 3) * 8;
    const int q = qt * 8 + g8;
    double d0 = 0.0, d1 = 0.0;
    tile_gemm_gather(d0, d1, Lr + s + qt * 8, 1, c, min(8, u - qt * 8), X, 0, s, f, s, U, n0, lane);
    if (q < u) {
      double* xr = X + (size_t)U[q] * kPanelW + n0 + 2 * t4;
      xr[0] -= d0;
      xr[1] -= d1;
    }
  }
}

// backward, big supernode r: x[S] = L_SS^{-T} (z[S] - L_US^T x[U]), chunks descending; each chunk
// takes the rows of S after it as part of its gather (they are final by then).  The gathered X rows
// (the B operand, shared by every output tile of the chunk) are staged in shared memory in K-chunks
// of kKc rows, double-buffered with cp.async; each warp keeps the accumulators of its tiles across
// K-chunks.  The A operand (panel L_r) streams from L2 with independent loads.
constexpr int kKc = 64;                  // gathered rows per staged K-chunk
constexpr int kMaxTasks = kChunk / 8 * 4 / 8;  // tiles per warp (8 warps, 128-row chunk, 4 RHS slices)

__device__ __forceinline__ void stage_gather(double* Bsb, const double* X, int kb0, int nrows, int f, int s,
                                             const int32_t* __restrict__ U, int tid, int nt) {
  for (int idx = tid; idx < kKc * 16; idx += nt) {  // 16 x 16-byte pieces per 256-byte row
    const int rr = idx >> 4, ch = idx & 15;
    const bool v = rr < nrows;
    const int row = v ? op_row(kb0 + rr, f, s, U) : 0;
    cp_async16(Bsb + rr * kVs + ch * 2, X + (size_t)row * kPanelW + ch * 2, v);
  }
  cp_async_commit();
}

__device__ void big_bwd(const double* __restrict__ Lr, int c, int s, int f, const int32_t* __restrict__ U,
                        double* X, bool onpath, double* Vs, double* Bs, int tid, int lane, int wid, int nw) {
  const int g8 = lane >> 2, t4 = lane & 3;
  const int nch = (s + kChunk - 1) / kChunk;
  for (int ch = nch - 1; ch >= 0; --ch) {
    const int t0 = ch * kChunk, w = min(kChunk, s - t0), t1 = t0 + w;
    const int ntt = (w + 7) >> 3, ntask = ntt * 4;
    const int K = c - t1;  // gathered rows: S after the chunk, then U
    if (w <= 16) {
      // thin chunk (e.g. the 8-13-column separator supernodes of a 3D torus with |U| ~ 1,400-2,900): the
      // K rows are split over the warps instead of the output tiles (each warp: both row tiles x four
      // RHS slices, operands straight from L2, no staging barriers), partial sums reduced through Bs
      const int Kw = ((K + 4 * nw - 1) / (4 * nw)) * 4, kb = wid * Kw, ke = min(K, kb + Kw);
      double d[2][4][2];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) d[mt][nt][0] = d[mt][nt][1] = 0.0;
#pragma unroll 2
      for (int k0 = kb; k0 < ke; k0 += 4) {
        const int q = t1 + k0 + t4;
        const bool kv = k0 + t4 < ke;
        const int row = kv ? op_row(q, f, s, U) : 0;
        double av[2], bv[4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) av[mt] = (kv && 8 * mt + g8 < w) ? Lr[q + (size_t)(t0 + 8 * mt + g8) * c] : 0.0;
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) bv[nt] = kv ? X[(size_t)row * kPanelW + 8 * nt + g8] : 0.0;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) dmma_8x8x4(d[mt][nt][0], d[mt][nt][1], av[mt], bv[nt]);
      }
      double* red = Bs + wid * (16 * 33);
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          red[(8 * mt + g8) * 33 + 8 * nt + 2 * t4] = d[mt][nt][0];
          red[(8 * mt + g8) * 33 + 8 * nt + 2 * t4 + 1] = d[mt][nt][1];
        }
      __syncthreads();
      for (int idx = tid; idx < w * kPanelW; idx += nw * 32) {
        const int r = idx >> 5, n = idx & 31;
        double sum = 0.0;
        for (int v = 0; v < nw; ++v) sum += Bs[v * (16 * 33) + r * 33 + n];
        Vs[r * kVs + n] = (onpath ? X[(size_t)(f + t0 + r) * kPanelW + n] : 0.0) - sum;
      }
    } else {
    double acc[kMaxTasks][2];
#pragma unroll
    for (int q = 0; q < kMaxTasks; ++q) acc[q][0] = acc[q][1] = 0.0;
    const int nkc = (K + kKc - 1) / kKc;
    if (nkc > 0) stage_gather(Bs, X, t1, min(kKc, K), f, s, U, tid, nw * 32);
    for (int kc = 0; kc < nkc; ++kc) {
      const double* Bb = Bs + (kc & 1) * kKc * kVs;
      if (kc + 1 < nkc) {
        stage_gather(Bs + ((kc + 1) & 1) * kKc * kVs, X, t1 + (kc + 1) * kKc, min(kKc, K - (kc + 1) * kKc), f, s,
                     U, tid, nw * 32);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const int kr = min(kKc, K - kc * kKc);
#pragma unroll
      for (int q = 0; q < kMaxTasks; ++q) {
        const int task = wid + q * nw;
        if (task < ntask) {
          const int tt = task >> 2, n0 = (task & 3) * 8;
          const bool tv = tt * 8 + g8 < w;
          // A(t, k) = L[t1 + kc*kKc + k][t0 + tt*8 + t]
          const double* ap = Lr + t1 + kc * kKc + t4 + (size_t)(t0 + tt * 8 + g8) * c;
          const double* bp = Bb + t4 * kVs + n0 + g8;
#pragma unroll 8
          for (int k0 = 0; k0 < kKc; k0 += 4) {
            const bool kv = k0 + t4 < kr;
            const double av = (tv && kv) ? ap[k0] : 0.0;
            const double bv = kv ? bp[k0 * kVs] : 0.0;
            dmma_8x8x4(acc[q][0], acc[q][1], av, bv);
          }
        }
      }
      __syncthreads();  // buffer (kc & 1) is refilled by the next iteration's prefetch
    }
#pragma unroll
    for (int q = 0; q < kMaxTasks; ++q) {
      const int task = wid + q * nw;
      if (task < ntask) {
        const int tt = task >> 2, n0 = (task & 3) * 8;
        const int r0 = tt * 8 + g8;
        if (r0 < w) {
          double z0 = 0.0, z1 = 0.0;
          if (onpath) {
            z0 = X[(size_t)(f + t0 + r0) * kPanelW + n0 + 2 * t4];
            z1 = X[(size_t)(f + t0 + r0) * kPanelW + n0 + 2 * t4 + 1];
          }
          Vs[r0 * kVs + n0 + 2 * t4] = z0 - acc[q][0];
          Vs[r0 * kVs + n0 + 2 * t4 + 1] = z1 - acc[q][1];
        }
      }
    }
    }  // (w > 16)
    __syncthreads();
    // chunk triangle L_cc^T, 16-row diagonal blocks from the bottom up
    const int nb = (w + 15) / 16;
    for (int bb = nb - 1; bb >= 0; --bb) {
      const int b0 = bb * 16, bw = min(16, w - b0);
      // stage L[t0 + b0 + j][t0 + t] (t < b0 + bw, j < 16) as Ls[j * kLs + t] (Bs is free here)
      for (int idx = tid; idx < 16 * (b0 + bw); idx += nw * 32) {
        const int t = idx >> 4, j = idx & 15;
        Bs[j * kLs + t] = j < bw ? Lr[(t0 + b0 + j) + (size_t)(t0 + t) * c] : 0.0;
      }
      __syncthreads();
      if (wid == 0) {
        double acc16[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) acc16[j] = j < bw ? Vs[(b0 + j) * kVs + lane] : 0.0;
#pragma unroll
        for (int j = 15; j >= 0; --j) {
          if (j < bw) {
#pragma unroll
            for (int jj = 0; jj < j; ++jj) acc16[jj] -= Bs[j * kLs + b0 + jj] * acc16[j];
          }
        }
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (j < bw) Vs[(b0 + j) * kVs + lane] = acc16[j];
      }
      __syncthreads();
      for (int t = wid; t < b0; t += nw) {
        double v = Vs[t * kVs + lane];
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (j < bw) v -= Bs[j * kLs + t] * Vs[(b0 + j) * kVs + lane];
        Vs[t * kVs + lane] = v;
      }
      __syncthreads();
    }
    for (int t = wid; t < w; t += nw) X[(size_t)(f + t0 + t) * kPanelW + lane] = Vs[t * kVs + lane];
    __syncthreads();
  }
}

// forward for a small supernode (s < kBigS), no barrier inside: every warp solves the unit-lower
// L_SS block for the 32 RHS in registers (redundantly: s <= 15) and updates its share of the rows U
// with that copy of z[S]; warp 0 parks z[S] in a shared-memory slot (zslot[j*32 + lane]), copied to
// X after the next barrier (writing X[S] here could race with a slower warp still reading it)
template <int kCh>
__device__ __forceinline__ void fwd_small(const double* __restrict__ Lr, int c, int s, int f,
                                          const int32_t* __restrict__ U, double* X, double* zslot, int lane,
                                          int wid, int nw, double* zw) {
  double zt[kCh];
#pragma unroll
  for (int j = 0; j < kCh; ++j) zt[j] = j < s ? xrow(X, f + j, lane) : 0.0;
#pragma unroll
  for (int j = 0; j < kCh; ++j)
#pragma unroll
    for (int jj = j + 1; jj < kCh; ++jj)
      if (jj < s) zt[jj] -= Lr[jj + (size_t)j * c] * zt[j];
  if (wid == 0) {
#pragma unroll
    for (int j = 0; j < kCh; ++j)
      if (j < s) zslot[j * kPanelW + lane] = zt[j];
  }
  const int u = c - s;
  constexpr int KQ = kCh >= 8 ? kCh / 4 : 1;
  if constexpr (kCh >= 8) if (u >= 128) {
    // tall supernode (e.g. the top separator chain of a 3D torus, |U| ~ 1,400-2,900): x[U] -= L_US z[S] as
    // m8n8k4 DMMA tiles (8 rows of U x 8 RHS), z[S] as B fragments through a per-warp shared square, two
    // row tiles per warp in flight
    const int g8 = lane >> 2, t4 = lane & 3;
#pragma unroll
    for (int j = 0; j < kCh; ++j) zw[j * 33 + lane] = zt[j];
    __syncwarp();
    double bv[KQ][4];
#pragma unroll
    for (int kq = 0; kq < KQ; ++kq)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) bv[kq][nt] = zw[(4 * kq + t4) * 33 + 8 * nt + g8];
    const int ntile = (u + 7) >> 3;
    for (int t = wid; t < ntile; t += 2 * nw) {
      int row[2];
      double av[2][KQ], cc[2][4][2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int q = 8 * (t + e * nw) + g8;
        const bool qv = t + e * nw < ntile && q < u;
        row[e] = qv ? U[q] : -1;
#pragma unroll
        for (int kq = 0; kq < KQ; ++kq)
          av[e][kq] = (qv && 4 * kq + t4 < s) ? -Lr[s + q + (size_t)(4 * kq + t4) * c] : 0.0;
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          cc[e][nt][0] = qv ? X[(size_t)row[e] * kPanelW + 8 * nt + 2 * t4] : 0.0;
          cc[e][nt][1] = qv ? X[(size_t)row[e] * kPanelW + 8 * nt + 2 * t4 + 1] : 0.0;
        }
      }
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int kq = 0; kq < KQ; ++kq)
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) dmma_8x8x4(cc[e][nt][0], cc[e][nt][1], av[e][kq], bv[kq][nt]);
#pragma unroll
      for (int e = 0; e < 2; ++e)
        if (row[e] >= 0)
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) {
            X[(size_t)row[e] * kPanelW + 8 * nt + 2 * t4] = cc[e][nt][0];
            X[(size_t)row[e] * kPanelW + 8 * nt + 2 * t4 + 1] = cc[e][nt][1];
          }
    }
    return;
  }
  // rows U in groups of 4 per warp: independent row / L loads in flight
  for (int q0 = 4 * wid; q0 < u; q0 += 4 * nw) {
    int row[4];
    double acc[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      row[e] = q0 + e < u ? U[q0 + e] : -1;
      acc[e] = row[e] >= 0 ? xrow(X, row[e], lane) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < kCh; ++j)
      if (j < s)
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (q0 + e < u) acc[e] -= Lr[s + q0 + e + (size_t)j * c] * zt[j];
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (row[e] >= 0) xrow(X, row[e], lane) = acc[e];
  }
}

__device__ __forceinline__ void solve_panel(const SolveArgs& a, const int P, const int fac, double* smem_solve) {
  double* Vs = smem_solve;                                                          // chunk of S rows
  double* Bs = smem_solve + kChunk * kVs;                                           // 2 staged K-chunks
  uint32_t* inreach = reinterpret_cast<uint32_t*>(smem_solve + (kChunk + 2 * kKc) * kVs);  // bitmap
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int NW = kSolveThreads / 32;
  const int n = a.n;
  const double* __restrict__ Lp = a.Lp[fac];
  const double* __restrict__ D = a.D[fac];
  double* X = a.out[fac] + (size_t)P * n * kPanelW;
  const int myrhs = a.rhs[P * kPanelW + lane];  // this lane's RHS: e_{myrhs} (all-zero column if -1)
  const bool gen = a.rhs_in != nullptr;
  const double* Xin = gen ? a.rhs_in + (size_t)P * n * kPanelW : nullptr;
  // truncated backward (SURVEY §8(a) note): only rows i >= pmin of this panel are read later, and
  // row i of x depends only on rows > i, so supernodes entirely below pmin are skipped
  const int pmin = (a.trunc && !gen) ? a.rhs[P * kPanelW] : -1;
  const int32_t* __restrict__ rowind = a.rowind;
  const int32_t* __restrict__ reach_sn = gen ? a.full_sn : a.reach_sn;

  const int nwords = (a.nsuper + 31) / 32;
  for (int i = tid; i < nwords; i += kSolveThreads) inreach[i] = 0;
  __syncthreads();
  const int rb = gen ? 0 : a.reach_ptr[P], re = gen ? a.nsuper : a.reach_ptr[P + 1];
  for (int q = rb + tid; q < re; q += kSolveThreads) {
    const int r = reach_sn[q];
    atomicOr(&inreach[r >> 5], 1u << (r & 31));
  }
  // initialise z rows on the paths: z[i][lane] = (i == myrhs), or the given dense panel
  for (int q = rb + wid; q < re; q += NW) {
    const int r = reach_sn[q];
    const int f = a.super_ptr[r], s = a.sns[r];
    if (gen) {
      if (Xin != X)
        for (int t = 0; t < s; ++t) xrow(X, f + t, lane) = Xin[(size_t)(f + t) * kPanelW + lane];
    } else {
      for (int t = 0; t < s; ++t) xrow(X, f + t, lane) = (f + t == myrhs) ? 1.0 : 0.0;
    }
  }
  __syncthreads();

  // forward L z = E_P over the paths, ascending supernodes.  Small supernodes park their z[S] in
  // one of two shared-memory slots (Bs is free during the forward), flushed after the next barrier.
  double* zslots = Bs;
  int pend_f = -1, pend_s = 0, pend_slot = 0, slot = 0;
  auto flush = [&](int wflush) {
    if (pend_f >= 0 && wid == wflush)
      for (int t = 0; t < pend_s; ++t) xrow(X, pend_f + t, lane) = zslots[(pend_slot * 16 + t) * kPanelW + lane];
    pend_f = -1;
  };
  for (int q = rb; q < re; ++q) {
    const int r = reach_sn[q];
    const int f = a.super_ptr[r], s = a.sns[r], c = a.snc[r];
    const double* Lr = Lp + a.panel_off[r];
    flush(NW - 1);
    if (s >= kBigS) {
      __syncthreads();
      big_fwd(Lr, c, s, f, rowind + a.colptr[f] + s, X, Vs, Bs, tid, lane, wid, NW);
    } else {
      const int32_t* U = rowind + a.colptr[f] + s;
      double* zs = zslots + slot * 16 * kPanelW;
      if (s <= 1) fwd_small<1>(Lr, c, s, f, U, X, zs, lane, wid, NW, Vs + wid * (16 * 33));
      else if (s <= 2) fwd_small<2>(Lr, c, s, f, U, X, zs, lane, wid, NW, Vs + wid * (16 * 33));
      else if (s <= 4) fwd_small<4>(Lr, c, s, f, U, X, zs, lane, wid, NW, Vs + wid * (16 * 33));
      else if (s <= 8) fwd_small<8>(Lr, c, s, f, U, X, zs, lane, wid, NW, Vs + wid * (16 * 33));
      else fwd_small<16>(Lr, c, s, f, U, X, zs, lane, wid, NW, Vs + wid * (16 * 33));
      pend_f = f;
      pend_s = s;
      pend_slot = slot;
      slot ^= 1;
    }
    __syncthreads();
  }
  flush(NW - 1);
  __syncthreads();
  // z <- D^{-1} z on the path rows (deferred: the U updates above use the unscaled z)
  for (int q = rb + wid; q < re; q += NW) {
    const int r = reach_sn[q];
    const int f = a.super_ptr[r], s = a.sns[r];
    for (int t = 0; t < s; ++t) xrow(X, f + t, lane) /= D[f + t];
  }
  __syncthreads();

  // backward L^T x = z.  (1) the top of the tree (big supernodes near the roots) in level order,
  // each supernode by the whole CTA; (2) the remaining subtrees, one warp per subtree in preorder,
  // claimed from a shared counter (no waiting: their only outside dependencies are in the top).
  // Rows off the paths have z = 0.
  for (int it = 0; it < a.ntop; ++it) {
    const int r = a.border[it];
    const int f = a.super_ptr[r], s = a.sns[r], c = a.snc[r];
    if (f + s - 1 < pmin) continue;  // uniform over the CTA
    const bool onpath = (inreach[r >> 5] >> (r & 31)) & 1u;
    const double* Lr = Lp + a.panel_off[r];
    const int32_t* U = rowind + a.colptr[f] + s;
    big_bwd(Lr, c, s, f, U, X, onpath, Vs, Bs, tid, lane, wid, NW);
  }
  int* ctr = reinterpret_cast<int*>(inreach + nwords);
  if (tid == 0) *ctr = 0;
  __syncthreads();
  for (;;) {
    int q = 0;
    if (lane == 0) q = atomicAdd(ctr, 1);
    q = __shfl_sync(0xffffffffu, q, 0);
    if (q >= a.nsub) break;
    for (int it = a.sub_ptr[q]; it < a.sub_ptr[q + 1]; ++it) {
      const int r = a.border[it];
      const int f = a.super_ptr[r], s = a.sns[r], c = a.snc[r];
      if (f + s - 1 < pmin) continue;
      const bool onpath = (inreach[r >> 5] >> (r & 31)) & 1u;
      const double* Lr = Lp + a.panel_off[r];
      const int32_t* U = rowind + a.colptr[f] + s;
      if (s <= 1) bwd_supernode<1>(Lr, c, s, f, U, X, lane, onpath);
      else if (s <= 2) bwd_supernode<2>(Lr, c, s, f, U, X, lane, onpath);
      else if (s <= 4) bwd_supernode<4>(Lr, c, s, f, U, X, lane, onpath);
      else if (s <= 8) bwd_supernode<8>(Lr, c, s, f, U, X, lane, onpath);
      else bwd_supernode_mma(Lr, c, s, f, U, X, lane, onpath, Vs + wid * (16 * 33));
    }
  }
}

// One CTA per (RHS panel, factor); with gridDim.x < npanels (the X-hat solves that overlap the
// tree-level (a2) launches leave SMs free for them) each CTA walks one panel per round of gridDim.x.
// MINB = 3 (80 registers, some spills) pays when the solve is CTA-wide DMMA sweeps over big supernodes
// (block-arrow: (b) 25.2 -> 20.0 ms); on the deep trees of the tori, where per-warp walks over small
// supernodes dominate, it is slower (configs[1] (b) done 5.8 -> 6.4 ms), so the launch picks.
template <int MINB>
__global__ void __launch_bounds__(kSolveThreads, MINB) inverse_panel_kernel(SolveArgs a) {
  extern __shared__ __align__(16) double smem_solve[];
  const int fac = blockIdx.y + a.fac0;
  // rounds of gridDim.x panels; odd rounds in reverse, so that the CTA with the most expensive panel of
  // one round (low elimination indices: long reach, little truncated) takes the cheapest of the next
  const int G = gridDim.x;
  for (int k = 0; k * G < a.npanels; ++k) {
    const int P = (k & 1) ? min((k + 1) * G, a.npanels) - 1 - (int)blockIdx.x : k * G + (int)blockIdx.x;
    if (P < k * G || P >= a.npanels) break;
    solve_panel(a, P, fac, smem_solve);
    __syncthreads();
  }
}

static int launch_panels(sdpc_ctx* h, cudaStream_t st, int fac0, int nfac, int max_ctas, const double* in,
                         double* out, bool trunc);

// Dynamic shared memory of the solve kernel for nsuper supernodes (the reach bitmap grows with nsuper);
// sdpc_create rejects problems beyond kSolveSmemCap.
size_t solve_smem_bytes(int64_t nsuper) {
  return sizeof(double) * (kChunk + 2 * kKc) * kVs + sizeof(uint32_t) * (((nsuper + 31) / 32) + 1);
}
bool solve_smem_fits(int64_t nsuper) { return solve_smem_bytes(nsuper) <= (size_t)kSolveSmemCap; }

int launch_inverse_panels(sdpc_ctx* h, cudaStream_t st, int fac0, int nfac, int max_ctas) {
  return launch_panels(h, st, fac0, nfac, max_ctas, nullptr, nullptr, h->trunc_active);
}

// out[P] = X-hat in[P] (factor 0) or Y^{-1} in[P] (factor 1) for every RHS panel P (in == out allowed)
int launch_apply_inverse(sdpc_ctx* h, cudaStream_t st, int fac, const double* in, double* out) {
  return launch_panels(h, st, fac, 1, 0, in, out, false);
}

static int launch_panels(sdpc_ctx* h, cudaStream_t st, int fac0, int nfac, int max_ctas, const double* in,
                         double* out, bool trunc) {
  SolveArgs a{};
  a.n = h->S.n;
  a.nsuper = h->S.nsuper;
  a.super_ptr = h->d.super_ptr;
  a.snc = h->d.snc;
  a.sns = h->d.sns;
  a.colptr = h->d.colptr;
  a.rowind = h->d.rowind;
  a.panel_off = h->d.panel_off;
  a.reach_ptr = h->d.reach_ptr;
  a.reach_sn = h->d.reach_sn;
  a.rhs = h->d.rhs;
  a.border = h->d.border;
  a.sub_ptr = h->d.sub_ptr;
  a.ntop = h->S.ntop;
  a.nsub = (int32_t)h->S.sub_ptr.size() - 1;
  a.trunc = trunc ? 1 : 0;
  a.Lp[0] = h->Lx;
  a.Lp[1] = h->Ly;
  a.D[0] = h->Dx;
  a.D[1] = h->Dy;
  a.out[0] = h->Xh;
  a.out[1] = h->Yh;
  if (in) {
    a.rhs_in = in;
    a.out[fac0] = out;
    a.full_sn = h->d.all_sn;
  }
  const size_t smem = solve_smem_bytes(h->S.nsuper);
  static std::atomic<uint64_t> attr{0};
  if (once_per_device(attr)) {
    cudaFuncSetAttribute(inverse_panel_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSolveSmemCap);
    cudaFuncSetAttribute(inverse_panel_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSolveSmemCap);
  }
  if (h->d.npanels == 0) return 0;
  a.fac0 = fac0;
  a.npanels = h->d.npanels;
  dim3 grid(max_ctas > 0 ? std::min(h->d.npanels, max_ctas) : h->d.npanels, nfac);
  // three CTAs per SM when three fit the SM's shared memory and the work is CTA-wide DMMA sweeps over big
  // supernodes (shallow elimination trees: block-arrow) or the panels are many
  const bool occ3 = (h->a2lev.size() < 8 || h->d.npanels >= kOcc3Panels) && 3 * (smem + 1024) <= (size_t)227 * 1024;
  if (occ3) inverse_panel_kernel<3><<<grid, kSolveThreads, smem, st>>>(a);
  else inverse_panel_kernel<2><<<grid, kSolveThreads, smem, st>>>(a);
  return 1;
}

}  // namespace sdpc
