// (b) Multi-RHS supernodal solves: dense X-hat = (L D L^T)^{-1} and Y^{-1} = (L_Y D_Y L_Y^T)^{-1},
// one RHS panel of 32 identity columns per CTA (lane <-> RHS column).
//
// PAPER.md P:320-330 (forward/backward substitution instead of forming X-hat),
// P:686-688 (Eq. newSCM2: x_p = L-hat^{-T} L-hat^{-1} e_p, v = N^{-T} N^{-1} [A_j]_{*k}),
// P:859-869 (reuse of x_p across a column of B; on B200 the whole X-hat fits in HBM, so the
// columns are materialised once and reused by every column of B, reading #21).
//
// Per panel P (columns p0 = 32P .. p0+31, elimination order):
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

namespace sdpc {

struct SolveArgs {
  int32_t n, nsuper, ndlev;
  const int32_t* super_ptr;
  const int32_t* snc;
  const int32_t* sns;
  const int64_t* colptr;
  const int32_t* rowind;
  const int64_t* panel_off;
  const int32_t* reach_ptr;
  const int32_t* reach_sn;
  const int32_t* dlev_ptr;
  const int32_t* dlev_sn;
  const int32_t* border;   // backward task order: top supernodes (level order), then subtrees (preorder)
  const int32_t* sub_ptr;  // [nsub+1] offsets of the subtrees in border (starting at ntop)
  int32_t ntop, nsub;
  const int32_t* sparent;
  const double* Lp[2];
  const double* D[2];
  double* out[2];
};

constexpr int kSolveThreads = 256;
constexpr int kCh = 16;  // register chunk of supernode columns (widest instantiation)

__device__ __forceinline__ double& xrow(double* X, int row, int lane) { return X[(size_t)row * kPanelW + lane]; }

// backward for one supernode, one warp: x[S] = L_SS^{-T} (y[S] - L_US^T x[U]); CH = register chunk
template <int kCh>
__device__ __forceinline__ void bwd_supernode(const double* __restrict__ Lr, int c, int s, int f,
                                              const int32_t* __restrict__ U, double* X, int lane, bool onpath) {
  const int u = c - s;
  for (int t1 = s; t1 > 0; t1 -= kCh) {
    const int t0 = t1 > kCh ? t1 - kCh : 0;
    const int w = t1 - t0;
    double acc[kCh];
#pragma unroll
    for (int j = 0; j < kCh; ++j) acc[j] = (j < w && onpath) ? xrow(X, f + t0 + j, lane) : 0.0;
    const double* Lc = Lr + (size_t)t0 * c;  // Lc[i + j*c] = L[i, t0+j]
    // U rows in blocks of 32: indices and L values loaded coalesced by the warp, broadcast by
    // shuffles; 8 independent row loads in flight
    for (int q0 = 0; q0 < u; q0 += 32) {
      const int nq = min(32, u - q0);
      const int myrow = lane < nq ? U[q0 + lane] : 0;
      double lv[kCh];
#pragma unroll
      for (int j = 0; j < kCh; ++j) lv[j] = (j < w && lane < nq) ? Lc[s + q0 + lane + (size_t)j * c] : 0.0;
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
    for (int tp = t1; tp < s; ++tp) {
      const double xq = xrow(X, f + tp, lane);
#pragma unroll
      for (int j = 0; j < kCh; ++j)
        if (j < w) acc[j] -= Lc[tp + (size_t)j * c] * xq;
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

// ---- CTA-cooperative pieces for big supernodes (all warps, CTA barriers) ----
// backward, step 1: X[f+t] = y_t - sum_q L[s+q, t] x[U_q] for all t in S (columns over warps, 8 per pass)
__device__ __forceinline__ void coop_bwd_gemv(const double* __restrict__ Lr, int c, int s, int f,
                                              const int32_t* __restrict__ U, double* X, int lane, int wid,
                                              int nw, bool onpath) {
  const int u = c - s;
  for (int tb = wid; tb < s; tb += 8 * nw) {  // columns tb, tb+nw, ..., tb+7nw
    double acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int t = tb + j * nw;
      acc[j] = (t < s && onpath) ? xrow(X, f + t, lane) : 0.0;
    }
    for (int q = 0; q < u; ++q) {
      const double xq = xrow(X, U[q], lane);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int t = tb + j * nw;
        if (t < s) acc[j] -= Lr[s + q + (size_t)t * c] * xq;
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int t = tb + j * nw;
      if (t < s) xrow(X, f + t, lane) = acc[j];
    }
  }
}

// backward, step 2: x[S] = L_SS^{-T} acc, blocked by 16 from the last block
__device__ __forceinline__ void coop_bwd_tri(const double* __restrict__ Lr, int c, int s, int f, double* X,
                                             int lane, int wid, int nw) {
  for (int t1 = s; t1 > 0; t1 -= 16) {
    const int t0 = t1 > 16 ? t1 - 16 : 0;
    if (wid == 0) {
      for (int t = t1 - 1; t >= t0; --t) {
        double v = xrow(X, f + t, lane);
        for (int tp = t + 1; tp < t1; ++tp) v -= Lr[tp + (size_t)t * c] * xrow(X, f + tp, lane);
        xrow(X, f + t, lane) = v;
      }
    }
    __syncthreads();
    for (int t = wid; t < t0; t += nw) {
      double v = xrow(X, f + t, lane);
      for (int tp = t0; tp < t1; ++tp) v -= Lr[tp + (size_t)t * c] * xrow(X, f + tp, lane);
      xrow(X, f + t, lane) = v;
    }
    __syncthreads();
  }
}

// forward triangle z[S] = L_SS^{-1} z[S] (unit lower), blocked by 16 from the first block
__device__ __forceinline__ void coop_fwd_tri(const double* __restrict__ Lr, int c, int s, int f, double* X,
                                             int lane, int wid, int nw) {
  for (int t0 = 0; t0 < s; t0 += 16) {
    const int t1 = min(s, t0 + 16);
    if (wid == 0) {
      for (int t = t0 + 1; t < t1; ++t) {
        double v = xrow(X, f + t, lane);
        for (int tp = t0; tp < t; ++tp) v -= Lr[t + (size_t)tp * c] * xrow(X, f + tp, lane);
        xrow(X, f + t, lane) = v;
      }
    }
    __syncthreads();
    for (int t = t1 + wid; t < s; t += nw) {
      double v = xrow(X, f + t, lane);
      for (int tp = t0; tp < t1; ++tp) v -= Lr[t + (size_t)tp * c] * xrow(X, f + tp, lane);
      xrow(X, f + t, lane) = v;
    }
    __syncthreads();
  }
}

// forward update of the U rows of one supernode by all warps: x[U] -= L_US z[S] (S rows final)
template <int kCh>
__device__ __forceinline__ void fwd_update(const double* __restrict__ Lr, int c, int s, int f,
                                           const int32_t* __restrict__ U, double* X, int lane, int wid, int nw) {
  const int u = c - s;
  for (int t0 = 0; t0 < s; t0 += kCh) {
    const int w = min(kCh, s - t0);
    double zt[kCh];
#pragma unroll
    for (int j = 0; j < kCh; ++j) zt[j] = j < w ? xrow(X, f + t0 + j, lane) : 0.0;
    const double* Lc = Lr + (size_t)t0 * c;
    for (int qq = wid; qq < u; qq += nw) {
      double acc = xrow(X, U[qq], lane);
#pragma unroll
      for (int j = 0; j < kCh; ++j)
        if (j < w) acc -= Lc[s + qq + (size_t)j * c] * zt[j];
      xrow(X, U[qq], lane) = acc;
    }
  }
}

__global__ void __launch_bounds__(kSolveThreads, 2) inverse_panel_kernel(SolveArgs a) {
  extern __shared__ uint32_t inreach[];  // bitmap over supernodes
  const int P = blockIdx.x, fac = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int NW = kSolveThreads / 32;
  const int n = a.n;
  const double* __restrict__ Lp = a.Lp[fac];
  const double* __restrict__ D = a.D[fac];
  double* X = a.out[fac] + (size_t)P * n * kPanelW;
  const int p0 = P * kPanelW;
  const int32_t* __restrict__ rowind = a.rowind;

  const int nwords = (a.nsuper + 31) / 32;
  for (int i = tid; i < nwords; i += kSolveThreads) inreach[i] = 0;
  __syncthreads();
  const int rb = a.reach_ptr[P], re = a.reach_ptr[P + 1];
  for (int q = rb + tid; q < re; q += kSolveThreads) {
    const int r = a.reach_sn[q];
    atomicOr(&inreach[r >> 5], 1u << (r & 31));
  }
  // initialise z rows on the paths: z[i][lane] = (i == p0 + lane)
  for (int q = rb + wid; q < re; q += NW) {
    const int r = a.reach_sn[q];
    const int f = a.super_ptr[r], s = a.sns[r];
    for (int t = 0; t < s; ++t) xrow(X, f + t, lane) = (f + t == p0 + lane) ? 1.0 : 0.0;
  }
  __syncthreads();

  // forward L z = E_P over the paths, ascending supernodes
  for (int q = rb; q < re; ++q) {
    const int r = a.reach_sn[q];
    const int f = a.super_ptr[r], s = a.sns[r], c = a.snc[r], u = c - s;
    const double* Lr = Lp + a.panel_off[r];
    if (s > 16) {
      coop_fwd_tri(Lr, c, s, f, X, lane, wid, NW);
    } else {
      if (wid == 0) {  // unit lower diagonal block in registers
        double acc[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = j < s ? xrow(X, f + j, lane) : 0.0;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (j < s) {
            const double zj = acc[j];
            xrow(X, f + j, lane) = zj;
#pragma unroll
            for (int jj = j + 1; jj < 16; ++jj)
              if (jj < s) acc[jj] -= Lr[jj + (size_t)j * c] * zj;
          }
        }
      }
      __syncthreads();
    }
    if (u > 0) {
      const int32_t* U = rowind + a.colptr[f] + s;
      if (s <= 1) fwd_update<1>(Lr, c, s, f, U, X, lane, wid, NW);
      else if (s <= 2) fwd_update<2>(Lr, c, s, f, U, X, lane, wid, NW);
      else if (s <= 4) fwd_update<4>(Lr, c, s, f, U, X, lane, wid, NW);
      else if (s <= 8) fwd_update<8>(Lr, c, s, f, U, X, lane, wid, NW);
      else fwd_update<16>(Lr, c, s, f, U, X, lane, wid, NW);
    }
    __syncthreads();
    for (int t = wid; t < s; t += NW) xrow(X, f + t, lane) /= D[f + t];
  }
  __syncthreads();

  // backward L^T x = z.  (1) the top of the tree (big supernodes near the roots) in level order,
  // each supernode by the whole CTA; (2) the remaining subtrees, one warp per subtree in preorder,
  // claimed from a shared counter (no waiting: their only outside dependencies are in the top).
  // Rows off the paths have z = 0.
  for (int it = 0; it < a.ntop; ++it) {
    const int r = a.border[it];
    const int f = a.super_ptr[r], s = a.sns[r], c = a.snc[r];
    const bool onpath = (inreach[r >> 5] >> (r & 31)) & 1u;
    const double* Lr = Lp + a.panel_off[r];
    coop_bwd_gemv(Lr, c, s, f, rowind + a.colptr[f] + s, X, lane, wid, NW, onpath);
    __syncthreads();
    coop_bwd_tri(Lr, c, s, f, X, lane, wid, NW);
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
      const bool onpath = (inreach[r >> 5] >> (r & 31)) & 1u;
      const double* Lr = Lp + a.panel_off[r];
      const int32_t* U = rowind + a.colptr[f] + s;
      if (s <= 1) bwd_supernode<1>(Lr, c, s, f, U, X, lane, onpath);
      else if (s <= 2) bwd_supernode<2>(Lr, c, s, f, U, X, lane, onpath);
      else if (s <= 4) bwd_supernode<4>(Lr, c, s, f, U, X, lane, onpath);
      else if (s <= 8) bwd_supernode<8>(Lr, c, s, f, U, X, lane, onpath);
      else bwd_supernode<16>(Lr, c, s, f, U, X, lane, onpath);
    }
  }
}

int launch_inverse_panels(sdpc_ctx* h, cudaStream_t st) {
  SolveArgs a{};
  a.n = h->S.n;
  a.nsuper = h->S.nsuper;
  a.ndlev = (int32_t)h->S.dlev_ptr.size() - 1;
  a.super_ptr = h->d.super_ptr;
  a.snc = h->d.snc;
  a.sns = h->d.sns;
  a.colptr = h->d.colptr;
  a.rowind = h->d.rowind;
  a.panel_off = h->d.panel_off;
  a.reach_ptr = h->d.reach_ptr;
  a.reach_sn = h->d.reach_sn;
  a.dlev_ptr = h->d.dlev_ptr;
  a.dlev_sn = h->d.dlev_sn;
  a.border = h->d.border;
  a.sub_ptr = h->d.sub_ptr;
  a.ntop = h->S.ntop;
  a.nsub = (int32_t)h->S.sub_ptr.size() - 1;
  a.sparent = h->d.sparent;
  a.Lp[0] = h->Lx;
  a.Lp[1] = h->Ly;
  a.D[0] = h->Dx;
  a.D[1] = h->Dy;
  a.out[0] = h->Xh;
  a.out[1] = h->Yh;
  size_t smem = sizeof(uint32_t) * (((h->S.nsuper + 31) / 32) + 1);
  static bool attr = false;
  if (!attr && smem > 48 * 1024) {
    cudaFuncSetAttribute(inverse_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  dim3 grid(h->d.npanels, 2);
  inverse_panel_kernel<<<grid, kSolveThreads, smem, st>>>(a);
  return 1;
}

}  // namespace sdpc
