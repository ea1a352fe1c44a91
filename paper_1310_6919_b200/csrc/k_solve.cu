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
  const int32_t* rhs;  // [npanels * 32] RHS vertex of each slot (elimination id), -1 = padding
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

// ---- CTA-cooperative pieces (all warps, CTA barriers), rows staged in shared memory ----
constexpr int kStageRows = 384;  // rows of 256 B staged per CTA (96 KB)

// stage rows S (zero if !s_valid) then U of a supernode into R[0..s+u) with cp.async
__device__ __forceinline__ void stage_rows(double* R, const double* X, int f, int s, const int32_t* __restrict__ U,
                                           int u, bool s_valid, int tid, int nt) {
  for (int idx = tid; idx < (s + u) * 16; idx += nt) {
    const int row = idx >> 4, ch = idx & 15;
    const int src = row < s ? f + row : U[row - s];
    const bool v = row < s ? s_valid : true;
    cp_async16(R + row * kPanelW + ch * 2, X + (size_t)src * kPanelW + ch * 2, v);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
}

// backward for a staged supernode: R[t] = y_t - sum_q L[s+q,t] R[s+q]; then x[S] = L_SS^{-T} R[S]
__device__ __forceinline__ void coop_bwd_staged(const double* __restrict__ Lr, int c, int s, double* R, int lane,
                                                int wid, int nw) {
  const int u = c - s;
  for (int t = wid; t < s; t += nw) {
    const double* Lt = Lr + s + (size_t)t * c;
    double a0 = R[t * kPanelW + lane], a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int q = 0;
    for (; q + 3 < u; q += 4) {
      a0 -= Lt[q] * R[(s + q) * kPanelW + lane];
      a1 -= Lt[q + 1] * R[(s + q + 1) * kPanelW + lane];
      a2 -= Lt[q + 2] * R[(s + q + 2) * kPanelW + lane];
      a3 -= Lt[q + 3] * R[(s + q + 3) * kPanelW + lane];
    }
    for (; q < u; ++q) a0 -= Lt[q] * R[(s + q) * kPanelW + lane];
    R[t * kPanelW + lane] = (a0 + a1) + (a2 + a3);
  }
  __syncthreads();
  for (int t1 = s; t1 > 0; t1 -= 16) {
    const int t0 = t1 > 16 ? t1 - 16 : 0;
    if (wid == 0) {
      for (int t = t1 - 1; t >= t0; --t) {
        double v = R[t * kPanelW + lane];
        for (int tp = t + 1; tp < t1; ++tp) v -= Lr[tp + (size_t)t * c] * R[tp * kPanelW + lane];
        R[t * kPanelW + lane] = v;
      }
    }
    __syncthreads();
    for (int t = wid; t < t0; t += nw) {
      double v = R[t * kPanelW + lane];
      for (int tp = t0; tp < t1; ++tp) v -= Lr[tp + (size_t)t * c] * R[tp * kPanelW + lane];
      R[t * kPanelW + lane] = v;
    }
    __syncthreads();
  }
}

// forward triangle on staged S rows: R[S] = L_SS^{-1} R[S] (unit lower), blocked by 16
__device__ __forceinline__ void coop_fwd_tri_staged(const double* __restrict__ Lr, int c, int s, double* R, int lane,
                                                    int wid, int nw) {
  for (int t0 = 0; t0 < s; t0 += 16) {
    const int t1 = min(s, t0 + 16);
    if (wid == 0) {
      for (int t = t0 + 1; t < t1; ++t) {
        double v = R[t * kPanelW + lane];
        for (int tp = t0; tp < t; ++tp) v -= Lr[t + (size_t)tp * c] * R[tp * kPanelW + lane];
        R[t * kPanelW + lane] = v;
      }
    }
    __syncthreads();
    for (int t = t1 + wid; t < s; t += nw) {
      double v = R[t * kPanelW + lane];
      for (int tp = t0; tp < t1; ++tp) v -= Lr[t + (size_t)tp * c] * R[tp * kPanelW + lane];
      R[t * kPanelW + lane] = v;
    }
    __syncthreads();
  }
}

// forward U update from staged S rows: x[U_q] -= sum_t L[s+q, t] R[t], 2 rows per warp in flight
__device__ __forceinline__ void coop_fwd_update_staged(const double* __restrict__ Lr, int c, int s,
                                                       const int32_t* __restrict__ U, const double* R, double* X,
                                                       int lane, int wid, int nw) {
  const int u = c - s;
  for (int qq = wid; qq < u; qq += 2 * nw) {
    const int q2 = qq + nw;
    const int r1 = U[qq], r2 = q2 < u ? U[q2] : r1;
    double x1 = xrow(X, r1, lane), x2 = q2 < u ? xrow(X, r2, lane) : 0.0;
    for (int t = 0; t < s; ++t) {
      const double z = R[t * kPanelW + lane];
      x1 -= Lr[s + qq + (size_t)t * c] * z;
      if (q2 < u) x2 -= Lr[s + q2 + (size_t)t * c] * z;
    }
    xrow(X, r1, lane) = x1;
    if (q2 < u) xrow(X, r2, lane) = x2;
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
  extern __shared__ __align__(16) double smem_solve[];
  double* R = smem_solve;                                                               // staged rows
  uint32_t* inreach = reinterpret_cast<uint32_t*>(smem_solve + kStageRows * kPanelW);  // bitmap
  const int P = blockIdx.x, fac = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int NW = kSolveThreads / 32;
  const int n = a.n;
  const double* __restrict__ Lp = a.Lp[fac];
  const double* __restrict__ D = a.D[fac];
  double* X = a.out[fac] + (size_t)P * n * kPanelW;
  const int myrhs = a.rhs[P * kPanelW + lane];  // this lane's RHS: e_{myrhs} (all-zero column if -1)
  const int32_t* __restrict__ rowind = a.rowind;

  const int nwords = (a.nsuper + 31) / 32;
  for (int i = tid; i < nwords; i += kSolveThreads) inreach[i] = 0;
  __syncthreads();
  const int rb = a.reach_ptr[P], re = a.reach_ptr[P + 1];
  for (int q = rb + tid; q < re; q += kSolveThreads) {
    const int r = a.reach_sn[q];
    atomicOr(&inreach[r >> 5], 1u << (r & 31));
  }
  // initialise z rows on the paths: z[i][lane] = (i == myrhs)
  for (int q = rb + wid; q < re; q += NW) {
    const int r = a.reach_sn[q];
    const int f = a.super_ptr[r], s = a.sns[r];
    for (int t = 0; t < s; ++t) xrow(X, f + t, lane) = (f + t == myrhs) ? 1.0 : 0.0;
  }
  __syncthreads();

  // forward L z = E_P over the paths, ascending supernodes
  for (int q = rb; q < re; ++q) {
    const int r = a.reach_sn[q];
    const int f = a.super_ptr[r], s = a.sns[r], c = a.snc[r], u = c - s;
    const double* Lr = Lp + a.panel_off[r];
    if (s > 16 && s <= kStageRows) {
      // big supernode: S rows staged in shared memory, triangle and U update from there
      stage_rows(R, X, f, s, nullptr, 0, true, tid, kSolveThreads);
      coop_fwd_tri_staged(Lr, c, s, R, lane, wid, NW);
      for (int t = wid; t < s; t += NW) xrow(X, f + t, lane) = R[t * kPanelW + lane];
      if (u > 0) coop_fwd_update_staged(Lr, c, s, rowind + a.colptr[f] + s, R, X, lane, wid, NW);
    } else {
      if (wid == 0) {  // unit lower diagonal block in registers, chunks of 16
        for (int t0 = 0; t0 < s; t0 += 16) {
          const int w = min(16, s - t0);
          double acc[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[j] = j < w ? xrow(X, f + t0 + j, lane) : 0.0;
          for (int tp = 0; tp < t0; ++tp) {
            const double zt = xrow(X, f + tp, lane);
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (j < w) acc[j] -= Lr[(t0 + j) + (size_t)tp * c] * zt;
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if (j < w) {
              const double zj = acc[j];
              xrow(X, f + t0 + j, lane) = zj;
#pragma unroll
              for (int jj = j + 1; jj < 16; ++jj)
                if (jj < w) acc[jj] -= Lr[(t0 + jj) + (size_t)(t0 + j) * c] * zj;
            }
          }
        }
      }
      __syncthreads();
      if (u > 0) {
        const int32_t* U = rowind + a.colptr[f] + s;
        if (s <= 1) fwd_update<1>(Lr, c, s, f, U, X, lane, wid, NW);
        else if (s <= 2) fwd_update<2>(Lr, c, s, f, U, X, lane, wid, NW);
        else if (s <= 4) fwd_update<4>(Lr, c, s, f, U, X, lane, wid, NW);
        else if (s <= 8) fwd_update<8>(Lr, c, s, f, U, X, lane, wid, NW);
        else fwd_update<16>(Lr, c, s, f, U, X, lane, wid, NW);
      }
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
    const int32_t* U = rowind + a.colptr[f] + s;
    if (c <= kStageRows) {
      stage_rows(R, X, f, s, U, c - s, onpath, tid, kSolveThreads);
      coop_bwd_staged(Lr, c, s, R, lane, wid, NW);
      for (int t = wid; t < s; t += NW) xrow(X, f + t, lane) = R[t * kPanelW + lane];
    } else if (wid == 0) {  // very large clique: one warp from global memory
      bwd_supernode<16>(Lr, c, s, f, U, X, lane, onpath);
    }
    __syncthreads();
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
  a.rhs = h->d.rhs;
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
  size_t smem = sizeof(double) * kStageRows * kPanelW + sizeof(uint32_t) * (((h->S.nsuper + 31) / 32) + 1);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(inverse_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
    attr = true;
  }
  if (h->d.npanels == 0) return 0;
  dim3 grid(h->d.npanels, 2);
  inverse_panel_kernel<<<grid, kSolveThreads, smem, st>>>(a);
  return 1;
}

}  // namespace sdpc
