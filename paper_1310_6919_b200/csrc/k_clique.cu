// Batched per-clique kernels: (a1) Algorithm 1 and (a2) multifrontal LDL^T of Y.
//
// (a1) PAPER.md P:493-530, Algorithm 1.  One CTA per clique r (fundamental supernode):
//      Step 2-1 gather P_r X-bar_{C_rC_r} P_r^T (reversal is index arithmetic),
//      Step 2-2 Cholesky = M_r M_r^T,
//      Step 2-3 L_r = P_r M_r^{-T} P_r^T: only its first |S_r| columns are needed (Step 3),
//      i.e. the last |S_r| rows of M_r^{-1}, obtained by back substitution M_r^T W = [0; I].
//      Output in the north-star unit form L-hat = L D^{1/2}: D_j = L-hat_jj^2, L = L-hat / L-hat_jj.
// (a2) PAPER.md P:221-225 / P:722-725 (type (v)): Y = L_Y D_Y L_Y^T on the same E, multifrontal:
//      frontal = Y[C_r, S_r] + extend-add of the children's update matrices, Cholesky of the
//      |S_r| pivot columns, Schur complement passed to the parent.  One launch per etree height.
// Both use the same CTA-cooperative dense routines, blocked by 32 columns: the 32 x 32 diagonal
// block is factored and inverted by one warp in registers (shuffles), the panel below is formed
// with the inverse, and the trailing matrix is updated with 4 x 4 register tiles per thread.
// Cliques whose working set exceeds shared memory live in an L2-resident global workspace; their
// current 32-column panel is staged in shared memory.
#include <cuda_runtime.h>

#include "common.cuh"
#include "ctx.hpp"

namespace sdpc {

struct CliqueArgs {
  const int32_t* super_ptr;
  const int32_t* snc;
  const int32_t* sns;
  const int64_t* colptr;
  const int64_t* panel_off;
  const int64_t* umap_off;
  const int32_t* umap;
  const int64_t* ws_off;
  double* ws;
  const double* vals;
  double* Lp;
  double* D;
  int32_t* err;
  const int32_t* child_ptr;
  const int32_t* child_list;
  const int64_t* relind_off;
  const int32_t* relind;
  const int64_t* upd_off;
  double* upd;
  const uint8_t* pre;  // front already holds its children's extend-add (pre-pass)
};

constexpr unsigned kFullMask = 0xffffffffu;
constexpr int kLdInv = 33;

// Shared-memory scratch layout for one CTA: inverse of the current 32 x 32 diagonal block, and
// (global-workspace cliques) the current panel P (c x 32, ld c).
struct Scratch {
  double* inv;    // 32 x 33
  double* l11;    // 32 x 33 staging of the factored diagonal block
  double* panel;  // c x 32 (only used when the matrix lives in global memory)
  int* flag;
};

// Warp 0: Cholesky of the jw x jw block at A[j0, j0] in registers (lane = row), write it back,
// then invert it (lane = column) into s.inv (lower).  NC >= jw is the unrolled block width (a
// power of two, identity-padded beyond jw), so a 1- or 2-column supernode does not pay for 32.
// Returns via *flag the failing local column (>= 0) or -1.  Every shuffle is executed by all lanes.
template <int NC>
__device__ __forceinline__ void warp_chol_inv(double* A, int ld, int j0, int jw, const Scratch& s) {
  const int lane = threadIdx.x & 31;
  double row[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c)
    row[c] = (lane < jw && c < jw) ? A[(j0 + lane) + (size_t)(j0 + c) * ld] : (lane == c ? 1.0 : 0.0);
  int fail = -1;
  double rinv = 0.0;  // lane j: 1 / L[j][j]
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    const double d = __shfl_sync(kFullMask, row[j], j);
    if (fail < 0) {  // uniform (d is a broadcast)
      if (!(d > 0.0)) {
        fail = j;
      } else {
        const double rl = rsqrt_nr(d);
        if (lane == j) {
          row[j] = d * rl;
          rinv = rl;
        } else if (lane > j) {
          row[j] *= rl;
        }
#pragma unroll
        for (int k = j + 1; k < NC; ++k) {
          const double akj = __shfl_sync(kFullMask, row[j], k);
          if (lane >= k) row[k] -= row[j] * akj;
        }
      }
    }
  }
  if (lane == 0) *s.flag = fail;
  if (fail >= 0) return;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const double v = (lane < NC && lane >= c) ? row[c] : 0.0;
    if (lane < NC) s.l11[lane + c * kLdInv] = v;
    if (lane < jw && c < jw) A[(j0 + lane) + (size_t)(j0 + c) * ld] = v;
  }
  __syncwarp();
  // inverse, lane = column: forward substitution, L11 broadcast from shared memory
  double x[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    double sacc = (i == lane) ? 1.0 : 0.0;
#pragma unroll
    for (int k = 0; k < i; ++k) sacc -= s.l11[i + k * kLdInv] * x[k];
    x[i] = sacc * __shfl_sync(kFullMask, rinv, i);
  }
  if (lane < NC) {
#pragma unroll
    for (int i = 0; i < NC; ++i) s.inv[i + lane * kLdInv] = i >= lane ? x[i] : 0.0;
  }
}

__device__ __forceinline__ void warp_chol_inv32(double* A, int ld, int j0, int jw, const Scratch& s) {
  if (jw <= 4) warp_chol_inv<4>(A, ld, j0, jw, s);
  else if (jw <= 16) warp_chol_inv<16>(A, ld, j0, jw, s);
  else warp_chol_inv<32>(A, ld, j0, jw, s);
}

// CTA-cooperative blocked Cholesky of the leading `ncols` columns of the symmetric c x c matrix A
// (lower triangle, column-major, leading dimension ld = c), with the trailing block updated.
// Returns the failing column index, or -1.
// lim: the trailing update is restricted to columns < lim (the big-front path factors only the pivot
// panel here and forms the Schur complement in front_schur_kernel; lim = c otherwise).
template <int NT, bool GLOBAL>
__device__ int cta_chol_partial(double* A, int c, int ncols, const Scratch& s, int lim = 0x7fffffff) {
  const int tid = threadIdx.x, wid = tid >> 5;
  const int ld = c;
  for (int j0 = 0; j0 < ncols; j0 += 32) {
    const int jw = min(32, ncols - j0);
    if (wid == 0) warp_chol_inv32(A, ld, j0, jw, s);
    __syncthreads();
    const int f = *s.flag;
    if (f >= 0) return j0 + f;
    // panel below the diagonal block: L[i, j0:j0+jw] = A[i, j0:j0+jw] L11^{-T}
    const int r0 = j0 + jw, nr = c - r0;
    double* P = GLOBAL ? s.panel : A + (size_t)j0 * ld;  // P[i + k*ld] = L[i, j0+k]
    if (nr > 0) {
      // rows in groups of 2 x (jw outputs) per thread would need registers; do row-per-thread-chunk:
      for (int idx = tid; idx < nr; idx += NT) {
        const int i = r0 + idx;
        double a[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) a[k] = k < jw ? A[i + (size_t)(j0 + k) * ld] : 0.0;
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          if (q < jw) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k <= q; ++k) acc += a[k] * s.inv[q + k * kLdInv];
            P[i + (size_t)q * ld] = acc;
            if (GLOBAL) A[i + (size_t)(j0 + q) * ld] = acc;
          }
        }
      }
      __syncthreads();
      // trailing update of rows/cols >= r0: A[i,j] -= sum_k P[i,k] P[j,k] on the FP64 tensor cores,
      // one 8 x 8 lower tile per warp task (m8n8k4 DMMA, K = jw), C read-modify-written in place
      const int lane = tid & 31, g8 = lane >> 2, t4 = lane & 3;
      const int nb8 = (nr + 7) >> 3;
      const int jl = min(lim, c);                             // columns < jl are updated
      const int nbj = min(nb8, (jl - r0 + 7) >> 3);            // tile columns kept
      const int ntri = nbj * (nbj + 1) / 2, ntile = ntri + (nb8 - nbj) * nbj;
      constexpr int kB = 8;  // tiles per warp batch: their C loads are in flight together
      for (int t0 = wid * kB; t0 < ntile; t0 += (NT / 32) * kB) {
        double c0[kB], c1[kB];
        int ii[kB], jj[kB];
#pragma unroll
        for (int b = 0; b < kB; ++b) {
          const int t = t0 + b;
          int ti, tj;
          if (t < ntri) {  // triangle of the kept tile columns, then the rectangle below it
            ti = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
            while (ti * (ti + 1) / 2 > t) --ti;
            while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
            tj = t - ti * (ti + 1) / 2;
          } else {
            ti = nbj + (t - ntri) / nbj;
            tj = (t - ntri) % nbj;
          }
          ii[b] = t < ntile ? r0 + ti * 8 : c;  // c: empty tile
          jj[b] = r0 + tj * 8;
          const int i = ii[b] + g8, j = jj[b] + 2 * t4;
          const bool iv = i < c;
          c0[b] = (iv && j < jl && j <= i) ? A[i + (size_t)j * ld] : 0.0;
          c1[b] = (iv && j + 1 < jl && j + 1 <= i) ? A[i + (size_t)(j + 1) * ld] : 0.0;
        }
#pragma unroll
        for (int b = 0; b < kB; ++b) {
          const int ia = ii[b] + g8, ja = jj[b] + g8;
#pragma unroll 4
          for (int k0 = 0; k0 < jw; k0 += 4) {
            const int k = k0 + t4;
            const double av = (ia < c && k < jw) ? P[ia + (size_t)k * ld] : 0.0;
            const double bv = (ja < c && k < jw) ? P[ja + (size_t)k * ld] : 0.0;
            dmma_8x8x4(c0[b], c1[b], -av, bv);
          }
        }
#pragma unroll
        for (int b = 0; b < kB; ++b) {
          const int i = ii[b] + g8, j = jj[b] + 2 * t4;
          const bool iv = i < c;
          if (iv && j < jl && j <= i) A[i + (size_t)j * ld] = c0[b];
          if (iv && j + 1 < jl && j + 1 <= i) A[i + (size_t)(j + 1) * ld] = c1[b];
        }
      }
    }
    __syncthreads();
  }
  return -1;
}

// inverse of the 32 x 32 (jw valid) lower diagonal block M[J,J] at row jb, lane = column, into dst
// (ld kLdInv): one warp.  It does not depend on W, so the back substitution runs it one block ahead.
__device__ __noinline__ void warp_tri_inv32(const double* A, int lda, int jb, int jw, double* dst) {
  const int lane = threadIdx.x & 31;
  double x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    double sacc = (i == lane) ? 1.0 : 0.0;
#pragma unroll
    for (int k = 0; k < i; ++k) sacc -= ((i < jw && k < jw) ? A[(jb + i) + (size_t)(jb + k) * lda] : 0.0) * x[k];
    const double dii = (i < jw) ? A[(jb + i) + (size_t)(jb + i) * lda] : 1.0;
    x[i] = sacc / dii;
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) dst[i + lane * kLdInv] = i >= lane ? x[i] : 0.0;
}

// W (c x s, ld c) = M^{-T} [0; I_s]: blocked back substitution from the last 32-row block up.
// M lower (A, ld c).  Column t of W is nonzero only in rows <= u + t.
template <int NT>
__device__ void cta_backsub_last_rows(const double* A, double* W, int c, int s, const Scratch& sc, int lda = 0) {
  if (lda == 0) lda = c;  // leading dimension of M (W: ld c)
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const int u = c - s;
  for (int idx = tid; idx < c * s; idx += NT) {
    const int i = idx % c, t = idx / c;
    W[idx] = (i == u + t) ? 1.0 : 0.0;
  }
  const int nblk = (c + 31) / 32;
  // warp 0 inverts the diagonal block of step bI - 1 (into the other of two buffers; sc.l11 is free
  // after the Cholesky) while the other warps apply the DMMA update of step bI
  double* ibuf[2] = {sc.inv, sc.l11};
  constexpr int kUpdW = NT > 32 ? NT / 32 - 1 : 1;  // warps on the update
  if (wid == 0) warp_tri_inv32(A, lda, (nblk - 1) * 32, min(32, c - (nblk - 1) * 32), ibuf[(nblk - 1) & 1]);
  __syncthreads();
  for (int bI = nblk - 1; bI >= 0; --bI) {
    const int jb = bI * 32, jw = min(32, c - jb);
    const int t0 = jb > u ? jb - u : 0;  // columns t < t0 are zero in rows >= jb
    const int ns = s - t0;
    // W[J, t] -= sum_{i >= jb+jw} M[i, jb+q] W[i, t]
    const int lo = jb + jw;
    if (NT > 32 && wid == 0) {
      if (bI > 0) warp_tri_inv32(A, lda, jb - 32, 32, ibuf[(bI - 1) & 1]);
    } else if (lo < c && ns > 0) {
      // DMMA 8 x 8 tiles (q block x t block), K = c - lo; rows i > u + t of W are zero, so the
      // full K range adds nothing there
      const int g8 = lane >> 2, t4 = lane & 3;
      const int nq8 = (jw + 7) >> 3, nt8 = (ns + 7) >> 3, K = c - lo;
      for (int task = (NT > 32 ? wid - 1 : 0); task < nq8 * nt8; task += kUpdW) {
        const int qb = (task % nq8) * 8, tb = t0 + (task / nq8) * 8;
        const int qa = qb + g8, ta = tb + g8;
        const double* Ap = A + lo + (size_t)(jb + qa) * lda;
        const double* Bp = W + lo + (size_t)ta * c;
        double c0 = 0.0, c1 = 0.0;
#pragma unroll 4
        for (int k0 = 0; k0 < K; k0 += 4) {
          const int k = k0 + t4;
          const double av = (qa < jw && k < K) ? Ap[k] : 0.0;
          const double bv = (ta < s && k < K) ? Bp[k] : 0.0;
          dmma_8x8x4(c0, c1, av, bv);
        }
        const int q = qb + g8, t = tb + 2 * t4;
        if (q < jw && t < s) W[jb + q + (size_t)t * c] -= c0;
        if (q < jw && t + 1 < s) W[jb + q + (size_t)(t + 1) * c] -= c1;
      }
    }
    __syncthreads();
    const double* binv = ibuf[bI & 1];
    // W[J, t] = M[J,J]^{-T} W[J, t]:  W_new[q] = sum_{p >= q} inv[p][q] W_old[p], one thread per column t
    for (int t = t0 + tid; t < s; t += NT) {
      double w[32];
#pragma unroll
      for (int p = 0; p < 32; ++p) w[p] = p < jw ? W[jb + p + (size_t)t * c] : 0.0;
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        if (q < jw) {
          double acc = 0.0;
#pragma unroll
          for (int p = q; p < 32; ++p) acc += binv[p + q * kLdInv] * w[p];
          W[jb + q + (size_t)t * c] = acc;
        }
      }
    }
    __syncthreads();
  }
}

template <int NT>
__global__ void __launch_bounds__(NT) alg1_kernel(CliqueArgs a, const int32_t* __restrict__ list, int pbytes) {
  extern __shared__ double smem[];
  __shared__ double inv[32 * kLdInv], l11[32 * kLdInv];
  __shared__ int flag;
  const int r = list[blockIdx.x];
  const int f = a.super_ptr[r], s = a.sns[r], c = a.snc[r], u = c - s;
  const bool glob = a.ws_off[r] >= 0;
  double* A = glob ? a.ws + a.ws_off[r] : smem;
  double* W = A + (size_t)c * c;
  const int tid = threadIdx.x;
  const int64_t* __restrict__ colptr = a.colptr;
  const double* __restrict__ X = a.vals;

  // Step 2-1: A = P_r X-bar_{C_rC_r} P_r^T, lower triangle (A[i'+j'c] = X[c-1-i', c-1-j']).
  const int64_t uo = a.umap_off[r];
  for (int idx = tid; idx < c * c; idx += NT) {
    const int ip = idx % c, jp = idx / c;
    if (ip < jp) continue;
    const int ai = c - 1 - ip, bi = c - 1 - jp;  // ai <= bi: need X[bi, ai] (lower)
    double v;
    if (ai < s) {
      v = X[colptr[f + ai] + (bi - ai)];
    } else {
      const int64_t ap = ai - s, bp = bi - s;
      v = X[a.umap[uo + ap * u - ap * (ap - 1) / 2 + (bp - ap)]];
    }
    A[idx] = v;
  }
  __syncthreads();
  // global cliques: the current 32-column panel goes to shared memory if it fits, else after W
  double* panel = ((size_t)c * 32 * sizeof(double) <= (size_t)pbytes) ? smem : W + (size_t)c * s;
  Scratch sc{inv, l11, panel, &flag};
  // Step 2-2: Cholesky A = M M^T
  int fail = glob ? cta_chol_partial<NT, true>(A, c, c, sc) : cta_chol_partial<NT, false>(A, c, c, sc);
  if (fail >= 0) {
    if (tid == 0) report_error(a.err, r);
    return;
  }
  // Step 2-3 (first |S_r| columns only): M^T W = [0; I_s]
  cta_backsub_last_rows<NT>(A, W, c, s, sc);

  // Step 3: L-hat[a, t] = W[c-1-a, s-1-t]; unit form L = L-hat / L-hat_tt, D = L-hat_tt^2.
  double* Lp = a.Lp + a.panel_off[r];
  for (int idx = tid; idx < c * s; idx += NT) {
    const int ar = idx % c, t = idx / c;
    const double dg = W[(c - 1 - t) + (size_t)(s - 1 - t) * c];
    double v;
    if (ar > t) v = W[(c - 1 - ar) + (size_t)(s - 1 - t) * c] / dg;
    else v = (ar == t) ? 1.0 : 0.0;
    Lp[idx] = v;
  }
  for (int t = tid; t < s; t += NT) {
    const double dg = W[(c - 1 - t) + (size_t)(s - 1 - t) * c];
    a.D[f + t] = dg * dg;
  }
}

template <int NT>
__global__ void __launch_bounds__(NT) mf_kernel(CliqueArgs a, const int32_t* __restrict__ list, int pbytes) {
  extern __shared__ double smem[];
  __shared__ double inv[32 * kLdInv], l11[32 * kLdInv];
  __shared__ int flag;
  const int r = list[blockIdx.x];
  const int f = a.super_ptr[r], s = a.sns[r], c = a.snc[r], u = c - s;
  const bool glob = a.ws_off[r] >= 0;
  double* F = glob ? a.ws + a.ws_off[r] : smem;
  const int tid = threadIdx.x;
  const int64_t* __restrict__ colptr = a.colptr;

  // frontal matrix: pivot columns from Y on E, the U x U block starts at zero (pre-pass fronts
  // already hold the extend-add of their children: add instead of overwrite)
  const bool pre = a.pre[r] != 0;
  for (int idx = tid; idx < c * c; idx += NT) {
    const int i = idx % c, j = idx / c;
    const double yv = (j < s && i >= j) ? a.vals[colptr[f + j] + (i - j)] : 0.0;
    if (pre) F[idx] += yv;
    else F[idx] = yv;
  }
  __syncthreads();
  // extend-add of the children's update matrices, one child at a time in a fixed order (warp per
  // column; the columns of one child map to distinct columns of F): deterministic summation order, so
  // L_Y, D_Y and B are bitwise reproducible
  {
    const int c0 = pre ? 0 : a.child_ptr[r], c1 = pre ? 0 : a.child_ptr[r + 1];
    const int lane = tid & 31, wid = tid >> 5;
    for (int q = c0; q < c1; ++q) {
      const int ch = a.child_list[q];
      const int uc = a.snc[ch] - a.sns[ch];
      const int32_t* rel = a.relind + a.relind_off[ch];
      const double* Uc = a.upd + a.upd_off[ch];
      for (int ib = wid; ib < uc; ib += NT / 32) {
        double* Fc = F + (size_t)rel[ib] * c;
        const double* Ucol = Uc + (size_t)ib * uc;
        for (int ia = ib + lane; ia < uc; ia += 32) Fc[rel[ia]] += Ucol[ia];
      }
      __syncthreads();
    }
  }
  // Cholesky of the |S_r| pivot columns (L~ = L D^{1/2}) with the Schur complement in F_UU
  double* panel = ((size_t)c * 32 * sizeof(double) <= (size_t)pbytes) ? smem : F + (size_t)c * c + (size_t)c * s;
  Scratch sc{inv, l11, panel, &flag};
  const int fail = glob ? cta_chol_partial<NT, true>(F, c, s, sc) : cta_chol_partial<NT, false>(F, c, s, sc);
  if (fail >= 0) {
    if (tid == 0) report_error(a.err, f + fail);
    return;
  }
  double* Lp = a.Lp + a.panel_off[r];
  for (int idx = tid; idx < c * s; idx += NT) {
    const int ar = idx % c, t = idx / c;
    const double dg = F[t + (size_t)t * c];
    Lp[idx] = ar > t ? F[idx] / dg : (ar == t ? 1.0 : 0.0);
  }
  for (int t = tid; t < s; t += NT) {
    const double dg = F[t + (size_t)t * c];
    a.D[f + t] = dg * dg;
  }
  if (u > 0) {
    double* Ur = a.upd + a.upd_off[r];
    for (int idx = tid; idx < u * u; idx += NT) {
      const int ia = idx % u, ib = idx / u;
      Ur[idx] = ia >= ib ? F[(s + ia) + (size_t)(s + ib) * c] : 0.0;
    }
  }
}

// (a2) pre-pass for global fronts with many children (the block-arrow border front has 200): CTA (front,
// q) zeroes the front's columns of chunk q and adds, child by child in a fixed order, the children's
// update columns that land there (warp per column, distinct columns within a child, a barrier between
// children).  Columns are owned by one CTA: no atomics, deterministic summation order.
constexpr int kPreChunks = 128;  // column ranges per front: parallelism of the fixed-order child loop
__global__ void __launch_bounds__(256) pre_extend_add_kernel(CliqueArgs a, const int32_t* __restrict__ list) {
  const int r = list[blockIdx.x];
  const int c = a.snc[r];
  double* F = a.ws + a.ws_off[r];
  const int j0 = (int)((int64_t)c * blockIdx.y / kPreChunks), j1 = (int)((int64_t)c * (blockIdx.y + 1) / kPreChunks);
  for (int64_t i = threadIdx.x; i < (int64_t)(j1 - j0) * c; i += blockDim.x) F[(int64_t)j0 * c + i] = 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int q = a.child_ptr[r]; q < a.child_ptr[r + 1]; ++q) {
    const int ch = a.child_list[q];
    const int uc = a.snc[ch] - a.sns[ch];
    const int32_t* rel = a.relind + a.relind_off[ch];
    const double* Uc = a.upd + a.upd_off[ch];
    // child columns ib with rel[ib] in [j0, j1) (rel ascending: a contiguous range)
    int lo = 0, hi = uc;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (rel[mid] < j0) lo = mid + 1;
      else hi = mid;
    }
    for (int ib = lo + wid; ib < uc && rel[ib] < j1; ib += blockDim.x / 32) {
      double* __restrict__ Fc = F + (size_t)rel[ib] * c;
      const double* __restrict__ Ucol = Uc + (size_t)ib * uc;
      for (int ia = ib + lane; ia < uc; ia += 32) Fc[rel[ia]] += Ucol[ia];
    }
    __syncthreads();
  }
}

// (a2) big fronts (global workspace), one front over many CTAs: the pre-pass assembles the front
// (zero + children's extend-add, column ranges per CTA); front_panel_kernel (one CTA per front) adds
// Y's pivot columns and factors the |S_r| pivot columns only (L~ = L D^{1/2} in place, L_Y, D_Y out);
// front_schur_kernel (64 x 64 tiles of the update matrix over CTAs) forms U_r = F_UU - L~_U L~_U^T on the
// tensor cores straight into the update-matrix storage.  Same arithmetic as mf_kernel,
// with the Schur complement no longer streamed through a single SM.
constexpr int kThinS = 32;  // fronts with at most this many pivots: front_thin_kernel
#ifndef SDPC_PANEL_NT
#define SDPC_PANEL_NT 512
#endif
constexpr int kPanelNT = SDPC_PANEL_NT;  // threads of front_panel_kernel (one CTA per front)

template <int NT>
__global__ void __launch_bounds__(NT) front_panel_kernel(CliqueArgs a, const int32_t* __restrict__ list, int pbytes) {
  extern __shared__ double smem[];
  __shared__ double inv[32 * kLdInv], l11[32 * kLdInv];
  __shared__ int flag;
  const int r = list[blockIdx.x];
  const int f = a.super_ptr[r], s = a.sns[r], c = a.snc[r];
  if (s <= kThinS) return;  // front_thin_kernel
  double* F = a.ws + a.ws_off[r];
  const int tid = threadIdx.x;
  const int64_t* __restrict__ colptr = a.colptr;
  // Y's pivot columns into the front: a thread owns row i and takes 8 columns at a time, loads first
  // (a column-by-column loop exposes one memory round trip per pivot column to the whole CTA)
  {
    const double* __restrict__ vals = a.vals;
    for (int i = tid; i < c; i += NT) {
      const int jm = min(i, s - 1);
      for (int j0 = 0; j0 <= jm; j0 += 8) {
        double y[8], fv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (j0 + u <= jm) {
            y[u] = vals[colptr[f + j0 + u] - (j0 + u) + i];
            fv[u] = F[i + (size_t)(j0 + u) * c];
          }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (j0 + u <= jm) F[i + (size_t)(j0 + u) * c] = fv[u] + y[u];
      }
    }
  }
  __syncthreads();
  double* panel = ((size_t)c * 32 * sizeof(double) <= (size_t)pbytes) ? smem : F + (size_t)c * c + (size_t)c * s;
  Scratch sc{inv, l11, panel, &flag};
  const int fail = cta_chol_partial<NT, true>(F, c, s, sc, s);
  if (fail >= 0) {
    if (tid == 0) report_error(a.err, f + fail);
    return;
  }
  // L_Y = L~ D^{-1/2}, D_Y = diag(L~)^2 out: row-owning threads, 8 pivot columns per batch of loads
  __syncthreads();
  double* __restrict__ Lp = a.Lp + a.panel_off[r];
  for (int ar = tid; ar < c; ar += NT) {
    for (int t0 = 0; t0 < s; t0 += 8) {
      double dgv[8], fv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (t0 + u < s) {
          dgv[u] = F[(t0 + u) + (size_t)(t0 + u) * c];
          fv[u] = F[ar + (size_t)(t0 + u) * c];
        }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (t0 + u < s) {
          const int t = t0 + u;
          const double rdg = 1.0 / dgv[u];
          Lp[ar + (size_t)t * c] = ar > t ? fv[u] * rdg : (ar == t ? 1.0 : 0.0);
        }
    }
  }
  for (int t = tid; t < s; t += NT) {
    const double dg = F[t + (size_t)t * c];
    a.D[f + t] = dg * dg;
  }
}

constexpr int kSchurT = 64, kSchurK = 32, kSchurLd = kSchurT + 4;
__global__ void __launch_bounds__(256) front_schur_kernel(CliqueArgs a, const int32_t* __restrict__ list) {
  __shared__ __align__(16) double As[kSchurK * kSchurLd], Bs[kSchurK * kSchurLd];
  const int r = list[blockIdx.y];
  const int s = a.sns[r], c = a.snc[r], u = c - s;
  const int nt = (u + kSchurT - 1) / kSchurT;
  const int t = blockIdx.x;
  if (s <= kThinS || t >= nt * (nt + 1) / 2 || *(const volatile int32_t*)a.err != kNoError) return;
  int ti = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while (ti * (ti + 1) / 2 > t) --ti;
  while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
  const int tj = t - ti * (ti + 1) / 2;
  const double* F = a.ws + a.ws_off[r];
  double* Ur = a.upd + a.upd_off[r];
  const int a0 = ti * kSchurT, b0 = tj * kSchurT;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int g8 = lane >> 2, t4 = lane & 3;
  const int wm = wid & 1, wn = wid >> 1;  // warp tile: rows 32 wm .. +32, columns 16 wn .. +16
  double acc[4][2][2];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 2; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  for (int k0 = 0; k0 < s; k0 += kSchurK) {
    __syncthreads();
    for (int q = tid; q < kSchurK * kSchurT; q += 256) {
      const int kk = q / kSchurT, i = q % kSchurT;
      const bool kv = k0 + kk < s;
      As[kk * kSchurLd + i] = (kv && a0 + i < u) ? F[(s + a0 + i) + (size_t)(k0 + kk) * c] : 0.0;
      Bs[kk * kSchurLd + i] = (kv && b0 + i < u) ? F[(s + b0 + i) + (size_t)(k0 + kk) * c] : 0.0;
    }
    __syncthreads();
#pragma unroll 2
    for (int k4 = 0; k4 < kSchurK; k4 += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int x = 0; x < 4; ++x) af[x] = As[(k4 + t4) * kSchurLd + 32 * wm + 8 * x + g8];
#pragma unroll
      for (int y = 0; y < 2; ++y) bf[y] = Bs[(k4 + t4) * kSchurLd + 16 * wn + 8 * y + g8];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 2; ++y) dmma_8x8x4(acc[x][y][0], acc[x][y][1], af[x], bf[y]);
    }
  }
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const int ia = a0 + 32 * wm + 8 * x + g8;
#pragma unroll
    for (int y = 0; y < 2; ++y)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int ib = b0 + 16 * wn + 8 * y + 2 * t4 + e;
        if (ia < u && ib <= ia) Ur[ia + (size_t)ib * u] = F[(s + ia) + (size_t)(s + ib) * c] - acc[x][y][e];
      }
  }
}

// (a1) big cliques (global workspace), Algorithm 1 over many CTAs: Step 2-1 (gather of the reversed
// clique matrix) by CTAs owning column ranges; Step 2-2 (Cholesky M M^T) by the batched task kernels
// of k_chol_dag.cu (POTRF / TRSM / UPD steps over every big clique at once); Step 2-3 (last |S_r| rows
// of M^{-1}) and Step 3 by one CTA per clique.  The same arithmetic as alg1_kernel.
// Workspace of big clique b: A (c x ld, ld = c + (c & 1), 16-byte aligned) then W (c x s, ld c).
constexpr int kBigGatherChunks = 32;
__global__ void __launch_bounds__(256) big_gather_kernel(CliqueArgs a, const int32_t* __restrict__ list,
                                                         const int64_t* __restrict__ off, double* base) {
  const int r = list[blockIdx.y];
  const int f = a.super_ptr[r], s = a.sns[r], c = a.snc[r], u = c - s, ld = c + (c & 1);
  double* A = base + off[blockIdx.y];
  const int j0 = (int)((int64_t)c * blockIdx.x / kBigGatherChunks), j1 = (int)((int64_t)c * (blockIdx.x + 1) / kBigGatherChunks);
  const int64_t uo = a.umap_off[r];
  for (int jp = j0; jp < j1; ++jp)
    for (int ip = jp + threadIdx.x; ip < c; ip += blockDim.x) {
      const int ai = c - 1 - ip, bi = c - 1 - jp;  // ai <= bi: X[bi, ai] (lower)
      double v;
      if (ai < s) {
        v = a.vals[a.colptr[f + ai] + (bi - ai)];
      } else {
        const int64_t ap = ai - s, bp = bi - s;
        v = a.vals[a.umap[uo + ap * u - ap * (ap - 1) / 2 + (bp - ap)]];
      }
      A[ip + (size_t)jp * ld] = v;
    }
}

__global__ void __launch_bounds__(256) big_backsub_kernel(CliqueArgs a, const int32_t* __restrict__ list,
                                                          const int64_t* __restrict__ off, double* base,
                                                          const int32_t* __restrict__ err_slot) {
  __shared__ double inv[32 * kLdInv], l11[32 * kLdInv];
  __shared__ int flag;
  const int b = blockIdx.x;
  if (err_slot[b] != kNoError) return;
  const int r = list[b];
  const int f = a.super_ptr[r], s = a.sns[r], c = a.snc[r], ld = c + (c & 1);
  const double* A = base + off[b];
  double* W = base + off[b] + (size_t)c * ld;
  Scratch sc{inv, l11, nullptr, &flag};
  cta_backsub_last_rows<256>(A, W, c, s, sc, ld);
  const int tid = threadIdx.x;
  double* __restrict__ Lp = a.Lp + a.panel_off[r];
  for (int idx0 = tid; idx0 < c * s; idx0 += 256 * 4) {  // 4 elements per batch of (global) loads
    double dg[4], wv[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = idx0 + e * 256;
      if (idx < c * s) {
        const int ar = idx % c, t = idx / c;
        dg[e] = W[(c - 1 - t) + (size_t)(s - 1 - t) * c];
        wv[e] = W[(c - 1 - ar) + (size_t)(s - 1 - t) * c];
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = idx0 + e * 256;
      if (idx < c * s) {
        const int ar = idx % c, t = idx / c;
        Lp[idx] = ar > t ? wv[e] / dg[e] : (ar == t ? 1.0 : 0.0);
      }
    }
  }
  for (int t = tid; t < s; t += 256) {
    const double dg = W[(c - 1 - t) + (size_t)(s - 1 - t) * c];
    a.D[f + t] = dg * dg;
  }
}

// Thin big fronts (|S_r| <= 32, e.g. the separator chain of a 3D torus: s ~ 8-13, |C_r| ~ 1,400-2,900):
// pivot panel and update matrix in ONE launch.  Every CTA (a 64 x 64 tile of U_r) factors the s x s
// pivot block F_SS + Y_SS itself (one warp, registers: a few microseconds), forms the L~ rows of its
// tile rows and columns, L~_U = F_US L~_SS^{-T}, and applies U_r = F_UU - L~_U L~_U^T on the tensor cores;
// diagonal tiles also write their L rows (unit form) and CTA 0 the pivot block and D_Y.  Same arithmetic
// as front_panel_kernel + front_schur_kernel.
__global__ void __launch_bounds__(256) front_thin_kernel(CliqueArgs a, const int32_t* __restrict__ list) {
  __shared__ __align__(16) double As[kSchurK * kSchurLd], Bs[kSchurK * kSchurLd];
  __shared__ double inv[32 * kLdInv], dg[32];
  __shared__ int flag;
  double* a11 = Bs;  // the pivot block and the warp's staging square live in Bs / As until the L~ rows
  const int r = list[blockIdx.y];
  const int f = a.super_ptr[r], s = a.sns[r], c = a.snc[r], u = c - s;
  if (s > kThinS) return;
  const int nt = (u + kSchurT - 1) / kSchurT;
  const int t = blockIdx.x;
  if (t >= max(1, nt * (nt + 1) / 2)) return;
  const double* F = a.ws + a.ws_off[r];
  const double* __restrict__ Y = a.vals;
  const int64_t* __restrict__ colptr = a.colptr;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // pivot block F_SS + Y_SS (lower), factored and inverted by warp 0
  for (int idx = tid; idx < 32 * 32; idx += 256) {
    const int i = idx & 31, j = idx >> 5;
    a11[i + j * kLdInv] = (i < s && j < s && i >= j) ? F[i + (size_t)j * c] + Y[colptr[f + j] + (i - j)] : 0.0;
  }
  __syncthreads();
  Scratch sc{inv, As, nullptr, &flag};
  if (wid == 0) warp_chol_inv32(a11, kLdInv, 0, s, sc);
  __syncthreads();
  if (flag >= 0) {
    if (t == 0 && tid == 0) report_error(a.err, f + flag);
    return;
  }
  double* Lp = a.Lp + a.panel_off[r];
  if (t == 0) {  // pivot block rows of the unit-form panel, D_Y
    for (int idx = tid; idx < s * s; idx += 256) {
      const int ar = idx % s, k = idx / s;
      Lp[ar + (size_t)k * c] = ar > k ? a11[ar + k * kLdInv] / a11[k + k * kLdInv] : (ar == k ? 1.0 : 0.0);
    }
    for (int k = tid; k < s; k += 256) a.D[f + k] = a11[k + k * kLdInv] * a11[k + k * kLdInv];
  }
  if (tid < 32) dg[tid] = tid < s ? a11[tid + tid * kLdInv] : 1.0;
  __syncthreads();  // a11 (Bs) and the staging square (As) are overwritten below
  int ti = 0, tj = 0;
  if (u > 0) {
    ti = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while (ti * (ti + 1) / 2 > t) --ti;
    while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
    tj = t - ti * (ti + 1) / 2;
  }
  const int a0 = ti * kSchurT, b0 = tj * kSchurT;
  // L~ rows: L~[s + a][k] = sum_{q <= k} (F + Y)[s + a][q] Linv[k][q]   (inv(k, q) at inv[k + q * kLdInv])
  for (int idx = tid; idx < 2 * kSchurT * kSchurK; idx += 256) {
    const int which = idx / (kSchurT * kSchurK), rem = idx % (kSchurT * kSchurK);
    const int i = rem % kSchurT, k = rem / kSchurT;
    const int aa = (which ? b0 : a0) + i;
    double v = 0.0;
    if (aa < u && k < s) {
      const int row = s + aa;
      for (int q = 0; q <= k; ++q) v += (F[row + (size_t)q * c] + Y[colptr[f + q] + (row - q)]) * inv[k + q * kLdInv];
    }
    (which ? Bs : As)[k * kSchurLd + i] = v;
  }
  __syncthreads();
  if (u == 0) return;
  if (ti == tj)
    for (int idx = tid; idx < kSchurT * s; idx += 256) {
      const int i = idx % kSchurT, k = idx / kSchurT;
      if (a0 + i < u) Lp[(s + a0 + i) + (size_t)k * c] = As[k * kSchurLd + i] / dg[k];
    }
  double* Ur = a.upd + a.upd_off[r];
  const int g8 = lane >> 2, t4 = lane & 3;
  const int wm = wid & 1, wn = wid >> 1;
  double acc[4][2][2];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 2; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
#pragma unroll 2
  for (int k4 = 0; k4 < kSchurK; k4 += 4) {
    if (k4 >= s) break;
    double af[4], bf[2];
#pragma unroll
    for (int x = 0; x < 4; ++x) af[x] = As[(k4 + t4) * kSchurLd + 32 * wm + 8 * x + g8];
#pragma unroll
    for (int y = 0; y < 2; ++y) bf[y] = Bs[(k4 + t4) * kSchurLd + 16 * wn + 8 * y + g8];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y) dmma_8x8x4(acc[x][y][0], acc[x][y][1], af[x], bf[y]);
  }
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const int ia = a0 + 32 * wm + 8 * x + g8;
#pragma unroll
    for (int y = 0; y < 2; ++y)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int ib = b0 + 16 * wn + 8 * y + 2 * t4 + e;
        if (ia < u && ib <= ia) Ur[ia + (size_t)ib * u] = F[(s + ia) + (size_t)(s + ib) * c] - acc[x][y][e];
      }
  }
}

static CliqueArgs base_args(sdpc_ctx* h) {
  CliqueArgs a{};
  a.super_ptr = h->d.super_ptr;
  a.snc = h->d.snc;
  a.sns = h->d.sns;
  a.colptr = h->d.colptr;
  a.panel_off = h->d.panel_off;
  a.umap_off = h->d.umap_off;
  a.umap = h->d.umap;
  a.ws_off = h->d_ws_off;
  a.ws = h->ws;
  a.err = h->d_err;
  a.child_ptr = h->d.child_ptr;
  a.child_list = h->d.child_list;
  a.relind_off = h->d.relind_off;
  a.relind = h->d.relind;
  a.upd_off = h->d.upd_off;
  a.upd = h->upd;
  a.pre = h->d_pre;
  return a;
}

template <int NT, bool ALG1>
static void launch_one(const CliqueArgs& a, const CliqueClass& k, cudaStream_t st) {
  static std::atomic<uint64_t> attr{0};
  auto fn = ALG1 ? alg1_kernel<NT> : mf_kernel<NT>;
  if (once_per_device(attr)) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  fn<<<(unsigned)k.sn.size(), NT, k.smem, st>>>(a, k.d_sn, (int)k.smem);
}

template <bool ALG1>
static int launch_classes(const CliqueArgs& a, const std::vector<CliqueClass>& cls, cudaStream_t st) {
  int n = 0;
  for (const auto& k : cls) {
    if (k.sn.empty()) continue;
    switch (k.threads) {
      case 64: launch_one<64, ALG1>(a, k, st); break;
      case 128: launch_one<128, ALG1>(a, k, st); break;
      case 256: launch_one<256, ALG1>(a, k, st); break;
      default: launch_one<512, ALG1>(a, k, st); break;
    }
    ++n;
  }
  return n;
}

static void ensure_side_streams(sdpc_ctx* h) {
  if (h->side[0]) return;
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  for (int q = 0; q < 2; ++q)
    for (int i = 0; i < 4; ++i) {
      // set 1 carries (a2) inside sdpc_iteration: high priority like its parent stream
      cudaStreamCreateWithPriority(&h->sides[q][i], cudaStreamNonBlocking, q == 1 ? hi : lo);
      cudaEventCreateWithFlags(&h->sides_ev[q][i], cudaEventDisableTiming);
    }
  for (int i = 0; i < 4; ++i) {
    h->side[i] = h->sides[0][i];
    h->side_ev[i] = h->sides_ev[0][i];
  }
  cudaEventCreateWithFlags(&h->fork_ev, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&h->fork_ev2, cudaEventDisableTiming);
}

int launch_alg1(sdpc_ctx* h, const double* xbar, cudaStream_t st) {
  CliqueArgs a = base_args(h);
  a.vals = xbar;
  a.Lp = h->Lx;
  a.D = h->Dx;
  // the cliques are independent (Algorithm 1 works clique by clique): the size classes run
  // concurrently on side streams, so the many small cliques fill the SMs the few big ones leave idle
  ensure_side_streams(h);
  cudaEventRecord(h->fork_ev, st);
  int n = 0;
  for (int q = 0; q < (int)h->a1cls.size() && q < 4; ++q) {
    cudaStreamWaitEvent(h->side[q], h->fork_ev, 0);
    if (q == 3 && h->nbig1 > 0) {  // global-workspace cliques: the multi-CTA big-clique pipeline
      cudaStream_t s3 = h->side[q];
      cudaMemsetAsync(h->big1_err, 0x7f, (size_t)h->nbig1 * sizeof(int32_t), s3);
      big_gather_kernel<<<dim3(kBigGatherChunks, h->nbig1), 256, 0, s3>>>(a, h->a1cls[3].d_sn, h->big1_off, h->big1_ws);
      BatchDesc d{h->big1_ws, h->big1_off, h->big1_dim, h->big1_err, h->a1cls[3].d_sn, h->d_err, h->big1_linv};
      n += 2;
      for (int stp = 0; 128 * stp < h->big1_c[0]; ++stp) {
        int nact = 0;
        while (nact < h->nbig1 && h->big1_c[nact] > 128 * stp) ++nact;
        n += batched_chol_step(d, stp, nact, h->big1_c[0], s3);
      }
      big_backsub_kernel<<<h->nbig1, 256, 0, s3>>>(a, h->a1cls[3].d_sn, h->big1_off, h->big1_ws, h->big1_err);
      cudaEventRecord(h->side_ev[q], s3);
      cudaStreamWaitEvent(st, h->side_ev[q], 0);
      continue;
    }
    std::vector<CliqueClass> one(1, h->a1cls[q]);
    n += launch_classes<true>(a, one, h->side[q]);
    one[0].d_sn = nullptr;  // not owned here
    cudaEventRecord(h->side_ev[q], h->side[q]);
    cudaStreamWaitEvent(st, h->side_ev[q], 0);
  }
  return n;
}

int launch_ldl_y(sdpc_ctx* h, const double* y, cudaStream_t st, int32_t* err, int set) {
  CliqueArgs a = base_args(h);
  a.ws = h->ws2;  // own workspace: (a2) may run concurrently with (a1)
  if (err) a.err = err;
  a.vals = y;
  a.Lp = h->Ly;
  a.D = h->Dy;
  // levels are sequential (a front needs its children's update matrices); the size classes of one
  // level are independent fronts and run concurrently on the side streams
  ensure_side_streams(h);
  int n = 0;
  for (int lvi = 0; lvi < (int)h->a2lev.size(); ++lvi) {
    const auto& lev = h->a2lev[lvi];
    const int z0 = h->zero_ptr[lvi], z1 = h->zero_ptr[lvi + 1];
    if (z1 > z0) {
      pre_extend_add_kernel<<<dim3(z1 - z0, kPreChunks), 256, 0, st>>>(a, h->d_zero_list + z0);
      n += 1;
    }
    int used = 0;
    for (const auto& k : lev) used += k.sn.empty() ? 0 : 1;
    const int b0 = h->big_ptr[lvi], nbig = h->big_ptr[lvi + 1] - b0;
    if (nbig == 0 && used <= 1) {
      n += launch_classes<false>(a, lev, st);
      continue;
    }
    cudaEvent_t fk = set ? h->fork_ev2 : h->fork_ev;
    if (used > 0) cudaEventRecord(fk, st);
    if (nbig > 0) {  // big fronts on the level's own stream, concurrent with the class kernels
      static std::atomic<uint64_t> attr{0};
      if (once_per_device(attr))
        cudaFuncSetAttribute(front_panel_kernel<kPanelNT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      if (h->big_wide[lvi]) {
        front_panel_kernel<kPanelNT><<<nbig, kPanelNT, h->big_smem, st>>>(a, h->d_big_list + b0, (int)h->big_smem);
        if (h->big_tiles[lvi] > 0)
          front_schur_kernel<<<dim3(h->big_tiles[lvi], nbig), 256, 0, st>>>(a, h->d_big_list + b0);
        n += 1 + (h->big_tiles[lvi] > 0);
      }
      if (h->big_thin[lvi]) {
        front_thin_kernel<<<dim3(std::max(1, h->big_tiles[lvi]), nbig), 256, 0, st>>>(a, h->d_big_list + b0);
        n += 1;
      }
    }
    for (int q = 0; q < (int)lev.size() && q < 4; ++q) {
      if (lev[q].sn.empty()) continue;
      cudaStreamWaitEvent(h->sides[set][q], fk, 0);
      std::vector<CliqueClass> one(1, lev[q]);
      n += launch_classes<false>(a, one, h->sides[set][q]);
      one[0].d_sn = nullptr;
      cudaEventRecord(h->sides_ev[set][q], h->sides[set][q]);
      cudaStreamWaitEvent(st, h->sides_ev[set][q], 0);
    }
  }
  return n;
}

}  // namespace sdpc
