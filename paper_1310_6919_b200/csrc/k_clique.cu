// Batched per-clique kernels: (a1) Algorithm 1 and (a2) multifrontal LDL^T of Y.
//
// (a1) PAPER.md P:493-530, Algorithm 1.  One CTA per clique r (fundamental supernode):
//      Step 2-1 gather P_r X-bar_{C_rC_r} P_r^T (reversal is index arithmetic),
//      Step 2-2 Cholesky = M_r M_r^T in shared memory (global workspace for big cliques),
//      Step 2-3 L_r = P_r M_r^{-T} P_r^T: only its first |S_r| columns are needed (Step 3),
//      i.e. the last |S_r| rows of M_r^{-1}, obtained by back substitution M_r^T W = [0; I].
//      Output in the north-star unit form L-hat = L D^{1/2}: D_j = L-hat_jj^2, L = L-hat / L-hat_jj.
// (a2) PAPER.md P:221-225 / P:722-725 (type (v)): Y = L_Y D_Y L_Y^T on the same E, multifrontal:
//      frontal = Y[C_r, S_r] + extend-add of the children's update matrices, partial LDL^T of
//      the |S_r| pivot columns, Schur complement passed to the parent.  One launch per etree height.
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
};

template <int NT>
__global__ void __launch_bounds__(NT) alg1_kernel(CliqueArgs a, const int32_t* __restrict__ list) {
  extern __shared__ double smem[];
  __shared__ int bad;
  const int r = list[blockIdx.x];
  const int f = a.super_ptr[r], s = a.sns[r], c = a.snc[r], u = c - s;
  double* A = (a.ws_off[r] >= 0) ? a.ws + a.ws_off[r] : smem;
  double* W = A + (size_t)c * c;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int NW = NT / 32;
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
  for (int idx = tid; idx < c * s; idx += NT) {
    const int i = idx % c, t = idx / c;
    W[idx] = (i == u + t) ? 1.0 : 0.0;
  }
  if (tid == 0) bad = 0;
  __syncthreads();

  // Step 2-2: Cholesky A = M M^T (right-looking, lower).
  for (int k = 0; k < c; ++k) {
    if (tid == 0) {
      const double d = A[k + (size_t)k * c];
      if (!(d > 0.0)) bad = 1;
      else A[k + (size_t)k * c] = sqrt(d);
    }
    __syncthreads();
    if (bad) {
      if (tid == 0) report_error(a.err, r);
      return;
    }
    const double inv = 1.0 / A[k + (size_t)k * c];
    for (int i = k + 1 + tid; i < c; i += NT) A[i + (size_t)k * c] *= inv;
    __syncthreads();
    for (int j = k + 1 + wid; j < c; j += NW) {
      const double ajk = A[j + (size_t)k * c];
      for (int i = j + lane; i < c; i += 32) A[i + (size_t)j * c] -= A[i + (size_t)k * c] * ajk;
    }
    __syncthreads();
  }

  // Step 2-3 (first |S_r| columns only): M^T W = [0; I_s], back substitution.
  for (int jp = c - 1; jp >= 0; --jp) {
    const int t0 = jp > u ? jp - u : 0;  // W[jp, t] = 0 for u + t < jp
    const double inv = 1.0 / A[jp + (size_t)jp * c];
    for (int t = t0 + tid; t < s; t += NT) W[jp + (size_t)t * c] *= inv;
    __syncthreads();
    const int ns = s - t0;
    for (int idx = tid; idx < jp * ns; idx += NT) {
      const int i = idx % jp, t = t0 + idx / jp;
      W[i + (size_t)t * c] -= A[jp + (size_t)i * c] * W[jp + (size_t)t * c];
    }
    __syncthreads();
  }

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
__global__ void __launch_bounds__(NT) mf_kernel(CliqueArgs a, const int32_t* __restrict__ list) {
  extern __shared__ double smem[];
  __shared__ int bad;
  const int r = list[blockIdx.x];
  const int f = a.super_ptr[r], s = a.sns[r], c = a.snc[r], u = c - s;
  double* F = (a.ws_off[r] >= 0) ? a.ws + a.ws_off[r] : smem;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int NW = NT / 32;
  const int64_t* __restrict__ colptr = a.colptr;

  // frontal matrix: pivot columns from Y on E, the U x U block starts at zero
  for (int idx = tid; idx < c * c; idx += NT) {
    const int i = idx % c, j = idx / c;
    F[idx] = (j < s && i >= j) ? a.vals[colptr[f + j] + (i - j)] : 0.0;
  }
  if (tid == 0) bad = 0;
  __syncthreads();
  // extend-add of the children's update matrices (sequential over children: deterministic)
  for (int q = a.child_ptr[r]; q < a.child_ptr[r + 1]; ++q) {
    const int ch = a.child_list[q];
    const int uc = a.snc[ch] - a.sns[ch];
    const int32_t* rel = a.relind + a.relind_off[ch];
    const double* Uc = a.upd + a.upd_off[ch];
    for (int idx = tid; idx < uc * uc; idx += NT) {
      const int ia = idx % uc, ib = idx / uc;
      if (ia >= ib) F[rel[ia] + (size_t)rel[ib] * c] += Uc[idx];
    }
    __syncthreads();
  }
  // partial LDL^T of the |S_r| pivot columns
  for (int k = 0; k < s; ++k) {
    const double d = F[k + (size_t)k * c];
    if (!(d > 0.0)) {
      if (tid == 0) report_error(a.err, f + k);
      return;
    }
    const double inv = 1.0 / d;
    __syncthreads();
    for (int i = k + 1 + tid; i < c; i += NT) F[i + (size_t)k * c] *= inv;
    __syncthreads();
    for (int j = k + 1 + wid; j < c; j += NW) {
      const double ljd = F[j + (size_t)k * c] * d;
      for (int i = j + lane; i < c; i += 32) F[i + (size_t)j * c] -= F[i + (size_t)k * c] * ljd;
    }
    __syncthreads();
  }
  double* Lp = a.Lp + a.panel_off[r];
  for (int idx = tid; idx < c * s; idx += NT) {
    const int ar = idx % c, t = idx / c;
    Lp[idx] = ar > t ? F[idx] : (ar == t ? 1.0 : 0.0);
  }
  for (int t = tid; t < s; t += NT) a.D[f + t] = F[t + (size_t)t * c];
  if (u > 0) {
    double* Ur = a.upd + a.upd_off[r];
    for (int idx = tid; idx < u * u; idx += NT) {
      const int ia = idx % u, ib = idx / u;
      Ur[idx] = ia >= ib ? F[(s + ia) + (size_t)(s + ib) * c] : 0.0;
    }
  }
  (void)bad;
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
  return a;
}

template <int NT, bool ALG1>
static void launch_one(const CliqueArgs& a, const CliqueClass& k, cudaStream_t st) {
  static bool attr_done = false;
  auto fn = ALG1 ? alg1_kernel<NT> : mf_kernel<NT>;
  if (!attr_done) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024);
    attr_done = true;
  }
  fn<<<(unsigned)k.sn.size(), NT, k.smem, st>>>(a, k.d_sn);
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

int launch_alg1(sdpc_ctx* h, const double* xbar, cudaStream_t st) {
  CliqueArgs a = base_args(h);
  a.vals = xbar;
  a.Lp = h->Lx;
  a.D = h->Dx;
  return launch_classes<true>(a, h->a1cls, st);
}

int launch_ldl_y(sdpc_ctx* h, const double* y, cudaStream_t st) {
  CliqueArgs a = base_args(h);
  a.vals = y;
  a.Lp = h->Ly;
  a.D = h->Dy;
  int n = 0;
  for (const auto& lev : h->a2lev) n += launch_classes<false>(a, lev, st);
  return n;
}

}  // namespace sdpc
