// Small support kernels: factor export (panels -> E), inverse-column export, diag(R),
// and the FP64 roof microbenchmarks (DMMA via mma.sync m8n8k4 f64, and DFMA).
#include <cuda_runtime.h>

#include "common.cuh"
#include "ctx.hpp"

namespace sdpc {

__global__ void panels_to_E_kernel(int64_t nnz, const int32_t* __restrict__ e2p, const double* __restrict__ P,
                                   double* __restrict__ E) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x)
    E[e] = P[e2p[e]];
}

int launch_panels_to_E(sdpc_ctx* h, const double* panels, double* E, cudaStream_t st) {
  int64_t nnz = h->S.nnzE();
  int blocks = (int)std::min<int64_t>((nnz + 255) / 256, 148 * 16);
  panels_to_E_kernel<<<blocks, 256, 0, st>>>(nnz, h->d.e2p, panels, E);
  return 1;
}

// out[o + c*n] = M_orig[o, col_c] for original row o; M is panel-major by RHS slot, rows in
// elimination order.  Every requested column has a slot (checked on the host).
__global__ void gather_columns_kernel(int n, int ncols, const int32_t* __restrict__ cols_new,
                                      const int32_t* __restrict__ slot_of, const int32_t* __restrict__ iperm,
                                      const double* __restrict__ Xh, const double* __restrict__ Yh, double* Xo,
                                      double* Yo) {
  const int c = blockIdx.y;
  const int j = slot_of[cols_new[c]];
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < n; o += gridDim.x * blockDim.x) {
    const int i = iperm[o];
    const size_t idx = ((size_t)(j >> 5) * n + i) * kPanelW + (j & 31);
    Xo[o + (size_t)c * n] = Xh[idx];
    Yo[o + (size_t)c * n] = Yh[idx];
  }
}

int launch_gather_columns(sdpc_ctx* h, const int32_t* d_cols_new, int32_t ncols, double* Xo, double* Yo,
                          cudaStream_t st) {
  dim3 grid((h->S.n + 255) / 256, ncols);
  gather_columns_kernel<<<grid, 256, 0, st>>>(h->S.n, ncols, d_cols_new, h->d.slot_of, h->d.iperm, h->Xh, h->Yh, Xo, Yo);
  return 1;
}

__global__ void diag_copy_kernel(const double* B, int64_t m, int64_t ld, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = B[i + i * ld];
}

int launch_diag_copy(double* B, int64_t m, int64_t ld, double* out, cudaStream_t st) {
  diag_copy_kernel<<<(int)std::min<int64_t>((m + 255) / 256, 1024), 256, 0, st>>>(B, m, ld, out);
  return 1;
}

// ---------------------------------------------------------------- FP64 roof microbenchmarks
__global__ void __launch_bounds__(256) dmma_peak_kernel(int iters, double* sink) {
  const int lane = threadIdx.x & 31;
  double a = 1.0 + 1e-9 * lane, b = 1.0 - 1e-9 * lane;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma_8x8x4(c[i][0], c[i][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) sink[0] = s;
}

__global__ void __launch_bounds__(256) dfma_peak_kernel(int iters, double* sink) {
  double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-12;
  double c[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 12345.678) sink[0] = s;
}

cudaError_t fp64_peak(int device, double ms, double* dmma, double* dfma) {
  cudaSetDevice(device);
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, device);
  const int sms = prop.multiProcessorCount;
  double* sink;
  cudaMalloc(&sink, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 4, threads = 256;
  auto run = [&](bool mma, int iters) {
    cudaEventRecord(e0);
    if (mma) dmma_peak_kernel<<<blocks, threads>>>(iters, sink);
    else dfma_peak_kernel<<<blocks, threads>>>(iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float t = 0;
    cudaEventElapsedTime(&t, e0, e1);
    return (double)t;
  };
  for (int pass = 0; pass < 2; ++pass) {
    const bool mma = pass == 0;
    int iters = 1000;
    run(mma, iters);
    double t = run(mma, iters);
    while (t < ms && iters < (1 << 28)) {
      iters = (int)std::min<double>((double)(1 << 28), iters * std::max(2.0, ms / std::max(t, 1e-3)));
      t = run(mma, iters);
    }
    const double warps = (double)blocks * threads / 32;
    const double flops = mma ? warps * iters * 8 * 512.0 : (double)blocks * threads * iters * 8 * 2.0;
    const double tf = flops / (t * 1e-3) / 1e12;
    if (mma) *dmma = tf;
    else *dfma = tf;
  }
  cudaFree(sink);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return cudaGetLastError();
}

}  // namespace sdpc
