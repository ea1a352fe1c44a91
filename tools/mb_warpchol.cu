// Microbenchmark: cycles of the 32x32 warp Cholesky + inverse used by the Cholesky diagonal kernel
// (variants: noinline generic pointers vs inline shared).  Build: nvcc -arch=sm_100a -O3.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kLdD = 132;
__device__ __forceinline__ double rsqrt_nr(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  y = y * (1.5 - 0.5 * d * y * y);
  y = y * (1.5 - 0.5 * d * y * y);
  return y;
}
__device__ __forceinline__ int chol_body(double* Ab, double (*Tinv)[33], int lane) {
  double row[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) row[c] = c <= lane ? Ab[lane + c * kLdD] : 0.0;
  int fail = -1;
  double rinv = 0.0;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const double d = __shfl_sync(0xffffffffu, row[j], j);
    if (fail < 0 && !(d > 0.0)) fail = j;
    const double rl = rsqrt_nr(d);
    if (lane == j) { row[j] = d * rl; rinv = rl; } else if (lane > j) { row[j] *= rl; }
#pragma unroll
    for (int k = j + 1; k < 32; ++k) {
      const double lkj = __shfl_sync(0xffffffffu, row[j], k);
      if (lane >= k) row[k] -= row[j] * lkj;
    }
  }
  if (fail >= 0) return fail;
#pragma unroll
  for (int c = 0; c < 32; ++c) if (c <= lane) Ab[lane + c * kLdD] = row[c];
  __syncwarp();
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
__device__ __noinline__ int chol_noinline(double* Ab, double (*Tinv)[33], int lane) { return chol_body(Ab, Tinv, lane); }
// factor only (no inverse)
__device__ __forceinline__ int factor_only(double* Ab, int lane) {
  double row[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) row[c] = c <= lane ? Ab[lane + c * kLdD] : 0.0;
  int fail = -1;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const double d = __shfl_sync(0xffffffffu, row[j], j);
    if (fail < 0 && !(d > 0.0)) fail = j;
    const double rl = rsqrt_nr(d);
    if (lane == j) row[j] = d * rl; else if (lane > j) row[j] *= rl;
#pragma unroll
    for (int k = j + 1; k < 32; ++k) {
      const double lkj = __shfl_sync(0xffffffffu, row[j], k);
      if (lane >= k) row[k] -= row[j] * lkj;
    }
  }
#pragma unroll
  for (int c = 0; c < 32; ++c) if (c <= lane) Ab[lane + c * kLdD] = row[c];
  return fail;
}
// factor with the scaled column broadcast through shared memory (no shuffles)
__device__ __forceinline__ int factor_lds(double* Ab, double* colbuf, int lane) {
  double row[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) row[c] = c <= lane ? Ab[lane + c * kLdD] : 0.0;
  int fail = -1;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    // lane j: pivot; everyone needs rl = 1/sqrt(d)
    if (lane == j) colbuf[32] = rsqrt_nr(row[j]);
    __syncwarp();
    const double rl = colbuf[32];
    const double lj = row[j] * rl;  // L[lane][j] for lane > j
    if (lane == j) row[j] = row[j] * rl;
    else if (lane > j) row[j] = lj;
    colbuf[lane] = lj;
    __syncwarp();
#pragma unroll
    for (int k = j + 1; k < 32; ++k)
      if (lane >= k) row[k] -= lj * colbuf[k];
    __syncwarp();
  }
#pragma unroll
  for (int c = 0; c < 32; ++c) if (c <= lane) Ab[lane + c * kLdD] = row[c];
  return fail;
}
// inverse only (L given in Ab, unit diag scaling by 1/L_ii from smem)
__device__ __forceinline__ void inverse_only(const double* Ab, double (*Tinv)[33], int lane) {
  double x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = (i == lane) ? 1.0 : 0.0;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    x[i] *= 1.0 / Ab[i + i * kLdD];
#pragma unroll
    for (int k = i + 1; k < 32; ++k) x[k] -= Ab[k + i * kLdD] * x[i];
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) Tinv[i][lane] = i >= lane ? x[i] : 0.0;
}
template <int V>
__global__ void k(const double* g, long long* cyc, double* out) {
  __shared__ double A[32 * kLdD];
  __shared__ double T[32][33];
  for (int i = threadIdx.x; i < 32 * kLdD; i += blockDim.x) A[i] = g[i];
  __syncthreads();
  long long t0 = clock64();
  int r = 0;
  if (threadIdx.x < 32) {
    if (V == 0) r = chol_noinline(A, T, threadIdx.x);
    else if (V == 1) r = chol_body(A, T, threadIdx.x);
    else if (V == 2) r = factor_only(A, threadIdx.x);
    else if (V == 4) r = factor_lds(A, &T[0][0], threadIdx.x);
    else inverse_only(A, T, threadIdx.x);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[V] = t1 - t0; out[V] = T[31][0] + r; }
}
int main() {
  double h[32 * kLdD];
  for (int i = 0; i < 32; ++i) for (int j = 0; j < 32; ++j) h[i + j * kLdD] = (i == j ? 40.0 : 0.0) + 1.0 / (1 + i + j);
  double *g, *o; long long* c;
  cudaMalloc(&g, sizeof h); cudaMalloc(&o, 64); cudaMalloc(&c, 64);
  cudaMemcpy(g, h, sizeof h, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep) { k<0><<<1, 256>>>(g, c, o); k<1><<<1, 256>>>(g, c, o); k<2><<<1, 256>>>(g, c, o); k<3><<<1, 256>>>(g, c, o); k<4><<<1, 256>>>(g, c, o); }
  long long hc[5]; cudaMemcpy(hc, c, 40, cudaMemcpyDeviceToHost);
  printf("warp_chol_inv32 cycles: noinline %lld, inline %lld, factor only %lld, inverse only %lld, factor lds %lld\n", hc[0], hc[1], hc[2], hc[3], hc[4]);
  return 0;
}
