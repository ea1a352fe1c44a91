// Microbenchmark (not product code): one-warp 32x32 Cholesky (+ inverse) variants in shared memory.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rsqrt_nr(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  y = y * (1.5 - 0.5 * d * y * y);
  y = y * (1.5 - 0.5 * d * y * y);
  return y;
}
constexpr int LD = 36;

// V1: lane = row in registers, columns by shuffles (current product code)
__device__ void v1(double* Ab, int lane) {
  double row[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) row[c] = c <= lane ? Ab[lane + c * LD] : 0.0;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const double d = __shfl_sync(0xffffffffu, row[j], j);
    const double rl = rsqrt_nr(d);
    row[j] *= rl;
#pragma unroll
    for (int k = j + 1; k < 32; ++k) row[k] = fma(-row[j], __shfl_sync(0xffffffffu, row[j], k), row[k]);
  }
#pragma unroll
  for (int c = 0; c < 32; ++c)
    if (c <= lane) Ab[lane + c * LD] = row[c];
}

// V2: lane = row in registers, the scaled column broadcast through shared memory (LDS.128)
__device__ void v2(double* Ab, double* col, int lane) {
  double row[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) row[c] = c <= lane ? Ab[lane + c * LD] : 0.0;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    // pivot: lane j's diagonal, broadcast via shared memory
    if (lane == j) col[32 + (j & 1)] = row[j];
    __syncwarp();
    const double d = col[32 + (j & 1)];
    const double rl = rsqrt_nr(d);
    row[j] *= rl;
    col[lane] = row[j];
    __syncwarp();
#pragma unroll
    for (int k = j + 1; k < 32; ++k) row[k] = fma(-row[j], col[k], row[k]);
    __syncwarp();
  }
#pragma unroll
  for (int c = 0; c < 32; ++c)
    if (c <= lane) Ab[lane + c * LD] = row[c];
}

// V3: 256 threads, column steps on the 32x32 block in shared memory
__device__ void v3(double* Ab, int tid) {
  for (int j = 0; j < 32; ++j) {
    const double d = Ab[j + j * LD];
    const double rl = rsqrt_nr(d);
    __syncthreads();
    if (tid >= j && tid < 32) Ab[tid + j * LD] *= rl;
    __syncthreads();
    // trailing update: (31-j)(32-j)/2 elements
    const int n = 31 - j;
    for (int e = tid; e < n * n; e += blockDim.x) {
      const int r = j + 1 + e % n, c = j + 1 + e / n;
      if (r >= c) Ab[r + c * LD] -= Ab[r + j * LD] * Ab[c + j * LD];
    }
  }
  __syncthreads();
}

// inverse of the lower factor, lane = column, right-looking (current product code)
__device__ void inv1(const double* Ab, double* X, int lane) {
  double x[32];
  double rinv = 1.0 / Ab[lane + lane * LD];
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = (i == lane) ? 1.0 : 0.0;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    x[i] *= __shfl_sync(0xffffffffu, rinv, i);
#pragma unroll
    for (int k = i + 1; k < 32; ++k) x[k] -= Ab[k + i * LD] * x[i];
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) X[i * 33 + lane] = x[i];
}

template <int V>
__global__ void kern(const double* in, double* out, long long* cyc, int reps) {
  __shared__ double A[32 * LD];
  __shared__ double col[64];
  __shared__ double X[32 * 33];
  const int tid = threadIdx.x, lane = tid & 31;
  long long tot = 0, tinv = 0;
  for (int r = 0; r < reps; ++r) {
    for (int e = tid; e < 1024; e += blockDim.x) A[(e & 31) + (e >> 5) * LD] = in[e];
    __syncthreads();
    long long t0 = clock64();
    if (V == 1 && tid < 32) v1(A, lane);
    if (V == 2 && tid < 32) v2(A, col, lane);
    if (V == 3) v3(A, tid);
    __syncthreads();
    long long t1 = clock64();
    if (tid < 32) inv1(A, X, lane);
    __syncthreads();
    long long t2 = clock64();
    tot += t1 - t0;
    tinv += t2 - t1;
  }
  for (int e = tid; e < 1024; e += blockDim.x) out[e] = A[(e & 31) + (e >> 5) * LD] + 1e-300 * X[e];
  if (tid == 0) {
    cyc[0] = tot / reps;
    cyc[1] = tinv / reps;
  }
}

int main() {
  double h[1024];
  for (int i = 0; i < 32; ++i)
    for (int j = 0; j < 32; ++j) h[i + 32 * j] = (i == j ? 40.0 : 0.0) + 1.0 / (1 + i + j);
  double *in, *out;
  long long *cyc, hc[2];
  cudaMalloc(&in, 8192);
  cudaMalloc(&out, 8192);
  cudaMalloc(&cyc, 16);
  cudaMemcpy(in, h, 8192, cudaMemcpyHostToDevice);
  double ref[1024];
  for (int v = 1; v <= 3; ++v) {
    for (int w = 0; w < 2; ++w) {
      if (v == 1) kern<1><<<1, 256>>>(in, out, cyc, 20);
      if (v == 2) kern<2><<<1, 256>>>(in, out, cyc, 20);
      if (v == 3) kern<3><<<1, 256>>>(in, out, cyc, 20);
    }
    cudaMemcpy(hc, cyc, 16, cudaMemcpyDeviceToHost);
    double o[1024];
    cudaMemcpy(o, out, 8192, cudaMemcpyDeviceToHost);
    if (v == 1) for (int e = 0; e < 1024; ++e) ref[e] = o[e];
    double err = 0;
    for (int i = 0; i < 32; ++i)
      for (int j = 0; j <= i; ++j) err = fmax(err, fabs(o[i + 32 * j] - ref[i + 32 * j]));
    printf("V%d: factor %lld clk, inverse %lld clk, max diff vs V1 %.2e (%s)\n", v, hc[0], hc[1], err,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
