// Latency microbenchmark (not product code): dependent chains of DMMA.8x8x4, DFMA, SHFL (double),
// LDS.64 and BAR.SYNC on one CTA, and DMMA issue rate with independent chains, in SM clocks.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int CH>
__global__ void k_dmma(double* out, long long* cyc, int n) {
  double c0[CH], c1[CH];
  for (int i = 0; i < CH; ++i) c0[i] = c1[i] = threadIdx.x * 1e-3 + i;
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999;
  long long t0 = clock64();
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) dmma(c0[i], c1[i], a, b);
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < CH; ++i) s += c0[i] + c1[i];
  out[threadIdx.x + blockIdx.x * blockDim.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_dfma(double* out, long long* cyc, int n) {
  double x = threadIdx.x * 1e-3, a = 1.0000001, b = 1e-9;
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) x = fma(x, a, b);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_shfl(double* out, long long* cyc, int n) {
  double x = threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 1e-9;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_shfl_tp(double* out, long long* cyc, int n) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  long long t0 = clock64();
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = __shfl_sync(0xffffffffu, x[i], (threadIdx.x + i) & 31);
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_lds(double* out, long long* cyc, int n) {
  __shared__ double sm[64];
  sm[threadIdx.x] = 0.0;
  sm[threadIdx.x + 32] = 0.0;
  __syncwarp();
  int idx = threadIdx.x & 31;
  long long t0 = clock64();
  double x = 0;
  for (int it = 0; it < n; ++it) {
    x += sm[idx];
    idx = ((int)x + threadIdx.x) & 31;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_bar(long long* cyc, int n) {
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

static long long get(long long* cyc) {
  long long h;
  cudaDeviceSynchronize();
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  return h;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&cyc, 8);
  const int n = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    k_dmma<1><<<1, 32>>>(out, cyc, n);
    printf("DMMA latency (1 chain, 1 warp): %.1f clk\n", (double)get(cyc) / n);
    k_dmma<4><<<1, 32>>>(out, cyc, n);
    printf("DMMA 4 chains, 1 warp: %.1f clk per DMMA\n", (double)get(cyc) / n / 4);
    k_dmma<8><<<1, 32>>>(out, cyc, n);
    printf("DMMA 8 chains, 1 warp: %.1f clk per DMMA\n", (double)get(cyc) / n / 8);
    k_dmma<16><<<1, 32>>>(out, cyc, n);
    printf("DMMA 16 chains, 1 warp: %.1f clk per DMMA\n", (double)get(cyc) / n / 16);
    k_dmma<8><<<1, 128>>>(out, cyc, n);
    printf("DMMA 8 chains, 4 warps: %.1f clk per warp-DMMA\n", (double)get(cyc) / n / 8);
    k_dmma<8><<<1, 256>>>(out, cyc, n);
    printf("DMMA 8 chains, 8 warps: %.1f clk per warp-DMMA\n", (double)get(cyc) / n / 8);
    k_dfma<<<1, 32>>>(out, cyc, n);
    printf("DFMA latency: %.1f clk\n", (double)get(cyc) / n);
    k_shfl<<<1, 32>>>(out, cyc, n);
    printf("SHFL(double)+DADD latency: %.1f clk\n", (double)get(cyc) / n);
    k_shfl_tp<<<1, 32>>>(out, cyc, n);
    printf("SHFL(double) throughput, 1 warp: %.1f clk per shuffle\n", (double)get(cyc) / n / 8);
    k_lds<<<1, 32>>>(out, cyc, n);
    printf("LDS.64 dependent (+DADD+cvt): %.1f clk\n", (double)get(cyc) / n);
    k_bar<<<1, 256>>>(cyc, n);
    printf("BAR.SYNC 256 threads: %.1f clk\n", (double)get(cyc) / n);
  }
  return 0;
}
