// accuracy of rsqrt.approx.ftz.f64 (+ Newton steps) against correctly rounded 1/sqrt (diagnostic)
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
__global__ void k(const double* d, double* o, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x = d[i], y0;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(x));
  double y1 = y0 * (1.5 - 0.5 * x * y0 * y0);
  double y2 = y1 * (1.5 - 0.5 * x * y1 * y1);
  double h = 0.5 * x * y2; // refined: y3 = y2 + y2*(0.5 - x*y2*y2/2) with fma residual
  double r = fma(-x * y2, y2, 1.0);
  double y3 = fma(0.5 * y2, r, y2);
  o[4 * i] = y0; o[4 * i + 1] = y1; o[4 * i + 2] = y2; o[4 * i + 3] = y3;
  (void)h;
}
int main() {
  const int n = 1 << 16;
  double *d, *o; cudaMallocManaged(&d, n * 8); cudaMallocManaged(&o, 4 * n * 8);
  unsigned long long s = 88172645463325252ull;
  for (int i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; d[i] = 0.01 + 10.0 * (double)(s >> 11) / 9007199254740992.0; }
  k<<<n / 256, 256>>>(d, o, n); cudaDeviceSynchronize();
  double mx[4] = {0, 0, 0, 0};
  for (int i = 0; i < n; ++i) {
    long double ref = 1.0L / sqrtl((long double)d[i]);
    for (int t = 0; t < 4; ++t) { double e = (double)fabsl(((long double)o[4 * i + t] - ref) / ref); if (e > mx[t]) mx[t] = e; }
  }
  printf("max rel err: approx %.3e  NR1 %.3e  NR2 %.3e  NR2+fma-refine %.3e  (u = %.3e)\n", mx[0], mx[1], mx[2], mx[3], 1.1102230246251565e-16);
}
