// Microbenchmark (not product code): the task-graph kernel's POTRF task alone in a one-CTA kernel, per-phase
// globaltimer stamps, at two register budgets (launch bounds (256, 2) as in the product, and (256, 1)).
#include "../paper_1310_6919_b200/csrc/k_chol_dag.cu"

namespace sdpc {
namespace dag {
template <int MINB>
__global__ void __launch_bounds__(kThreads, MINB) potrf_only(Args a, int k) {
  extern __shared__ double sm[];
  const long long c0 = clock64();
  const unsigned long long g0 = gtimer();
  run_potrf(a, k, sm);
  __syncthreads();
  if (threadIdx.x == 0) {
    a.ptrace[15] = clock64() - c0;
    a.ptrace[14] = gtimer() - g0;
  }
}
}  // namespace dag
}  // namespace sdpc

int main() {
  using namespace sdpc;
  using namespace sdpc::dag;
  const int m = 256, ld = 256;
  std::vector<double> hB((size_t)m * ld, 0.0);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j <= i; ++j) hB[i + (size_t)j * ld] = (i == j ? m : 0.0) + 1.0 / (1.0 + i + j);
  double *B, *Linv;
  unsigned long long* pt;
  int32_t* err;
  cudaMalloc(&B, hB.size() * 8);
  cudaMalloc(&Linv, 2 * NB * NB * 8);
  cudaMalloc(&pt, 64 * 8);
  cudaMemset(pt, 0, 64 * 8);
  cudaMalloc(&err, 4);
  Args a{};
  a.B = B;
  a.ld = ld;
  a.m = m;
  a.T = 2;
  a.Linv = Linv;
  a.err = err;
  a.ptrace = pt;
  cudaFuncSetAttribute(potrf_only<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem * 8);
  cudaFuncSetAttribute(potrf_only<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem * 8);
  const char* names[] = {"load", "p0", "p1", "p2", "p3", "Lstore", "Linv"};
  for (int v = 0; v < 2; ++v) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemcpy(B, hB.data(), hB.size() * 8, cudaMemcpyHostToDevice);
      cudaMemset(err, 0x7f, 4);
      if (v == 0) potrf_only<2><<<1, kThreads, kSmem * 8>>>(a, 0);
      else potrf_only<1><<<1, kThreads, kSmem * 8>>>(a, 0);
      cudaDeviceSynchronize();
    }
    unsigned long long h[16];
    cudaMemcpy(h, pt, 128, cudaMemcpyDeviceToHost);
    printf("launch_bounds(256,%d): total %.1f us |", v == 0 ? 2 : 1, (h[7] - h[0]) / 1e3);
    for (int i = 0; i < 7; ++i) printf(" %s %.1f", names[i], (h[i + 1] - h[i]) / 1e3);
    printf(" | inverse pairs:");
    unsigned long long prev = h[6];
    for (int i = 9; i < 15; ++i) { printf(" %.1f", (h[i] - prev) / 1e3); prev = h[i]; }
    printf(" write-out %.1f | %llu clk in %llu ns = %.0f MHz", (h[7] - h[8]) / 1e3, h[15], h[14], 1e3 * h[15] / (double)h[14]);
    printf("  (%s)\n", cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
