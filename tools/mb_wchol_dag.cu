// Microbenchmark (not product code): clock cycles of the task-graph POTRF's 32 x 32 warp Cholesky +
// inverse (dag::wchol32) and of the inverse alone (dag::wtrtri32), one warp, operands in shared memory.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 [-DSDPC_WCHOL_V2=0|1] tools/mb_wchol_dag.cu
#include "../paper_1310_6919_b200/csrc/k_chol_dag.cu"

namespace sdpc {
namespace dag {
__global__ void wchol_only(const double* g, long long* cyc, double* out) {
  __shared__ double A[32 * 132];
  __shared__ double W[32 * 36 + 64 + 32];
  for (int i = threadIdx.x; i < 32 * 132; i += blockDim.x) A[i] = g[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  long long t0 = clock64(), t1 = 0, t2 = 0;
  int r = 0;
  if (threadIdx.x < 32) {
    r = wchol32(A, 132, W + 32 * 36 + 64, W, W + 32 * 36, lane);
    __syncwarp();
    t1 = clock64();
    wtrtri32(A, 132, W + 32 * 36 + 64, W, W + 32 * 36, lane);
    __syncwarp();
    t2 = clock64();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
  }
  if (threadIdx.x < 32) out[lane] = A[lane + lane * 132] + W[lane] + r;
}
}  // namespace dag
}  // namespace sdpc

int main() {
  double h[32 * 132];
  for (int i = 0; i < 32; ++i)
    for (int j = 0; j < 132; ++j) h[i + 32 * 0 + j * 0] = 0;
  for (int j = 0; j < 32; ++j)
    for (int i = 0; i < 32; ++i) h[i + j * 132] = (i == j ? 40.0 : 0.0) + 1.0 / (1 + i + j);
  double *g, *o;
  long long* c;
  cudaMalloc(&g, sizeof h);
  cudaMalloc(&o, 32 * 8);
  cudaMalloc(&c, 16);
  cudaMemcpy(g, h, sizeof h, cudaMemcpyHostToDevice);
  long long hc[2];
  for (int rep = 0; rep < 5; ++rep) sdpc::dag::wchol_only<<<1, 256>>>(g, c, o);
  cudaMemcpy(hc, c, 16, cudaMemcpyDeviceToHost);
  printf("SDPC_WCHOL_V2=%d: wchol32 (factor + inverse) %lld clk, wtrtri32 (inverse only) %lld clk (%s)\n",
         SDPC_WCHOL_V2, hc[0], hc[1], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
