// Shared device/host helpers for libsdpc kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>
#include <cstdio>

namespace sdpc {

// True the first time it is called for the current device with this flag set (kernel attributes such as
// the dynamic shared-memory opt-in are per device: a handle on a second GPU must set them again).
inline bool once_per_device(std::atomic<uint64_t>& mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  return (mask.fetch_or(bit) & bit) == 0;
}

constexpr int kWarp = 32;
constexpr int kPanelW = 32;  // RHS panel width of the multi-RHS solves: lane <-> RHS column
constexpr int kScmNB = 256;  // tile size of the 2D block-cyclic distribution of B

// 2D block-cyclic ownership of B (ScaLAPACK convention, rank = myrow * Pc + mycol): tile (I, J) of
// size kScmNB lives on process (I mod Pr, J mod Pc) at local tile (I / Pr, J / Pc).  Pr = Pc = 1
// reduces to the plain column-major B.
struct Grid {
  int Pr = 1, Pc = 1, pr = 0, pc = 0;
  __host__ __device__ __forceinline__ bool own_row(int k) const { return (k / kScmNB) % Pr == pr; }
  __host__ __device__ __forceinline__ bool own_col(int l) const { return (l / kScmNB) % Pc == pc; }
  __host__ __device__ __forceinline__ int64_t lrow(int k) const {
    return Pr == 1 ? k : (int64_t)(k / kScmNB / Pr) * kScmNB + k % kScmNB;
  }
  __host__ __device__ __forceinline__ int64_t lcol(int l) const {
    return Pc == 1 ? l : (int64_t)(l / kScmNB / Pc) * kScmNB + l % kScmNB;
  }
};

// Device error flag protocol: kernels atomicMin the failing index into *err
// (initialised to kNoError by a byte memset).  Host reads it after the phase.
constexpr int32_t kNoError = 0x7f7f7f7f;  // = cudaMemset(.., 0x7f, 4)

__device__ __forceinline__ void report_error(int32_t* err, int32_t idx) { atomicMin(err, idx); }

// FP64 tensor-core MMA: D(8x8) = A(8x4, row) * B(4x8, col) + C.  Lowers to DMMA.8x8x4 on sm_100a.
// Fragments (PTX ISA, mma.m8n8k4 .f64): a = A[lane>>2][lane&3], b = B[lane&3][lane>>2],
// c/d = C[lane>>2][2*(lane&3) + {0,1}].
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// 1/sqrt(d) for a positive normal d without the library's out-of-line slow path (whose call forces
// live registers to the stack): MUFU seed (rsqrt.approx.f64) + two Newton steps, ~1 ulp.
__device__ __forceinline__ double rsqrt_nr(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  y = y * (1.5 - 0.5 * d * y * y);
  y = y * (1.5 - 0.5 * d * y * y);
  return y;
}

// 1/d for a positive normal d: MUFU seed (rcp.approx.f64) + two Newton steps (r += r (1 - d r)).
__device__ __forceinline__ double rcp_nr(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

}  // namespace sdpc
