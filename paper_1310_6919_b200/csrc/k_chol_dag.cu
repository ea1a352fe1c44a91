// (d) Dense FP64 Cholesky of the SCM, B = R R^T (lower, in place), as ONE persistent kernel that
// executes the tile task graph of the blocked right-looking factorisation.
// PAPER.md P:711-713 / P:735-736 (type (i): dense Cholesky of the SCM), P:978-979 (S-CHOLESKY).
//
// Tiles are 128 x 128 (T = ceil(m / 128) tile rows).  Tasks, each run by one 256-thread CTA:
//   POTRF(k)       factor tile (k, k) in shared memory and form L_kk^{-1} (kept in a workspace);
//   TRSM(i, k, r)  rows [64 r, 64 r + 64) of tile (i, k) <- A L_kk^{-T}  (GEMM with L_kk^{-1}, K = 128);
//   UPD(i, j, k, h) columns [64 h, 64 h + 64) of tile (i, j) -= L_ik L_jk^T (k < j <= i, K = 128).
// Dependencies are counted per task in global memory; a task whose last input completes is pushed on
// one of three ready queues (0: POTRF, TRSM and the update of the next panel's tile column, 1: the
// column after that, 2: the rest) and the CTAs of the persistent grid pop the most urgent ready task.
// This replaces round 1's 37 shrinking launches (each with a tail of partly idle SMs) and its fixed
// lookahead depth: the panel chain runs as soon as its inputs are ready, overlapped with the bulk of
// the trailing updates, and no CTA ever waits on a dependency while holding a task (a popped task is
// ready), so the scheme is deadlock-free whatever the number of co-resident CTAs.
//
// GEMMs: mma.sync m8n8k4 f64 (DMMA.8x8x4 on sm_100a; tcgen05 has no f64 kind), 8 warps x (32 x 32),
// operands staged by a double-buffered cp.async.cg pipeline of 32-deep k-chunks.  Data written by other CTAs is
// read only through L2 (cp.async.cg / ld.global.cg): L1 is not coherent across SMs.  Requires B
// 16-byte aligned with an even leading dimension (the caller falls back to the multi-launch schedule
// of k_potrf.cu otherwise).
// Non-PD: the first failing column (1-based, LAPACK potrf rule) is atomicMin'ed into *err; every CTA
// then leaves at its next pop (later panels depend on the failing one, so the index is the first).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "ctx.hpp"

namespace sdpc {
namespace dag {

constexpr int NB = 128;          // tile
constexpr int kThreads = 256;    // 8 warps
#ifndef SDPC_DAG_BK  // (16-deep x 4 stages measured 2.4% more update time on configs[1])
#define SDPC_DAG_BK 32
#define SDPC_DAG_STAGES 2
#endif
constexpr int kBK = SDPC_DAG_BK;          // k-chunk per pipeline stage
constexpr int kStages = SDPC_DAG_STAGES;
constexpr int kGemmSmem = kStages * kBK * ((NB + 4) + (NB / 2 + 4));  // doubles (both tile shapes)
// POTRF: the lower 128 x 128 tile as four packed 32-column panels (panel p = rows 32p..127, ld 132 - 32p),
// the diagonal of L^{-1}, the current 32 x 32 diagonal-block inverse as a full square (later the scratch
// block of the in-place L^{-1})
constexpr int kPackN = 32 * (132 + 100 + 68 + 36);
constexpr int kPotrfSmem = kPackN + NB + 32 * 36 + 64;  // (col: two 32-double broadcast buffers)
constexpr int kCtl = 32;         // uint32 stride between queue counters (one 128-byte line each)
constexpr int kQ = 5;            // ready queues
#ifndef SDPC_WCHOL_V2
#define SDPC_WCHOL_V2 1
#endif
#ifndef SDPC_DAG_BLOCKED_TRSM
#define SDPC_DAG_BLOCKED_TRSM 1
#endif
#ifndef SDPC_DAG_FUSED_DIAG
#define SDPC_DAG_FUSED_DIAG SDPC_DAG_BLOCKED_TRSM
#endif
#ifndef SDPC_DAG_CHAIN_SMS
#if SDPC_DAG_FUSED_DIAG
#define SDPC_DAG_CHAIN_SMS 4
#elif SDPC_DAG_BLOCKED_TRSM
#define SDPC_DAG_CHAIN_SMS 3
#else
#define SDPC_DAG_CHAIN_SMS 2
#endif
#endif
#ifndef SDPC_DAG_FRAG_PIPE  // explicit fragment double-buffering (volatile LDS): configs[1] 15.35 -> 15.30 ms, not kept
#define SDPC_DAG_FRAG_PIPE 0
#endif
#ifndef SDPC_DAG_MAX_STEPS
#define SDPC_DAG_MAX_STEPS 4
#endif
constexpr int kLX = 132;                                            // fused diagonal update: 16 staged columns
constexpr int kPotrfAll = kPotrfSmem + (SDPC_DAG_FUSED_DIAG ? 16 * kLX : 0);  // (<= 112 KB: 2 CTAs per SM)
constexpr int kSmem = kGemmSmem > kPotrfAll ? kGemmSmem : kPotrfAll;
constexpr int kChainSms = SDPC_DAG_CHAIN_SMS;  // SMs whose CTAs run only the panel chain
constexpr int kMaxSteps = SDPC_DAG_MAX_STEPS;  // an update task applies up to this many consecutive panel steps

enum : uint64_t { kPotrf = 1, kTrsm = 2, kUpd = 3 };

__host__ __device__ __forceinline__ uint64_t enc(uint64_t type, uint64_t h, uint64_t k, uint64_t i, uint64_t j) {
  return (type << 60) | (h << 56) | (k << 32) | (i << 16) | j;
}

struct Args {
  double* B;
  int64_t ld;
  int m, T;
  double* Linv;          // [T][NB * NB] column-major, zero above the diagonal.  SDPC_DAG_BLOCKED_TRSM:
                         // "Lmix" = the 32 x 32 diagonal blocks hold D_p^{-1} (the inverses of L's
                         // diagonal blocks), the blocks below hold L; otherwise L_kk^{-1}
  unsigned* pflag;       // [T] or null: column blocks of L_kk published so far by POTRF(k) (the chain
                         // TRSM(k + 1, k, *) is released when POTRF(k) starts and follows it block by block)
  unsigned* tflag;       // [2 T] or null (SDPC_DAG_FUSED_DIAG): column blocks of L_{k+1,k} rows [64 r, 64 r + 64)
                         // stored so far by TRSM(k + 1, k, r); POTRF(k + 1) is released when both start and
                         // applies the step-k update of its tile itself, block by block
  unsigned* ctl;         // head[q] = ctl[q * kCtl], tail[q] = ctl[(kQ + q) * kCtl]; ctl[2 kQ kCtl + r] = chain SM r;
                         // ctl[(2 kQ + 1) kCtl + q] = tasks of queue q absorbed into earlier updates (never pushed)
  uint64_t* slots[5];    // ready queues (see qof)
  int* cnt_p;            // [T]        POTRF(k) inputs seen
  int* cnt_t;            // [T(T-1)/2 x 2]  TRSM(i, k, r)
  int* cnt_u;            // [NU x 2]   UPD(i, j, k, h)
  const int64_t* koff;   // [T] first UPD index of step k
  unsigned total;        // number of tasks
  unsigned qcap[5];      // exact number of tasks each queue receives
  int32_t* err;
  unsigned long long* trace;  // optional: per task {task, t_start, t_end, smid} (globaltimer ns)
  unsigned long long* ptrace; // optional: [T][8] POTRF phase stamps
  unsigned* trace_n;
  unsigned trace_cap;
};

__device__ __forceinline__ int64_t tidx(int i, int k) { return (int64_t)i * (i - 1) / 2 + k; }  // i > k
__device__ __forceinline__ int64_t uidx(const Args& a, int k, int i, int j) {  // k < j <= i
  const int64_t r = i - k - 1;
  return a.koff[k] + r * (r + 1) / 2 + (j - k - 1);
}
__device__ __forceinline__ int need_t(int k) { return k > 0 ? 3 : 1; }
// POTRF(k), k >= 1: the two halves of UPD(k, k, k - 1); fused: the starts of TRSM(k, k - 1, *) and UPD(k, k, k - 2, *)
__device__ __forceinline__ int need_p(const Args& a, int k) {
  return (SDPC_DAG_FUSED_DIAG && a.tflag) ? 2 + (k >= 2 ? 2 : 0) : 2;
}
__device__ __forceinline__ int need_u(int i, int j, int k) { return (i != j ? 3 : 2) + (k > 0 ? 1 : 0); }
// Queue of a task.  The panel chain POTRF(k) -> TRSM(k+1, k, *) -> UPD(k+1, k+1, k, *) -> POTRF(k+1) is
// the critical path; it runs on the CTAs of kChainSms elected SMs that take nothing else, so the
// latency-bound POTRF never shares an SM's FP64 pipe with a bulk GEMM.  0: POTRF (chain CTAs),
// 1: the chain's TRSM / UPD tasks (chain CTAs), 2: the other TRSM tasks and the other updates of the
// next panel's tile column, 3: updates of the column after that, 4: the rest (2-4: bulk CTAs).
__device__ __forceinline__ int qof(uint64_t t) {
  const int type = (int)(t >> 60);
  const int k = (int)((t >> 32) & 0xffff), i = (int)((t >> 16) & 0xffff), j = (int)(t & 0xffff);
  if (type == kPotrf) return 0;
  if (type == kTrsm) return i == k + 1 ? 1 : 2;
  if (j == k + 1) return i == j ? 1 : 2;
  return j == k + 2 ? 3 : 4;
}

__device__ __forceinline__ void cp_async16_n(void* smem, const void* gmem, int bytes) {  // src bytes 0..16
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned ld_vol(const unsigned* p) { return *(const volatile unsigned*)p; }
__device__ __forceinline__ uint64_t ld_vol64(const uint64_t* p) { return *(const volatile uint64_t*)p; }

__device__ void push(const Args& a, uint64_t task) {
  const int q = qof(task);
  const unsigned t = atomicAdd(&a.ctl[(kQ + q) * kCtl], 1u);
  atomicExch(reinterpret_cast<unsigned long long*>(&a.slots[q][t]), (unsigned long long)task);
}

// one more input of a task is complete; the last one makes it ready
__device__ __forceinline__ void dep(const Args& a, int* cnt, int need, uint64_t task) {
  if (atomicAdd(cnt, 1) + 1 == need) {
    __threadfence();
    push(a, task);
  }
}

// Ticket queues.  A CTA takes a ticket (one atomicAdd on the queue head, never retried: no CAS
// contention among hundreds of CTAs) when the queue looks non-empty, and owns the task that lands in
// that slot.  It holds at most one ticket per queue; while waiting for a slot it keeps polling the other
// queues, so a held ticket never blocks a ready task elsewhere (no deadlock), and every ticket below the
// queue's exact capacity is eventually filled.  Returns the most urgent task whose slot is filled, or 0
// when every ticket is spent (or the factorisation failed).
constexpr unsigned kNone = 0xffffffffu, kSpent = 0xfffffffeu;

__device__ __forceinline__ unsigned live_cap(const Args& a, int q) {  // tasks queue q will still receive
  return a.qcap[q] - ld_vol(&a.ctl[(2 * kQ + 1) * kCtl + q]);
}

__device__ uint64_t pop(const Args& a, unsigned* tk, int q0, int q1) {  // tk: this CTA's tickets (shared)
  for (unsigned spin = 0;; ++spin) {
    if (*(const volatile int32_t*)a.err != kNoError) return 0;
    bool live = false;
#pragma unroll 1
    for (int q = q0; q < q1; ++q) {
      if (tk[q] == kSpent) continue;
      if (tk[q] == kNone) {
        const unsigned h = ld_vol(&a.ctl[q * kCtl]);
        if (h < ld_vol(&a.ctl[(kQ + q) * kCtl])) {
          const unsigned x = atomicAdd(&a.ctl[q * kCtl], 1u);
          tk[q] = x < a.qcap[q] ? x : kSpent;  // (slots beyond the static capacity are another queue's)
          if (tk[q] == kSpent) continue;
        } else {
          if (h < live_cap(a, q)) live = true;  // more tasks to come
          continue;
        }
      }
      const uint64_t v = ld_vol64(&a.slots[q][tk[q]]);
      if (v != 0) {
        tk[q] = kNone;
        __threadfence();
        return v;
      }
      if (tk[q] >= live_cap(a, q)) {
        tk[q] = kSpent;  // beyond the last task this queue will receive (heads only grow, capacities shrink)
      } else {
        live = true;
      }
    }
    if (!live) return 0;
    __nanosleep(spin < 8 ? 20 : 100);
  }
}

__device__ void notify(const Args& a, uint64_t task, int lane) {
  const int type = (int)(task >> 60), hh = (int)((task >> 56) & 15);
  const int k = (int)((task >> 32) & 0xffff), i = (int)((task >> 16) & 0xffff), j = (int)(task & 0xffff);
  const int T = a.T;
  if (type == kPotrf) {
    const int x0 = (SDPC_DAG_BLOCKED_TRSM && a.pflag) ? 2 : 0;  // TRSM(k + 1, k, *): released at the POTRF's start
    for (int x = x0 + lane; x < 2 * (T - k - 1); x += 32) {
      const int ii = k + 1 + (x >> 1), r = x & 1;
      dep(a, &a.cnt_t[2 * tidx(ii, k) + r], need_t(k), enc(kTrsm, r, k, ii, 0));
    }
  } else if (type == kTrsm) {
    // rows of L_ik are the A operand of UPD(i, j, k, *) for k < j <= i ...
    // (fused: the diagonal tile's update UPD(k + 1, k + 1, k, *) is done by POTRF(k + 1))
    const int xu0 = (SDPC_DAG_FUSED_DIAG && a.tflag && i == k + 1) ? 2 : 0;
    for (int x = xu0 + lane; x < 2 * (i - k); x += 32) {
      const int jj = k + 1 + (x >> 1), h = x & 1;
      dep(a, &a.cnt_u[2 * uidx(a, k, i, jj) + h], need_u(i, jj, k), enc(kUpd, h, k, i, jj));
    }
    // ... and rows [64 r, 64 r + 64) of L_ik the B operand of UPD(l, i, k, r) for l > i
    for (int l = i + 1 + lane; l < T; l += 32)
      dep(a, &a.cnt_u[2 * uidx(a, k, l, i) + hh], need_u(l, i, k), enc(kUpd, hh, k, l, i));
  } else if (lane == 0) {
    if (SDPC_DAG_FUSED_DIAG && a.tflag && i == j && j == k + 2) {
      dep(a, &a.cnt_p[j], need_p(a, j), enc(kPotrf, 0, j, j, j));
    } else if (j > k + 1) {
      dep(a, &a.cnt_u[2 * uidx(a, k + 1, i, j) + hh], need_u(i, j, k + 1), enc(kUpd, hh, k + 1, i, j));
    } else if (i == j) {
      dep(a, &a.cnt_p[k + 1], need_p(a, k + 1), enc(kPotrf, 0, k + 1, k + 1, k + 1));
    } else {
      dep(a, &a.cnt_t[2 * tidx(i, k + 1)], need_t(k + 1), enc(kTrsm, 0, k + 1, i, 0));
      dep(a, &a.cnt_t[2 * tidx(i, k + 1) + 1], need_t(k + 1), enc(kTrsm, 1, k + 1, i, 0));
    }
  }
}

__device__ __forceinline__ double neg(double x) {  // sign flip on the integer pipe
  return __hiloint2double(__double2hiint(x) ^ 0x80000000, __double2loint(x));
}

// ------------------------------------------------------------------ GEMM tasks
// UPD: C (BM x BN) <- C - A Bm^T; TRSM (in place, C == A allowed): C <- A Bm^T.  K = 128.
// A(i, kk) = A[i + kk lda], Bm(j, kk) = Bm[j + kk ldbm], C(i, j) = C[i + j ldc]; na / nbv valid rows of
// A (and C) / of Bm; a diagonal tile keeps j + doff <= i only (mask).
template <int BM, int BN, bool UPD>
__device__ __forceinline__ void tile_gemm(const double* A, int64_t lda, const double* Bm, int64_t ldbm, double* C,
                                          int64_t ldc, int na, int nbv, int doff, bool mask, int K, double* sm) {
  constexpr int LA = BM + 4, LB = BN + 4;  // conflict-free m8n8k4 fragment loads
  constexpr int WM = BM / 32;
  const int nk = K / kBK;  // K: a multiple of 128
  double* As = sm;
  double* Bs = sm + kStages * kBK * LA;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int wm = wid % WM, wn = wid / WM;
  const int g8 = lane >> 2, t4 = lane & 3;

  auto load_stage = [&](int stage, int k0) {
    double* as = As + stage * kBK * LA;
    double* bs = Bs + stage * kBK * LB;
#pragma unroll
    for (int q = 0; q < (kBK * BM / 2) / kThreads; ++q) {
      const int cid = tid + q * kThreads;
      const int kk = cid / (BM / 2), rp = (cid % (BM / 2)) * 2;
      const bool v = rp < na;
      cp_async16(as + kk * LA + rp, v ? A + rp + (int64_t)(k0 + kk) * lda : A, v);
    }
#pragma unroll
    for (int q = 0; q < (kBK * BN / 2) / kThreads; ++q) {
      const int cid = tid + q * kThreads;
      const int kk = cid / (BN / 2), rp = (cid % (BN / 2)) * 2;
      const bool v = rp < nbv;
      cp_async16(bs + kk * LB + rp, v ? Bm + rp + (int64_t)(k0 + kk) * ldbm : Bm, v);
    }
  };
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    load_stage(s, s * kBK);
    cp_async_commit();
  }
  // Tiles off the diagonal accumulate into C (the textbook update order).  A diagonal tile's
  // accumulators start at zero and C is added once in the epilogue: its O(1) entries meet the K-sum of
  // small products in one rounding per task instead of one per DMMA (which put the backward error of
  // B = R R^T at ~1e-14, 40x cuSOLVER's, entirely in the diagonal tiles); C is prefetched into L2 meanwhile.
  const bool cadd = UPD && mask;
  if (cadd)
    for (int q = tid; q < nbv * (BM / 16); q += kThreads) {
      const int c = q / (BM / 16), r = (q % (BM / 16)) * 16;
      if (r < na) prefetch_l2(C + r + (int64_t)c * ldc);
    }
  double acc[4][4][2];
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const int i = wm * 32 + x * 8 + g8;
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int jc = wn * 32 + y * 8 + 2 * t4 + e;
        acc[x][y][e] = (UPD && !mask && i < na && jc < nbv) ? __ldcg(C + i + (int64_t)jc * ldc) : 0.0;
      }
  }
  // a diagonal tile adds each 128-deep step's sum to C separately (the same rounding whatever the number
  // of steps a task applies: bitwise reproducible under the run-dependent absorption); each thread
  // owns its C entries, so no barrier is needed
  auto flush_c = [&]() {
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const int i = wm * 32 + x * 8 + g8;
#pragma unroll
      for (int y = 0; y < 4; ++y)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int jc = wn * 32 + y * 8 + 2 * t4 + e;
          if (i < na && jc < nbv && jc + doff <= i) {
            double* cp = C + i + (int64_t)jc * ldc;
            __stcg(cp, __ldcg(cp) + acc[x][y][e]);
          }
          acc[x][y][e] = 0.0;
        }
    }
  };
#pragma unroll 1
  for (int kc = 0; kc < nk; ++kc) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    const int nxt = kc + kStages - 1;
    if (nxt < nk) load_stage(nxt % kStages, nxt * kBK);
    cp_async_commit();
    const double* as = As + (kc % kStages) * kBK * LA;
    const double* bs = Bs + (kc % kStages) * kBK * LB;
#if SDPC_DAG_FRAG_PIPE
    // fragments of step k4 + 1 are loaded before the DMMAs of step k4 are issued (two register sets):
    // without this the compiler loads each B fragment right before the four DMMAs that use it
    double af[2][4], bf[2][4];
    const unsigned as_u = (unsigned)__cvta_generic_to_shared(as + t4 * LA + wm * 32 + g8);
    const unsigned bs_u = (unsigned)__cvta_generic_to_shared(bs + t4 * LB + wn * 32 + g8);
    auto ldfrag = [&](int buf, int k4) {  // volatile loads: kept in this order relative to the DMMAs
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        double v;
        asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(v) : "r"(as_u + (unsigned)((k4 * 4 * LA + x * 8) * 8)));
        af[buf][x] = UPD ? neg(v) : v;
      }
#pragma unroll
      for (int y = 0; y < 4; ++y)
        asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(bf[buf][y]) : "r"(bs_u + (unsigned)((k4 * 4 * LB + y * 8) * 8)));
    };
    ldfrag(0, 0);
#pragma unroll
    for (int k4 = 0; k4 < kBK / 4; ++k4) {
      if (k4 + 1 < kBK / 4) ldfrag((k4 + 1) & 1, k4 + 1);
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) dmma_8x8x4(acc[x][y][0], acc[x][y][1], af[k4 & 1][x], bf[k4 & 1][y]);
    }
#else
#pragma unroll
    for (int k4 = 0; k4 < kBK / 4; ++k4) {
      double af[4], bf[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const double v = as[(k4 * 4 + t4) * LA + wm * 32 + x * 8 + g8];
        af[x] = UPD ? neg(v) : v;
      }
#pragma unroll
      for (int y = 0; y < 4; ++y) bf[y] = bs[(k4 * 4 + t4) * LB + wn * 32 + y * 8 + g8];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) dmma_8x8x4(acc[x][y][0], acc[x][y][1], af[x], bf[y]);
    }
#endif
    if (cadd && (kc + 1) % (NB / kBK) == 0 && kc + 1 < nk) flush_c();
  }
  cp_async_wait<0>();
  if (!UPD) __syncthreads();  // in place: every warp has staged its A rows before any is overwritten
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const int i = wm * 32 + x * 8 + g8;
    if (i >= na) continue;
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int jc = wn * 32 + y * 8 + 2 * t4 + e;
        if (jc < nbv && (!mask || jc + doff <= i)) {
          double* cp = C + i + (int64_t)jc * ldc;
          __stcg(cp, cadd ? __ldcg(cp) + acc[x][y][e] : acc[x][y][e]);
        }
      }
  }
}

// steps k .. k + ns - 1 on tile (i, j), columns [64 h, 64 h + 64): K = 128 ns (tile columns k.. are adjacent)
__device__ __forceinline__ void run_upd(const Args& a, int k, int ns, int i, int j, int h, double* sm) {
  const int64_t ri = (int64_t)i * NB, cj = (int64_t)j * NB + h * 64, ck = (int64_t)k * NB;
  const int na = a.m - ri < NB ? (int)(a.m - ri) : NB;
  const int nbv = a.m - cj < 64 ? (int)(a.m - cj) : 64;
  if (nbv <= 0) return;
  const int doff = (int)(cj - ri);
  tile_gemm<NB, 64, true>(a.B + ri + ck * a.ld, a.ld, a.B + cj + ck * a.ld, a.ld, a.B + ri + cj * a.ld, a.ld, na, nbv,
                          doff, i == j, NB * ns, sm);
}

#if SDPC_DAG_BLOCKED_TRSM
// TRSM(i, k, r): rows [64 r, 64 r + 64) of tile (i, k) <- A L_kk^{-T}, by 32-column blocks against Lmix
// (forward substitution over the blocks, P:711-713 type (i) Cholesky): X_p = (A_p - sum_{q<p} X_q L_pq^T)
// D_p^{-T}.  Warp (wm, wn) owns rows 32 wm .. 32 wm + 31 of column block wn, in registers; X_p goes through
// shared memory (double-buffered) as the A operand of the later blocks' updates; column block p of Lmix
// (rows 32 p ..) is staged in shared memory per stage.  The chain TRSM (i == k + 1, a.pflag set) waits
// before stage p until POTRF(k) has published column block p, so it runs alongside its POTRF.
__device__ __forceinline__ void run_trsm(const Args& a, int k, int i, int r, double* sm) {
  constexpr int LX = 68, LL = 132;  // conflict-free fragment loads
  __shared__ int s_stop;
  const int64_t ri = (int64_t)i * NB + r * 64, ck = (int64_t)k * NB;
  const int na = a.m - ri < 64 ? (int)(a.m - ri) : 64;
  double* Ap = a.B + ri + ck * a.ld;
  const double* Lm = a.Linv + (int64_t)k * NB * NB;
  double* Xs = sm;             // [2][32 columns][LX]: X_p column-major, rows 0..63
  double* Ls = sm + 2 * 32 * LX;  // [32 columns][LL]: rows 32 p .. 127 of column block p of Lmix
  const bool early = a.pflag != nullptr && i == k + 1;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int wm = wid & 1, wn = wid >> 1;
  if (SDPC_DAG_FUSED_DIAG && early && a.tflag && tid == 0) {  // POTRF(k + 1) follows this TRSM block by block
    dep(a, &a.cnt_p[k + 1], need_p(a, k + 1), enc(kPotrf, 0, k + 1, k + 1, k + 1));
    if (na <= 0) {  // no rows (ragged last tile): nothing for POTRF(k + 1) to wait for
      __threadfence();
      atomicExch(a.tflag + 2 * k + r, 4u);
    }
  }
  if (na <= 0) return;
  const int g8 = lane >> 2, t4 = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const int row = 32 * wm + 8 * x + g8;
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = 32 * wn + 8 * y + 2 * t4 + e;
        acc[x][y][e] = row < na ? __ldcg(Ap + row + (int64_t)col * a.ld) : 0.0;
      }
  }
#pragma unroll 1
  for (int p = 0; p < 4; ++p) {
    if (early) {
      if (tid == 0) {
        unsigned spin = 0;
        while (ld_vol(a.pflag + k) < (unsigned)(p + 1) && *(const volatile int32_t*)a.err == kNoError)
          __nanosleep(spin++ < 16 ? 20 : 64);
        __threadfence();  // acquire: column block p of Lmix is visible
        s_stop = *(const volatile int32_t*)a.err != kNoError;
      }
    }
    __syncthreads();  // (also: every warp is done with the previous stage's Ls)
    if (early && s_stop) return;
    // column block p of Lmix, rows 32 p .. 127, into Ls (16-byte cp.async, pairs of rows)
    const int nrow2 = (NB - 32 * p) / 2;
    for (int c = tid; c < 32 * nrow2; c += kThreads) {
      const int col = c / nrow2, rr = 2 * (c % nrow2);
      cp_async16(Ls + rr + col * LL, Lm + (32 * p + rr) + (int64_t)(32 * p + col) * NB, true);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    double* X = Xs + (p & 1) * 32 * LX;
    if (wn == p) {
      // X_p = acc D_p^{-T}: acc to shared as the A operand, then B(kk, n) = D_p^{-1}[n][kk] from Ls
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            X[(8 * y + 2 * t4 + e) * LX + 32 * wm + 8 * x + g8] = acc[x][y][e];
            acc[x][y][e] = 0.0;
          }
      __syncwarp();
#pragma unroll
      for (int k4 = 0; k4 < 8; ++k4) {
        double af[4], bf[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) af[x] = X[(4 * k4 + t4) * LX + 32 * wm + 8 * x + g8];
#pragma unroll
        for (int y = 0; y < 4; ++y) bf[y] = Ls[(8 * y + g8) + (4 * k4 + t4) * LL];
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) dmma_8x8x4(acc[x][y][0], acc[x][y][1], af[x], bf[y]);
      }
      __syncwarp();
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const int row = 32 * wm + 8 * x + g8;
#pragma unroll
        for (int y = 0; y < 4; ++y)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int cl = 8 * y + 2 * t4 + e;
            X[cl * LX + row] = acc[x][y][e];
            if (row < na) __stcg(Ap + row + (int64_t)(32 * p + cl) * a.ld, acc[x][y][e]);
          }
      }
    }
    __syncthreads();
    if (SDPC_DAG_FUSED_DIAG && early && a.tflag && tid == 0) {  // column block p of these rows is stored
      __threadfence();
      atomicExch(a.tflag + 2 * k + r, (unsigned)(p + 1));
    }
    if (wn > p) {
      // acc -= X_p L_{wn,p}^T: B(kk, n) = L[32 wn + n][32 p + kk] at Ls row 32 (wn - p) + n
#pragma unroll
      for (int k4 = 0; k4 < 8; ++k4) {
        double af[4], bf[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) af[x] = neg(X[(4 * k4 + t4) * LX + 32 * wm + 8 * x + g8]);
#pragma unroll
        for (int y = 0; y < 4; ++y) bf[y] = Ls[(32 * (wn - p) + 8 * y + g8) + (4 * k4 + t4) * LL];
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) dmma_8x8x4(acc[x][y][0], acc[x][y][1], af[x], bf[y]);
      }
    }
  }
}
#else
__device__ __forceinline__ void run_trsm(const Args& a, int k, int i, int r, double* sm) {
  const int64_t ri = (int64_t)i * NB + r * 64, ck = (int64_t)k * NB;
  const int na = a.m - ri < 64 ? (int)(a.m - ri) : 64;
  if (na <= 0) return;
  double* Ap = a.B + ri + ck * a.ld;
  tile_gemm<64, NB, false>(Ap, a.ld, a.Linv + (int64_t)k * NB * NB, NB, Ap, a.ld, na, NB, 0, false, NB, sm);
}
#endif

// ------------------------------------------------------------------ POTRF task
__device__ __forceinline__ int pofs(int p) { return 32 * (132 * p - 16 * p * (p - 1)); }
__device__ __forceinline__ int pld(int p) { return 132 - 32 * p; }
// element (r, c) of the lower tile, r >= 32 (c / 32)
__device__ __forceinline__ double* pel(double* S, int r, int c) {
  const int p = c >> 5;
  return S + pofs(p) + (r - 32 * p) + (c & 31) * pld(p);
}

// warp shuffle of a double by inline PTX (the caller guarantees a converged warp)
__device__ __forceinline__ double shfl_d(double v, int src) {
  unsigned lo = __double2loint(v), hi = __double2hiint(v), rlo, rhi;
  asm volatile("shfl.sync.idx.b32 %0, %1, %2, 0x1f, 0xffffffff;" : "=r"(rlo) : "r"(lo), "r"(src));
  asm volatile("shfl.sync.idx.b32 %0, %1, %2, 0x1f, 0xffffffff;" : "=r"(rhi) : "r"(hi), "r"(src));
  return __hiloint2double((int)rhi, (int)rlo);
}

// Warp Cholesky + inverse of the 32 x 32 diagonal block at Ab (ld), lane = row with the row in registers.
// Per column: the pivot by one shuffle, the scaled column broadcast through shared memory (col, 16-byte
// aligned, 16-byte loads): no per-element shuffles (SHFL of a double costs ~9 clk of issue, and
// shuffles make ptxas emit a second, non-converged copy of the code).  Out: strict lower(Ab) <- L;
// ldiag[a] <- L[a][a]; upper(Ab) incl. the diagonal (row b, column a >= b) <- Linv[a][b];
// Dq[a * 33 + b] <- Linv[a][b] (zero above the diagonal).  Returns the failing local column or -1.
__device__ __forceinline__ int wchol32(double* Ab, int ld, double* ldiag, double* Dq, double* col, int lane) {
  double row[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) row[c] = c <= lane ? Ab[lane + c * ld] : 0.0;
  int fail = -1;
  double rinv = 0.0;
#if SDPC_WCHOL_V2
  // The critical chain per column is pivot (shuffle) -> 1/d (MUFU seed + two Newton FMAs) -> multiplier
  // -> update of the next pivot.  The column goes out UNSCALED (a_kj, independent of the pivot's
  // reciprocal), so its shared-memory round trip overlaps the reciprocal: a_ik -= (a_ij / d_j) a_kj.
  // The two broadcast buffers alternate (one warp barrier per column); 1/sqrt(d_j) scales row j's L
  // entry off the chain.
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const double d = shfl_d(row[j], j);
    fail = (fail < 0 && !(d > 0.0)) ? j : fail;
    double* cb = col + 32 * (j & 1);
    if (j < 31) cb[lane] = row[j];
    const double r = rcp_nr(d);
    const double rl = rsqrt_nr(d);
    rinv = lane == j ? rl : rinv;
    if (j < 31) {
      __syncwarp();
      const double s = row[j] * r;
      const double2* col2 = reinterpret_cast<const double2*>(cb);
      // lanes < k update entries above the diagonal, which are never read
#pragma unroll
      for (int k2 = (j + 1) / 2; k2 < 16; ++k2) {
        const double2 c = col2[k2];
        if (2 * k2 > j) row[2 * k2] = fma(-s, c.x, row[2 * k2]);
        row[2 * k2 + 1] = fma(-s, c.y, row[2 * k2 + 1]);
      }
    }
    row[j] *= rl;
  }
  __syncwarp();
#else
  const double2* col2 = reinterpret_cast<const double2*>(col);
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const double d = shfl_d(row[j], j);
    fail = (fail < 0 && !(d > 0.0)) ? j : fail;
    const double rl = rsqrt_nr(d);
    rinv = lane == j ? rl : rinv;
    row[j] *= rl;
    if (j < 31) {
      col[lane] = row[j];
      __syncwarp();
      // lanes < k update entries above the diagonal, which are never read
#pragma unroll
      for (int k2 = (j + 1) / 2; k2 < 16; ++k2) {
        const double2 c = col2[k2];
        if (2 * k2 > j) row[2 * k2] = fma(-row[j], c.x, row[2 * k2]);
        row[2 * k2 + 1] = fma(-row[j], c.y, row[2 * k2 + 1]);
      }
      __syncwarp();
    }
  }
#endif
  if (fail >= 0) return fail;
  double dl = 0.0;
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    if (c < lane) Ab[lane + c * ld] = row[c];
    dl = c == lane ? row[c] : dl;
  }
  ldiag[lane] = dl;
  col[lane] = rinv;
  __syncwarp();
  // inverse, lane = column c: right-looking forward substitution (x_i final at step i)
  double x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = (i == lane) ? 1.0 : 0.0;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    x[i] *= col[i];
#pragma unroll
    for (int k = i + 1; k < 32; ++k) x[k] -= Ab[k + i * ld] * x[i];
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    Dq[i * 33 + lane] = i >= lane ? x[i] : 0.0;
    if (i >= lane) Ab[lane + i * ld] = x[i];
  }
  return -1;
}

// Inverse only (the block is already factored): lower(Ab) incl. the diagonal holds L.  Outputs as wchol32.
__device__ __forceinline__ void wtrtri32(double* Ab, int ld, double* ldiag, double* Dq, double* col, int lane) {
  const double dl = Ab[lane + lane * ld];
  ldiag[lane] = dl;
  col[lane] = 1.0 / dl;
  __syncwarp();
  double x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = (i == lane) ? 1.0 : 0.0;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    x[i] *= col[i];
#pragma unroll
    for (int k = i + 1; k < 32; ++k) x[k] -= Ab[k + i * ld] * x[i];
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    Dq[i * 33 + lane] = i >= lane ? x[i] : 0.0;
    if (i >= lane) Ab[lane + i * ld] = x[i];
  }
}

// INV_ONLY: the tile is already a Cholesky factor (R of sdpc_scm_cholesky): only its inverse is formed
// (the SCE solve's diagonal-block inverses), also for the last tile.
template <bool INV_ONLY = false>
__device__ void run_potrf(const Args& a, int k, double* sm) {
  __shared__ int fail_col;
  const int k0 = k * NB, kb = a.m - k0 < NB ? a.m - k0 : NB;
  double* Bd = a.B + k0 + (int64_t)k0 * a.ld;
  double* S = sm;
  double* ldiag = sm + kPackN;  // diagonal of L (the block diagonals hold that of L^{-1})
  double* Dq = ldiag + NB;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int g8 = lane >> 2, t4 = lane & 3;
  unsigned long long* pt = a.ptrace ? a.ptrace + 16 * k : nullptr;
  if (pt && tid == 0) pt[0] = gtimer();
  // Lmix column blocks are published for the TRSMs of the panel below (not for the last tile)
  const bool publish = SDPC_DAG_BLOCKED_TRSM && !INV_ONLY && k + 1 < a.T;
  double* Lmx = a.Linv + (int64_t)k * NB * NB;
  if (publish && a.pflag && tid == 0)  // the chain TRSM(k + 1, k, *) follows this POTRF block by block
    for (int r = 0; r < 2; ++r) dep(a, &a.cnt_t[2 * tidx(k + 1, k) + r], need_t(k), enc(kTrsm, r, k, k + 1, 0));
  // the lower tile into the packed panels by 16-byte cp.async (pairs of rows of one column); chunks
  // entirely above the diagonal or outside the kb x kb tile are zero-filled
  for (int c = tid; c < 16 * (128 + 96 + 64 + 32); c += kThreads) {
    int p = 0, cc = c;
    while (cc >= 16 * (128 - 32 * p)) {
      cc -= 16 * (128 - 32 * p);
      ++p;
    }
    const int rows2 = (128 - 32 * p) / 2;
    const int jc = cc / rows2, r = 32 * p + 2 * (cc % rows2), j = 32 * p + jc;
    int bytes = 0;
    if (j < kb && r + 1 >= j) bytes = r + 1 < kb ? 16 : (r < kb ? 8 : 0);
    cp_async16_n(S + pofs(p) + (r - 32 * p) + jc * pld(p), bytes ? Bd + r + (int64_t)j * a.ld : Bd, bytes);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  for (int i = kb + tid; i < NB; i += kThreads) *pel(S, i, i) = 1.0;  // identity padding of a ragged tile
  __syncthreads();
#if SDPC_DAG_FUSED_DIAG
  if (!INV_ONLY && a.tflag && k >= 1) {
    // The step-(k-1) update of this diagonal tile, C -= L_{k,k-1} L_{k,k-1}^T, applied here (no separate
    // UPD task on the chain), 16 columns of L_{k,k-1} at a time as TRSM(k, k-1, *) stores them.  The
    // K-sum is accumulated from zero and subtracted once (as the diagonal update tasks do).  Warps 0-5:
    // the off-diagonal 32 x 32 blocks (I, J); warps 6, 7: the lower 8 x 8 tiles of two diagonal blocks each.
    __shared__ int s_stop2;
    if (pt && tid == 0) pt[9] = gtimer();
    const double* X = a.B + k0 + (int64_t)(k0 - NB) * a.ld;  // tile (k, k - 1)
    double* Xst = sm + kPotrfSmem;                          // [16 columns][kLX], rows 0..127
    const bool offd = wid < 6;
    const int bI = offd ? (wid < 3 ? wid + 1 : (wid < 5 ? wid - 1 : 3)) : (wid == 6 ? 0 : 1);
    const int bJ = offd ? (wid < 3 ? 0 : (wid < 5 ? 1 : 2)) : (wid == 6 ? 3 : 2);  // diag warps: 2nd block
    double acc[20][2];
#pragma unroll
    for (int t = 0; t < 20; ++t) acc[t][0] = acc[t][1] = 0.0;
#pragma unroll 1
    for (int hs = 0; hs < 8; ++hs) {
      if ((hs & 1) == 0 && tid == 0) {
        const unsigned want = (unsigned)(hs / 2 + 1);
        const unsigned* f = a.tflag + 2 * (k - 1);
        unsigned spin = 0;
        while ((ld_vol(f) < want || ld_vol(f + 1) < want) && *(const volatile int32_t*)a.err == kNoError)
          __nanosleep(spin++ < 16 ? 20 : 64);
        __threadfence();  // acquire: the block's columns are visible
        s_stop2 = *(const volatile int32_t*)a.err != kNoError;
      }
      __syncthreads();  // (also: the previous half-slice is consumed)
      if (s_stop2) return;
      for (int c = tid; c < 16 * (NB / 2); c += kThreads) {
        const int col = c / (NB / 2), rr = 2 * (c % (NB / 2));
        const int bytes = rr + 1 < kb ? 16 : (rr < kb ? 8 : 0);  // rows beyond the matrix: zeros
        cp_async16_n(Xst + rr + col * kLX, bytes ? X + rr + (int64_t)(16 * hs + col) * a.ld : X, bytes);
      }
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
#pragma unroll
      for (int k4 = 0; k4 < 4; ++k4) {
        const double* xr = Xst + (4 * k4 + t4) * kLX + g8;
        if (offd) {
          double af[4], bf[4];
#pragma unroll
          for (int x = 0; x < 4; ++x) af[x] = xr[32 * bI + 8 * x];
#pragma unroll
          for (int y = 0; y < 4; ++y) bf[y] = xr[32 * bJ + 8 * y];
#pragma unroll
          for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) dmma_8x8x4(acc[4 * x + y][0], acc[4 * x + y][1], af[x], bf[y]);
        } else {
          double f0[4], f1[4];
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            f0[x] = xr[32 * bI + 8 * x];
            f1[x] = xr[32 * bJ + 8 * x];
          }
          int t = 0;
#pragma unroll
          for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y <= x; ++y, ++t) {
              dmma_8x8x4(acc[t][0], acc[t][1], f0[x], f0[y]);
              dmma_8x8x4(acc[10 + t][0], acc[10 + t][1], f1[x], f1[y]);
            }
        }
      }
    }
    // C -= acc in the packed tile (diagonal 8 x 8 tiles: the entries above their diagonal are never read)
    if (offd) {
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y)
#pragma unroll
          for (int e = 0; e < 2; ++e) *pel(S, 32 * bI + 8 * x + g8, 32 * bJ + 8 * y + 2 * t4 + e) -= acc[4 * x + y][e];
    } else {
      int t = 0;
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y <= x; ++y, ++t)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            *pel(S, 32 * bI + 8 * x + g8, 32 * bI + 8 * y + 2 * t4 + e) -= acc[t][e];
            *pel(S, 32 * bJ + 8 * x + g8, 32 * bJ + 8 * y + 2 * t4 + e) -= acc[10 + t][e];
          }
    }
    __syncthreads();
  }
#endif
  if (pt && tid == 0) pt[1] = gtimer();
#pragma unroll 1
  for (int p = 0; p < 4; ++p) {
    const int c0 = 32 * p, ldp = pld(p);
    double* P = S + pofs(p);  // panel p: element (r, c0 + c) at P[(r - c0) + c ldp]
    if (INV_ONLY) {
      if (wid == 0) wtrtri32(P, ldp, ldiag + c0, Dq, Dq + 32 * 36, lane);
      __syncthreads();
      continue;
    }
    if (wid == 0) {
      const int f = wchol32(P, ldp, ldiag + c0, Dq, Dq + 32 * 36, lane);
      if (lane == 0) fail_col = f;
    }
    __syncthreads();
    if (fail_col >= 0) {
      if (tid == 0) report_error(a.err, k0 + c0 + fail_col + 1);
      return;
    }
    if (pt && tid == 0) pt[2 + p] = gtimer();
    const int r0 = c0 + 32, nr = NB - r0;
    // column block p of Lmix (rows 32 p .. 127): D_p^{-1} (row b, column a of the diagonal block holds
    // D_p^{-1}[a][b]) and L below; then released to the waiting TRSMs
    auto publish_block = [&]() {
      for (int x = tid; x < 32 * (NB - c0); x += kThreads) {
        const int jc = x / (NB - c0), i = c0 + x % (NB - c0);
        const int ic = i - c0;
        const double v = ic < 32 ? (ic >= jc ? P[jc + ic * ldp] : 0.0) : P[ic + jc * ldp];
        __stcg(Lmx + i + (int64_t)(c0 + jc) * NB, v);
      }
      __syncthreads();
      if (a.pflag && tid == 0) {
        __threadfence();
        atomicExch(a.pflag + k, (unsigned)(p + 1));
      }
    };
    if (nr == 0) {
      if (publish) publish_block();
      break;
    }
    // panel rows below the diagonal block, in place: X = A Dinv^T (one warp per 8-row strip)
    for (int tr = wid; tr < nr / 8; tr += kThreads / 32) {
      double* Ar = P + (r0 + tr * 8 - c0);
      double af[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) af[q] = Ar[g8 + (q * 4 + t4) * ldp];
      __syncwarp();
#pragma unroll
      for (int tc = 0; tc < 4; ++tc) {
        double e0 = 0.0, e1 = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) dmma_8x8x4(e0, e1, af[q], Dq[(tc * 8 + g8) * 33 + q * 4 + t4]);
        Ar[g8 + (tc * 8 + 2 * t4) * ldp] = e0;
        Ar[g8 + (tc * 8 + 2 * t4 + 1) * ldp] = e1;
      }
    }
    __syncthreads();
    if (publish) publish_block();
    // trailing update A22 -= X X^T on the 8 x 8 tiles (ti >= tj) of rows / columns r0..127; tiles are
    // dealt to the warps round-robin in row-major order
    const int nb8 = nr / 8;
    int t = 0;
#pragma unroll 1
    for (int ti = 0; ti < nb8; ++ti) {
#pragma unroll 1
      for (int tj = 0; tj <= ti; ++tj, ++t) {
        if ((t & 7) != wid) continue;
        const int i0 = r0 + ti * 8, j0 = r0 + tj * 8;
        const int pj = j0 >> 5, ldc = pld(pj);
        double* Cp = S + pofs(pj) + (i0 + g8 - 32 * pj) + ((j0 & 31) + 2 * t4) * ldc;
        double e0 = Cp[0], e1 = Cp[ldc];
        const double* Xi = P + (i0 + g8 - c0) + t4 * ldp;
        const double* Xj = P + (j0 + g8 - c0) + t4 * ldp;
        double xa[8], xb[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          xa[q] = neg(Xi[q * 4 * ldp]);
          xb[q] = Xj[q * 4 * ldp];
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) dmma_8x8x4(e0, e1, xa[q], xb[q]);
        Cp[0] = e0;
        Cp[ldc] = e1;
      }
    }
    __syncthreads();
  }
  // L to B: warp w writes columns w, w + 8, ..., lanes over rows (coalesced)
#pragma unroll 1
  for (int j = INV_ONLY ? kb : wid; j < kb; j += kThreads / 32) {
    const int p = j >> 5;
    const double* col = S + pofs(p) + (j & 31) * pld(p) - 32 * p;  // element i at col[i], i >= 32 p
    for (int i = j + lane; i < kb; i += 32) __stcg(Bd + i + (int64_t)j * a.ld, i == j ? ldiag[i] : col[i]);
  }
  if (pt && tid == 0) pt[6] = gtimer();
  if (!INV_ONLY && (SDPC_DAG_BLOCKED_TRSM || k == a.T - 1)) {
    if (pt && tid == 0) pt[7] = pt[8] = gtimer();
    return;
  }  // (Lmix is published; the last tile has no panel below)
  // L^{-1} in shared memory, in place by block rows I = 1..3 and columns J < I (ascending):
  //   T = sum_{K=J}^{I-1} L[I,K] Linv[K,J]  (L[I,K] for K >= J is still L: only columns < J of row I are
  //   overwritten yet);  Linv[I,J] = -Dinv_I T  replaces L[I,J] (panel J, rows 32 I ..).
  // Two phases per (I, J), 6 (I, J) pairs; T (32 x 32, transposed, ld 36) reuses the Dinv square.
  // Dinv_p[x][y] (x >= y) sits at row y, column x of diagonal block p (diagonal included), so an operand
  // fragment is one unconditional load and a select.
  double* Tt = Dq;  // Tt[n + kk * 36] = T[kk][n]
#pragma unroll 1
  for (int I = 1; I < 4; ++I) {
#pragma unroll 1
    for (int J = 0; J < I; ++J) {
      for (int t = wid; t < 16; t += kThreads / 32) {
        const int tr = t >> 2, tc = t & 3, n = tc * 8 + g8;
        double e0 = 0.0, e1 = 0.0;
#pragma unroll 1
        for (int Kb = J; Kb < I; ++Kb) {
          const int lk = pld(Kb), lj = pld(J);
          // A: L[I, Kb](row, kk) at panel Kb, row 32 I + tr 8 + g8; B: Linv[Kb, J](kk, n)
          const double* Ap = S + pofs(Kb) + (32 * I + tr * 8 + g8 - 32 * Kb) + t4 * lk;
          const double* Bp = Kb == J ? S + pofs(J) + n + t4 * lj : S + pofs(J) + (32 * Kb - 32 * J + t4) + n * lj;
          const int bs = Kb == J ? 4 * lj : 4;  // B fragment stride per q
          double av[8], bv[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            av[q] = Ap[q * 4 * lk];
            const double v = Bp[q * bs];
            bv[q] = (Kb != J || q * 4 + t4 >= n) ? v : 0.0;
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) dmma_8x8x4(e0, e1, av[q], bv[q]);
        }
        const int ra = tr * 8 + g8, cb = tc * 8 + 2 * t4;
        Tt[cb + ra * 36] = e0;
        Tt[cb + 1 + ra * 36] = e1;
      }
      __syncthreads();
      for (int t = wid; t < 16; t += kThreads / 32) {
        const int tr = t >> 2, tc = t & 3;
        const int li = pld(I), lj = pld(J), xr = tr * 8 + g8;
        // A: Dinv_I[xr][kk] at row kk, column xr of block I
        const double* Ap = S + pofs(I) + t4 + xr * li;
        double e0 = 0.0, e1 = 0.0, av[8], bv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const double v = Ap[q * 4];
          av[q] = (xr >= q * 4 + t4) ? neg(v) : 0.0;
          bv[q] = Tt[(tc * 8 + g8) + (q * 4 + t4) * 36];
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) dmma_8x8x4(e0, e1, av[q], bv[q]);
        double* o = S + pofs(J) + (32 * I + xr - 32 * J) + (tc * 8 + 2 * t4) * lj;
        o[0] = e0;
        o[lj] = e1;
      }
      __syncthreads();
      if (pt && tid == 0) pt[9 + (I * (I - 1)) / 2 + J] = gtimer();
    }
  }
  if (pt && tid == 0) pt[8] = gtimer();
  // L^{-1} (column-major, ld 128, zero above the diagonal) into the workspace: warp w writes columns
  // w, w + 8, ...; lanes over rows
  double* Li = a.Linv + (int64_t)k * NB * NB;
#pragma unroll 1
  for (int j = wid; j < NB; j += kThreads / 32) {
    const int p = j >> 5, lp = pld(p);
    const double* col = S + pofs(p) + (j & 31) * lp - 32 * p;     // below the block: Linv in place
    const double* drow = S + pofs(p) + (j & 31) - 32 * p * lp;     // diagonal block: Linv[i][j] at (j, i)
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = lane + 32 * r;
      double v = 0.0;
      if (i >= j) v = (i >> 5) == p ? drow[i * lp] : col[i];
      __stcg(Li + i + j * NB, v);
    }
  }
  if (pt && tid == 0) pt[7] = gtimer();
}

// ------------------------------------------------------------------ the persistent kernel
__global__ void __launch_bounds__(kThreads, 2) chol_dag_kernel(Args a) {
  extern __shared__ double sm[];
  __shared__ uint64_t s_task;
  const int tid = threadIdx.x;
  __shared__ unsigned tk[kQ];  // tickets held by this CTA (used by thread 32, the popping thread)
  __shared__ int s_chain;
  if (tid < kQ) tk[tid] = kNone;
  if (tid == 0) {
    // role: the first CTAs to arrive elect kChainSms SMs; every CTA on an elected SM serves the chain
    unsigned smid;
    asm("mov.u32 %0, %%smid;" : "=r"(smid));
    // one CTA per elected SM serves the chain; another CTA on an elected SM leaves at once, so the two
    // halves of a chain TRSM / update never share an SM (-1 = leave, 0 = bulk, 1 = chain)
    int role = 0;
    for (int r = 0; r < kChainSms && role == 0; ++r) {
      const unsigned o = atomicCAS(&a.ctl[2 * kQ * kCtl + r], 0u, smid + 1);
      role = o == 0 ? 1 : (o == smid + 1 ? -1 : 0);
    }
    s_chain = role;
    if (blockIdx.x == 0) push(a, enc(kPotrf, 0, 0, 0, 0));
  }
  __syncthreads();
  if (s_chain < 0) return;
  const int q0 = s_chain ? 0 : 2, q1 = s_chain ? 2 : kQ;
  if (tid == 32) s_task = pop(a, tk, q0, q1);
  __syncthreads();
  __shared__ int s_ns;
#pragma unroll 1
  for (;;) {
    const uint64_t task0 = s_task;
    if (task0 == 0) break;
    unsigned long long t1 = 0;
    if (tid == 0 && a.trace) t1 = gtimer();
    const int type = (int)(task0 >> 60), hh = (int)((task0 >> 56) & 15);
    const int k = (int)((task0 >> 32) & 0xffff), i = (int)((task0 >> 16) & 0xffff), j = (int)(task0 & 0xffff);
    if (type == kUpd && j >= k + 3) {
      // a bulk update absorbs the next steps of its tile whose panel inputs are already complete
      // (counter = need - 1: only this tile's previous step is missing); they are never pushed
      if (tid == 0) {
        int ns = 1;
        while (ns < kMaxSteps && j >= k + ns + 3 &&
               ld_vol(reinterpret_cast<const unsigned*>(&a.cnt_u[2 * uidx(a, k + ns, i, j) + hh])) ==
                   (unsigned)(need_u(i, j, k + ns) - 1))
          ++ns;
        if (ns > 1) {
          atomicAdd(&a.ctl[(2 * kQ + 1) * kCtl + 4], (unsigned)(ns - 1));
          __threadfence();  // acquire: the absorbed steps' panel rows are visible
        }
        s_ns = ns;
      }
      __syncthreads();
    } else if (tid == 0) {
      s_ns = 1;
    }
    if (type == kUpd) {
      if (j >= k + 3) run_upd(a, k, s_ns, i, j, hh, sm);
      else run_upd(a, k, 1, i, j, hh, sm);
    } else if (type == kTrsm) {
      run_trsm(a, k, i, hh, sm);
    } else {
      run_potrf(a, k, sm);
    }
    __syncthreads();  // every thread's results are issued; s_task may be overwritten
    const int ns = type == kUpd ? s_ns : 1;
    const uint64_t task = type == kUpd ? enc(kUpd, hh, k + ns - 1, i, j) : task0;  // the last step applied
    unsigned long long t2 = 0;
    if (tid < 32) {
      // warp 0 reports the task done (release: one fence after the CTA barrier, as in a grid sync) ...
      if (tid == 0) {
        __threadfence();
        if (a.trace) t2 = gtimer();
      }
      __syncwarp();
      if (*(const volatile int32_t*)a.err == kNoError) notify(a, task, tid);
    } else if (tid == 32) {
      // ... while warp 1 takes the next task
      s_task = pop(a, tk, q0, q1);
    }
    if (tid == 0 && a.trace) {
      const unsigned x = atomicAdd(a.trace_n, 1u);
      if (x < a.trace_cap) {
        unsigned smid;
        asm("mov.u32 %0, %%smid;" : "=r"(smid));
        a.trace[4 * x] = task0;
        a.trace[4 * x + 1] = t1;
        a.trace[4 * x + 2] = t2;
        a.trace[4 * x + 3] = smid | ((unsigned long long)blockIdx.x << 32) | ((unsigned long long)ns << 48);
      }
    }
    __syncthreads();
  }
}

// The inverses of the T diagonal 128-tiles of a Cholesky factor, one CTA per tile (all in parallel).
__global__ void __launch_bounds__(kThreads, 2) tile_inverse_kernel(Args a) {
  extern __shared__ double sm[];
  run_potrf<true>(a, blockIdx.x, sm);
}

// ------------------------------------------------------------------ batched dense Cholesky steps
// Step q of the blocked right-looking Cholesky of many independent matrices at once (the big cliques
// of Algorithm 1, Step 2-2): matrix b is dim[b] x dim[b] at base + off[b] (column-major, ld = dim + (dim
// & 1), 16-byte aligned); the matrices are sorted by decreasing dim, so the ones still active at step q
// are a prefix (gridDim.y).  Three launches per step, each a batch of the task-graph kernel's own
// tasks: POTRF(q) of every matrix (L_qq^{-1} to its own 128 x 128 buffer), TRSM(i, q, *) and
// UPD(i, j, q, *).  A failing matrix reports err_id[b] (its clique) into *err and its later steps are
// skipped.
__device__ __forceinline__ bool batch_args(const BatchDesc& d, int b, int q, Args& a) {
  const int m = d.dim[b];
  if (*(const volatile int32_t*)(d.err_slot + b) != kNoError || 128 * q >= m) return false;
  a = Args{};
  a.B = d.base + d.off[b];
  a.ld = m + (m & 1);
  a.m = m;
  a.T = (m + NB - 1) / NB;
  a.Linv = d.linv + (int64_t)b * NB * NB - (int64_t)q * NB * NB;  // run_* index Linv + q NB NB
  a.err = d.err_slot + b;
  return true;
}

__global__ void __launch_bounds__(kThreads, 2) batch_potrf_kernel(BatchDesc d, int q) {
  extern __shared__ double sm[];
  Args a;
  const int b = blockIdx.x;
  if (!batch_args(d, b, q, a)) return;
  run_potrf(a, q, sm);
  __syncthreads();
  if (threadIdx.x == 0 && *(volatile int32_t*)a.err != kNoError) report_error(d.err, d.err_id[b]);
}

__global__ void __launch_bounds__(kThreads, 2) batch_trsm_kernel(BatchDesc d, int q) {
  extern __shared__ double sm[];
  Args a;
  if (!batch_args(d, blockIdx.y, q, a)) return;
  const int i = q + 1 + (int)(blockIdx.x >> 1);
  if (i >= a.T) return;
  run_trsm(a, q, i, blockIdx.x & 1, sm);
}

__global__ void __launch_bounds__(kThreads, 2) batch_upd_kernel(BatchDesc d, int q) {
  extern __shared__ double sm[];
  Args a;
  if (!batch_args(d, blockIdx.y, q, a)) return;
  const int t = blockIdx.x >> 1;  // lower-triangle tile (i, j), q < j <= i < T, row-major
  int r = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while (r * (r + 1) / 2 > t) --r;
  while ((r + 1) * (r + 2) / 2 <= t) ++r;
  const int i = q + 1 + r, j = q + 1 + (t - r * (r + 1) / 2);
  if (i >= a.T) return;
  run_upd(a, q, 1, i, j, blockIdx.x & 1, sm);
}

}  // namespace dag

int batched_chol_step(const BatchDesc& d, int q, int nact, int maxdim, cudaStream_t st) {
  using namespace dag;
  static std::atomic<uint64_t> attr{0};
  if (once_per_device(attr)) {
    cudaFuncSetAttribute(batch_potrf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem * (int)sizeof(double));
    cudaFuncSetAttribute(batch_trsm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem * (int)sizeof(double));
    cudaFuncSetAttribute(batch_upd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem * (int)sizeof(double));
  }
  if (nact <= 0) return 0;
  const int T = (maxdim + NB - 1) / NB, below = T - q - 1;
  const size_t smem = kSmem * sizeof(double);
  batch_potrf_kernel<<<nact, kThreads, smem, st>>>(d, q);
  if (below <= 0) return 1;
  batch_trsm_kernel<<<dim3(2 * below, nact), kThreads, smem, st>>>(d, q);
  batch_upd_kernel<<<dim3(below * (below + 1), nact), kThreads, smem, st>>>(d, q);
  return 3;
}

// out[k] (128 x 128 column-major, zero above the diagonal, identity-padded for a ragged last tile) <- the
// inverse of the k-th 128 x 128 diagonal block of the lower factor R (m x m, ldr).  Needs 16-byte staging
// (potrf_dag_usable); returns launches or -1.
int tile_inverses(const double* R, int64_t ldr, int64_t m, double* out, cudaStream_t st) {
  using namespace dag;
  if (!potrf_dag_usable(R, ldr) || m <= 0) return -1;
  static std::atomic<uint64_t> attr{0};
  if (once_per_device(attr))
    cudaFuncSetAttribute(tile_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem * (int)sizeof(double));
  Args a{};
  a.B = const_cast<double*>(R);
  a.ld = ldr;
  a.m = (int)m;
  a.T = (int)((m + NB - 1) / NB);
  a.Linv = out;
  tile_inverse_kernel<<<a.T, kThreads, kSmem * sizeof(double), st>>>(a);
  return 1;
}

// Workspace sizes for T tiles.
struct DagSizes {
  int64_t nu = 0, nt = 0, ctl_b = 0, cnt_b = 0, q_n[dag::kQ] = {0, 0, 0, 0, 0}, total = 0;
};
static DagSizes dag_sizes(int T) {
  DagSizes s;
  for (int k = 0; k < T; ++k) s.nu += (int64_t)(T - k - 1) * (T - k) / 2;
  s.nt = (int64_t)T * (T - 1) / 2;
  s.total = T + 2 * s.nt + 2 * s.nu - (SDPC_DAG_FUSED_DIAG ? 2 * (int64_t)std::max(0, T - 1) : 0);  // (fused: no UPD(k+1, k+1, k, *))
  int64_t c1 = 0, c2 = 0;  // tiles of the next panel's column / the column after, over all steps
  for (int k = 0; k < T; ++k) {
    c1 += std::max(0, T - k - 1);
    c2 += std::max(0, T - k - 2);
  }
  const int64_t chain = 4 * (int64_t)std::max(0, T - 1);  // TRSM(k+1, k, *) + UPD(k+1, k+1, k, *)
  s.q_n[0] = T;
  s.q_n[1] = SDPC_DAG_FUSED_DIAG ? chain / 2 : chain;
  s.q_n[2] = 2 * s.nt + 2 * c1 - chain;
  s.q_n[3] = 2 * c2;
  s.q_n[4] = s.total - s.q_n[0] - s.q_n[1] - s.q_n[2] - s.q_n[3];
  s.ctl_b = (2 * dag::kQ * dag::kCtl + 2 * dag::kCtl) * 4;
  s.cnt_b = 4 * ((int64_t)T + 2 * s.nt + 2 * s.nu + 3 * T);  // (+ T: pflag, + 2 T: tflag)
  return s;
}

bool potrf_dag_usable(const double* B, int64_t ld) {
  return ld % 2 == 0 && (reinterpret_cast<uintptr_t>(B) & 15) == 0;
}

int potrf_dag(sdpc_ctx* h, double* B, int64_t m, int64_t ld, int32_t* d_err, cudaStream_t st) {
  using namespace dag;
  if (m <= 0) return 0;
  const int T = (int)((m + NB - 1) / NB);
  const DagSizes s = dag_sizes(T);
  int dev = 0;
  cudaGetDevice(&dev);
  if (h->dag_T != T || h->dag_dev != dev) {
    // (re)size the workspace: control + counters + queues (zeroed per call), L^{-1} tiles, scratch
    if (h->dag_ws) cudaFree(h->dag_ws);
    if (h->dag_linv) cudaFree(h->dag_linv);
    if (h->dag_koff) cudaFree(h->dag_koff);
    h->dag_ws = nullptr;
    h->dag_linv = nullptr;
    h->dag_koff = nullptr;
    h->dag_T = -1;
    cudaFuncSetAttribute(chol_dag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem * (int)sizeof(double));
    int nsm = 0, per = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, chol_dag_kernel, kThreads, kSmem * sizeof(double));
    h->dag_grid = std::max(1, nsm * std::max(per, 1));
    h->dag_zero_bytes = (size_t)(s.ctl_b + ((s.cnt_b + 7) / 8) * 8 + 8 * s.total);
    if (cudaMalloc(&h->dag_ws, h->dag_zero_bytes) != cudaSuccess) return -1;
    const size_t linv = (size_t)T * NB * NB;
    if (cudaMalloc(&h->dag_linv, linv * sizeof(double)) != cudaSuccess) return -1;
    if (cudaMalloc(&h->dag_koff, (size_t)T * sizeof(int64_t)) != cudaSuccess) return -1;
    std::vector<int64_t> koff(T);
    int64_t acc = 0;
    for (int k = 0; k < T; ++k) {
      koff[k] = acc;
      acc += (int64_t)(T - k - 1) * (T - k) / 2;
    }
    cudaMemcpy(h->dag_koff, koff.data(), T * sizeof(int64_t), cudaMemcpyHostToDevice);
    h->dag_T = T;
    h->dag_dev = dev;
  }
  Args a{};
  a.B = B;
  a.ld = ld;
  a.m = (int)m;
  a.T = T;
  a.Linv = h->dag_linv;
  char* base = static_cast<char*>(h->dag_ws);
  a.ctl = reinterpret_cast<unsigned*>(base);
  int* cnt = reinterpret_cast<int*>(base + s.ctl_b);
  a.cnt_p = cnt;
  a.cnt_t = cnt + T;
  a.cnt_u = cnt + T + 2 * s.nt;
  a.pflag = SDPC_DAG_BLOCKED_TRSM ? reinterpret_cast<unsigned*>(cnt + T + 2 * s.nt + 2 * s.nu) : nullptr;
  a.tflag = SDPC_DAG_FUSED_DIAG ? reinterpret_cast<unsigned*>(cnt + 2 * T + 2 * s.nt + 2 * s.nu) : nullptr;
  uint64_t* q = reinterpret_cast<uint64_t*>(base + s.ctl_b + ((s.cnt_b + 7) / 8) * 8);
  for (int x = 0; x < kQ; ++x) {
    a.slots[x] = q;
    q += s.q_n[x];
  }
  a.koff = h->dag_koff;
  a.total = (unsigned)s.total;
  for (int x = 0; x < kQ; ++x) a.qcap[x] = (unsigned)s.q_n[x];
  a.err = d_err;
  if (h->dag_trace) {
    a.trace = h->dag_trace;
    a.trace_n = reinterpret_cast<unsigned*>(h->dag_trace + 4 * h->dag_trace_cap);
    a.trace_cap = (unsigned)h->dag_trace_cap;
    cudaMemsetAsync(a.trace_n, 0, sizeof(unsigned), st);
    if (h->dag_trace_cap >= 1 + 4 * (int64_t)T) a.ptrace = h->dag_trace + 4 * h->dag_trace_cap - 16 * (int64_t)T;
  }
  cudaMemsetAsync(h->dag_ws, 0, h->dag_zero_bytes, st);
  chol_dag_kernel<<<h->dag_grid, kThreads, kSmem * sizeof(double), st>>>(a);
  return 1;
}

}  // namespace sdpc
