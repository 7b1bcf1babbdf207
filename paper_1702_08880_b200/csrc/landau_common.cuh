// landau_common.cuh -- launch constants, scratch budget, record layout, species coupling
// and the PTX helpers (mbarrier, 1-D TMA bulk copy) shared by the kernels.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "../../include/landau_b200.h"

// Device bounds checks for debug builds (-DLB_DEBUG=1): a failed check traps
// the kernel (the host sees a CUDA error).  Used where compute-sanitizer is
// not available; compiled out otherwise.
#ifndef LB_DEBUG
#define LB_DEBUG 0
#endif
#if LB_DEBUG
#include <cstdio>
#define LB_DCHECK(cond)                                                              \
  do {                                                                               \
    if (!(cond)) {                                                                   \
      printf("LB_DCHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__,  \
             __LINE__, (int)blockIdx.x, (int)threadIdx.x);                           \
      __trap();                                                                      \
    }                                                                                \
  } while (0)
#else
#define LB_DCHECK(cond) \
  do {                  \
  } while (0)
#endif
#include "landau_pair.cuh"

namespace lb {


constexpr int kTI = 128;        // outer points per CTA (one per thread)
#ifndef LB_MINB
#define LB_MINB 4
#endif
#ifndef LB_UNROLL
#define LB_UNROLL 1
#endif
constexpr int kMinBlocks = LB_MINB;  // CTAs per SM the register budget targets
constexpr int kUnroll = LB_UNROLL;   // inner pairs interleaved per loop trip
constexpr int kMaxChunks = 64;  // inner chunks per sweep (sets the JC length)
constexpr int kChunkAlign = 128;
// Scratch budgets for partial sums (bytes): general-path chunk partials per
// outer batch and symmetric-path i/j-side partials per row batch.  The
// batch sizes only depend on the problem size and these budgets; the
// LB_PARTIAL_BUDGET_MB environment variable lowers them (tests use it to
// exercise multi-batch runs at moderate N).
inline size_t partial_budget() {
  static size_t b = [] {
    const char* e = std::getenv("LB_PARTIAL_BUDGET_MB");
    const long long mb = e ? std::atoll(e) : 0;
    return mb > 0 ? size_t(mb) << 20 : size_t(2) << 30;
  }();
  return b;
}

// Record stride in doubles: the smallest even count >= 4 + 3S whose half is
// odd.  The symmetric sweep reads records at lane-varying addresses (lane l
// takes record (l + s) mod 32); a 16-byte load then hits bank group
// (RS/2 * k) mod 8, so RS/2 odd spreads 32 lanes over all 8 groups (4
// wavefronts, the minimum) while e.g. RS = 8 would put them on 2 (16-way
// conflict).
__host__ __device__ constexpr int rec_stride(int S) {
  return (((4 + 3 * S) + 1) & ~1) + (((((4 + 3 * S) + 1) & ~1) / 2) % 2 == 0 ? 2 : 0);
}
template <int S>
struct TileCfg {
  static constexpr int RS = rec_stride(S);
  static constexpr int TJ = S <= 4 ? 128 : 64;  // inner records per stage
};

// Species coupling (kernel.py:496-501) and the record layout it implies.
// When coK and coD are rank one -- always for the reference's own tables:
// nu_ab ~ e_a^2 e_b^2 (physics.py:77-94), so coK_ab = k_a k_b with
// k_a = sqrt(nu_aa) m_o/m_a and coD_ab = al_a be_b -- the S species collapse
// into ONE accumulator set: each inner point carries the pre-weighted fields
// gr' = sum_b k_b w df_r,b, gz' = sum_b k_b w df_z,b, f' = sum_b be_b w f_b
// (formed once per point in K0), the pair loop runs at S = 1 cost, and the
// combine expands K[a] = k_a A'_{0:2}, D[a] = al_a A'_{2:5}.  Algebraically
// identical to summing per species then coupling (the reference's order);
// the rank-one test admits only tables factoring to ~4 ulp.
struct Coupling {
  int S = 1;          // species
  int Se = 1;         // accumulator species sets (1 when collapsed)
  int collapsed = 0;
  double coK4[LB_MAX_SPECIES * LB_MAX_SPECIES];  // 4 * coK (the pulled-out 4)
  double coD4[LB_MAX_SPECIES * LB_MAX_SPECIES];
  double kw[LB_MAX_SPECIES], dw[LB_MAX_SPECIES];      // per-point field weights
  double kout[LB_MAX_SPECIES], dout[LB_MAX_SPECIES];  // 4 k_a, 4 al_a
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "LB_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra LB_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 1-D TMA bulk copy global -> shared, completion counted on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

}  // namespace lb
