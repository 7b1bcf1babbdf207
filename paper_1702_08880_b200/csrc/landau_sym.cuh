// landau_sym.cuh -- symmetric all-points sweep (outer set == inner set).
//
// The reference evaluates every ordered pair (i, j) independently
// (kernel.py:443-493).  Everything expensive in a pair -- d^2, P, m, x, ln x,
// K, E, Em1, S2, S3 and B1, B3, B4, B5 -- is symmetric under i <-> j, and the
// swapped pair's tensors are permutations of the direct ones except UD_xx
// (SURVEY section 0 fact 4):
//   UK_rr(j,i) = UK_rr(i,j)   UD_zz(j,i) = UD_zz(i,j)
//   UD_xz(j,i) = UK_zr(i,j)   UK_zr(j,i) = UD_xz(i,j)
//   UD_xx(j,i) = B1 - rj^2 B3 + 2 ri rj B4 - ri^2 B5
// so each unordered pair is evaluated once and feeds both accumulators.
//
// Decomposition (points Morton-sorted, tiles of 128):
//  * tile pairs {I, J} are enumerated by the circular schedule: row I takes
//    partners J = I + d (mod nt), d = 1..H(I) with H = floor((nt-1)/2), plus
//    d = nt/2 for I < nt/2 when nt is even -- every unordered tile pair once,
//    every row the same length (balanced across CTAs and GPUs);
//  * d = 0 is the diagonal tile, evaluated as ordered pairs (i-side only);
//  * a work item is (row I, a segment of sym_seglen(nt) consecutive d);
//  * inside a CTA each thread owns one i of I (registers), each warp walks
//    the 128 j of J as 4 blocks of 32 in a rotated ("diagonal") order: at
//    step s lane l takes j = (l + s) mod 32, so the 32 lanes touch 32
//    distinct j and the j-side accumulators travel one lane per step with a
//    register shuffle -- no cross-lane reduction trees;
//  * the four warps' j-side sums meet in shared memory (fixed warp order) and
//    are written per (I, d) to HBM; the i-side sums per (I, segment);
//  * a reduction kernel adds, per point and in a fixed order, its i-side
//    segments and the j-side blocks of every row that has its tile as a
//    partner.  No atomics: results are bitwise reproducible.
//
// Summation order (independent of the GPU count): the rows are cut into
// kSymGroups = 8 fixed row groups (boundaries nt*g/8).  A point's total is
// ((T_0 + T_1) + ...) + T_7 in group order, where T_g adds, by increasing row
// I of group g, the j-side block of row I (if the point's tile is one of its
// partners) or, at I = the point's own row, its i-side segments.  A rank of a
// G-GPU split owns whole groups (groups 8r/G .. 8(r+1)/G - 1, the same rows
// as an even split when G divides 8), computes their T_g, and the owner of a
// point adds all eight in group order -- so every bit of K and D is the same
// for G = 1, 2, 4, 8 (and any G <= 8), as the reference promises for its
// `workers` (kernel.py:508-511, test_kernel.py:197-212).
#pragma once
#include "landau_sweep.cuh"

namespace lb {

constexpr int kSymTile = 128;   // points per tile (== threads per CTA)
#ifndef LB_SYM_STAGES
#define LB_SYM_STAGES 2
#endif
constexpr int kSymStages = LB_SYM_STAGES;  // TMA ring depth (one J tile per stage)
#ifndef LB_SEGLEN
#define LB_SEGLEN 2
#endif
constexpr int kSegLenMax = LB_SEGLEN;  // partner tiles per work item (large n)
#ifndef LB_CLAIM_FULL_FIRST
#define LB_CLAIM_FULL_FIRST 0  // 1: claim full segments of every row before the short last ones (measured: 17.09 vs 16.92 ms, and no better G = 8 share)
#endif
#ifndef LB_SYM_MINB
#define LB_SYM_MINB 5  // CTAs per SM of lb_symsweep_kernel<1> (LB_SYM_IB=0; 94 registers)
#endif
#ifndef LB_SYM_UNROLL
#define LB_SYM_UNROLL 1
#endif
constexpr int kSymMinBlocks = LB_SYM_MINB;
// register budget per accumulator-set count (measured: Se = 1 at 5 CTAs/SM,
// Se = 2 spills above 4, Se = 3 needs ~184 registers)
__host__ __device__ constexpr int sym_min_blocks(int Se) {
  return Se == 1 ? kSymMinBlocks : (Se == 2 ? 4 : 2);
}
constexpr int kSymUnroll = LB_SYM_UNROLL;
#ifndef LB_SYM_MAXS
#define LB_SYM_MAXS 3  // measured: S = 4 symmetric (210 regs, 2 CTAs/SM) loses to the general sweep
#endif
constexpr int kSymMaxS = LB_SYM_MAXS;  // register / shared-memory budget bounds S

// partner count of row I (d = 1..H(I)); nt tiles
__host__ __device__ __forceinline__ int sym_h(int I, int nt) {
  const int h = (nt - 1) / 2;
  return ((nt & 1) == 0 && I < nt / 2) ? h + 1 : h;
}
__host__ __device__ __forceinline__ int sym_hmax(int nt) { return nt / 2; }
// Segment length: 8 partner tiles per item for large n, shorter for small n
// so there are enough items to fill the GPU (a function of n only, so the
// summation order -- hence every bit of the result -- depends on n alone).
__host__ __device__ __forceinline__ int sym_seglen(int nt) {
  return max(1, min(kSegLenMax, nt / 64));
}
__host__ __device__ __forceinline__ int sym_nseg(int nt) {
  const int L = sym_seglen(nt);
  return (sym_hmax(nt) + 1 + L - 1) / L;
}

// fixed row groups: the outer level of every point's summation order
constexpr int kSymGroups = 8;
__host__ __device__ __forceinline__ int sym_group_row(int g, int nt) {
  return (int)((long long)nt * g / kSymGroups);
}
// groups [g0, g1) of rank `rank` among `world` (contiguous, whole groups)
__host__ __device__ __forceinline__ void sym_rank_groups(int rank, int world, int& g0, int& g1) {
  g0 = (int)((long long)kSymGroups * rank / world);
  g1 = (int)((long long)kSymGroups * (rank + 1) / world);
}
// device pointers of the eight group sums T_g ([5S][npad] each), in group order
struct SymGroupPtrs {
  const double* p[kSymGroups];
};

#ifndef LB_SYM_IB
#define LB_SYM_IB 1  // species-collapsed sweep: two outer points per thread (lb_symsweep_ib_kernel)
#endif
constexpr int kIbThreads = kSymTile / 2;
template <int S>
__host__ __device__ constexpr int sym_threads() {
  return (S == 1 && LB_SYM_IB) ? kIbThreads : kSymTile;
}

// TMA stages + log table + j-side exchange (2 x warps x 32 j x 5S doubles)
#ifndef LB_IB_ROT_SMEM
#define LB_IB_ROT_SMEM 0  // 1: j-side rotation through shared memory instead of shuffles
#endif
template <int S>
constexpr size_t sym_smem_bytes() {
  return size_t(kSymStages) * kSymTile * rec_stride(S) * sizeof(double) +
         size_t(2 << LB_LOGT_BITS) * sizeof(double) +
         size_t(2) * (sym_threads<S>() / 32) * 32 * 5 * S * sizeof(double) +
         ((S == 1 && LB_SYM_IB && LB_IB_ROT_SMEM) ? size_t(2) * kIbThreads * 10 * sizeof(double) : 0);
}

struct SymArgs {
  const double* rec;  // sorted records, nt*128 x RS (padding records are inert)
  double* iside;      // [row - row0][nseg][5S][128]
  double* jside;      // [row - row0][hmax][5S][128]
  int* next_item;     // work counter (zero at launch): items past the first wave
  // optional execution counters (species-collapsed kernel; NULL: off):
  // [0] off-diagonal thread-steps, [1] diagonal thread-steps, [2] thread-steps
  // that took the m < 0.01 series branch -- with the per-step FP64
  // instruction counts read from this kernel's SASS they give the executed
  // FP64 work of a launch (bench.py, tools/sass_fp64.py)
  unsigned long long* stats;
  int nt, row0, row1, nseg, hmax;
  long long gthr;
};

// Producer of both symmetric sweeps (thread 0 of the CTA): walks the (item,
// d) partner tiles of its work items, issuing each tile into the TMA ring
// once the stage is free.  Items after the first wave (item = blockIdx.x)
// are claimed from a global counter, so CTAs that the warp schedulers favour
// take more items and all CTAs of an SM stay resident until the end; every
// item writes its own partial slot, so the result does not depend on which
// CTA ran it.  Each stage carries its (item, d) to the consumers; item -1
// ends the sweep.
template <int RS>
struct SymProducer {
  const SymArgs& a;
  long long nitems;
  double* smem;
  uint64_t *full, *empty;
  int *stage_item, *stage_d;
  int p_item, p_d = -1;
  uint32_t p_k = 0;
  bool p_done = false;

  long long nclaim;  // items that exist (rows x their segments); nitems = rows x nseg slots

  __device__ SymProducer(const SymArgs& args, long long n, double* sm, uint64_t* f, uint64_t* e, int* si,
                         int* sd)
      : a(args), nitems(n), smem(sm), full(f), empty(e), stage_item(si), stage_d(sd) {
    const int nt = a.nt, L = sym_seglen(nt);
    const int mid = (nt & 1) ? a.row1 : max(a.row0, min(a.row1, nt / 2));
    const int tA = sym_h(a.row0 < mid ? a.row0 : mid, nt) + 1, tB = sym_h(max(mid, a.row0), nt) + 1;
    nclaim = (long long)(mid - a.row0) * ((tA + L - 1) / L) + (long long)(a.row1 - mid) * ((tB + L - 1) / L);
    p_item = (int)blockIdx.x < nclaim ? claimed_item((int)blockIdx.x) : (int)nitems;
  }

  __device__ void seg_range(int item, int& I, int& d0, int& d1) const {
    I = a.row0 + item / a.nseg;
    const int seg = item % a.nseg;
    const int L = sym_seglen(a.nt);
    d0 = seg * L;
    d1 = min(sym_h(I, a.nt) + 1, d0 + L);
  }

  // Claim order -> work item (row-major slot (I - row0) nseg + seg).  The
  // full L-tile segments of all rows come first, then the short last
  // segments (rows whose H + 1 tiles are not a multiple of L), so the final
  // wave is made of the smallest items (a shorter tail, most visible on the
  // 1/G row share of a G-GPU split).  Every item still writes its own
  // partial slot: the order changes the schedule, never a bit of the result.
  __device__ int claimed_item(int c) const {
#if !LB_CLAIM_FULL_FIRST
    {  // row-major claim order (the item's own slot order)
      const int nt = a.nt, L = sym_seglen(nt);
      const int mid = (nt & 1) ? a.row1 : max(a.row0, min(a.row1, nt / 2));
      const int tA = sym_h(a.row0 < mid ? a.row0 : mid, nt) + 1, tB = sym_h(max(mid, a.row0), nt) + 1;
      const int sA = (tA + L - 1) / L, sB = (tB + L - 1) / L, rowsA = mid - a.row0;
      if (c < rowsA * sA) return (c / sA) * a.nseg + c % sA;
      c -= rowsA * sA;
      return (rowsA + c / sB) * a.nseg + c % sB;
    }
#endif
    const int nt = a.nt, L = sym_seglen(nt);
    const int mid = (nt & 1) ? a.row1 : max(a.row0, min(a.row1, nt / 2));  // rows below mid: H + 1 = nt/2 + 1
    const int tA = sym_h(a.row0 < mid ? a.row0 : mid, nt) + 1;             // tiles per row, class A
    const int tB = sym_h(max(mid, a.row0), nt) + 1;                         // class B (rows >= mid)
    const int rowsA = mid - a.row0, rowsB = a.row1 - mid;
    const int fA = tA / L, fB = tB / L;
    const long long nfA = (long long)rowsA * fA, nfB = (long long)rowsB * fB;
    if (c < nfA) return (c / fA) * a.nseg + c % fA;
    c -= (int)nfA;
    if (c < nfB) return (rowsA + c / fB) * a.nseg + c % fB;
    c -= (int)nfB;
    const int sA = (tA % L) ? rowsA : 0;  // short segments: class A rows first, then B
    if (c < sA) return c * a.nseg + fA;
    c -= sA;
    return (rowsA + c) * a.nseg + fB;
  }

  __device__ void issue_next() {
    if (p_done) return;
    int I = 0, d0, d1;
    while (p_item < nitems) {
      seg_range(p_item, I, d0, d1);
      if (p_d < 0) p_d = d0;
      if (p_d < d1) break;
      // segment done: claim the next one
      const int c = (int)gridDim.x + atomicAdd(a.next_item, 1);
      p_item = c < nclaim ? claimed_item(c) : (int)nitems;
      p_d = -1;
    }
    const uint32_t s = p_k % kSymStages;
    if (p_k >= kSymStages) mbar_wait(&empty[s], ((p_k / kSymStages) - 1) & 1);
    ++p_k;
    if (p_item >= nitems) {
      stage_item[s] = -1;
      mbar_arrive(&full[s]);
      p_done = true;
      return;
    }
    stage_item[s] = p_item;
    stage_d[s] = p_d;
    const int J = (I + p_d) % a.nt;
    LB_DCHECK(I >= a.row0 && I < a.row1 && p_d >= 0 && p_d <= sym_h(I, a.nt) && J >= 0 && J < a.nt);
    const uint32_t bytes = kSymTile * RS * sizeof(double);
    mbar_expect_tx(&full[s], bytes);
    bulk_g2s(smem + s * (kSymTile * RS), a.rec + (size_t)J * kSymTile * RS, bytes, &full[s]);
    ++p_d;
  }
};

template <int S>
__device__ __forceinline__ void load_point(const double* rp, Outer& o, double (&gi)[S][3]) {
  o = make_outer(rp[0], rp[1]);
#pragma unroll
  for (int b = 0; b < S; ++b) {
    gi[b][0] = rp[4 + 3 * b];
    gi[b][1] = rp[5 + 3 * b];
    gi[b][2] = rp[6 + 3 * b];
  }
}

template <int S>
__global__ void __launch_bounds__(kSymTile, sym_min_blocks(S)) lb_symsweep_kernel(const SymArgs a) {
  constexpr int RS = rec_stride(S);
  constexpr int NW = kSymTile / 32;
  extern __shared__ __align__(128) double lb_smem[];
  __shared__ __align__(8) uint64_t full[kSymStages], empty[kSymStages];
  __shared__ int stage_item[kSymStages], stage_d[kSymStages];  // what each stage holds (-1: end)
  double2* logt = reinterpret_cast<double2*>(lb_smem + kSymStages * kSymTile * RS);
  double* jred = lb_smem + kSymStages * kSymTile * RS + (2 << LB_LOGT_BITS);  // [2][NW][32][5S]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nrows = a.row1 - a.row0;
  const long long nitems = (long long)nrows * a.nseg;

  for (int t = tid; t < (2 << LB_LOGT_BITS); t += kSymTile)
    lb_smem[kSymStages * kSymTile * RS + t] = c_logt[t];
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < kSymStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  SymProducer<RS> prod(a, nitems, lb_smem, full, empty, stage_item, stage_d);
  if (tid == 0) prod.issue_next();

  Outer o;
  double gi[S][3];
  double acc[S][5];
  int cur = -1, I = 0;
  auto flush_iside = [&]() {
    double* dst = a.iside + ((size_t)(I - a.row0) * a.nseg + (cur % a.nseg)) * (5 * S) * kSymTile + tid;
#pragma unroll
    for (int b = 0; b < S; ++b)
#pragma unroll
      for (int q = 0; q < 5; ++q) dst[(size_t)(b * 5 + q) * kSymTile] = acc[b][q];
  };
  for (uint32_t k = 0;; ++k) {
    if (tid == 0) prod.issue_next();
    const uint32_t s = k % kSymStages;
    mbar_wait(&full[s], (k / kSymStages) & 1);
    const int item = stage_item[s], d = stage_d[s];
    if (item < 0) break;
    if (item != cur) {
      if (cur >= 0) flush_iside();
      cur = item;
      I = a.row0 + item / a.nseg;
      load_point<S>(a.rec + ((size_t)I * kSymTile + tid) * RS, o, gi);
#pragma unroll
      for (int b = 0; b < S; ++b)
#pragma unroll
        for (int q = 0; q < 5; ++q) acc[b][q] = 0.0;
    }
    {
      const double* tile = lb_smem + s * (kSymTile * RS);
      const bool diag = (d == 0);
#pragma unroll 1
      for (int jb = 0; jb < kSymTile / 32; ++jb) {
        double jacc[S][5];
#pragma unroll
        for (int b = 0; b < S; ++b)
#pragma unroll
          for (int q = 0; q < 5; ++q) jacc[b][q] = 0.0;
        // (r, z) of the next step's record are loaded one step ahead so the
        // shared-memory latency is off the pair's dependency chain
        double2 rz_next = *reinterpret_cast<const double2*>(tile + (jb * 32 + lane) * RS);
#pragma unroll kSymUnroll
        for (int st = 0; st < 32; ++st) {
          const int jl = (lane + st) & 31;
          const double* rp = tile + (jb * 32 + jl) * RS;
          const double2 rz = rz_next;
          rz_next = *reinterpret_cast<const double2*>(tile + (jb * 32 + ((jl + 1) & 31)) * RS);
          const double2 aux = *reinterpret_cast<const double2*>(rp + 2);
          T5 t;
          const double txx2 = pair_tensor_sym(o, rz.x, rz.y, aux.x, aux.y, a.gthr, logt, t);
#pragma unroll
          for (int b = 0; b < S; ++b) {
            const double gr = rp[4 + 3 * b], gz = rp[5 + 3 * b], fw = rp[6 + 3 * b];
            acc[b][0] = fma(t.xz, gz, fma(t.kr, gr, acc[b][0]));
            acc[b][1] = fma(t.zz, gz, fma(t.zr, gr, acc[b][1]));
            acc[b][2] = fma(fw, t.xx, acc[b][2]);
            acc[b][3] = fma(fw, t.xz, acc[b][3]);
            acc[b][4] = fma(fw, t.zz, acc[b][4]);
          }
          if (!diag) {
            // outer j, inner i (kernel.py:411-415 with the swapped tensors)
#pragma unroll
            for (int b = 0; b < S; ++b) {
              jacc[b][0] = fma(t.zr, gi[b][1], fma(t.kr, gi[b][0], jacc[b][0]));
              jacc[b][1] = fma(t.zz, gi[b][1], fma(t.xz, gi[b][0], jacc[b][1]));
              jacc[b][2] = fma(gi[b][2], txx2, jacc[b][2]);
              jacc[b][3] = fma(gi[b][2], t.zr, jacc[b][3]);
              jacc[b][4] = fma(gi[b][2], t.zz, jacc[b][4]);
            }
            // the accumulator of j = (lane + st + 1) mod 32 comes from lane + 1
#pragma unroll
            for (int b = 0; b < S; ++b)
#pragma unroll
              for (int q = 0; q < 5; ++q)
                jacc[b][q] = __shfl_sync(0xffffffffu, jacc[b][q], (lane + 1) & 31);
          }
        }
        if (!diag) {
          // lane holds this warp's sum for j = jb*32 + lane; the four warps'
          // sums meet in a double-buffered exchange slot and are added in
          // fixed warp order (one CTA barrier per 32 j).  (A barrier-free
          // variant -- per-slot mbarriers, each warp reducing the previous
          // exchange -- measured 14% slower.)
          double* slot = jred + (size_t)(jb & 1) * NW * 32 * (5 * S);
          double* dst = slot + ((size_t)warp * 32 + lane) * (5 * S);
#pragma unroll
          for (int b = 0; b < S; ++b)
#pragma unroll
            for (int q = 0; q < 5; ++q) dst[b * 5 + q] = jacc[b][q];
          __syncthreads();
          LB_DCHECK(d >= 1 && d <= a.hmax);
          double* out = a.jside + ((size_t)(I - a.row0) * a.hmax + (d - 1)) * (5 * S) * kSymTile +
                        jb * 32;
          for (int v = tid; v < 32 * 5 * S; v += kSymTile) {
            const int c = v >> 5, jj = v & 31;
            double x = slot[(size_t)jj * (5 * S) + c];
#pragma unroll
            for (int w = 1; w < NW; ++w) x = __dadd_rn(x, slot[((size_t)w * 32 + jj) * (5 * S) + c]);
            out[(size_t)c * kSymTile + jj] = x;
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
  if (cur >= 0) flush_iside();
}

// Species-collapsed variant with two OUTER points per thread (i-blocking):
// 64 threads own the 128 points of the row tile (lane l of warp w: points
// 64w + l and 64w + 32 + l) and every step pairs both with the same partner
// j = (l + s) mod 32, so the partner's record loads, the coefficient loads
// and the one j-side accumulator shuffle are shared by two pairs.  Same
// work items, schedule, TMA ring and partial layouts as lb_symsweep_kernel.
#ifndef LB_IB_PAIRS
#define LB_IB_PAIRS 2  // partners per step, each paired with both outer points (4 pairs)
#endif
#ifndef LB_IB_ROT_TOP
#define LB_IB_ROT_TOP 0  // 1: j-side rotation at the top of the next step (measured no gain)
#endif
#ifndef LB_IB_MINB
#define LB_IB_MINB (LB_IB_PAIRS == 2 ? 4 : 6)  // CTAs per SM (240 / 168 registers)
#endif

template <int S, bool MG>
#ifdef LB_IB_MAXNREG
__global__ void __maxnreg__(LB_IB_MAXNREG) lb_symsweep_ib_kernel(const SymArgs a) {
#else
__global__ void __launch_bounds__(kIbThreads, LB_IB_MINB) lb_symsweep_ib_kernel(const SymArgs a) {
#endif
  constexpr int RS = rec_stride(S);
  constexpr int NW = kIbThreads / 32;
  extern __shared__ __align__(128) double lb_smem[];
  __shared__ __align__(8) uint64_t full[kSymStages], empty[kSymStages];
  __shared__ int stage_item[kSymStages], stage_d[kSymStages];
  double2* logt = reinterpret_cast<double2*>(lb_smem + kSymStages * kSymTile * RS);
  double* jred = lb_smem + kSymStages * kSymTile * RS + (2 << LB_LOGT_BITS);  // [2][NW][32][5S]
#if LB_IB_ROT_SMEM
  double* jrot = jred + 2 * NW * 32 * (5 * S);  // [2][kIbThreads][10]
#endif

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nrows = a.row1 - a.row0;
  const long long nitems = (long long)nrows * a.nseg;
  for (int t = tid; t < (2 << LB_LOGT_BITS); t += kIbThreads)
    lb_smem[kSymStages * kSymTile * RS + t] = c_logt[t];
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < kSymStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  SymProducer<RS> prod(a, nitems, lb_smem, full, empty, stage_item, stage_d);
  if (tid == 0) prod.issue_next();

  Outer o[2];
  double gi[2][S][3];
  double acc[2][S][5];
  int cur = -1, I = 0;
  unsigned n_off = 0, n_diag = 0, n_ser = 0;  // thread-steps (execution counters)
  auto pidx = [&](int ib) { return warp * 64 + ib * 32 + lane; };
  auto flush_iside = [&]() {
#pragma unroll
    for (int ib = 0; ib < 2; ++ib) {
      LB_DCHECK(pidx(ib) < kSymTile && I >= a.row0 && I < a.row1);
      double* dst = a.iside + ((size_t)(I - a.row0) * a.nseg + (cur % a.nseg)) * (5 * S) * kSymTile + pidx(ib);
#pragma unroll
      for (int b = 0; b < S; ++b)
#pragma unroll
        for (int q = 0; q < 5; ++q) dst[(size_t)(b * 5 + q) * kSymTile] = acc[ib][b][q];
    }
  };
  for (uint32_t k = 0;; ++k) {
    if (tid == 0) prod.issue_next();
    const uint32_t s = k % kSymStages;
    mbar_wait(&full[s], (k / kSymStages) & 1);
    const int item = stage_item[s], d = stage_d[s];
    if (item < 0) break;
    if (item != cur) {
      if (cur >= 0) flush_iside();
      cur = item;
      I = a.row0 + item / a.nseg;
#pragma unroll
      for (int ib = 0; ib < 2; ++ib) {
        load_point<S>(a.rec + ((size_t)I * kSymTile + pidx(ib)) * RS, o[ib], gi[ib]);
#pragma unroll
        for (int b = 0; b < S; ++b)
#pragma unroll
          for (int q = 0; q < 5; ++q) acc[ib][b][q] = 0.0;
      }
    }
    const double* tile = lb_smem + s * (kSymTile * RS);
    const bool diag = (d == 0);
#pragma unroll 1
    for (int jb = 0; jb < kSymTile / 32; ++jb) {
      // JU partners per step (j = (lane + st + u L) mod 32, L = 32 / JU) for
      // both outer points: 2 JU pairs in lockstep, JU j-side accumulators
      constexpr int JU = LB_IB_PAIRS, L = 32 / JU, P2 = 2 * JU;
      double ju[JU][S][5];
#pragma unroll
      for (int u = 0; u < JU; ++u)
#pragma unroll
        for (int b = 0; b < S; ++b)
#pragma unroll
          for (int q = 0; q < 5; ++q) ju[u][b][q] = 0.0;
      double2 rzn[JU];
#pragma unroll
      for (int u = 0; u < JU; ++u)
        rzn[u] = *reinterpret_cast<const double2*>(tile + (jb * 32 + ((lane + u * L) & 31)) * RS);
#pragma unroll 1
      for (int st = 0; st < L; ++st) {
#if LB_IB_ROT_TOP
        // rotate the j-side sums of the previous step here (a no-op on the
        // zeros at st == 0) rather than after its accumulation, so the
        // shuffles share a basic block with, and hide under, this step's
        // pair arithmetic
#pragma unroll
        for (int u = 0; u < JU; ++u)
#pragma unroll
          for (int b = 0; b < S; ++b)
#pragma unroll
            for (int q = 0; q < 5; ++q) ju[u][b][q] = __shfl_sync(0xffffffffu, ju[u][b][q], (lane + 1) & 31);
#endif
        const double* rp[JU];
        Outer oo[P2];
        double rn[P2], zn[P2], rn2[P2], rcpr[P2], rnx[P2];
#pragma unroll
        for (int u = 0; u < JU; ++u) {
          const int jl = (lane + st + u * L) & 31;
          rp[u] = tile + (jb * 32 + jl) * RS;
          const double2 rz = rzn[u];
          rzn[u] = *reinterpret_cast<const double2*>(tile + (jb * 32 + ((jl + 1) & 31)) * RS);
          const double2 aux = *reinterpret_cast<const double2*>(rp[u] + 2);
          const double r2x = rp[u][7];  // 2 rn (species-collapsed record)
#pragma unroll
          for (int ib = 0; ib < 2; ++ib) {
            oo[2 * u + ib] = o[ib];
            rn[2 * u + ib] = rz.x;
            zn[2 * u + ib] = rz.y;
            rn2[2 * u + ib] = aux.x;
            rcpr[2 * u + ib] = aux.y;
            rnx[2 * u + ib] = r2x;
          }
        }
        T5 t[P2];
        double txx2[P2];
        pair_tensor_sym_x<P2, MG>(oo, rn, zn, rn2, rnx, rcpr, a.gthr, logt, t, txx2, n_ser);
#pragma unroll
        for (int u = 0; u < JU; ++u)
#pragma unroll
          for (int b = 0; b < S; ++b) {
            const double gr = rp[u][4 + 3 * b], gz = rp[u][5 + 3 * b], fw = rp[u][6 + 3 * b];
#pragma unroll
            for (int ib = 0; ib < 2; ++ib) {
              const T5& tt = t[2 * u + ib];
              acc[ib][b][0] = fma(tt.xz, gz, fma(tt.kr, gr, acc[ib][b][0]));
              acc[ib][b][1] = fma(tt.zz, gz, fma(tt.zr, gr, acc[ib][b][1]));
              acc[ib][b][2] = fma(fw, tt.xx, acc[ib][b][2]);
              acc[ib][b][3] = fma(fw, tt.xz, acc[ib][b][3]);
              acc[ib][b][4] = fma(fw, tt.zz, acc[ib][b][4]);
            }
          }
        if (!diag) {
#pragma unroll
          for (int u = 0; u < JU; ++u)
#pragma unroll
            for (int b = 0; b < S; ++b)
#pragma unroll
              for (int ib = 0; ib < 2; ++ib) {
                const T5& tt = t[2 * u + ib];
                ju[u][b][0] = fma(tt.zr, gi[ib][b][1], fma(tt.kr, gi[ib][b][0], ju[u][b][0]));
                ju[u][b][1] = fma(tt.zz, gi[ib][b][1], fma(tt.xz, gi[ib][b][0], ju[u][b][1]));
                ju[u][b][2] = fma(gi[ib][b][2], txx2[2 * u + ib], ju[u][b][2]);
                ju[u][b][3] = fma(gi[ib][b][2], tt.zr, ju[u][b][3]);
                ju[u][b][4] = fma(gi[ib][b][2], tt.zz, ju[u][b][4]);
              }
#if LB_IB_ROT_SMEM
          {
            // rotate through a double-buffered per-thread slot (80 B stride:
            // conflict-free 16-byte accesses); one __syncwarp per step
            static_assert(JU * S * 5 == 10, "shared-memory rotation assumes 10 j-side sums");
            double* own = jrot + ((size_t)(st & 1) * kIbThreads + tid) * 10;
            const double* nb = jrot + ((size_t)(st & 1) * kIbThreads + warp * 32 + ((lane + 1) & 31)) * 10;
            double* flat = &ju[0][0][0];
#pragma unroll
            for (int q = 0; q < 10; q += 2)
              *reinterpret_cast<double2*>(own + q) = make_double2(flat[q], flat[q + 1]);
            __syncwarp();
#pragma unroll
            for (int q = 0; q < 10; q += 2) {
              const double2 v = *reinterpret_cast<const double2*>(nb + q);
              flat[q] = v.x;
              flat[q + 1] = v.y;
            }
          }
#elif !LB_IB_ROT_TOP
#pragma unroll
          for (int u = 0; u < JU; ++u)
#pragma unroll
            for (int b = 0; b < S; ++b)
#pragma unroll
              for (int q = 0; q < 5; ++q) ju[u][b][q] = __shfl_sync(0xffffffffu, ju[u][b][q], (lane + 1) & 31);
#endif
        }
      }
#if LB_IB_ROT_TOP
      // the last step's rotation
#pragma unroll
      for (int u = 0; u < JU; ++u)
#pragma unroll
        for (int b = 0; b < S; ++b)
#pragma unroll
          for (int q = 0; q < 5; ++q) ju[u][b][q] = __shfl_sync(0xffffffffu, ju[u][b][q], (lane + 1) & 31);
#endif
      if (diag) n_diag += L; else n_off += L;
      // lane l holds accumulator u of j = l + (u+1)L: gather j = l in u order
      double jacc[S][5];
#pragma unroll
      for (int b = 0; b < S; ++b)
#pragma unroll
        for (int q = 0; q < 5; ++q) {
          double x = 0.0;
#pragma unroll
          for (int u = 0; u < JU; ++u) {
            const double v = (u + 1) * L == 32 ? ju[u][b][q]
                                               : __shfl_sync(0xffffffffu, ju[u][b][q], (lane - (u + 1) * L) & 31);
            x = u == 0 ? v : __dadd_rn(x, v);
          }
          jacc[b][q] = x;
        }
      if (!diag) {
        double* slot = jred + (size_t)(jb & 1) * NW * 32 * (5 * S);
        double* dst = slot + ((size_t)warp * 32 + lane) * (5 * S);
#pragma unroll
        for (int b = 0; b < S; ++b)
#pragma unroll
          for (int q = 0; q < 5; ++q) dst[b * 5 + q] = jacc[b][q];
        __syncthreads();
        LB_DCHECK(d >= 1 && d <= a.hmax);
        double* out = a.jside + ((size_t)(I - a.row0) * a.hmax + (d - 1)) * (5 * S) * kSymTile + jb * 32;
        for (int v = tid; v < 32 * 5 * S; v += kIbThreads) {
          const int c = v >> 5, jj = v & 31;
          double x = slot[(size_t)jj * (5 * S) + c];
#pragma unroll
          for (int w = 1; w < NW; ++w) x = __dadd_rn(x, slot[((size_t)w * 32 + jj) * (5 * S) + c]);
          out[(size_t)c * kSymTile + jj] = x;
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (cur >= 0) flush_iside();
  if (a.stats) {
    unsigned long long c0 = n_off, c1 = n_diag, c2 = n_ser;
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) {
      c0 += __shfl_xor_sync(0xffffffffu, c0, o2);
      c1 += __shfl_xor_sync(0xffffffffu, c1, o2);
      c2 += __shfl_xor_sync(0xffffffffu, c2, o2);
    }
    if (lane == 0) {
      atomicAdd(a.stats + 0, c0);
      atomicAdd(a.stats + 1, c1);
      atomicAdd(a.stats + 2, c2);
    }
  }
}

// Fixed-order reduction of one row batch [row0, row1) into the group sums
// T_g (tot + (g - gbase) [5S][npad], SoA) of every group the batch touches:
// per point, by increasing row I within the group, the j-side block of row
// I when the point's tile P is one of its partners (d = P - I mod nt in
// 1..H(I)) or, at I = P, the sum of the point's own i-side segments (added
// among themselves in segment order).  A group's first
// batch starts its sums from zero.  The order depends only on n, never on
// the batching or on which rank runs the group (landau_sym.cuh header).
template <int S>
__global__ void lb_symreduce_kernel(const double* __restrict__ iside, const double* __restrict__ jside,
                                    int nt, int row0, int row1, int nseg, int hmax, int gbase,
                                    double* __restrict__ tot) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  const int npad = nt * kSymTile;
  if (p >= npad) return;
  const int P = p / kSymTile, t = p % kSymTile;
#ifndef LB_RED_G
#define LB_RED_G 8
#endif
  constexpr int G = LB_RED_G;
  // the point's own i-side segments (its row's partners, in segment order),
  // added into the group sum at I = P
  double own[5 * S];
  const bool has_own = P >= row0 && P < row1;
  if (has_own) {
    const int nsg = min(nseg, sym_h(P, nt) / sym_seglen(nt) + 1);
    const double* src = iside + (size_t)(P - row0) * nseg * (5 * S) * kSymTile + t;
#pragma unroll
    for (int c = 0; c < 5 * S; ++c) own[c] = src[(size_t)c * kSymTile];
#pragma unroll 1
    for (int s1 = 1; s1 < nsg; s1 += G) {
      double x[G][5 * S];
#pragma unroll
      for (int k = 0; k < G; ++k)
        if (s1 + k < nsg) {
          const double* sp = src + (size_t)(s1 + k) * (5 * S) * kSymTile;
#pragma unroll
          for (int c = 0; c < 5 * S; ++c) x[k][c] = sp[(size_t)c * kSymTile];
        }
#pragma unroll
      for (int k = 0; k < G; ++k)
        if (s1 + k < nsg) {
#pragma unroll
          for (int c = 0; c < 5 * S; ++c) own[c] = __dadd_rn(own[c], x[k][c]);
        }
    }
  }
#pragma unroll 1
  for (int g = 0; g < kSymGroups; ++g) {
    const int gb0 = sym_group_row(g, nt), gb1 = sym_group_row(g + 1, nt);
    const int lo = max(row0, gb0), hi = min(row1, gb1);
    if (lo >= hi) continue;
    LB_DCHECK(g >= gbase);
    double* T = tot + (size_t)(g - gbase) * (5 * S) * npad;
    double v[5 * S];
#pragma unroll
    for (int c = 0; c < 5 * S; ++c) v[c] = lo == gb0 ? 0.0 : T[(size_t)c * npad + p];
    // d = (P - I) mod nt, stepped down with I (no integer division per row);
    // rows in groups of G: the group's loads are issued before its adds, which
    // stay in increasing-I order (the conditions are uniform across the block)
    int d = (P - lo) % nt;
    if (d < 0) d += nt;
#pragma unroll 1
    for (int I0 = lo; I0 < hi; I0 += G) {
      double x[G][5 * S];
      bool on[G];
#pragma unroll
      for (int k = 0; k < G; ++k) {
        const int I = I0 + k;
        on[k] = I < hi && d >= 1 && d <= sym_h(I, nt);
        if (on[k]) {
          LB_DCHECK(d >= 1 && d <= hmax);
          const double* src = jside + ((size_t)(I - row0) * hmax + (d - 1)) * (5 * S) * kSymTile + t;
#pragma unroll
          for (int c = 0; c < 5 * S; ++c) x[k][c] = src[(size_t)c * kSymTile];
        }
        d = d == 0 ? nt - 1 : d - 1;
      }
#pragma unroll
      for (int k = 0; k < G; ++k) {
        if (has_own && I0 + k == P && P < hi) {
#pragma unroll
          for (int c = 0; c < 5 * S; ++c) v[c] = __dadd_rn(v[c], own[c]);
        }
        if (on[k]) {
#pragma unroll
          for (int c = 0; c < 5 * S; ++c) v[c] = __dadd_rn(v[c], x[k][c]);
        }
      }
    }
#pragma unroll
    for (int c = 0; c < 5 * S; ++c) T[(size_t)c * npad + p] = v[c];
  }
}

// Tile interleave.  The Morton order keeps each 128-point tile spatially
// coherent (warp-coherent series branch), but consecutive tiles -- hence a
// row group, hence a rank's share of a G-GPU split -- would cover one region
// of velocity space, and regions differ in work (rows near the axis take the
// m < 0.01 series more often: groups 0, 1, 4, 5 ran 4 % slower than 2, 3, 6,
// 7).  So the sorted order deals the Morton tiles to the tile positions by
// residue class: position T holds Morton tile c + 8 k, classes c = 0..7 in
// turn (class c at positions off(c) .. off(c) + cnt(c) - 1).  Every row group
// then draws its tiles evenly from the whole curve.  A function of nt alone:
// the summation order, hence every bit of K and D, stays GPU-count invariant.
__host__ __device__ __forceinline__ int sym_class_off(int c, int nt) {
  return c * (nt / kSymGroups) + min(c, nt % kSymGroups);
}
// Morton tile -> sorted tile position
__host__ __device__ __forceinline__ int sym_tile_pos(int To, int nt) {
  return sym_class_off(To % kSymGroups, nt) + To / kSymGroups;
}
// sorted tile position -> Morton tile
__host__ __device__ __forceinline__ int sym_tile_src(int Tn, int nt) {
  int c = 0;
#pragma unroll 1
  while (c + 1 < kSymGroups && sym_class_off(c + 1, nt) <= Tn) ++c;
  return c + kSymGroups * (Tn - sym_class_off(c, nt));
}

// Sorted, padded records: rec_s[p'] = rec[perm[p]] where p is the Morton
// position of sorted position p' (tile interleave above) and p < n; inert
// records for the padding positions p >= n (far away on the axis side, zero
// fields: they add exact zeros).
__global__ void lb_sym_gather_kernel(int n, int npad, int RS, const int* __restrict__ perm,
                                     const double* __restrict__ rec, double* __restrict__ rec_s) {
  const int pn = blockIdx.x * blockDim.x + threadIdx.x;
  if (pn >= npad) return;
  const int nt = npad / kSymTile;
  const int p = sym_tile_src(pn / kSymTile, nt) * kSymTile + pn % kSymTile;
  double* o = rec_s + (size_t)pn * RS;
  if (p < n) {
    const double* src = rec + (size_t)perm[p] * RS;
    for (int c = 0; c < RS; ++c) o[c] = src[c];
  } else {  // r = 1: r, z, 4 r^2, 1/r, zero fields (and 2 r in a collapsed record's slot 7)
    o[0] = 1.0;
    o[1] = 1.0e6;
    o[2] = 4.0;
    o[3] = 1.0;
    for (int c = 4; c < RS; ++c) o[c] = c == 7 ? 2.0 : 0.0;
  }
}

// K/D for original points [q0, q1) from the eight group sums (sorted point
// order, through the inverse permutation), added in group order; coupling as
// _combine (kernel.py:419-440).  The group sums may live on other GPUs: with
// peer pointers (CUDA IPC over NVLink) this kernel is the cross-rank
// reduction and the combine in one, reading only this rank's points.
template <int Se>
__global__ void lb_sym_combine_kernel(const SymGroupPtrs gp, int npad, const int* __restrict__ inv,
                                      int q0, int q1, const Coupling cp, double* __restrict__ K,
                                      double* __restrict__ D) {
  const int q = q0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= q1) return;
  const int p = inv[q];
  double A[Se][5];
#pragma unroll
  for (int b = 0; b < Se; ++b)
#pragma unroll
    for (int c = 0; c < 5; ++c) {
      const size_t off = (size_t)(b * 5 + c) * npad + p;
      double v = gp.p[0][off];
#pragma unroll
      for (int g = 1; g < kSymGroups; ++g) v = __dadd_rn(v, gp.p[g][off]);
      A[b][c] = v;
    }
  write_kd<Se>(A, cp, (size_t)(q - q0), K, D);
}

// inv[q] = sorted position of original point q (Morton position perm^-1[q]
// through the tile interleave)
__global__ void lb_invert_perm_kernel(int n, int nt, const int* __restrict__ perm, int* __restrict__ inv) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) inv[perm[p]] = sym_tile_pos(p / kSymTile, nt) * kSymTile + p % kSymTile;
}

}  // namespace lb
