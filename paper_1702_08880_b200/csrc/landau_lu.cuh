// landau_lu.cuh -- batched dense LU with partial pivoting and the solves of
// the Crank-Nicolson block cyclic reduction (landau_b200.cu, cn_factor_issue
// / cn_solve_issue), replacing cuBLAS getrfBatched / getrsBatched /
// trsmBatched at the solver's block sizes (nb <= 384; 68..354 here).
//
// cuBLAS's batched getrf is a latency-bound chain of small launches per
// column panel (~4.6 us per column at nb = 260, 1.2 ms per call whatever
// the batch), and its batched getrs with 2 nb right-hand sides runs at a few
// TFLOP/s.  Here:
//  * lb_getrf_kernel: one CTA per matrix, right-looking blocked LU with a
//    KB-column panel in shared memory.  Panel: per column one CTA-wide
//    pivot search (LAPACK idamax: first maximum of |a|), row swap, and a
//    row-owned scale + rank-1 update fused with the next column's pivot
//    candidates (2 barriers per column).  Then the panel's swaps on the
//    other columns (warp-per-column gather on six warps while two warps
//    invert the diagonal blocks of L and U), U12 = L11^-1 A12 and the
//    trailing update A22 -= L21 U12 on the FP64 tensor path
//    (mma.sync.m8n8k4.f64).  Output in LAPACK layout (unit L below the
//    diagonal, U on and above it, 1-based ipiv) so the vector solves
//    (lb_small_solve_kernel, getrs) consume it unchanged; also the row
//    permutation and the inverses of the KB x KB diagonal blocks.
//  * lb_getrs_slab_kernel: X := A^-1 X for an n x m block of right-hand
//    sides (the cyclic reduction's [L U], m = 2 nb), one CTA per (matrix,
//    W-column slab): rows gathered through the permutation into shared
//    memory, then block forward / backward substitution in which every
//    step is two small DMMA GEMMs (the diagonal block through its stored
//    inverse, then the factor column block streamed in by cp.async).
//  * lb_lu_vsolve_kernel: one vector per matrix (blocks > 96 rows).
#pragma once
#include <climits>
#include <cstdint>

#ifndef LB_DCHECK  // standalone use (tools/microbench): bounds checks off
#define LB_DCHECK(cond) \
  do {                  \
  } while (0)
#endif

namespace lb {

constexpr int kLuThreads = 256;
#ifndef LB_LU_REGPANEL
#define LB_LU_REGPANEL 1  // panel factorisation in registers (one row per thread); 0: shared-memory panel
#endif
// lb_getrf_kernel: one thread per panel row (n <= 384) with the register panel
constexpr int kGetrfThreads = LB_LU_REGPANEL ? 384 : kLuThreads;
#ifndef LB_LU_LOOKAHEAD_WARPS
#define LB_LU_LOOKAHEAD_WARPS 4  // idle warps needed to run a deferred trailing update beside a panel
#endif
constexpr int kLookAheadWarps = LB_LU_LOOKAHEAD_WARPS;
#ifdef LB_LU_PROF
#ifndef LB_LU_PROF_TID
#define LB_LU_PROF_TID 0  // the thread whose phase cycles are recorded
#endif
// cycles per phase (block 0, thread LB_LU_PROF_TID): accumulated in registers, written by LU_FLUSH
__device__ long long lu_prof[8];
#define LU_T(k)                                                        \
  do {                                                                 \
    const long long t1_ = clock64();                                   \
    pacc_[k] += t1_ - t0_;                                             \
    t0_ = t1_;                                                         \
  } while (0)
#define LU_FLUSH()                                                                   \
  do {                                                                               \
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == LB_LU_PROF_TID) {       \
      for (int k_ = 0; k_ < 8; ++k_) lu_prof[k_] += pacc_[k_];                       \
      for (int k_ = 0; k_ < 4; ++k_) lu_prof2[k_] += pcol_[k_];                      \
    }                                                                                \
  } while (0)
// column-loop breakdown of the register panel (reduction, pivot row, update)
__device__ long long lu_prof2[4];
#define LU_TC(k)                                                       \
  do {                                                                 \
    const long long t1_ = clock64();                                   \
    pcol_[k] += t1_ - t0_;                                             \
    t0_ = t1_;                                                         \
  } while (0)
#else
#define LU_T(k) \
  do {          \
  } while (0)
#define LU_FLUSH() \
  do {             \
  } while (0)
#define LU_TC(k) \
  do {           \
  } while (0)
#endif

template <int KB>
__host__ __device__ constexpr int lu_ld(int n) {
  return (n + 7) & ~7;  // panel / slab leading dimension (8-row padding for the 8x8 tiles)
}

// shared memory of lb_getrf_kernel<KB>: panel [KB][ld] + U12 rows [KB][ld] + reduction scratch
template <int KB>
inline size_t getrf_smem_bytes(int n) {
  constexpr int NW = kGetrfThreads / 32;
  return sizeof(double) * (2 * (size_t)KB * lu_ld<KB>(n) + 2 * 32 + KB * KB + 2 * NW * (KB + 2)) +
         sizeof(int) * (KB + 32 + 2 * lu_ld<KB>(n) + 4 * KB + 4 * NW);
}

// Inverse diagonal blocks: per matrix, per panel p, invL[p] (KB x KB, unit
// lower, column-major) then invU[p]; inv_stride = 2 * npanel * KB * KB.
template <int KB>
__host__ __device__ inline int lu_inv_stride(int n) {
  return 2 * ((n + KB - 1) / KB) * KB * KB;
}

// D += A B for one 8x8x4 FP64 tile (mma.sync, SASS DMMA): lane l holds
// A[l/4][l%4], B[l%4][l/4] and D[l/4][2(l%4) + {0,1}]
__device__ __forceinline__ void dmma_884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <int KB>
__global__ void __launch_bounds__(kGetrfThreads) lb_getrf_kernel(int n, double* const* __restrict__ As,
                                                              int* __restrict__ ipiv_all,
                                                              int* __restrict__ perm_all,
                                                              int* __restrict__ info_all,
                                                              double* __restrict__ inv_all, int pivot) {
  extern __shared__ __align__(16) double lu_sm[];
  const int ld = lu_ld<KB>(n);
  double* P = lu_sm;                   // panel, column-major [KB][ld] (row offset from c0)
  double* Ub = lu_sm + (size_t)KB * ld;  // U12 rows, row-major [KB][ld] (column offset from c0 + w)
  double* redv = Ub + (size_t)KB * ld;   // [32]
  double* iLs = redv + 64;               // [KB][KB] L11^-1 of the current panel (column-major)
  // register panel: the warps' pivot candidates, double-buffered by column parity
  constexpr int NT = kGetrfThreads;
  constexpr int NW = NT / 32;
  double* pr_rows = iLs + KB * KB;                            // [2][NW][KB] candidate rows
  double* pr_rcp = pr_rows + 2 * NW * KB;                     // [2][NW] 1 / a of the candidates
  unsigned long long* pr_key = reinterpret_cast<unsigned long long*>(pr_rcp + 2 * NW);  // [2][NW]
  int* pr_slot = reinterpret_cast<int*>(pr_key + 2 * NW);     // [2][NW]
  int* pr_thr = pr_slot + 2 * NW;                             // [2][NW]
  int* redi = pr_thr + 2 * NW;                                // [32]
  int* pv_sh = redi + 32;                         // [KB]
  int* lp = pv_sh + KB;                           // [ld] panel-local row permutation
  int* tl_dst = lp + ld;                          // [2 KB] rows a panel's swaps touch
  int* tl_src = tl_dst + 2 * KB;                  // [2 KB] and where their values come from
  int* perm_s = tl_src + 2 * KB;                  // [ld] cumulative row permutation (register panel)
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* A = As[b];
  int* ipiv = ipiv_all ? ipiv_all + (size_t)b * n : nullptr;
  double* inv = inv_all + (size_t)b * lu_inv_stride<KB>(n);
  int info = 0;
#ifdef LB_LU_PROF
  long long t0_ = clock64(), pacc_[8] = {}, pcol_[4] = {};
#endif

#if LB_LU_REGPANEL
  for (int i = tid; i < ld; i += NT) perm_s[i] = i;  // (ordered before use by the first panel's barriers)
#endif
  // trailing update A22 -= L21 U12 of the panel at (uc0, uw) for the warp
  // tiles (16 rows x 32 columns) in tile columns [tc0, tc1), distributed over
  // warps [wb, wb + nwk); L21 from P, U12 from Ub (shared memory)
  auto trailing_update = [&](int uc0, int uw, int um2, int un2, int tc0, int tc1, int wb, int nwk) {
    const int lk = lane & 3;
    const int twr = (um2 + 15) >> 4, twc = tc1 - tc0;
    for (int t = warp - wb; t < twr * twc; t += nwk) {
      const int R0 = (t / twc) * 16, C0 = (tc0 + t - (t / twc) * twc) * 32;
      double acc[2][4][2];
#pragma unroll
      for (int mm = 0; mm < 2; ++mm) {
        const int R = R0 + 8 * mm + (lane >> 2);
#pragma unroll
        for (int nn = 0; nn < 4; ++nn)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int C = C0 + 8 * nn + 2 * lk + e;
            acc[mm][nn][e] = (R < um2 && C < un2) ? A[(size_t)(uc0 + uw + C) * n + uc0 + uw + R] : 0.0;
          }
      }
#pragma unroll
      for (int k0 = 0; k0 < KB; k0 += 4) {
        const int k = k0 + lk;
        double av[2], bv[4];
#pragma unroll
        for (int mm = 0; mm < 2; ++mm) av[mm] = -P[(size_t)k * ld + uw + R0 + 8 * mm + (lane >> 2)];
#pragma unroll
        for (int nn = 0; nn < 4; ++nn) bv[nn] = Ub[(size_t)k * ld + C0 + 8 * nn + (lane >> 2)];
#pragma unroll
        for (int mm = 0; mm < 2; ++mm)
#pragma unroll
          for (int nn = 0; nn < 4; ++nn) dmma_884(acc[mm][nn], av[mm], bv[nn]);
      }
#pragma unroll
      for (int mm = 0; mm < 2; ++mm) {
        const int R = R0 + 8 * mm + (lane >> 2);
        if (R >= um2) continue;
#pragma unroll
        for (int nn = 0; nn < 4; ++nn)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int C = C0 + 8 * nn + 2 * lk + e;
            if (C < un2) A[(size_t)(uc0 + uw + C) * n + uc0 + uw + R] = acc[mm][nn][e];
          }
      }
    }
  };
  // look-ahead: the previous panel's update of the columns right of the
  // current panel (tile columns 1..), deferred so that the warps the current
  // panel leaves idle (those past its rows) run it during the factorisation
  int def_c0 = 0, def_w = 0, def_m2 = 0, def_n2 = 0, def_twc = 0;
  for (int c0 = 0, p = 0; c0 < n; c0 += KB, ++p) {
    const int w = min(KB, n - c0), m = n - c0;
#if LB_LU_REGPANEL
    // 1-3. Panel in registers: thread t holds panel row t (its KB columns,
    //    compile-time indexed: the column loop is unrolled).  Rows never
    //    move during the panel: the row chosen as pivot of column j retires
    //    (it is row j of U); every other row takes l = a_j / d and its
    //    rank-1 update in registers.  The LAPACK view is bookkeeping: each
    //    thread tracks its row's slot, and the pivot is the largest |a| among
    //    the live rows, ties to the smallest slot (idamax's first maximum
    //    over slots j..m-1), so pivots and factors (the same operations in
    //    the same order) are those of the shared-memory panel.  ONE barrier
    //    per column, over the warps that own rows (named barrier 1): every
    //    warp publishes its best candidate -- key, slot, thread, 1/a and the
    //    row itself -- double-buffered by column parity, and after the
    //    barrier every warp picks the winner among them.  Warp-level picks
    //    are three redux.sync (max |a| as the high and low words of its bit
    //    pattern, then the smallest slot) instead of shuffle trees.
    const bool own = tid < m;
    int slot = tid;
    bool done = false;  // this row is a pivot (a row of U) already
    // only the warps that own panel rows take part: the per-column overhead
    // is issue- and latency-bound, and the panel shrinks by 32 rows a step
    const int nact = (m + 31) >> 5;
    __syncthreads();
    LU_T(0);
    // the previous panel's deferred update (tile columns 1.., columns right
    // of this panel): beside the panel on its idle warps, or -- too few of
    // them -- by everyone first
    const bool lookahead = def_twc > 1 && NW - nact >= kLookAheadWarps;
    if (def_twc > 1 && !lookahead) {
      trailing_update(def_c0, def_w, def_m2, def_n2, 1, def_twc, 0, NW);
      __syncthreads();
    }
    double v[KB];
    if (warp >= nact) {  // (no panel rows; separate branch: v and the update's
                         // accumulators are never live together)
#pragma unroll
      for (int k = 0; k < KB; ++k) v[k] = 0.0;
      if (lookahead) trailing_update(def_c0, def_w, def_m2, def_n2, 1, def_twc, nact, NW - nact);
    } else {
    {
      const double* src = A + (size_t)c0 * n + c0 + tid;
#pragma unroll
      for (int k = 0; k < KB; ++k) v[k] = (own && k < w) ? src[(size_t)k * n] : 0.0;
    }
    // every live row's 1 / a_j, computed as soon as a_j is final (the IEEE
    // division overlaps the pivot search; the winner's is published)
    double rcp = v[0] != 0.0 ? 1.0 / v[0] : 0.0;
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      if (j >= w) break;
      const int buf = j & 1;
      double* rows = pr_rows + (size_t)buf * NW * KB;  // [NW][KB]
      int wq = 0;  // entry of the pivot row
      bool pub;    // this thread publishes its row
      if (pivot) {
        // key: live non-NaN rows by |a| (bit pattern, top bit set); the row
        // holding slot j is the fallback when no row has a comparable |a|
        const double av = fabs(v[j]);
        const bool live = own && !done;
        const unsigned long long key =
            (live && av >= 0.0) ? (__double_as_longlong(av) | (1ull << 63)) : ((live && slot == j) ? 1ull : 0ull);
        const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
        const unsigned m1 = __reduce_max_sync(0xffffffffu, hi);
        const unsigned m2 = __reduce_max_sync(0xffffffffu, hi == m1 ? lo : 0u);
        const bool top = hi == m1 && lo == m2;
        const unsigned ms = __reduce_min_sync(0xffffffffu, top ? (unsigned)slot : 0xffffffffu);
        pub = top && (unsigned)slot == ms;  // this warp's candidate (one lane: slots are distinct)
        if (pub) pr_key[buf * NW + warp] = key;
      } else {
        pub = tid == j;  // no pivoting: the row at slot j (thread j) is the pivot
      }
      if (pub) {
        const int e = pivot ? warp : 0;
        pr_slot[buf * NW + e] = slot;
        pr_thr[buf * NW + e] = tid;
        pr_rcp[buf * NW + e] = rcp;
        double2* dst = reinterpret_cast<double2*>(rows + e * KB);
#pragma unroll
        for (int k = 2 * (j / 2); k < KB; k += 2) dst[k / 2] = make_double2(v[k], v[k + 1]);
      }
      LU_TC(1);
      asm volatile("bar.sync 1, %0;" ::"r"(nact * 32) : "memory");
      LU_TC(3);
      if (pivot) {  // the winner among the warps' candidates (every warp, same answer)
        const unsigned long long kq = lane < nact ? pr_key[buf * NW + lane] : 0ull;
        const int sq = lane < nact ? pr_slot[buf * NW + lane] : INT_MAX;
        const unsigned qh = (unsigned)(kq >> 32), ql = (unsigned)kq;
        const unsigned g1 = __reduce_max_sync(0xffffffffu, qh);
        const unsigned g2 = __reduce_max_sync(0xffffffffu, qh == g1 ? ql : 0u);
        const bool gt = lane < nact && qh == g1 && ql == g2;
        const unsigned gs = __reduce_min_sync(0xffffffffu, gt ? (unsigned)sq : 0xffffffffu);
        wq = __ffs(__ballot_sync(0xffffffffu, gt && (unsigned)sq == gs)) - 1;
      }
      const int ps = pr_slot[buf * NW + wq], ph = pr_thr[buf * NW + wq];
      LB_DCHECK(ps >= j && ps < m && ph >= 0 && ph < m);
      const double* ur = rows + wq * KB;  // the pivot row: U row j
      const double r = pr_rcp[buf * NW + wq];
      LU_TC(0);
      if (tid == 0) {
        if (ur[j] == 0.0 && info == 0) info = c0 + j + 1;  // LAPACK info (first zero pivot)
        pv_sh[j] = ps;
      }
      if (tid == ph) {
        slot = j;
        done = true;
      } else if (slot == j) {
        slot = ps;
      }
      if (own && !done) {  // zero pivot: r = 0, the column below is zero too
        const double l = v[j] * r;
        v[j] = l;
#pragma unroll
        for (int k = j + 1; k < KB; ++k) v[k] = fma(-l, ur[k], v[k]);
        if (j + 1 < KB) rcp = v[j + 1] != 0.0 ? 1.0 / v[j + 1] : 0.0;
      }
      LU_TC(2);
    }
    }  // warp < nact
    __syncthreads();
    // the factored panel by LAPACK slot in P (zero padding: rows m..ld,
    // columns w..KB are zero in v)
    if (own) {
#pragma unroll
      for (int k = 0; k < KB; ++k) P[(size_t)k * ld + slot] = v[k];
      lp[slot] = tid;  // slot -> panel-local row: each row knows where the LAPACK swaps took it
    } else if (tid < ld) {
#pragma unroll
      for (int k = 0; k < KB; ++k) P[(size_t)k * ld + tid] = 0.0;
      lp[tid] = tid;
    }
    __syncthreads();  // pv_sh / lp final
    LU_T(1);
    // cumulative row permutation: row c0 + s of P A is row c0 + lp[s] before
    // this panel's swaps
    const int perm_new = own ? perm_s[c0 + lp[tid]] : 0;
    // the factored panel back to A (LAPACK layout)
    for (int t = tid; t < w * m; t += NT) {
      const int k = t / m, i = t - k * m;
      A[(size_t)(c0 + k) * n + c0 + i] = P[(size_t)k * ld + i];
    }
    if (ipiv && tid < w) ipiv[c0 + tid] = c0 + pv_sh[tid] + 1;
    __syncthreads();
    if (own) perm_s[c0 + tid] = perm_new;
#else
    // 1. panel rows c0..n, columns c0..c0+w -> P (zero padding to ld rows /
    //    KB columns); rows tid + 256 h, eight columns of loads in flight
    for (int i = tid; i < ld; i += NT) lp[i] = i;  // panel-local row permutation
    for (int h = 0; h * NT < ld; ++h) {
      const int i = tid + h * NT;
      if (i >= ld) break;
      const double* src = A + (size_t)c0 * n + c0 + i;
#pragma unroll
      for (int j0 = 0; j0 < KB; j0 += 8) {
        double v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = (j0 + j < w && i < m) ? src[(size_t)(j0 + j) * n] : 0.0;
#pragma unroll
        for (int j = 0; j < 8; ++j) P[(size_t)(j0 + j) * ld + i] = v[j];
      }
    }
    __syncthreads();
    LU_T(0);
    // 2. unblocked LU of the panel.  The rank-1 update of column j and the
    //    pivot search of column j+1 are one pass (each thread takes the
    //    largest |a| of column j+1 over the rows it just updated), so a
    //    column costs two barriers: after the warps' pivot candidates, and
    //    after the row swap.
    double best = -1.0;
    int bi = m;
    if (pivot)
      for (int i = tid; i < m; i += NT) {
        const double v = fabs(P[i]);
        if (v > best) { best = v; bi = i; }  // rows visited in increasing order
      }
    for (int j = 0; j < w; ++j) {
      int piv = j;
      if (pivot) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
        }
        if (lane == 0) { redv[warp] = best; redi[warp] = bi; }
        __syncthreads();
        best = redv[0];
        bi = redi[0];
#pragma unroll
        for (int q = 1; q < NW; ++q) {
          const double ov = redv[q];
          const int oi = redi[q];
          if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
        }
        // idamax: the first index of the largest |a|; a column with no
        // comparable entry (all NaN, after a singular block upstream) keeps
        // row j -- never the sentinel m, which would index past the block
        piv = bi < m ? bi : j;
        LB_DCHECK(piv >= j && piv < m);
        if (piv != j && tid < w) {
          const double t0 = P[(size_t)tid * ld + j];
          P[(size_t)tid * ld + j] = P[(size_t)tid * ld + piv];
          P[(size_t)tid * ld + piv] = t0;
        }
      }
      if (tid == 0) {
        pv_sh[j] = piv;
        const int t0 = lp[j];  // the same swap on the row permutation
        lp[j] = lp[piv];
        lp[piv] = t0;
      }
      __syncthreads();
      const double d = P[(size_t)j * ld + j];
      if (d == 0.0 && info == 0) info = c0 + j + 1;  // LAPACK info (first zero pivot)
      const double r = d != 0.0 ? 1.0 / d : 0.0;     // zero pivot: the column below is zero too
      best = -1.0;
      bi = m;
      for (int i = j + 1 + tid; i < m; i += NT) {
        const double l = P[(size_t)j * ld + i] * r;
        P[(size_t)j * ld + i] = l;
        int k = j + 1;
        if (k < w) {  // column j+1 first: the next pivot candidate
          const double v = fma(-l, P[(size_t)k * ld + j], P[(size_t)k * ld + i]);
          P[(size_t)k * ld + i] = v;
          if (fabs(v) > best) { best = fabs(v); bi = i; }
          ++k;
        }
        for (; k + 4 <= w; k += 4) {  // four independent read-modify-writes per round
          double a4[4], u4[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            a4[q] = P[(size_t)(k + q) * ld + i];
            u4[q] = P[(size_t)(k + q) * ld + j];
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) P[(size_t)(k + q) * ld + i] = fma(-l, u4[q], a4[q]);
        }
        for (; k < w; ++k) P[(size_t)k * ld + i] = fma(-l, P[(size_t)k * ld + j], P[(size_t)k * ld + i]);
      }
      if (!pivot) __syncthreads();  // (pivoting: the next column's first barrier orders these writes)
    }
    __syncthreads();
    LU_T(1);
    // 3. panel back; pivots (1-based, global rows)
    for (int j = 0; j < w; ++j)
      for (int i = tid; i < m; i += NT) A[(size_t)(c0 + j) * n + c0 + i] = P[(size_t)j * ld + i];
    if (ipiv && tid < w) ipiv[c0 + tid] = c0 + pv_sh[tid] + 1;
#endif
    // 4. inverses of the diagonal blocks: unit lower L11 and upper U11 (one
    //    column of each inverse per thread)
    {
      double* iL = inv + (size_t)(2 * p) * KB * KB;
      double* iU = iL + KB * KB;
#ifdef LB_LU_PROF_SKIP_INV  // profiling experiment only (wrong results)
      if (false) {
#else
      if (tid < KB) {  // column tid of L11^-1: right-looking forward substitution of e_tid
#endif
        const int c = tid;
        double x[KB];
#pragma unroll
        for (int i = 0; i < KB; ++i) x[i] = (i == c) ? 1.0 : 0.0;
#pragma unroll
        for (int k = 0; k < KB; ++k)  // x[k] is final; eliminate it from the rows below
#pragma unroll
          for (int i = k + 1; i < KB; ++i) x[i] = fma(-P[(size_t)k * ld + i], x[k], x[i]);
#pragma unroll
        for (int i = 0; i < KB; ++i) {
          const double v = (c < w && i < w) ? x[i] : 0.0;
          iL[(size_t)c * KB + i] = v;
          iLs[(size_t)c * KB + i] = v;
        }
      } else if (tid >= 32 && tid < 32 + KB) {  // column c of U11^-1: right-looking back substitution of e_c
        const int c = tid - 32;
        // 1/u_kk: lane k divides once, the substitution multiplies (a
        // 32-step chain of IEEE divisions was the longest path of the
        // panel's tail: the other warps waited for it at the next barrier)
        const double rme = 1.0 / ((c < w) ? P[(size_t)c * ld + c] : 1.0);
        double x[KB];
#pragma unroll
        for (int i = 0; i < KB; ++i) x[i] = (i == c) ? 1.0 : 0.0;
#pragma unroll
        for (int k = KB - 1; k >= 0; --k) {
          x[k] = x[k] * __shfl_sync(0xffffffffu, rme, k);
#pragma unroll
          for (int i = 0; i < k; ++i) x[i] = fma(-P[(size_t)k * ld + i], x[k], x[i]);
        }
#pragma unroll
        for (int i = 0; i < KB; ++i) iU[(size_t)c * KB + i] = (c < w && i < w) ? x[i] : 0.0;
      }
    }
    LU_T(2);
    // 5. the panel's row swaps on every other column, as one gather of the
    //    <= 2 KB rows they touch (all loads before any store); U12 =
    //    L11^-1 A12 on the columns right of the panel (one column per thread)
    // list: entries 0..w-1 are rows 0..w-1 (sources lp[j]); entry w + j is
    // pivot row pv[j] when it lies below the panel's first w rows (first
    // occurrence only), its source lp[pv[j]] (always one of rows 0..w-1);
    // unused entries have source -1
    // (warps 0 and 1 are still computing the diagonal-block inverses: the
    // list and the gather run on warps 2..7, synchronised by named barrier 1)
    const int cnt = 2 * w;
    const int n2 = n - c0 - w;
    constexpr int kGW = NW - 2;  // gather warps
    if (warp >= 2) {
      const int j = tid - 64;
      if (j < w) {
        tl_dst[j] = j;
        tl_src[j] = lp[j];
        const int r = pv_sh[j];
        bool first = pivot && r >= w;
        for (int q = 0; q < j && first; ++q) first = pv_sh[q] != r;
        tl_dst[w + j] = r;
        tl_src[w + j] = first ? lp[r] : -1;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kGW * 32) : "memory");
    // gather: one warp per column, lane q (and q + 32) owns list entry q:
    // the column's touched rows are read together (one coalesced segment
    // for rows c0..c0+w, a few sectors for the pivot rows), then written;
    // the first w rows of a right column go to Ub for the U12 product
    {
      const int s0 = lane < cnt ? tl_src[lane] : -1, s1 = lane + 32 < cnt ? tl_src[lane + 32] : -1;
      const int d0 = tl_dst[lane], d1 = tl_dst[lane + 32];
      const int kbeg = pivot ? 0 : c0;  // left columns only need the swaps
      constexpr int CB = 16;            // columns in flight per warp
#ifdef LB_LU_PROF_SKIP_GATHER  // profiling experiment only (wrong results)
      for (int kb0 = n; kb0 < n - w; kb0 += kGW * CB) {
#else
      for (int kb0 = kbeg + (warp - 2) * CB; kb0 < n - w; kb0 += kGW * CB) {
#endif
        double v0[CB], v1[CB];
#pragma unroll
        for (int u = 0; u < CB; ++u) {
          const int k = kb0 + u;
          const int col = k < c0 ? k : k + w;  // skip the panel's own columns
          const double* Ac = A + (size_t)col * n + c0;
          const bool ok = k < n - w;
          v0[u] = (ok && s0 >= 0) ? Ac[s0] : 0.0;
          v1[u] = (ok && s1 >= 0) ? Ac[s1] : 0.0;
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < CB; ++u) {
          const int k = kb0 + u;
          if (k >= n - w) break;
          const int col = k < c0 ? k : k + w;
          double* Ac = A + (size_t)col * n + c0;
          const bool right = col >= c0 + w;
          if (s0 >= 0 && !(right && lane < w)) Ac[d0] = v0[u];
          if (s1 >= 0 && !(right && lane + 32 < w)) Ac[d1] = v1[u];
          if (right) Ub[(size_t)lane * ld + (col - c0 - w)] = (lane < w) ? v0[u] : 0.0;
        }
      }
    }
    }
    __syncthreads();
    LU_T(5);
    // U12 = L11^-1 A12 on the FP64 tensor path: warp tiles of 32 rows x TN
    // columns (4 x TN/8 MMA tiles), written to Ub and back to A's rows c0..c0+w.
    // TN = 32: 16 independent accumulators per warp, so consecutive MMAs of a
    // k-step do not wait on each other (with 4 x 2 tiles ptxas grouped them
    // into 4 chains and the loop ran at a third of the pipe in place)
    {
#ifndef LB_U12_TN
#define LB_U12_TN 32
#endif
      constexpr int TN = LB_U12_TN, NNT = TN / 8;
      const int lk = lane & 3, lr = lane >> 2;
      constexpr int kMaxU = ((383 + TN - 1) / TN + NW - 1) / NW;
      double acc[kMaxU][4][NNT][2];
      const int nwt = (n2 + TN - 1) / TN;
#pragma unroll
      for (int u = 0; u < kMaxU; ++u) {
        const int t = warp + u * NW;
        if (t >= nwt) break;
        const int C0 = t * TN;
#pragma unroll
        for (int mm = 0; mm < 4; ++mm)
#pragma unroll
          for (int nn = 0; nn < NNT; ++nn) acc[u][mm][nn][0] = acc[u][mm][nn][1] = 0.0;
#ifdef LB_LU_PROF_SKIP_U12  // profiling experiment only (wrong results)
        continue;
#endif
#pragma unroll
        for (int k0 = 0; k0 < KB; k0 += 4) {
          const int k = k0 + lk;
          double av[4], bv[NNT];
#pragma unroll
          for (int mm = 0; mm < 4; ++mm) av[mm] = iLs[(size_t)k * KB + 8 * mm + lr];
#pragma unroll
          for (int nn = 0; nn < NNT; ++nn) {
            const int C = C0 + 8 * nn + lr;
            bv[nn] = C < n2 ? Ub[(size_t)k * ld + C] : 0.0;
          }
#pragma unroll
          for (int mm = 0; mm < 4; ++mm)
#pragma unroll
            for (int nn = 0; nn < NNT; ++nn) dmma_884(acc[u][mm][nn], av[mm], bv[nn]);
        }
      }
      __syncthreads();  // every Ub read done
      LU_T(6);
#pragma unroll
      for (int u = 0; u < kMaxU; ++u) {
        const int t = warp + u * NW;
        if (t >= nwt) break;
        const int C0 = t * TN;
#pragma unroll
        for (int mm = 0; mm < 4; ++mm) {
          const int i = 8 * mm + lr;
#pragma unroll
          for (int nn = 0; nn < NNT; ++nn)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int C = C0 + 8 * nn + 2 * lk + e;
              if (C < n2) {
                Ub[(size_t)i * ld + C] = acc[u][mm][nn][e];
                if (i < w) A[(size_t)(c0 + w + C) * n + c0 + i] = acc[u][mm][nn][e];
              }
            }
        }
      }
    }
    // zero padding of Ub's columns n2..n2+31 (32-column warp tiles read them)
    for (int t = tid; t < KB * 32; t += NT) {
      const int i = t >> 5, k2 = n2 + (t & 31);
      if (k2 < ld) Ub[(size_t)i * ld + k2] = 0.0;
    }
    __syncthreads();
    LU_T(3);
    // 6. trailing update A22 -= L21 U12 on the FP64 tensor path
    //    (mma.m8n8k4.f64): warp tiles of 16 rows x 32 columns, accumulators
    //    start from the tile's current values.  Tile column 0 is the next
    //    panel: updated now by every warp; the rest is deferred to the next
    //    panel's idle warps (look-ahead) -- or done now on the last panel /
    //    the shared-memory-panel build
    const int m2 = m - w;
    def_twc = 0;
#ifdef LB_LU_PROF_SKIP_UPD  // profiling experiment only (wrong results)
    if (false) {
#else
    if (m2 > 0 && n2 > 0) {
#endif
      static_assert(KB % 4 == 0, "k steps of 4");
      const int twc = (n2 + 31) >> 5;
      const bool defer = LB_LU_REGPANEL && c0 + KB < n && twc > 1;
      trailing_update(c0, w, m2, n2, 0, defer ? 1 : twc, 0, NW);
      if (defer) {
        def_c0 = c0;
        def_w = w;
        def_m2 = m2;
        def_n2 = n2;
        def_twc = twc;
      }
    }
    __syncthreads();
    LU_T(4);
  }
  LU_FLUSH();
  if (tid == 0) {
    if (info_all) info_all[b] = info;
#if !LB_LU_REGPANEL
    if (perm_all) {  // row i of P A is row perm[i] of A
      int* perm = perm_all + (size_t)b * n;
      for (int i = 0; i < n; ++i) perm[i] = i;
      if (pivot && ipiv)
        for (int i = 0; i < n; ++i) {
          const int q = ipiv[i] - 1;
          const int t0 = perm[i];
          perm[i] = perm[q];
          perm[q] = t0;
        }
    }
#endif
  }
#if LB_LU_REGPANEL
  if (perm_all) {  // row i of P A is row perm[i] of A (built per panel in shared memory)
    __syncthreads();
    int* perm = perm_all + (size_t)b * n;
    for (int i = tid; i < n; i += NT) perm[i] = perm_s[i];
  }
#endif
}

// X := A^-1 X for X = the n x m column-major block at Xs[b] (leading
// dimension n), A the factors of lb_getrf_kernel.  CTA (b, s) owns columns
// [s W, s W + W).  Shared memory: the slab X [ld][W + 4] (row-major: a row
// of W columns is contiguous), the factor column block of the current step
// in two k-halves H0/H1 [KB/2][ldh] (column-major, only the rows the step
// updates) and the diagonal-block inverse; the scaled block Y replaces the
// block's rows of X in place.
//
// 2 np block steps (forward p = 0..np-1 with L, backward p = np-1..0 with U).
// Step q:   Y = Di(q) X[block]   (X rows of the block := Y)
//           X[rows] -= F(q)[rows][0:KB/2] Y[0:KB/2]      (H0)
//           X[rows] -= F(q)[rows][KB/2:KB] Y[KB/2:KB]   (H1)
// The factor halves arrive by cp.async, each one phase ahead: H0 of step
// q+1 streams in during the H1 pass of step q, H1 of step q+1 (and Di)
// during the Di product of step q+1.
// Shared-memory strides chosen so that the FP64 MMA fragment loads are bank
// conflict free (a half-warp reads 4 k x 4 rows/columns of 8 bytes: the
// k-stride must be 4 or 12 mod 16 doubles): X and Y rows of W + 4, the
// diagonal-block inverse in columns of KB + 4, and the factor halves in
// columns of slab_ldh(n) holding only the rows a step updates (at most
// n - KB of them, stored from row 0).  (Strides of W, KB and lu_ld(n) made
// the Di product and the update 4-way / 4-way / 2-way conflicted: 64 k + 125 k
// of a 260-row slab's 252 k cycles.)
template <int KB>
__host__ __device__ constexpr int slab_ldh(int n) {
  int r = ((n + KB - 1) / KB - 1) * KB;  // most rows a step updates: above the last (ragged) block
  r = r < 16 ? 16 : r;
  r = (r + 3) & ~3;              // even (16-byte copies of row pairs), multiple of 4
  return (r & 7) == 4 ? r : r + 4;  // 4 or 12 mod 16
}
template <int KB, int W>
inline size_t getrs_smem_bytes(int n) {
  return sizeof(double) * ((size_t)lu_ld<KB>(n) * (W + 4) + (size_t)KB * slab_ldh<KB>(n) + 16 + KB * (KB + 4));
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}

__device__ __forceinline__ void cp_async16(double* dst, const double* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// MWT: warp tiles (16 rows x 32 columns) of the update a warp may hold --
// 0: sized for 383 rows; the host passes slab_mwt() when the block is small
// enough for fewer (fewer accumulator registers).
template <int KB, int W, int NT>
__host__ __device__ constexpr int slab_mwt(int n) {
  return ((((n + KB - 1) / KB - 1) * KB + 15) / 16 * (W / 32) + NT / 32 - 1) / (NT / 32);
}
template <int KB, int W, int NT = kLuThreads, int MWT = 0>
__global__ void __launch_bounds__(NT) lb_getrs_slab_kernel(int n, int m, double* const* __restrict__ As,
                                                                   const int* __restrict__ perm_all,
                                                                   const double* __restrict__ inv_all,
                                                                   double* const* __restrict__ Xs) {
  constexpr int KH = KB / 2;  // k-half
  extern __shared__ __align__(16) double lu_sm[];
  constexpr int XS = W + 4, DS = KB + 4;   // row stride of X and Y, column stride of Di (conflict-free)
  const int ld = lu_ld<KB>(n), ldh = slab_ldh<KB>(n);
  double* X = lu_sm;                       // [ld][XS]
  double* H[2] = {X + (size_t)ld * XS, X + (size_t)ld * XS + (size_t)KH * ldh};  // [KH][ldh] each, rows from lo
  double* Dis = H[1] + (size_t)KH * ldh + 16;  // [KB][DS] (streamed in with the first half; 16: tile reads past the last row)
  const int b = blockIdx.x, s = blockIdx.y, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int col0 = s * W, wc = min(W, m - col0);
  if (wc <= 0) return;
  const double* A = As[b];
  double* Xg = Xs[b] + (size_t)col0 * n;
  const int* perm = perm_all ? perm_all + (size_t)b * n : nullptr;
  const double* inv = inv_all + (size_t)b * lu_inv_stride<KB>(n);
  const int np = (n + KB - 1) / KB, nsteps = 2 * np;
  auto geom = [&](int q, int& p, int& r0, int& kb, int& lo, int& hi) {
    const bool fwd = q < np;
    p = fwd ? q : nsteps - 1 - q;
    r0 = p * KB;
    kb = min(KB, n - r0);
    lo = fwd ? r0 + kb : 0;  // rows the step updates: below the block (L) / above it (U)
    hi = fwd ? n : r0;
  };
  // issue the copies of half h of step q's factor block (and its Di when h == 1)
  // 16-byte copies of row pairs when every column start is 16-byte aligned
  // (n even; the row ranges start at multiples of KB or at n - r0 = kb even)
  const bool pairs = (n & 1) == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0;
  auto issue = [&](int q, int h) {
    int p, r0, kb, lo, hi;
    geom(q, p, r0, kb, lo, hi);
    double* dst = H[h];
    const int k_end = min(KH, kb - h * KH);
    if (pairs) {
      const int np2 = (hi - lo) >> 1;  // row pairs (hi - lo is even)
      for (int t = tid; t < k_end * np2; t += NT) {
        const int k = t / np2, i = lo + 2 * (t - k * np2);
        cp_async16(dst + (size_t)k * ldh + (i - lo), A + (size_t)(r0 + h * KH + k) * n + i);
      }
    } else {
      for (int k = 0; k < k_end; ++k) {
        const double* src = A + (size_t)(r0 + h * KH + k) * n;
        for (int i = lo + tid; i < hi; i += NT) cp_async8(dst + (size_t)k * ldh + (i - lo), src + i);
      }
    }
    if (h == 0) {  // Di of step q: its buffer is free once step q-1's Di product is done
      const double* di = inv + (size_t)(q < np ? 2 * p : 2 * p + 1) * KB * KB;
      for (int t = 2 * tid; t < KB * KB; t += 2 * NT) cp_async16(Dis + (t / KB) * DS + (t % KB), di + t);
    }
    cp_async_commit();
  };
  issue(0, 0);
  issue(0, 1);
  // gather P X into shared memory (zero rows n..ld, zero columns wc..W) by
  // cp.async: the whole slab is in flight at once (a register-staged gather
  // of 8 columns at a time left each CTA -- one per SM -- waiting on 8
  // successive HBM round trips, 16 % of the kernel at 256 blocks); the first
  // step's wait covers this group
  for (int i = tid; i < ld; i += NT) {  // consecutive threads: consecutive rows of a column
    const int src = (i < n) ? (perm ? perm[i] : i) : 0;
    for (int c = 0; c < W; ++c) {
      if (i < n && c < wc)
        cp_async8(X + (size_t)i * XS + c, Xg + (size_t)c * n + src);
      else
        X[(size_t)i * XS + c] = 0.0;
    }
  }
  cp_async_commit();
#ifdef LB_LU_PROF
  long long t0_ = clock64(), pacc_[8] = {}, pcol_[4] = {};
#endif
  for (int q = 0; q < nsteps; ++q) {
    int p, r0, kb, lo, hi;
    geom(q, p, r0, kb, lo, hi);
    cp_async_wait<0>();  // H1(q) and Di(q) (H0(q) landed earlier)
    __syncthreads();
    LU_T(1);
    // Y = Di X[r0 : r0 + kb] on the FP64 tensor path (mma.m8n8k4.f64):
    // 4 x (W/8) tiles of 8 x 8, W/16 per warp
    const double* Di = Dis;
    {
      static_assert(KB == 32 && (W == 32 || W == 64), "DMMA tiling assumes 32-row blocks, 32/64-column slabs");
      constexpr int NWS = NT / 32;
      static_assert(NWS % 4 == 0 && (W / 8) % (NWS / 4) == 0, "4 row tiles x (W/8) column tiles over the warps");
      constexpr int TPW = (W / 8) / (NWS / 4);  // column tiles per warp
      const int m = warp & 3, n0 = (warp >> 2) * TPW, lr = lane >> 2, lk = lane & 3;
      double d[TPW][2];
#pragma unroll
      for (int nn = 0; nn < TPW; ++nn) d[nn][0] = d[nn][1] = 0.0;
#pragma unroll
      for (int k0 = 0; k0 < KB; k0 += 4) {
        const int k = k0 + lk;
        const double av = Di[(size_t)k * DS + 8 * m + lr];
#pragma unroll
        for (int nn = 0; nn < TPW; ++nn) {
          const double bv = k < kb ? X[(size_t)(r0 + k) * XS + 8 * (n0 + nn) + lr] : 0.0;
          dmma_884(d[nn], av, bv);
        }
      }
      __syncthreads();  // every warp has read the block's rows of X: they become Y in place
      if (8 * m + lr < kb) {
#pragma unroll
        for (int nn = 0; nn < TPW; ++nn)
          *reinterpret_cast<double2*>(X + (size_t)(r0 + 8 * m + lr) * XS + 8 * (n0 + nn) + 2 * lk) =
              make_double2(d[nn][0], d[nn][1]);
      }
    }
    __syncthreads();
    const double* Y = X + (size_t)r0 * XS;  // [kb][XS]
    LU_T(2);
    // X[lo:hi] -= F Y in two k-halves on the FP64 tensor path: warp tiles of
    // 16 rows x 32 columns (2 x 4 MMA tiles of 8 x 8), acc kept across halves
    constexpr int CGW = W / 32;            // 32-column groups
    const int nr = hi - lo, nwt = ((nr + 15) >> 4) * CGW;
    constexpr int kMaxWt = MWT ? MWT : (24 * CGW + NT / 32 - 1) / (NT / 32);  // ceil(ceil(383 / 16) CGW / warps)
    LB_DCHECK(nwt <= kMaxWt * (NT / 32));
    double acc[kMaxWt][2][4][2];
#pragma unroll
    for (int u = 0; u < kMaxWt; ++u)
#pragma unroll
      for (int mm = 0; mm < 2; ++mm)
#pragma unroll
        for (int nn = 0; nn < 4; ++nn) acc[u][mm][nn][0] = acc[u][mm][nn][1] = 0.0;
    const int lr = lane >> 2, lk = lane & 3;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int k1 = min(kb, (h + 1) * KH);
      const double* Hh = H[h];  // rows stored from lo
#pragma unroll
      for (int u = 0; u < kMaxWt; ++u) {
        const int t = warp + u * (NT / 32);
        if (t >= nwt) break;
        const int wt = t / CGW, cg = t - (t / CGW) * CGW;
#pragma unroll
        for (int kq = 0; kq < KH; kq += 4) {
          const int k = h * KH + kq + lk;
          double av[2], bv[4];
#pragma unroll
          for (int mm = 0; mm < 2; ++mm)
            av[mm] = k < k1 ? Hh[(size_t)(kq + lk) * ldh + 16 * wt + 8 * mm + lr] : 0.0;
#pragma unroll
          for (int nn = 0; nn < 4; ++nn) bv[nn] = k < k1 ? Y[(size_t)k * XS + 32 * cg + 8 * nn + lr] : 0.0;
#pragma unroll
          for (int mm = 0; mm < 2; ++mm)
#pragma unroll
            for (int nn = 0; nn < 4; ++nn) dmma_884(acc[u][mm][nn], av[mm], bv[nn]);
        }
      }
      if (h == 0) {
        __syncthreads();  // H0 free: stream in the next step's first half
        if (q + 1 < nsteps) issue(q + 1, 0);
      }
    }
    LU_T(3);
#pragma unroll
    for (int u = 0; u < kMaxWt; ++u) {
      const int t = warp + u * (NT / 32);
      if (t >= nwt) break;
      const int wt = t / CGW, cg = t - (t / CGW) * CGW;
#pragma unroll
      for (int mm = 0; mm < 2; ++mm) {
        const int R = 16 * wt + 8 * mm + lr;
        if (R >= nr) continue;
#pragma unroll
        for (int nn = 0; nn < 4; ++nn) {
          double* xr = X + (size_t)(lo + R) * XS + 32 * cg + 8 * nn + 2 * lk;
          const double2 x2 = *reinterpret_cast<const double2*>(xr);
          *reinterpret_cast<double2*>(xr) = make_double2(x2.x - acc[u][mm][nn][0], x2.y - acc[u][mm][nn][1]);
        }
      }
    }
    LU_T(4);
    __syncthreads();  // H1 and Y free
    if (q + 1 < nsteps) issue(q + 1, 1);
    LU_T(5);
  }
  LU_FLUSH();
  cp_async_wait<0>();
  __syncthreads();
  for (int c = 0; c < wc; ++c)
    for (int i = tid; i < n; i += NT) Xg[(size_t)c * n + i] = X[(size_t)i * XS + c];
}

// v := A^-1 v for one vector per block (the cyclic reduction's vector
// passes), A the factors of lb_getrf_kernel: permuted gather into shared
// memory, then block forward / backward substitution -- per 32-row block a
// warp-synchronous substitution with the block's triangle (lane r holds
// x_r; the same operation order as LAPACK's trsv, divisions by the U
// diagonal), then the rows still to update by one thread per row, the
// block's 32 factor entries of that row read in one round of coalesced
// loads.  (The explicit diagonal-block inverses of the many-column solve
// are not used here: for the ill-conditioned electron systems of config 4
// the vector pass needs the substitution's accuracy.)
template <int KB>
__global__ void __launch_bounds__(kLuThreads) lb_lu_vsolve_kernel(int n, int count, double* const* __restrict__ As,
                                                                  const int* __restrict__ perm_all,
                                                                  const double* __restrict__ inv_all,
                                                                  double* const* __restrict__ Vs) {
  extern __shared__ __align__(16) double lu_sm[];
  double* x = lu_sm;  // [n]
  const int b = blockIdx.x, tid = threadIdx.x;
  if (b >= count) return;
  const double* A = As[b];
  const int* perm = perm_all + (size_t)b * n;
  const double* inv = inv_all + (size_t)b * lu_inv_stride<KB>(n);
  double* v = Vs[b];
  for (int i = tid; i < n; i += kLuThreads) x[i] = v[perm[i]];
  const int np = (n + KB - 1) / KB;
  for (int q = 0; q < 2 * np; ++q) {
    const bool fwd = q < np;
    const int p = fwd ? q : 2 * np - 1 - q;
    const int r0 = p * KB, kb = min(KB, n - r0);
    const int lo = fwd ? r0 + kb : 0, hi = fwd ? n : r0;
    __syncthreads();
    // this thread's rows of the update (<= 2 for n <= 384): their 32 factor
    // entries are loaded first, so the load latency overlaps the triangle
    const int i0 = lo + tid, i1 = i0 + kLuThreads;
    double f0[KB], f1[KB];
#pragma unroll
    for (int k = 0; k < KB; ++k) {
      f0[k] = (k < kb && i0 < hi) ? A[(size_t)(r0 + k) * n + i0] : 0.0;
      f1[k] = (k < kb && i1 < hi) ? A[(size_t)(r0 + k) * n + i1] : 0.0;
    }
    if (tid < 32) {  // the diagonal block's triangle, warp 0
      static_assert(KB == 32, "one lane per block row");
      const int r = tid;
      double xr = r < kb ? x[r0 + r] : 0.0;
      double t[KB];  // column k of the block at row r
#pragma unroll
      for (int k = 0; k < KB; ++k) t[k] = (k < kb && r < kb) ? A[(size_t)(r0 + k) * n + r0 + r] : 0.0;
      if (fwd) {
#pragma unroll
        for (int k = 0; k < KB; ++k) {
          const double xk = __shfl_sync(0xffffffffu, xr, k);
          if (r > k && k < kb) xr = fma(-t[k], xk, xr);
        }
      } else {
        // 1/u_rr per lane up front (overlapping the loads): the chain then
        // multiplies instead of running 32 dependent IEEE divisions
        const double rinv = 1.0 / (r < kb ? A[(size_t)(r0 + r) * n + r0 + r] : 1.0);
#pragma unroll
        for (int k = KB - 1; k >= 0; --k) {
          if (r == k && k < kb) xr = xr * rinv;
          const double xk = __shfl_sync(0xffffffffu, xr, k);
          if (r < k && k < kb) xr = fma(-t[k], xk, xr);
        }
      }
      if (r < kb) x[r0 + r] = xr;
    }
    __syncthreads();
    if (i0 < hi) {
      double acc = x[i0];
#pragma unroll
      for (int k = 0; k < KB; ++k) acc = fma(-f0[k], x[r0 + (k < kb ? k : 0)], acc);
      x[i0] = acc;
    }
    if (i1 < hi) {
      double acc = x[i1];
#pragma unroll
      for (int k = 0; k < KB; ++k) acc = fma(-f1[k], x[r0 + (k < kb ? k : 0)], acc);
      x[i1] = acc;
    }
  }
  __syncthreads();
  for (int i = tid; i < n; i += kLuThreads) v[i] = x[i];
}

}  // namespace lb
