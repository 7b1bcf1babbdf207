// landau_lu.cuh -- batched dense LU with partial pivoting and the
// many-right-hand-side solve of the Crank-Nicolson block cyclic reduction
// (landau_b200.cu, cn_factor_issue), replacing cuBLAS getrfBatched /
// getrsBatched / trsmBatched at the solver's block sizes (nb = 68..354).
//
// cuBLAS's batched getrf is a latency-bound chain of small launches per
// column panel (~4.6 us per column at nb = 260, 1.2 ms per call whatever
// the batch), and its batched trsm + laswp with 2 nb right-hand sides runs
// at ~4 TFLOP/s.  Here:
//  * lb_getrf_kernel: one CTA per matrix, right-looking blocked LU with a
//    KB-column panel in shared memory.  Panel: per column one CTA-wide
//    pivot search (LAPACK idamax: first maximum of |a|), row swap, and a
//    row-owned scale + rank-1 update (3 barriers per column).  Then the
//    panel's swaps on the other columns, U12 = L11^-1 A12 (one column per
//    thread, L11 broadcast from shared memory) and the trailing update
//    A22 -= L21 U12 with 8x8 register tiles.  Output in LAPACK layout (unit
//    L below the diagonal, U on and above it, 1-based ipiv) so the vector
//    solves (lb_small_solve_kernel, getrs) consume it unchanged; also the
//    row permutation and the inverses of the KB x KB diagonal blocks of L
//    and U (for the solve below).
//  * lb_getrs_slab_kernel: X := A^-1 X for an n x m block of right-hand
//    sides (the cyclic reduction's [L U], m = 2 nb), one CTA per (matrix,
//    W-column slab): rows gathered through the permutation into shared
//    memory, then block forward / backward substitution in which every
//    step is a small GEMM (the diagonal block through its stored inverse,
//    the off-diagonal column block staged in shared memory).
#pragma once
#include <cstdint>

namespace lb {

constexpr int kLuThreads = 256;
#ifdef LB_LU_PROF
__device__ long long lu_prof[8];  // cycles per phase (block 0, thread 0), accumulated
#define LU_T(k)                                                        \
  do {                                                                 \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                         \
      const long long t1_ = clock64();                                 \
      lu_prof[k] += t1_ - t0_;                                         \
      t0_ = t1_;                                                       \
    }                                                                  \
  } while (0)
#else
#define LU_T(k) \
  do {          \
  } while (0)
#endif

template <int KB>
__host__ __device__ constexpr int lu_ld(int n) {
  return (n + 7) & ~7;  // panel / slab leading dimension (8-row padding for the 8x8 tiles)
}

// shared memory of lb_getrf_kernel<KB>: panel [KB][ld] + U12 rows [KB][ld] + reduction scratch
template <int KB>
inline size_t getrf_smem_bytes(int n) {
  return sizeof(double) * (2 * (size_t)KB * lu_ld<KB>(n) + 2 * 32) +
         sizeof(int) * (KB + 32 + lu_ld<KB>(n) + 4 * KB);
}

// Inverse diagonal blocks: per matrix, per panel p, invL[p] (KB x KB, unit
// lower, column-major) then invU[p]; inv_stride = 2 * npanel * KB * KB.
template <int KB>
__host__ __device__ inline int lu_inv_stride(int n) {
  return 2 * ((n + KB - 1) / KB) * KB * KB;
}

template <int KB>
__global__ void __launch_bounds__(kLuThreads) lb_getrf_kernel(int n, double* const* __restrict__ As,
                                                              int* __restrict__ ipiv_all,
                                                              int* __restrict__ perm_all,
                                                              int* __restrict__ info_all,
                                                              double* __restrict__ inv_all, int pivot) {
  extern __shared__ __align__(16) double lu_sm[];
  const int ld = lu_ld<KB>(n);
  double* P = lu_sm;                   // panel, column-major [KB][ld] (row offset from c0)
  double* Ub = lu_sm + (size_t)KB * ld;  // U12 rows, row-major [KB][ld] (column offset from c0 + w)
  double* redv = Ub + (size_t)KB * ld;   // [32]
  int* redi = reinterpret_cast<int*>(redv + 32);  // [32]
  int* pv_sh = redi + 32;                         // [KB]
  int* lp = pv_sh + KB;                           // [ld] panel-local row permutation
  int* tl_dst = lp + ld;                          // [2 KB] rows a panel's swaps touch
  int* tl_src = tl_dst + 2 * KB;                  // [2 KB] and where their values come from
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kLuThreads / 32;
  double* A = As[b];
  int* ipiv = ipiv_all ? ipiv_all + (size_t)b * n : nullptr;
  double* inv = inv_all + (size_t)b * lu_inv_stride<KB>(n);
  int info = 0;
#ifdef LB_LU_PROF
  long long t0_ = clock64();
#endif

  for (int c0 = 0, p = 0; c0 < n; c0 += KB, ++p) {
    const int w = min(KB, n - c0), m = n - c0;
    // 1. panel rows c0..n, columns c0..c0+w -> P (zero padding to ld rows /
    //    KB columns); rows tid + 256 h, eight columns of loads in flight
    for (int i = tid; i < ld; i += kLuThreads) lp[i] = i;  // panel-local row permutation
    for (int h = 0; h * kLuThreads < ld; ++h) {
      const int i = tid + h * kLuThreads;
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
    // 2. unblocked LU of the panel
    for (int j = 0; j < w; ++j) {
      int piv = j;
      if (pivot) {
        double best = -1.0;
        int bi = m;
        for (int i = j + tid; i < m; i += kLuThreads) {
          const double v = fabs(P[(size_t)j * ld + i]);
          if (v > best) { best = v; bi = i; }  // rows visited in increasing order
        }
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
        piv = bi;  // idamax: the first index of the largest |a|
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
      for (int i = j + 1 + tid; i < m; i += kLuThreads) {
        const double l = P[(size_t)j * ld + i] * r;
        P[(size_t)j * ld + i] = l;
        int k = j + 1;
        for (; k + 4 <= w; k += 4) {  // four independent read-modify-writes per round
          double a[4], u[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            a[q] = P[(size_t)(k + q) * ld + i];
            u[q] = P[(size_t)(k + q) * ld + j];
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) P[(size_t)(k + q) * ld + i] = fma(-l, u[q], a[q]);
        }
        for (; k < w; ++k) P[(size_t)k * ld + i] = fma(-l, P[(size_t)k * ld + j], P[(size_t)k * ld + i]);
      }
      __syncthreads();
    }
    LU_T(1);
    // 3. panel back; pivots (1-based, global rows)
    for (int j = 0; j < w; ++j)
      for (int i = tid; i < m; i += kLuThreads) A[(size_t)(c0 + j) * n + c0 + i] = P[(size_t)j * ld + i];
    if (ipiv && tid < w) ipiv[c0 + tid] = c0 + pv_sh[tid] + 1;
    // 4. inverses of the diagonal blocks: unit lower L11 and upper U11 (one
    //    column of each inverse per thread)
    {
      double* iL = inv + (size_t)(2 * p) * KB * KB;
      double* iU = iL + KB * KB;
      if (tid < KB) {  // column tid of L11^-1: forward substitution of e_tid
        const int c = tid;
        double x[KB];
#pragma unroll
        for (int i = 0; i < KB; ++i) {
          double s = (i == c) ? 1.0 : 0.0;
#pragma unroll
          for (int k = 0; k < i; ++k) s = fma(-P[(size_t)k * ld + i], x[k], s);
          x[i] = (i < w) ? s : 0.0;
        }
#pragma unroll
        for (int i = 0; i < KB; ++i) iL[(size_t)c * KB + i] = (c < w) ? x[i] : 0.0;
      } else if (tid >= 32 && tid < 32 + KB) {  // column c of U11^-1: back substitution of e_c
        const int c = tid - 32;
        double x[KB];
#pragma unroll
        for (int i = KB - 1; i >= 0; --i) {
          double s = (i == c) ? 1.0 : 0.0;
#pragma unroll
          for (int k = i + 1; k < KB; ++k) s = fma(-P[(size_t)k * ld + i], x[k], s);
          const double dii = (i < w) ? P[(size_t)i * ld + i] : 1.0;
          x[i] = (i < w && c < w) ? s / dii : 0.0;
        }
#pragma unroll
        for (int i = 0; i < KB; ++i) iU[(size_t)c * KB + i] = x[i];
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
    if (tid < w) {
      tl_dst[tid] = tid;
      tl_src[tid] = lp[tid];
      const int r = pv_sh[tid];
      bool first = pivot && r >= w;
      for (int q = 0; q < tid && first; ++q) first = pv_sh[q] != r;
      tl_dst[w + tid] = r;
      tl_src[w + tid] = first ? lp[r] : -1;
    }
    __syncthreads();
    const int cnt = 2 * w;
    const int n2 = n - c0 - w;
    for (int k = tid; k < n - w; k += kLuThreads) {
      const int col = k < c0 ? k : k + w;  // skip the panel's own columns
      double* Ac = A + (size_t)col * n + c0;
      double v[2 * KB];
#pragma unroll
      for (int q = 0; q < 2 * KB; ++q) {
        const int sq = q < cnt ? tl_src[q] : -1;
        v[q] = sq >= 0 ? Ac[sq] : 0.0;
      }
      if (col >= c0 + w) {  // the first w entries are rows 0..w-1 in order
#pragma unroll
        for (int i = 0; i < KB; ++i) {
          double sacc = v[i];
#pragma unroll
          for (int q = 0; q < i; ++q) sacc = fma(-P[(size_t)q * ld + i], v[q], sacc);
          v[i] = (i < w) ? sacc : 0.0;
        }
        const int k2 = col - c0 - w;
#pragma unroll
        for (int i = 0; i < KB; ++i) Ub[(size_t)i * ld + k2] = v[i];
      } else if (!pivot) {
        continue;  // left columns: nothing to do without swaps
      }
#pragma unroll
      for (int q = 0; q < 2 * KB; ++q)
        if (q < cnt && tl_src[q] >= 0) Ac[tl_dst[q]] = v[q];
    }
    // zero padding of Ub's columns n2..ld (8-column tiles read them)
    for (int t = tid; t < KB * 8; t += kLuThreads) {
      const int i = t >> 3, k2 = n2 + (t & 7);
      if (k2 < ld) Ub[(size_t)i * ld + k2] = 0.0;
    }
    __syncthreads();
    LU_T(3);
    // 6. trailing update A22 -= L21 U12 (8 x 8 register tiles)
    const int m2 = m - w;
    if (m2 > 0 && n2 > 0) {
      const int tr = (m2 + 7) >> 3, tc = (n2 + 7) >> 3;
      for (int t = tid; t < tr * tc; t += kLuThreads) {
        const int ti = (t / tc) * 8, tk = (t - (t / tc) * tc) * 8;
        // the tile's current values first (one round of independent loads)
        double acc[8][8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const double* Ac = A + (size_t)(c0 + w + tk + c) * n + c0 + w + ti;
#pragma unroll
          for (int r = 0; r < 8; ++r) acc[c][r] = (tk + c < n2 && ti + r < m2) ? Ac[r] : 0.0;
        }
        for (int j = 0; j < w; ++j) {
          const double* lp = P + (size_t)j * ld + w + ti;  // L21[ti..ti+8][j]
          const double* up = Ub + (size_t)j * ld + tk;     // U12[j][tk..tk+8]
          double lv[8], uv[8];
#pragma unroll
          for (int q = 0; q < 8; q += 2) {
            const double2 a2 = *reinterpret_cast<const double2*>(lp + q);
            const double2 u2 = *reinterpret_cast<const double2*>(up + q);
            lv[q] = a2.x; lv[q + 1] = a2.y;
            uv[q] = u2.x; uv[q + 1] = u2.y;
          }
#pragma unroll
          for (int c = 0; c < 8; ++c)
#pragma unroll
            for (int r = 0; r < 8; ++r) acc[c][r] = fma(-lv[r], uv[c], acc[c][r]);
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          if (tk + c >= n2) break;
          double* Ac = A + (size_t)(c0 + w + tk + c) * n + c0 + w + ti;
#pragma unroll
          for (int r = 0; r < 8; ++r)
            if (ti + r < m2) Ac[r] = acc[c][r];
        }
      }
    }
    __syncthreads();
    LU_T(4);
  }
  if (tid == 0) {
    if (info_all) info_all[b] = info;
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
  }
}

// X := A^-1 X for X = the n x m column-major block at Xs[b] (leading
// dimension n), A the factors of lb_getrf_kernel.  CTA (b, s) owns columns
// [s W, s W + W).  Shared memory: the slab [ld][W] (row-major: a row of W
// columns is contiguous), one staged factor column block [KB][ld], the
// diagonal inverse [KB][KB].
template <int KB, int W>
inline size_t getrs_smem_bytes(int n) {
  return sizeof(double) * ((size_t)lu_ld<KB>(n) * W + (size_t)KB * lu_ld<KB>(n) + KB * KB);
}

template <int KB, int W>
__global__ void __launch_bounds__(kLuThreads) lb_getrs_slab_kernel(int n, int m, double* const* __restrict__ As,
                                                                   const int* __restrict__ perm_all,
                                                                   const double* __restrict__ inv_all,
                                                                   double* const* __restrict__ Xs) {
  static_assert(KB * W / 4 <= kLuThreads, "one diagonal-block output group per thread");
  extern __shared__ __align__(16) double lu_sm[];
  const int ld = lu_ld<KB>(n);
  double* X = lu_sm;                       // [ld][W]
  double* F = X + (size_t)ld * W;          // [KB][ld]: factor columns, column-major
  double* Di = F + (size_t)KB * ld;        // [KB][KB] diagonal-block inverse, column-major
  const int b = blockIdx.x, s = blockIdx.y, tid = threadIdx.x;
  const int col0 = s * W, wc = min(W, m - col0);
  if (wc <= 0) return;
  const double* A = As[b];
  double* Xg = Xs[b] + (size_t)col0 * n;
  const int* perm = perm_all ? perm_all + (size_t)b * n : nullptr;
  const double* inv = inv_all + (size_t)b * lu_inv_stride<KB>(n);
  const int np = (n + KB - 1) / KB;
  // gather P X into shared memory (zero rows n..ld, zero columns wc..W)
  for (int i = tid; i < ld; i += kLuThreads) {  // consecutive threads: consecutive rows of a column
    const int src = (i < n) ? (perm ? perm[i] : i) : 0;
#pragma unroll 4
    for (int c = 0; c < W; ++c) X[(size_t)i * W + c] = (i < n && c < wc) ? Xg[(size_t)c * n + src] : 0.0;
  }
  // Per block step: Y = Di * X[r0:r0+KB] (KB x W, one thread per 4 outputs),
  // then X[rows] -= F[rows][0:KB] * Y for the rows still to update.
  auto step = [&](int r0, int kb, int u0, int u1) {
    // X[r0:r0+kb] := Di X[r0:r0+kb]  (KB x KB times KB x W)
    __syncthreads();
    double y[4];
    const int nout = KB * W / 4;
    int yi = -1, yc = 0;
    for (int t = tid; t < nout; t += kLuThreads) {
      const int i = t / (W / 4), c = (t - i * (W / 4)) * 4;
      double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
      for (int k = 0; k < kb; ++k) {
        const double dk = Di[(size_t)k * KB + i];
        const double* xr = X + (size_t)(r0 + k) * W + c;
        a0 = fma(dk, xr[0], a0);
        a1 = fma(dk, xr[1], a1);
        a2 = fma(dk, xr[2], a2);
        a3 = fma(dk, xr[3], a3);
      }
      y[0] = a0; y[1] = a1; y[2] = a2; y[3] = a3;
      yi = i;
      yc = c;
    }
    __syncthreads();
    if (yi >= 0 && yi < kb) {
      double* xr = X + (size_t)(r0 + yi) * W + yc;
      xr[0] = y[0]; xr[1] = y[1]; xr[2] = y[2]; xr[3] = y[3];
    }
    __syncthreads();
    // X[u0:u1] -= F[u0:u1][0:kb] * X[r0:r0+kb]; 4 rows x 4 columns per thread
    const int nr = u1 - u0;
    if (nr <= 0) return;
    const int tr = (nr + 3) >> 2;
    for (int t = tid; t < tr * (W / 4); t += kLuThreads) {
      const int ri = (t / (W / 4)) * 4, c = (t - (t / (W / 4)) * (W / 4)) * 4;
      double acc[4][4] = {};
      for (int k = 0; k < kb; ++k) {
        const double* fp = F + (size_t)k * ld + u0 + ri;
        const double* xr = X + (size_t)(r0 + k) * W + c;
        const double2 x01 = *reinterpret_cast<const double2*>(xr);
        const double2 x23 = *reinterpret_cast<const double2*>(xr + 2);
        const double2 f01 = *reinterpret_cast<const double2*>(fp);
        const double2 f23 = *reinterpret_cast<const double2*>(fp + 2);
        const double xv[4] = {x01.x, x01.y, x23.x, x23.y};
        const double fv[4] = {f01.x, f01.y, f23.x, f23.y};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const double f = fv[r];
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[r][q] = fma(f, xv[q], acc[r][q]);
        }
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        if (ri + r >= nr) break;
        double* xr = X + (size_t)(u0 + ri + r) * W + c;
#pragma unroll
        for (int q = 0; q < 4; ++q) xr[q] -= acc[r][q];
      }
    }
  };
  // 2 np block steps: forward (L, unit lower) p = 0..np-1, then backward
  // (U) p = np-1..0.  Step q's factor column block F and diagonal inverse
  // Di are loaded into registers during step q-1 and stored after it.
  constexpr int kPf = (KB * 384) / kLuThreads;  // per-thread share of F (n <= 384)
  double fpf[kPf], dpf[KB * KB / kLuThreads];
  // element t = tid + e NT of F is (k, i) = divmod(t, ld): stepped without divisions
  const int k_0 = tid / ld, i_0 = tid - k_0 * ld, dk = kLuThreads / ld, di = kLuThreads - dk * ld;
  auto fetch = [&](int q) {
    const bool fwd = q < np;
    const int p = fwd ? q : 2 * np - 1 - q;
    const int r0 = p * KB, kb = min(KB, n - r0);
    const int lo = fwd ? r0 + kb : 0, hi = fwd ? n : r0;
    int k = k_0, i = i_0;
#pragma unroll
    for (int e = 0; e < kPf; ++e) {
      const bool in = k < kb && i >= lo && i < hi;
      fpf[e] = in ? A[(size_t)(r0 + k) * n + i] : 0.0;
      i += di;
      k += dk;
      if (i >= ld) { i -= ld; ++k; }
    }
#pragma unroll
    for (int e = 0; e < KB * KB / kLuThreads; ++e)
      dpf[e] = inv[(size_t)(fwd ? 2 * p : 2 * p + 1) * KB * KB + tid + e * kLuThreads];
  };
  auto stash = [&]() {
#pragma unroll
    for (int e = 0; e < kPf; ++e) {
      const int t = tid + e * kLuThreads;
      if (t < KB * ld) F[t] = fpf[e];
    }
#pragma unroll
    for (int e = 0; e < KB * KB / kLuThreads; ++e) Di[tid + e * kLuThreads] = dpf[e];
  };
  fetch(0);
  __syncthreads();  // the gather above is complete
  stash();
  for (int q = 0; q < 2 * np; ++q) {
    if (q + 1 < 2 * np) fetch(q + 1);
    const bool fwd = q < np;
    const int p = fwd ? q : 2 * np - 1 - q;
    const int r0 = p * KB, kb = min(KB, n - r0);
    if (fwd)
      step(r0, kb, r0 + kb, n);
    else
      step(r0, kb, 0, r0);
    __syncthreads();
    if (q + 1 < 2 * np) stash();
  }
  __syncthreads();
  for (int c = 0; c < wc; ++c)
    for (int i = tid; i < n; i += kLuThreads) Xg[(size_t)c * n + i] = X[(size_t)i * W + c];
}

}  // namespace lb
