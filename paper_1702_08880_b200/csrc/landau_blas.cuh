// landau_blas.cuh -- the batched dense products of the Crank-Nicolson block
// cyclic reduction (landau_b200.cu, cn_factor_issue / cn_solve_issue) on
// this package's own kernels, replacing cuBLAS gemmBatched / gemvBatched:
//
//  * lb_bgemm_kernel: C_b = beta C_b - A_b B_b for a batch of n x n
//    column-major blocks given by pointer arrays (the reduction's Schur
//    updates D -= L P^U + U P^L and its new couplings -L P^L, -U P^U).  One
//    CTA per (64 x 64 tile of C, matrix); A and B tiles of 16 k-columns are
//    double-buffered into shared memory by cp.async; four warps, each a
//    32 x 32 sub-tile of 4 x 4 FP64 MMA tiles (mma.sync.m8n8k4.f64, SASS
//    DMMA) with the accumulators in registers.  Edge tiles are zero-padded.
//  * lb_bgemv_kernel: y_b -= A_b x_b (the level passes of the block
//    substitution): one CTA per (32-row strip, matrix), eight column groups
//    per row reading A's columns coalesced, partial sums added in fixed
//    order.
#pragma once
#include "landau_lu.cuh"

namespace lb {

constexpr int kGemmTile = 64, kGemmKT = 16, kGemmThreads = 128;
constexpr int kGemmLdA = kGemmTile + 4;   // A tile [KT][64 + 4] (k-major)
constexpr int kGemmLdB = kGemmKT + 4;     // B tile [64][KT + 4] (column-major)

__device__ __forceinline__ void gemm_load_tile(double* __restrict__ As, double* __restrict__ Bs,
                                               const double* __restrict__ A, const double* __restrict__ B,
                                               int n, int i0, int j0, int k0, bool even, int tid) {
  // A[i0 .. i0+64, k0 .. k0+16]: per k, 64 contiguous rows
  if (even) {
    for (int t = tid; t < kGemmKT * (kGemmTile / 2); t += kGemmThreads) {
      const int kk = t / (kGemmTile / 2), ii = 2 * (t % (kGemmTile / 2));
      const int k = k0 + kk, i = i0 + ii;
      double* dst = As + kk * kGemmLdA + ii;
      if (k < n && i + 1 < n) {
        cp_async16(dst, A + (size_t)k * n + i);
      } else {
        dst[0] = (k < n && i < n) ? A[(size_t)k * n + i] : 0.0;
        dst[1] = 0.0;
      }
    }
    // B[k0 .. k0+16, j0 .. j0+64]: per column j, 16 contiguous k
    for (int t = tid; t < kGemmTile * (kGemmKT / 2); t += kGemmThreads) {
      const int jj = t / (kGemmKT / 2), kk = 2 * (t % (kGemmKT / 2));
      const int j = j0 + jj, k = k0 + kk;
      double* dst = Bs + jj * kGemmLdB + kk;
      if (j < n && k + 1 < n) {
        cp_async16(dst, B + (size_t)j * n + k);
      } else {
        dst[0] = (j < n && k < n) ? B[(size_t)j * n + k] : 0.0;
        dst[1] = 0.0;
      }
    }
  } else {  // odd n: 8-byte copies (columns are not 16-byte aligned)
    for (int t = tid; t < kGemmKT * kGemmTile; t += kGemmThreads) {
      const int kk = t / kGemmTile, ii = t % kGemmTile;
      const int k = k0 + kk, i = i0 + ii;
      double* dst = As + kk * kGemmLdA + ii;
      if (k < n && i < n) cp_async8(dst, A + (size_t)k * n + i);
      else *dst = 0.0;
    }
    for (int t = tid; t < kGemmTile * kGemmKT; t += kGemmThreads) {
      const int jj = t / kGemmKT, kk = t % kGemmKT;
      const int j = j0 + jj, k = k0 + kk;
      double* dst = Bs + jj * kGemmLdB + kk;
      if (j < n && k < n) cp_async8(dst, B + (size_t)j * n + k);
      else *dst = 0.0;
    }
  }
  cp_async_commit();
}

__global__ void __launch_bounds__(kGemmThreads) lb_bgemm_kernel(int n, double* const* __restrict__ As_,
                                                                double* const* __restrict__ Bs_,
                                                                double* const* __restrict__ Cs_, int beta) {
  __shared__ __align__(16) double As[2][kGemmKT * kGemmLdA];
  __shared__ __align__(16) double Bs[2][kGemmTile * kGemmLdB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tiles = (n + kGemmTile - 1) / kGemmTile;
  const int i0 = (blockIdx.x % tiles) * kGemmTile, j0 = (blockIdx.x / tiles) * kGemmTile;
  const double* __restrict__ A = As_[blockIdx.y];
  const double* __restrict__ B = Bs_[blockIdx.y];
  double* __restrict__ C = Cs_[blockIdx.y];
  const bool even = (n & 1) == 0;
  const int wr = (warp & 1) * 32, wc = (warp >> 1) * 32;  // warp sub-tile
  const int lr = lane >> 2, lk = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int nk = (n + kGemmKT - 1) / kGemmKT;
  gemm_load_tile(As[0], Bs[0], A, B, n, i0, j0, 0, even, tid);
  for (int s = 0; s < nk; ++s) {
    if (s + 1 < nk) {
      gemm_load_tile(As[(s + 1) & 1], Bs[(s + 1) & 1], A, B, n, i0, j0, (s + 1) * kGemmKT, even, tid);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* a_s = As[s & 1];
    const double* b_s = Bs[s & 1];
#pragma unroll
    for (int k4 = 0; k4 < kGemmKT; k4 += 4) {
      double av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = a_s[(k4 + lk) * kGemmLdA + wr + 8 * a + lr];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = b_s[(wc + 8 * b + lr) * kGemmLdB + k4 + lk];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma_884(acc[a][b], av[a], bv[b]);
    }
    __syncthreads();
  }
  // C = beta C - A B (lane holds D[lr][2 lk + e] of each 8 x 8 tile)
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int i = i0 + wr + 8 * a + lr;
    if (i >= n) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = j0 + wc + 8 * b + 2 * lk + e;
        if (j >= n) continue;
        double* c = C + (size_t)j * n + i;
        *c = beta ? *c - acc[a][b][e] : -acc[a][b][e];
      }
  }
}

// y_b -= A_b x_b, n x n column-major.  One CTA per (32-row strip, matrix):
// 32 rows x 8 column groups; thread (row, g) sums the columns k = g mod 8
// (reads of a column's 32 rows are one 256-byte segment per warp), the 8
// partial sums meet in shared memory in fixed order.
constexpr int kGemvRows = 32, kGemvGroups = 8, kGemvThreads = kGemvRows * kGemvGroups;
__global__ void __launch_bounds__(kGemvThreads) lb_bgemv_kernel(int n, double* const* __restrict__ As_,
                                                                double* const* __restrict__ xs_,
                                                                double* const* __restrict__ ys_) {
  __shared__ double part[kGemvGroups][kGemvRows];
  const double* __restrict__ A = As_[blockIdx.y];
  const double* __restrict__ x = xs_[blockIdx.y];
  double* __restrict__ y = ys_[blockIdx.y];
  const int r = threadIdx.x & (kGemvRows - 1), g = threadIdx.x / kGemvRows;
  const int i = blockIdx.x * kGemvRows + r;
  double s0 = 0.0, s1 = 0.0;
  if (i < n) {
    int k = g;
    for (; k + kGemvGroups < n; k += 2 * kGemvGroups) {
      s0 = fma(A[(size_t)k * n + i], x[k], s0);
      s1 = fma(A[(size_t)(k + kGemvGroups) * n + i], x[k + kGemvGroups], s1);
    }
    if (k < n) s0 = fma(A[(size_t)k * n + i], x[k], s0);
  }
  part[g][r] = s0 + s1;
  __syncthreads();
  if (g == 0 && i < n) {
    double s = part[0][r];
#pragma unroll
    for (int q = 1; q < kGemvGroups; ++q) s += part[q][r];
    y[i] -= s;
  }
}

}  // namespace lb
