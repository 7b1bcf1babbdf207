// landau_blas.cuh -- the batched dense products of the Crank-Nicolson block
// cyclic reduction (landau_b200.cu, cn_factor_issue / cn_solve_issue) on
// this package's own kernels, replacing cuBLAS gemmBatched / gemvBatched:
//
//  * lb_bgemm_kernel: [C0 | C1] = [b0 C0 | b1 C1] - A [B | B'] for a batch
//    of n x n column-major blocks given by pointer arrays, B' the block
//    after B (the reduction's products sharing A: L_k [P^L P^U]_{k-1} gives
//    the next level's coupling -L P^L and the Schur update D_k -= L P^U;
//    U_k [P^L P^U]_{k+1} gives D_k -= U P^L and -U P^U).  One CTA per
//    (64 x 64 tile of the product, matrix); A and B tiles of 16 k-columns are
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
                                               int n, int nc, int i0, int j0, int k0, bool even, int tid) {
  // A: n x n; B: n x nc (nc = n or 2n), both column-major with ld n
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
      if (j < nc && k + 1 < n) {
        cp_async16(dst, B + (size_t)j * n + k);
      } else {
        dst[0] = (j < nc && k < n) ? B[(size_t)j * n + k] : 0.0;
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
      if (j < nc && k < n) cp_async8(dst, B + (size_t)j * n + k);
      else *dst = 0.0;
    }
  }
  cp_async_commit();
}

// [C0_b | C1_b] = [beta0 C0_b | beta1 C1_b] - A_b [B_b | B_b + n^2]: A n x n,
// B the n x 2n pair of adjacent blocks (column-major, ld n), the product's
// first n columns into C0, the last n into C1 (C1 null: those columns are
// skipped).  The cyclic reduction's two products that share an A -- e.g.
// L_k P^L (the next level's coupling, beta 0) and L_k P^U (the Schur update
// of D_k, beta 1) -- are one launch reading A once.
// tri: the structure of A the caller vouches for -- 0 dense, 1 upper
// triangular (A[p][q] = 0 for p > q), 2 lower triangular (0 for q > p): the
// couplings of the reduction's level 0 are the band's own off-diagonal
// blocks, triangular when the block size covers the bandwidth.  The k-steps
// that only meet A's zeros are skipped; the sums that remain are formed in
// the same order, so the product is bitwise the dense one.
__global__ void __launch_bounds__(kGemmThreads) lb_bgemm_kernel(int n, double* const* __restrict__ As_,
                                                                double* const* __restrict__ Bs_,
                                                                double* const* __restrict__ C0s_, int beta0,
                                                                double* const* __restrict__ C1s_, int beta1,
                                                                int tri) {
  __shared__ __align__(16) double As[2][kGemmKT * kGemmLdA];
  __shared__ __align__(16) double Bs[2][kGemmTile * kGemmLdB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tiles = (n + kGemmTile - 1) / kGemmTile;
  const int i0 = (blockIdx.x % tiles) * kGemmTile, j0 = (blockIdx.x / tiles) * kGemmTile;
  double* __restrict__ C0 = C0s_[blockIdx.y];
  double* __restrict__ C1 = C1s_ ? C1s_[blockIdx.y] : nullptr;
  if (j0 >= n && !C1) return;
  const int nc = C1 ? 2 * n : n;  // product columns computed
  const double* __restrict__ A = As_[blockIdx.y];
  const double* __restrict__ B = Bs_[blockIdx.y];
  const bool even = (n & 1) == 0;
  const int wr = (warp & 1) * 32, wc = (warp >> 1) * 32;  // warp sub-tile
  const int lr = lane >> 2, lk = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  // 8 x 8 MMA tiles of this warp's 32 x 32 sub-tile that hold rows / columns
  // of the product (a prefix of the four; edge tiles of a 260-row block are
  // 4 rows of 64: the all-padding MMA tiles are skipped, warp-uniformly)
  const int na = min(4, max(0, (n - (i0 + wr) + 7) >> 3));
  const int nbt = min(4, max(0, (nc - (j0 + wc) + 7) >> 3));
  int ks = 0, nk = (n + kGemmKT - 1) / kGemmKT;
  // rows i0 .. i0+63 of an upper triangular A are zero left of column i0,
  // of a lower triangular one right of column i0+63
  if (tri == 1) ks = i0 / kGemmKT;
  else if (tri == 2) nk = min(nk, (i0 + kGemmTile + kGemmKT - 1) / kGemmKT);
  gemm_load_tile(As[0], Bs[0], A, B, n, nc, i0, j0, ks * kGemmKT, even, tid);
  for (int s = ks; s < nk; ++s) {
    const int cur = (s - ks) & 1;
    if (s + 1 < nk) {
      gemm_load_tile(As[cur ^ 1], Bs[cur ^ 1], A, B, n, nc, i0, j0, (s + 1) * kGemmKT, even, tid);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* a_s = As[cur];
    const double* b_s = Bs[cur];
    const int kv = min(kGemmKT, n - s * kGemmKT);  // k-columns of this step inside the matrix
#pragma unroll
    for (int k4 = 0; k4 < kGemmKT; k4 += 4) {
      if (k4 >= kv) break;  // zero padding only
      double av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = a_s[(k4 + lk) * kGemmLdA + wr + 8 * a + lr];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = b_s[(wc + 8 * b + lr) * kGemmLdB + k4 + lk];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        if (a >= na) break;
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if (b < nbt) dmma_884(acc[a][b], av[a], bv[b]);
      }
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
        int j = j0 + wc + 8 * b + 2 * lk + e;
        if (j >= nc) continue;
        const bool second = j >= n;
        double* c = (second ? C1 : C0) + (size_t)(second ? j - n : j) * n + i;
        *c = (second ? beta1 : beta0) ? *c - acc[a][b][e] : -acc[a][b][e];
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
  // four running sums (columns g + 8 (4 j + u)), loop unrolled twice: eight
  // independent column loads in flight per thread (a latency-bound pass:
  // the two-sum form waited out an L2 round trip every two columns)
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  if (i < n) {
    int k = g;
#pragma unroll 2
    for (; k + 3 * kGemvGroups < n; k += 4 * kGemvGroups) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        s[u] = fma(A[(size_t)(k + u * kGemvGroups) * n + i], x[k + u * kGemvGroups], s[u]);
    }
    for (; k < n; k += kGemvGroups) s[0] = fma(A[(size_t)k * n + i], x[k], s[0]);
  }
  part[g][r] = (s[0] + s[1]) + (s[2] + s[3]);
  __syncthreads();
  if (g == 0 && i < n) {
    double s = part[0][r];
#pragma unroll
    for (int q = 1; q < kGemvGroups; ++q) s += part[q][r];
    y[i] -= s;
  }
}

}  // namespace lb

namespace lb {

// ---------------------------------------------------------------------------
// Blocks above the shared-memory kernels' size (nb > 384, landau_lu.cuh):
// a plain right-looking LU with partial pivoting (LAPACK layout: unit L
// below the diagonal, U on and above it, 1-based ipiv, info = first zero
// pivot) worked in global memory by one CTA per matrix, and the matching
// substitution for blocks of right-hand sides.  O(n^3) L2 traffic per
// matrix: correct for any block size, meant for meshes whose banded order
// exceeds 384 rows (none of the BASELINE configurations does).
constexpr int kGmThreads = 1024;

__global__ void __launch_bounds__(kGmThreads) lb_getrf_gm_kernel(int n, double* const* __restrict__ As,
                                                                 int* __restrict__ ipiv_all,
                                                                 int* __restrict__ info_all, int pivot) {
  __shared__ double redv[32];
  __shared__ int redi[32];
  __shared__ int piv_sh;
  double* A = As[blockIdx.x];
  int* ipiv = ipiv_all + (size_t)blockIdx.x * n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int info = 0;
  for (int j = 0; j < n; ++j) {
    double* cj = A + (size_t)j * n;
    if (pivot) {  // idamax over rows j..n-1: the first largest |a|
      double best = -1.0;
      int bi = n;
      for (int i = j + tid; i < n; i += kGmThreads) {
        const double v = fabs(cj[i]);
        if (v > best) { best = v; bi = i; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
      }
      if (lane == 0) { redv[warp] = best; redi[warp] = bi; }
      __syncthreads();
      if (tid == 0) {
        for (int q = 1; q < kGmThreads / 32; ++q)
          if (redv[q] > best || (redv[q] == best && redi[q] < bi)) { best = redv[q]; bi = redi[q]; }
        piv_sh = bi < n ? bi : j;
      }
      __syncthreads();
      const int p = piv_sh;
      if (p != j)
        for (int k = tid; k < n; k += kGmThreads) {
          double* ck = A + (size_t)k * n;
          const double t = ck[j];
          ck[j] = ck[p];
          ck[p] = t;
        }
      if (tid == 0) ipiv[j] = p + 1;
      __syncthreads();
    } else if (tid == 0) {
      ipiv[j] = j + 1;
    }
    const double d = cj[j];
    if (d == 0.0 && info == 0) info = j + 1;
    const double r = d != 0.0 ? 1.0 / d : 0.0;
    for (int i = j + 1 + tid; i < n; i += kGmThreads) cj[i] *= r;
    __syncthreads();
    // A[j+1:, j+1:] -= A[j+1:, j] A[j, j+1:] (column-major: i runs fastest)
    const int m = n - j - 1;
    for (long long t = tid; t < (long long)m * m; t += kGmThreads) {
      const int i = j + 1 + (int)(t % m), k = j + 1 + (int)(t / m);
      double* ck = A + (size_t)k * n;
      ck[i] = fma(-cj[i], ck[j], ck[i]);
    }
    __syncthreads();
  }
  if (tid == 0) info_all[blockIdx.x] = info;
}

// X := A^-1 X for the factors of lb_getrf_gm_kernel, X (n x m, ld n,
// column-major) in place; one CTA per (matrix, 8-column chunk).
constexpr int kGmCols = 8;
__global__ void __launch_bounds__(256) lb_getrs_gm_kernel(int n, int m, double* const* __restrict__ As,
                                                          const int* __restrict__ ipiv_all,
                                                          double* const* __restrict__ Xs) {
  const double* A = As[blockIdx.x];
  const int* ipiv = ipiv_all + (size_t)blockIdx.x * n;
  double* X = Xs[blockIdx.x];
  const int c0 = blockIdx.y * kGmCols, nc = min(kGmCols, m - c0);
  const int tid = threadIdx.x;
  if (tid < nc) {  // row swaps in order (LAPACK laswp)
    double* x = X + (size_t)(c0 + tid) * n;
    for (int k = 0; k < n; ++k) {
      const int p = ipiv[k] - 1;
      if (p != k) {
        const double t = x[k];
        x[k] = x[p];
        x[p] = t;
      }
    }
  }
  __syncthreads();
  for (int k = 0; k < n; ++k) {  // unit lower L
    const double* lk = A + (size_t)k * n;
    for (int t = tid; t < (n - k - 1) * nc; t += blockDim.x) {
      const int i = k + 1 + t % (n - k - 1), c = t / (n - k - 1);
      double* x = X + (size_t)(c0 + c) * n;
      x[i] = fma(-lk[i], x[k], x[i]);
    }
    __syncthreads();
  }
  for (int k = n - 1; k >= 0; --k) {  // upper U
    const double* uk = A + (size_t)k * n;
    if (tid < nc) {
      double* x = X + (size_t)(c0 + tid) * n;
      x[k] = x[k] / uk[k];
    }
    __syncthreads();
    for (int t = tid; t < k * nc; t += blockDim.x) {
      const int i = t % k, c = t / k;
      double* x = X + (size_t)(c0 + c) * n;
      x[i] = fma(-uk[i], x[k], x[i]);
    }
    __syncthreads();
  }
}

}  // namespace lb
