// landau_cn.cuh -- device kernels of the Crank-Nicolson Newton step
// (reference solver.py:103-150): mass matrix, residual, the per-species
// block-banded system (M - dt/2 C_a) and its vector updates.
//
// The linear solve replaces SuperLU (solver.py:124-133) with block cyclic
// reduction of the banded matrix: the free nodes are permuted (natural or
// reverse Cuthill-McKee order, whichever has the smaller bandwidth b,
// chosen on the host once per mesh) and cut into blocks of nb >= b rows,
// so only the sub-, main- and super-diagonal nb x nb blocks are non-zero;
// the reduction levels run as batched dense block operations over rows and
// species (cuBLAS), blocks column-major in one pool (landau_b200.cu).
#pragma once
#include <cstdint>

namespace lb {

// r-weighted Q2 mass element matrices (fem.py:152-167):
// elem[c][i][j] = sum_q B[i][q] B[j][q] w[9c + q]
__global__ void lb_mass_elements_kernel(int ncell, const double* __restrict__ w,
                                        const double* __restrict__ B, double* __restrict__ elem) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 81 * ncell) return;
  const int c = t / 81, ij = t % 81, i = ij / 9, j = ij % 9;
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < 9; ++q) s = fma(B[i * 9 + q] * B[j * 9 + q], w[9 * c + q], s);
  elem[t] = s;
}

// sum_k vals[k] x[col_k] over one CSR row, in scipy's csr_matvec order (a
// sequential sum of unfused products over the row's entries).
__device__ __forceinline__ double csr_row_dot(const int* __restrict__ indptr,
                                              const int* __restrict__ indices,
                                              const double* __restrict__ vals,
                                              const double* __restrict__ x, int row) {
  double s = 0.0;
  for (int k = indptr[row]; k < indptr[row + 1]; ++k) s = __dadd_rn(s, __dmul_rn(vals[k], x[indices[k]]));
  return s;
}

// Crank-Nicolson residual (solver.py:87-100) and the norm terms:
//   R_a = M (g_a - f_a) - (dt/2) (Cg_a g_a + Co_a f_a)
//   Mf_a = M f_a (for the residual scale ||M f_old^T||)
// d = g - f is formed first, as numpy does before the product.
__global__ void lb_cn_residual_kernel(int n, int S, const int* __restrict__ indptr,
                                      const int* __restrict__ indices, long long nnz,
                                      const double* __restrict__ Mv, const double* __restrict__ Cg,
                                      const double* __restrict__ Co, const double* __restrict__ g,
                                      const double* __restrict__ f, const double* __restrict__ d,
                                      double h, double* __restrict__ R, double* __restrict__ Mf) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * S) return;
  const int a = t / n, row = t % n;
  const double* ga = g + (size_t)a * n;
  const double* fa = f + (size_t)a * n;
  const double mv = csr_row_dot(indptr, indices, Mv, d + (size_t)a * n, row);
  const double cg = csr_row_dot(indptr, indices, Cg + (size_t)a * nnz, ga, row);
  const double co = csr_row_dot(indptr, indices, Co + (size_t)a * nnz, fa, row);
  R[t] = __dsub_rn(mv, __dmul_rn(h, __dadd_rn(cg, co)));
  if (Mf) Mf[t] = csr_row_dot(indptr, indices, Mv, fa, row);
}

// Linear CN right-hand side (solver.py:146): rhs_a = (M + (dt/2) C_a) f_a,
// with the matrix sum formed entry-wise first, as scipy does.
__global__ void lb_cn_rhs_kernel(int n, int S, const int* __restrict__ indptr,
                                 const int* __restrict__ indices, long long nnz,
                                 const double* __restrict__ Mv, const double* __restrict__ C,
                                 const double* __restrict__ f, double h, double* __restrict__ rhs) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * S) return;
  const int a = t / n, row = t % n;
  const double* Ca = C + (size_t)a * nnz;
  const double* fa = f + (size_t)a * n;
  double s = 0.0;
  for (int k = indptr[row]; k < indptr[row + 1]; ++k)
    s = __dadd_rn(s, __dmul_rn(__dadd_rn(Mv[k], __dmul_rn(h, Ca[k])), fa[indices[k]]));
  rhs[t] = s;
}

// d = g - f (element-wise, as numpy forms f_new - f_old before the product)
__global__ void lb_axpby_kernel(int n, const double* __restrict__ g, const double* __restrict__ f,
                                double* __restrict__ d) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) d[t] = __dsub_rn(g[t], f[t]);
}

// Deterministic sum of squares of x[0..n) (one block, fixed order tree).
__global__ void lb_sumsq_kernel(long long n, const double* __restrict__ x, double* __restrict__ out) {
  __shared__ double red[1024];
  double s = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) s = fma(x[i], x[i], s);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

// Block-pool fill: the level-0 blocks hold A_a[k] = M[k] - h C_a[k],
// scattered through the slot -> pool offset map; the padded rows beyond n
// get an identity diagonal (in their D block).
__global__ void lb_band_identity_kernel(int S, long long sstride, int nb, int n, int npad,
                                        double* __restrict__ blk) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= S * (npad - n)) return;
  const int a = t / (npad - n), p = n + t % (npad - n);  // padded row p
  const int I = p / nb, l = p % nb;
  blk[a * sstride + (size_t)I * nb * nb + (size_t)l * nb + l] = 1.0;
}

__global__ void lb_band_fill_kernel(long long nnz, int S, long long sstride,
                                    const long long* __restrict__ off, const double* __restrict__ Mv,
                                    const double* __restrict__ C, double h, double* __restrict__ blk) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nnz * S) return;
  const int a = (int)(t / nnz);
  const long long k = t % nnz;
  const double c = C ? C[t] : 0.0;
  LB_DCHECK(off[k] >= 0 && off[k] < sstride);
  blk[a * sstride + off[k]] = __dsub_rn(Mv[k], __dmul_rn(h, c));
}

// Permute a species-major vector into / out of the padded block order:
// dst[a][p] = sign * src[a][perm[p]] for p < n, 0 beyond (gather), and the
// inverse scatter back.
__global__ void lb_perm_gather_kernel(int n, int npad, int S, const int* __restrict__ perm,
                                      const double* __restrict__ src, double sign,
                                      double* __restrict__ dst) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= S * npad) return;
  const int a = t / npad, p = t % npad;
  dst[t] = p < n ? sign * src[(size_t)a * n + perm[p]] : 0.0;
}

// out[a][perm[p]] = base[a][perm[p]] + x[a][p]  (f_next = guess + delta)
__global__ void lb_perm_update_kernel(int n, int npad, int S, const int* __restrict__ perm,
                                      const double* __restrict__ base, const double* __restrict__ x,
                                      double* __restrict__ out, double* __restrict__ dx_out,
                                      int* __restrict__ nonfinite) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= S * n) return;
  const int a = t / n, p = t % n;
  const double dx = x[(size_t)a * npad + p];
  if (!isfinite(dx)) atomicOr(nonfinite, 1);
  const size_t o = (size_t)a * n + perm[p];
  out[o] = base ? __dadd_rn(base[o], dx) : dx;
  if (dx_out) dx_out[o] = dx;
}

// Backward-error check of a solve of (M - h C_a) x_a = b_a (original order):
// e = (M - h C) x - b, written for a deterministic sum of squares.  With the
// unpivoted block LU the solver accepts the result only when ||e|| is at the
// level a pivoted factorisation reaches, else it refactorises with pivoting.
__global__ void lb_cn_check_kernel(int n, int S, const int* __restrict__ indptr,
                                   const int* __restrict__ indices, long long nnz,
                                   const double* __restrict__ Mv, const double* __restrict__ C, double h,
                                   const double* __restrict__ x, const double* __restrict__ b, double bsign,
                                   double* __restrict__ e) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * S) return;
  const int a = t / n, row = t % n;
  const double* Ca = C + (size_t)a * nnz;
  const double* xa = x + (size_t)a * n;
  double s = 0.0;
  for (int k = indptr[row]; k < indptr[row + 1]; ++k) s = fma(Mv[k] - h * Ca[k], xa[indices[k]], s);
  e[t] = s - bsign * b[t];
}

}  // namespace lb

namespace lb {

// ---------------------------------------------------------------- small-block solve
// Vector solves with small factor blocks (at most kSmallNb rows), where
// cuBLAS's batched getrs (1 right-hand side) spends ~0.1 ms per call in
// latency-bound kernels.  (A one-CTA shared-memory LU of the blocks was also
// written and measured slower than cuBLAS getrf: 228 vs ~160 us per level at
// 68 rows -- a latency-bound chain of 68 pivot steps on one SM.)
constexpr int kSmallNb = 96;
constexpr int kSmallThreads = 128;

// x := D^-1 x for one vector per matrix with getrf's factors (LAPACK
// layout, 1-based pivots): one CTA per vector, factors staged in shared memory,
// right-looking substitution parallel over rows.
__global__ void __launch_bounds__(kSmallThreads) lb_small_solve_kernel(int nb, int count,
                                                                       double* const* __restrict__ D,
                                                                       const int* __restrict__ piv_all,
                                                                       double* const* __restrict__ V) {
  extern __shared__ __align__(16) double sm[];
  double* A = sm;                  // [nb][nb]
  double* x = sm + (size_t)nb * nb;  // [nb]
  const int w = blockIdx.x, tid = threadIdx.x;
  if (w >= count) return;
  const double* Ag = D[w];
  const int* piv = piv_all ? piv_all + (size_t)w * nb : nullptr;
  double* xg = V[w];
  for (int t = tid; t < nb * nb; t += kSmallThreads) A[t] = Ag[t];
  for (int t = tid; t < nb; t += kSmallThreads) x[t] = xg[t];
  __syncthreads();
  if (tid == 0 && piv_all)  // no pivots: factors of the unpivoted LU
    for (int k = 0; k < nb; ++k) {
      const int p = piv[k] - 1;
      if (p != k) {
        const double t0 = x[k];
        x[k] = x[p];
        x[p] = t0;
      }
    }
  __syncthreads();
  for (int k = 0; k < nb - 1; ++k) {
    const double xk = x[k];
    const int i = k + 1 + tid;
    if (i < nb) x[i] = fma(-A[(size_t)k * nb + i], xk, x[i]);
    __syncthreads();
  }
  for (int k = nb - 1; k >= 0; --k) {
    const double xk = x[k] / A[(size_t)k * nb + k];
    __syncthreads();
    if (tid == 0) x[k] = xk;
    if (tid < k) x[tid] = fma(-A[(size_t)k * nb + tid], xk, x[tid]);
    __syncthreads();
  }
  for (int t = tid; t < nb; t += kSmallThreads) xg[t] = x[t];
}

inline size_t small_solve_smem_bytes(int nb) { return sizeof(double) * ((size_t)nb * nb + nb); }

}  // namespace lb
