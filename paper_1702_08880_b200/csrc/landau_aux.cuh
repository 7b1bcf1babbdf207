// landau_aux.cuh -- outer-point Morton ordering, K2 element contraction, K3 CSR
// gather, K4 state sampling, the per-pair entry and the FP64 peak probe.
#pragma once
#include "landau_common.cuh"

namespace lb {

// ------------------------------------------------------------------ outer ordering
// Outer points are visited in Morton (Z-curve) order of (r, z) so the 32
// outer points of a warp are spatial neighbours: the m < 0.01 series /
// closed-form branch of pair_tensor is then warp-coherent (random point
// clouds otherwise diverge on ~half the warps).  Each outer point's sum is
// computed identically wherever it lands, so the order changes no bit of
// the result; the combine kernel scatters rows back through `perm`.
// Bounding box of (r, z): grid-stride partial min/max per block (stage 1,
// gridDim.x blocks write part[4*block]), then one block folds the partials
// (stage 2, n = number of partials, stride 0 selects the partial layout).
__global__ void lb_bbox_kernel(int n, const double* __restrict__ r, const double* __restrict__ z,
                               int stride, double* __restrict__ box) {
  __shared__ double red[4][32];
  double v[4] = {1e308, -1e308, 1e308, -1e308};
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    if (stride > 0) {
      const double rp = r[(size_t)p * stride], zp = z[(size_t)p * stride];
      v[0] = fmin(v[0], rp);
      v[1] = fmax(v[1], rp);
      v[2] = fmin(v[2], zp);
      v[3] = fmax(v[3], zp);
    } else {  // fold stage-1 partials: r points at part[], z unused
      v[0] = fmin(v[0], r[4 * p + 0]);
      v[1] = fmax(v[1], r[4 * p + 1]);
      v[2] = fmin(v[2], r[4 * p + 2]);
      v[3] = fmax(v[3], r[4 * p + 3]);
    }
  }
  for (int o = 16; o; o >>= 1) {
    v[0] = fmin(v[0], __shfl_xor_sync(0xffffffffu, v[0], o));
    v[1] = fmax(v[1], __shfl_xor_sync(0xffffffffu, v[1], o));
    v[2] = fmin(v[2], __shfl_xor_sync(0xffffffffu, v[2], o));
    v[3] = fmax(v[3], __shfl_xor_sync(0xffffffffu, v[3], o));
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0)
    for (int q = 0; q < 4; ++q) red[q][w] = v[q];
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int ww = 1; ww < (int)(blockDim.x >> 5); ++ww) {
      v[0] = fmin(v[0], red[0][ww]);
      v[1] = fmax(v[1], red[1][ww]);
      v[2] = fmin(v[2], red[2][ww]);
      v[3] = fmax(v[3], red[3][ww]);
    }
    for (int q = 0; q < 4; ++q) box[4 * blockIdx.x + q] = v[q];
  }
}

__device__ __forceinline__ uint32_t spread16(uint32_t x) {
  x &= 0xFFFFu;
  x = (x | (x << 8)) & 0x00FF00FFu;
  x = (x | (x << 4)) & 0x0F0F0F0Fu;
  x = (x | (x << 2)) & 0x33333333u;
  x = (x | (x << 1)) & 0x55555555u;
  return x;
}

__global__ void lb_morton_kernel(int n, const double* __restrict__ r, const double* __restrict__ z,
                                 int stride, const double* __restrict__ box,
                                 uint32_t* __restrict__ key, int* __restrict__ idx) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const double rp = r[(size_t)p * stride], zp = z[(size_t)p * stride];
  const double sr = 65535.0 / fmax(box[1] - box[0], 1e-300);
  const double sz = 65535.0 / fmax(box[3] - box[2], 1e-300);
  const uint32_t qr = (uint32_t)fmin(fmax((rp - box[0]) * sr, 0.0), 65535.0);
  const uint32_t qz = (uint32_t)fmin(fmax((zp - box[2]) * sz, 0.0), 65535.0);
  key[p] = spread16(qr) | (spread16(qz) << 1);
  idx[p] = p;
}

__global__ void lb_gather_kernel(int n, const int* __restrict__ perm, const double* __restrict__ r,
                                 const double* __restrict__ z, double* __restrict__ rs,
                                 double* __restrict__ zs) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int q = perm[p];
  rs[p] = r[q];
  zs[p] = z[q];
}

// ------------------------------------------------------------------ K2 elements
// One thread per row i of two (cell e, species a) pairs of the element
// matrices: the nine entries of row i,
//   elem[a,e,i,j] = sum_q u[q] . (B[j,q], dB[j,q,0], dB[j,q,1]),
//   u[q] = (dB[i,q,:].G2[q], dB[i,q,:].G3[q][:,0], dB[i,q,:].G3[q][:,1]),
// with G2 = K Jinv w, G3 = Jinv D Jinv w (assembly.py:159-160, same factor
// grouping).  The 243 basis values (B, dB at the nine Gauss points) are a
// by-value kernel parameter: the row loop is fully unrolled with warp-uniform
// indices, so every one of the 243 DFMAs of a row takes its basis operand
// from the constant bank (uniform registers), not from a shared-memory load
// per FMA as the round-1 warp-per-cell form did (MIO-bound, 36 us at config
// 4).  A block takes 32 consecutive (e, a) pairs (tasks in (e, a, i) order:
// the cells' K/D/w are read contiguously); stage 1 forms G for its 288
// (e, a, q) in shared memory, stage 2 gives each of 144 threads row i of two
// pairs (c, c + 16), so each basis operand feeds two FMA chains (measured at
// config 4 under ncu's cache flush: 1 / 2 / 3 / 4 rows per thread 37 / 25 /
// 27 / 31 us -- fewer, fatter threads lose to latency: the kernel has ~2 waves
// of work).  Per (cell, species): 9 x 56 B in, 648 B out, 2772 FP64 ops; the
// (S, ncell, 81) result stays in L2 for K3.  Products and sums keep the
// round-1 kernel's order, so every entry is bitwise unchanged.
constexpr int kElemMaxS = 8;
#ifndef LB_ELEM_RPT
#define LB_ELEM_RPT 2  // rows per thread (pairs c and c + 16 of the block): the basis operands serve both
#endif
constexpr int kElemRpt = LB_ELEM_RPT;
constexpr int kElemPairs = 16 * kElemRpt;  // (cell, species) pairs per block
constexpr int kElemThreads = 144;          // row i of RPT pairs each
struct ElemBasis {
  double v[9][9][3];  // v[j][q] = (B[j,q], dB[j,q,0], dB[j,q,1])
};
__global__ void __launch_bounds__(kElemThreads) lb_elements_kernel(
    int ncell, int S, const double* __restrict__ sizes, const double* __restrict__ w,
    const double* __restrict__ K, const double* __restrict__ D, const ElemBasis V,
    const double* __restrict__ dBt, double* __restrict__ elem, int ncell_out, int c_out) {
  // cells e of this launch land at cell c_out + e of an (S, ncell_out, 81) buffer
  __shared__ double sG[kElemPairs][9][6];  // G2 r,z ; G3 rr, rz, zr, zz
  __shared__ double sdB[9][9][2];          // dB[i][q][:] (row-dependent, not uniform)
  __shared__ double sJ[kElemPairs + 1][2];  // 2 / sizes of the block's cells (fem.py:107-108)
  const int t = threadIdx.x;
  const int npair = ncell * S;  // host-checked < 2^31
  const int pr0 = blockIdx.x * kElemPairs, e_lo = pr0 / S;
  // stage 1 loads first (K, D, w of the thread's (pair, q) tasks in flight
  // while the block forms its cells' inverse sizes), then G
  double ld[kElemRpt][7];
#pragma unroll
  for (int r = 0; r < kElemRpt; ++r) {
    const int task = t + r * kElemThreads, c = task / 9, q = task % 9, pr = pr0 + c;
    if (pr < npair) {
      const int e = pr / S, a = pr - e * S;
      const size_t pnt = 9 * (size_t)e + q;
      const double* Kp = K + (pnt * S + a) * 2;  // (caller pointers: no alignment assumed)
      const double* Dp = D + (pnt * S + a) * 4;
      ld[r][0] = Kp[0];
      ld[r][1] = Kp[1];
      ld[r][2] = Dp[0];
      ld[r][3] = Dp[1];
      ld[r][4] = Dp[2];
      ld[r][5] = Dp[3];
      ld[r][6] = w[pnt];
    }
  }
  for (int k = t; k < 162; k += kElemThreads) (&sdB[0][0][0])[k] = dBt[k];
  for (int k = t; k < 2 * (kElemPairs + 1); k += kElemThreads) {
    const int e = e_lo + (k >> 1);
    if (e < ncell) sJ[k >> 1][k & 1] = 2.0 / sizes[2 * e + (k & 1)];
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kElemRpt; ++r) {
    const int task = t + r * kElemThreads, c = task / 9, q = task % 9, pr = pr0 + c;
    if (pr < npair) {
      const int e = pr / S;
      const double jr = sJ[e - e_lo][0], jz = sJ[e - e_lo][1], wp = ld[r][6];
      double* g = sG[c][q];
      g[0] = ld[r][0] * (jr * wp);
      g[1] = ld[r][1] * (jz * wp);
      g[2] = ld[r][2] * ((jr * jr) * wp);
      g[3] = ld[r][3] * ((jr * jz) * wp);
      g[4] = ld[r][4] * ((jz * jr) * wp);
      g[5] = ld[r][5] * ((jz * jz) * wp);
    }
  }
  __syncthreads();
  // stage 2: row i of pairs c0 + 16 r; u[q] formed per q (registers: the
  // RPT x 9 row sums and one q's u)
  const int c0 = t / 9, i = t % 9;
  constexpr int kStep = kElemPairs / kElemRpt;
  double s[kElemRpt][9];
#pragma unroll
  for (int r = 0; r < kElemRpt; ++r)
#pragma unroll
    for (int j = 0; j < 9; ++j) s[r][j] = 0.0;
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    const double2 b = *reinterpret_cast<const double2*>(sdB[i][q]);  // dB[i,q,:]
    double u[kElemRpt][3];
#pragma unroll
    for (int r = 0; r < kElemRpt; ++r) {
      const double* g = sG[c0 + r * kStep][q];
      u[r][0] = fma(b.y, g[1], b.x * g[0]);
      u[r][1] = fma(b.y, g[4], b.x * g[2]);
      u[r][2] = fma(b.y, g[5], b.x * g[3]);
    }
#pragma unroll
    for (int j = 0; j < 9; ++j)
#pragma unroll
      for (int r = 0; r < kElemRpt; ++r) {
        s[r][j] = fma(u[r][0], V.v[j][q][0], s[r][j]);
        s[r][j] = fma(u[r][1], V.v[j][q][1], s[r][j]);
        s[r][j] = fma(u[r][2], V.v[j][q][2], s[r][j]);
      }
  }
#pragma unroll
  for (int r = 0; r < kElemRpt; ++r) {
    const int pr = pr0 + c0 + r * kStep;
    if (pr < npair) {
      const int e = pr / S, a = pr - e * S;
      double* out = elem + ((size_t)a * ncell_out + c_out + e) * 81 + 9 * i;
#pragma unroll
      for (int j = 0; j < 9; ++j) out[j] = s[r][j];
    }
  }
}

// host: the by-value basis parameter from host copies of B (9 x 9, [j][q])
// and dB (9 x 9 x 2)
inline ElemBasis make_elem_basis(const double* hB, const double* hdB) {
  ElemBasis V;
  for (int t = 0; t < 81; ++t) {
    const int j = t / 9, q = t % 9;
    V.v[j][q][0] = hB[t];
    V.v[j][q][1] = hdB[2 * t];
    V.v[j][q][2] = hdB[2 * t + 1];
  }
  return V;
}

// ------------------------------------------------------------------ K3 CSR gather
// One thread per stored slot of C_free = P^T C P: the weighted sum of the
// element-matrix entries that land on it, in the map's fixed order
// (scatter.py builds the map once per mesh; assembly.py:115-129 is the
// reference's scipy COO->CSR + condensation).  HBM-bound gather.
// MAXS bounds S at compile time (2, 4 or 8: registers for the S running
// sums; fewer registers -> more resident warps -> more gathers in flight,
// which is what a latency-bound gather needs).
#ifndef LB_GATHER_MINB
#define LB_GATHER_MINB 8  // 32 registers, 8 blocks per SM (measured at config 4: 14.1 vs 17.7 us with 45 registers)
#endif
template <int MAXS>
__global__ void __launch_bounds__(256, LB_GATHER_MINB) lb_csr_gather_kernel(int nslots, int nent, int S,
                                                            const int* __restrict__ slot_ptr,
                                                            const int* __restrict__ gidx,
                                                            const double* __restrict__ gw,
                                                            const double* __restrict__ elem,
                                                            double* __restrict__ out) {
  const int slot = blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= nslots) return;
  const int k0 = slot_ptr[slot], k1 = slot_ptr[slot + 1];
  // contributions in groups of 4: the group's indices, weights and element
  // entries (all species) are loaded before the ordered adds (latency-bound
  // gather from L2; the order of the adds is the map's)
  double v[MAXS];
#pragma unroll
  for (int a = 0; a < MAXS; ++a) v[a] = 0.0;
  for (int kb = k0; kb < k1; kb += 4) {
    int ix[4];
    double ww[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool on = kb + u < k1;
      ix[u] = on ? gidx[kb + u] : 0;
      ww[u] = on ? gw[kb + u] : 0.0;
      LB_DCHECK(ix[u] >= 0 && ix[u] < nent);
    }
#pragma unroll
    for (int a = 0; a < MAXS; ++a) {
      if (a >= S) break;
      const double* ea = elem + (size_t)a * nent;
      double x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = kb + u < k1 ? ea[ix[u]] : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (kb + u < k1) v[a] = fma(ww[u], x[u], v[a]);
    }
  }
#pragma unroll
  for (int a = 0; a < MAXS; ++a)
    if (a < S) out[(size_t)a * nslots + slot] = v[a];
}

// host launcher of the gather (the S-bound instantiation)
inline void launch_csr_gather(int nslots, int nent, int S, const int* slot_ptr, const int* gidx,
                              const double* gw, const double* elem, double* out, cudaStream_t st) {
  const int blocks = (nslots + 255) / 256;
  if (S <= 2)
    lb_csr_gather_kernel<2><<<blocks, 256, 0, st>>>(nslots, nent, S, slot_ptr, gidx, gw, elem, out);
  else if (S <= 4)
    lb_csr_gather_kernel<4><<<blocks, 256, 0, st>>>(nslots, nent, S, slot_ptr, gidx, gw, elem, out);
  else
    lb_csr_gather_kernel<kElemMaxS><<<blocks, 256, 0, st>>>(nslots, nent, S, slot_ptr, gidx, gw, elem, out);
}

// ------------------------------------------------------------------ K4 sampling
// sample_state (fem.py:170-199) + element_geometry (fem.py:103-113) on the
// device: one thread per quadrature point (e, q) of cells [c0, c1).
// Coordinates / weights use the reference's exact operation order (no
// contraction), so r, z, w are bitwise those of the reference; nodal values
// go through the prolongation rows (hanging nodes: 3 weights).
__global__ void lb_sample_kernel(int c0, int c1, int S, int n_free, const double* __restrict__ origins,
                                 const double* __restrict__ sizes, const double* __restrict__ qgeo,
                                 const double* __restrict__ basis, const int* __restrict__ cell_nodes,
                                 const int* __restrict__ P_ptr, const int* __restrict__ P_idx,
                                 const double* __restrict__ P_w, const double* __restrict__ coeffs,
                                 double* __restrict__ r, double* __restrict__ z, double* __restrict__ w,
                                 double* __restrict__ f, double* __restrict__ dfr,
                                 double* __restrict__ dfz) {
  const int nloc = 9 * (c1 - c0);
  const int pl = blockIdx.x * blockDim.x + threadIdx.x;
  if (pl >= nloc) return;
  const int e = c0 + pl / 9, q = pl % 9;
  const double sr = sizes[2 * e], sz = sizes[2 * e + 1];
  // coords = origins + (qpts + 1) * 0.5 * sizes (fem.py:109-111)
  const double rq = __dadd_rn(origins[2 * e], __dmul_rn(__dmul_rn(__dadd_rn(qgeo[2 * q], 1.0), 0.5), sr));
  const double zq =
      __dadd_rn(origins[2 * e + 1], __dmul_rn(__dmul_rn(__dadd_rn(qgeo[2 * q + 1], 1.0), 0.5), sz));
  const double detJ = __ddiv_rn(__dmul_rn(sr, sz), 4.0);   // fem.py:105
  r[pl] = rq;
  z[pl] = zq;
  w[pl] = __dmul_rn(__dmul_rn(qgeo[18 + q], detJ), rq);   // fem.py:112
  const double jr = __ddiv_rn(2.0, sr), jz = __ddiv_rn(2.0, sz);  // fem.py:107-108
  for (int s = 0; s < S; ++s) {
    const double* cs = coeffs + (size_t)s * n_free;
    double fv = 0.0, gr = 0.0, gz = 0.0;
    for (int i = 0; i < 9; ++i) {
      const int node = cell_nodes[9 * e + i];
      double v = 0.0;  // (P @ coeffs^T)[node] (fem.py:182)
      for (int k = P_ptr[node]; k < P_ptr[node + 1]; ++k) v = __dadd_rn(v, __dmul_rn(P_w[k], cs[P_idx[k]]));
      // einsum("sei,iq->seq") / ("sei,iqd->seqd") (fem.py:185-186): numpy
      // sums the 9 products in i order, each rounded (no FMA), from zero --
      // the same here, so f and grad f are bitwise the reference's
      fv = __dadd_rn(fv, __dmul_rn(v, basis[9 * i + q]));
      gr = __dadd_rn(gr, __dmul_rn(v, basis[81 + 2 * (9 * i + q)]));
      gz = __dadd_rn(gz, __dmul_rn(v, basis[81 + 2 * (9 * i + q) + 1]));
    }
    f[(size_t)s * nloc + pl] = fv;
    dfr[(size_t)s * nloc + pl] = __dmul_rn(gr, jr);  // fem.py:188-189
    dfz[(size_t)s * nloc + pl] = __dmul_rn(gz, jz);
  }
}

// ------------------------------------------------------------------ per-pair
__global__ void lb_pairs_kernel(int npair, const double* __restrict__ r, const double* __restrict__ z,
                                const double* __restrict__ rb, const double* __restrict__ zb,
                                double* __restrict__ UK, double* __restrict__ UD) {
  __shared__ double2 logt[1 << LB_LOGT_BITS];
  for (int t = threadIdx.x; t < (1 << LB_LOGT_BITS); t += blockDim.x)
    logt[t] = make_double2(c_logt[2 * t], c_logt[2 * t + 1]);
  __syncthreads();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= npair) return;
  const Outer o = make_outer(r[p], z[p]);
  const double rn = rb[p];
  const T5 t = pair_tensor(o, rn, zb[p], 4.0 * (rn * rn), rn > 0.0 ? 1.0 / rn : 0.0, 1LL, logt);
  // restore the pulled-out factor 4 (exact) and lay out as kernel.py:227-234
  UD[4 * p + 0] = 4.0 * t.xx;
  UD[4 * p + 1] = 4.0 * t.xz;
  UD[4 * p + 2] = 4.0 * t.xz;
  UD[4 * p + 3] = 4.0 * t.zz;
  UK[4 * p + 0] = 4.0 * t.kr;
  UK[4 * p + 1] = 4.0 * t.xz;
  UK[4 * p + 2] = 4.0 * t.zr;
  UK[4 * p + 3] = 4.0 * t.zz;
}

// elliptic_KE (kernel.py:93-113): K(m), E(m) from x = 1 - m with the same
// table log and Horner chains as the pair kernels (pair_stage2)
__global__ void lb_elliptic_kernel(int n, const double* __restrict__ m, double* __restrict__ K,
                                   double* __restrict__ E) {
  __shared__ double2 logt[1 << LB_LOGT_BITS];
  for (int t = threadIdx.x; t < (1 << LB_LOGT_BITS); t += blockDim.x)
    logt[t] = make_double2(c_logt[2 * t], c_logt[2 * t + 1]);
  __syncthreads();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const double x = 1.0 - m[p];
  const double lx = log_table(x, logt);
  double pk = fma(c_pk[10], x, c_pk[9]), qk = c_qk[9];
  double pe = fma(c_pe[10], x, c_pe[9]), qe = c_qe[9];
#pragma unroll
  for (int k = 8; k >= 0; --k) {
    pk = fma(pk, x, c_pk[k]);
    qk = fma(qk, x, c_qk[k]);
    pe = fma(pe, x, c_pe[k]);
    if (k >= 1) qe = fma(qe, x, c_qe[k]);
  }
  qe = qe * x;
  K[p] = fma(-lx, qk, pk);
  E[p] = fma(-lx, qe, pe);
}

// ------------------------------------------------------------------ FP64 peak
constexpr int kDfmaChains = 8;
constexpr int kDfmaIters = 4096;
__global__ void __launch_bounds__(256) lb_dfma_kernel(double seed, double* sink) {
  double v[kDfmaChains];
#pragma unroll
  for (int c = 0; c < kDfmaChains; ++c) v[c] = seed + threadIdx.x * 1e-9 + c;
  const double m = 0.999999, add = 1e-7;
#pragma unroll 4
  for (int it = 0; it < kDfmaIters; ++it) {
#pragma unroll
    for (int c = 0; c < kDfmaChains; ++c) v[c] = fma(v[c], m, add);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kDfmaChains; ++c) s += v[c];
  if (s == 12345.6789) sink[threadIdx.x] = s;  // never true; keeps the chains live
}

}  // namespace lb
