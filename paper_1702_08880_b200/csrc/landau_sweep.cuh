// landau_sweep.cuh -- K0 record packing, K1 general pair sweep (any outer points)
// and K1b chunk-partial reduction + species coupling.
#pragma once
#include "landau_common.cuh"

namespace lb {

// ------------------------------------------------------------------ K0 pack
struct PackW {
  int collapsed;
  double kw[LB_MAX_SPECIES], dw[LB_MAX_SPECIES];
};

__global__ void lb_pack_kernel(int n, int S, int RS, const double* __restrict__ r,
                               const double* __restrict__ z, const double* __restrict__ w,
                               const double* __restrict__ f, const double* __restrict__ dfr,
                               const double* __restrict__ dfz, const PackW pw,
                               double* __restrict__ rec) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    const double rn = r[p], wn = w[p];
    double* o = rec + (size_t)p * RS;
    o[0] = rn;
    o[1] = z[p];
    o[2] = rn * rn;
    o[3] = rn > 0.0 ? 1.0 / rn : 0.0;
    if (pw.collapsed) {  // species-collapsed record (see Coupling)
      double gr = 0.0, gz = 0.0, fw = 0.0;
      for (int b = 0; b < S; ++b) {
        gr = fma(pw.kw[b], dfr[(size_t)b * n + p] * wn, gr);
        gz = fma(pw.kw[b], dfz[(size_t)b * n + p] * wn, gz);
        fw = fma(pw.dw[b], f[(size_t)b * n + p] * wn, fw);
      }
      o[4] = gr;
      o[5] = gz;
      o[6] = fw;
      for (int k = 7; k < RS; ++k) o[k] = 0.0;
    } else {
      for (int b = 0; b < S; ++b) {
        // same products as _accumulate_block (kernel.py:408-410)
        o[4 + 3 * b + 0] = dfr[(size_t)b * n + p] * wn;
        o[4 + 3 * b + 1] = dfz[(size_t)b * n + p] * wn;
        o[4 + 3 * b + 2] = f[(size_t)b * n + p] * wn;
      }
      for (int k = 4 + 3 * S; k < RS; ++k) o[k] = 0.0;
    }
  }
}

// ------------------------------------------------------------------ K1 sweep
struct SweepArgs {
  const double* ro;   // outer r (nout)
  const double* zo;   // outer z (nout)
  const double* rec;  // packed inner records (n x RS)
  double* partial;    // [nchunk][5S][nout_pad]
  int nout, nout_pad, n, jc, nchunk;
  long long gthr;     // mask threshold on bits(d^2)
};

constexpr int kStages = 4;     // shared-memory ring depth
constexpr int kLookahead = 2;  // tiles in flight ahead of the consumer
constexpr int kWarps = kTI / 32;

template <int S>
constexpr size_t sweep_smem_bytes() {
  return size_t(kStages) * TileCfg<S>::TJ * TileCfg<S>::RS * sizeof(double) +
         size_t(2 << LB_LOGT_BITS) * sizeof(double);
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Persistent CTAs walk work items (128 outer points x one inner chunk of jc
// points).  Inner records flow through a kStages ring: thread 0 issues the
// 1-D TMA bulk copy of tile k+kLookahead once every warp has released tile
// k+kLookahead-kStages (per-stage "empty" mbarriers, one arrival per warp),
// so warps drift independently instead of meeting at a CTA barrier per tile.
template <int S>
__global__ void __launch_bounds__(kTI, kMinBlocks) lb_sweep_kernel(const SweepArgs a) {
  constexpr int RS = TileCfg<S>::RS;
  constexpr int TJ = TileCfg<S>::TJ;
  extern __shared__ __align__(128) double lb_smem[];
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  double2* logt = reinterpret_cast<double2*>(lb_smem + kStages * TJ * RS);

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int nib = a.nout_pad / kTI;
  const long long nitems = (long long)nib * a.nchunk;

  for (int t = tid; t < (2 << LB_LOGT_BITS); t += kTI) lb_smem[kStages * TJ * RS + t] = c_logt[t];
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // producer cursor (thread 0 only): next (item, tile) to load, flat tile index
  long long p_item = blockIdx.x;
  int p_tile = 0;
  uint32_t p_k = 0;
  auto issue_next = [&]() {
    if (p_item >= nitems) return;
    const uint32_t s = p_k % kStages;
    if (p_k >= kStages) mbar_wait(&empty[s], ((p_k / kStages) - 1) & 1);
    const int c = (int)(p_item / nib);
    const int j0 = c * a.jc + p_tile * TJ;
    const int jend = min(a.n, (c + 1) * a.jc);
    const int cnt = min(TJ, jend - j0);
    const uint32_t bytes = (uint32_t)cnt * RS * sizeof(double);
    mbar_expect_tx(&full[s], bytes);
    bulk_g2s(lb_smem + s * (TJ * RS), a.rec + (size_t)j0 * RS, bytes, &full[s]);
    ++p_k;
    if (j0 + TJ >= jend) {
      p_tile = 0;
      p_item += gridDim.x;
    } else {
      ++p_tile;
    }
  };
  if (tid == 0)
    for (int q = 0; q < kLookahead; ++q) issue_next();

  uint32_t k = 0;  // consumer flat tile index (same sequence as the producer)
  for (long long item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int ib = (int)(item % nib);
    const int c = (int)(item / nib);
    const int i = ib * kTI + tid;
    const int il = min(i, a.nout - 1);
    const Outer o = make_outer(a.ro[il], a.zo[il]);
    double acc[S][5];
#pragma unroll
    for (int b = 0; b < S; ++b)
#pragma unroll
      for (int q = 0; q < 5; ++q) acc[b][q] = 0.0;

    const int jbeg = c * a.jc;
    const int jend = min(a.n, jbeg + a.jc);
    for (int j0 = jbeg; j0 < jend; j0 += TJ, ++k) {
      if (tid == 0) issue_next();
      const uint32_t s = k % kStages;
      mbar_wait(&full[s], (k / kStages) & 1);
      const double* tile = lb_smem + s * (TJ * RS);
      const int cnt = min(TJ, jend - j0);
#pragma unroll kUnroll
      for (int jj = 0; jj < cnt; ++jj) {
        const double* rp = tile + jj * RS;
        const double2 rz = *reinterpret_cast<const double2*>(rp);
        const double2 aux = *reinterpret_cast<const double2*>(rp + 2);
        const T5 t = pair_tensor(o, rz.x, rz.y, aux.x, aux.y, a.gthr, logt);
#pragma unroll
        for (int b = 0; b < S; ++b) {
          const double gr = rp[4 + 3 * b], gz = rp[5 + 3 * b], fw = rp[6 + 3 * b];
          // _accumulate_block (kernel.py:411-415)
          acc[b][0] = fma(t.xz, gz, fma(t.kr, gr, acc[b][0]));
          acc[b][1] = fma(t.zz, gz, fma(t.zr, gr, acc[b][1]));
          acc[b][2] = fma(fw, t.xx, acc[b][2]);
          acc[b][3] = fma(fw, t.xz, acc[b][3]);
          acc[b][4] = fma(fw, t.zz, acc[b][4]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);  // this warp is done with stage s
    }
    if (i < a.nout) {
      double* dst = a.partial + (size_t)c * (5 * S) * a.nout_pad + i;
#pragma unroll
      for (int b = 0; b < S; ++b)
#pragma unroll
        for (int q = 0; q < 5; ++q) dst[(size_t)(b * 5 + q) * a.nout_pad] = acc[b][q];
    }
  }
}

// ------------------------------------------------------------------ K1b combine
// Shared by both combine kernels: accumulators A[Se][5] -> K, D rows.
template <int Se>
__device__ __forceinline__ void write_kd(const double (&A)[Se][5], const Coupling& cp, size_t io,
                                         double* __restrict__ K, double* __restrict__ D) {
  const int S = cp.S;
  for (int a = 0; a < S; ++a) {
    double k0, k1, d0, d1, d2;
    if (cp.collapsed) {  // rank-one coupling: expand the single accumulator set
      k0 = __dmul_rn(cp.kout[a], A[0][0]);
      k1 = __dmul_rn(cp.kout[a], A[0][1]);
      d0 = __dmul_rn(cp.dout[a], A[0][2]);
      d1 = __dmul_rn(cp.dout[a], A[0][3]);
      d2 = __dmul_rn(cp.dout[a], A[0][4]);
    } else {  // _combine (kernel.py:419-440): strict order, no contraction
      k0 = 0.0, k1 = 0.0, d0 = 0.0, d1 = 0.0, d2 = 0.0;
#pragma unroll
      for (int b = 0; b < Se; ++b) {
        const double ck = cp.coK4[a * Se + b], cd = cp.coD4[a * Se + b];
        k0 = __dadd_rn(k0, __dmul_rn(ck, A[b][0]));
        k1 = __dadd_rn(k1, __dmul_rn(ck, A[b][1]));
        d0 = __dadd_rn(d0, __dmul_rn(cd, A[b][2]));
        d1 = __dadd_rn(d1, __dmul_rn(cd, A[b][3]));
        d2 = __dadd_rn(d2, __dmul_rn(cd, A[b][4]));
      }
    }
    double* Ko = K + (io * S + a) * 2;
    double* Do = D + (io * S + a) * 4;
    Ko[0] = k0;
    Ko[1] = k1;
    Do[0] = d0;
    Do[1] = d1;
    Do[2] = d1;
    Do[3] = d2;
  }
}

template <int Se>
__global__ void lb_combine_kernel(const double* __restrict__ partial, int nchunk, int nout,
                                  int nout_pad, const Coupling cp, const int* __restrict__ perm,
                                  double* __restrict__ K, double* __restrict__ D) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nout) return;
  const int io = perm ? perm[i] : i;  // output row of this (possibly reordered) outer point
  double A[Se][5];
#pragma unroll
  for (int b = 0; b < Se; ++b)
#pragma unroll
    for (int q = 0; q < 5; ++q) A[b][q] = 0.0;
  for (int c = 0; c < nchunk; ++c) {
    const double* src = partial + (size_t)c * (5 * Se) * nout_pad + i;
#pragma unroll
    for (int b = 0; b < Se; ++b)
#pragma unroll
      for (int q = 0; q < 5; ++q) A[b][q] = __dadd_rn(A[b][q], src[(size_t)(b * 5 + q) * nout_pad]);
  }
  write_kd<Se>(A, cp, (size_t)io, K, D);
}

}  // namespace lb
