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
    o[2] = 4.0 * (rn * rn);  // scaled (landau_pair.cuh): exactly 4 (rn rn)
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
    // one accumulator set (collapsed, or S = 1): slot 7 is free and carries
    // 2 rn for the species-collapsed symmetric sweep's tensor forms
    if ((pw.collapsed || S == 1) && RS > 7) o[7] = rn + rn;
  }
}

// ------------------------------------------------------------------ K1 sweep
struct SweepArgs {
  const double* ro;   // outer r (nout)
  const double* zo;   // outer z (nout)
  const double* rec;  // packed inner records (n x RS)
  double* partial;    // [nchunk][5S][nout_pad]
  int* next_item;     // work counter (zero at launch): items past the first wave
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
  const int nitems = nib * a.nchunk;

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

  // Producer (thread 0): walks the tiles of its items; items after the first
  // wave are claimed from a device counter (CTAs the schedulers favour take
  // more, every SM keeps its CTAs to the end; each item writes its own
  // partial slot, so results do not depend on the assignment).  Each stage
  // carries (item, first inner point, count); item -1 ends the sweep.
  __shared__ int stage_item[kStages], stage_j0[kStages], stage_cnt[kStages];
  int p_item = blockIdx.x, p_tile = 0;
  uint32_t p_k = 0;
  bool p_done = false;
  auto issue_next = [&]() {
    if (p_done) return;
    const uint32_t s = p_k % kStages;
    if (p_k >= kStages) mbar_wait(&empty[s], ((p_k / kStages) - 1) & 1);
    ++p_k;
    if (p_item >= nitems) {
      stage_item[s] = -1;
      mbar_arrive(&full[s]);
      p_done = true;
      return;
    }
    const int c = p_item / nib;
    const int j0 = c * a.jc + p_tile * TJ;
    const int jend = min(a.n, (c + 1) * a.jc);
    const int cnt = min(TJ, jend - j0);
    stage_item[s] = p_item;
    stage_j0[s] = j0;
    stage_cnt[s] = cnt;
    LB_DCHECK(j0 >= 0 && cnt >= 1 && cnt <= TJ && j0 + cnt <= a.n);
    const uint32_t bytes = (uint32_t)cnt * RS * sizeof(double);
    mbar_expect_tx(&full[s], bytes);
    bulk_g2s(lb_smem + s * (TJ * RS), a.rec + (size_t)j0 * RS, bytes, &full[s]);
    if (j0 + TJ >= jend) {
      p_tile = 0;
      p_item = (int)gridDim.x + atomicAdd(a.next_item, 1);
    } else {
      ++p_tile;
    }
  };
  if (tid == 0)
    for (int q = 0; q < kLookahead; ++q) issue_next();

  // partners per step: two for few accumulator sets (shared coefficient
  // loads, two overlapping chains), one where registers are short
  constexpr int GU = S <= 2 ? 2 : 1;
  Outer o;
  double acc[S][5];
  int cur = -1;
  auto flush = [&]() {
    const int i = (cur % nib) * kTI + tid;
    if (i < a.nout) {
      double* dst = a.partial + (size_t)(cur / nib) * (5 * S) * a.nout_pad + i;
#pragma unroll
      for (int b = 0; b < S; ++b)
#pragma unroll
        for (int q = 0; q < 5; ++q) dst[(size_t)(b * 5 + q) * a.nout_pad] = acc[b][q];
    }
  };
  auto accumulate = [&](const T5& t, const double* rp) {
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
  };
  for (uint32_t k = 0;; ++k) {
    if (tid == 0) issue_next();
    const uint32_t s = k % kStages;
    mbar_wait(&full[s], (k / kStages) & 1);
    const int item = stage_item[s];
    if (item < 0) break;
    if (item != cur) {
      if (cur >= 0) flush();
      cur = item;
      const int il = min((item % nib) * kTI + tid, a.nout - 1);
      o = make_outer(a.ro[il], a.zo[il]);
#pragma unroll
      for (int b = 0; b < S; ++b)
#pragma unroll
        for (int q = 0; q < 5; ++q) acc[b][q] = 0.0;
    }
    const double* tile = lb_smem + s * (TJ * RS);
    const int cnt = stage_cnt[s];
    int jj = 0;
    if constexpr (GU == 2) {
      const Outer oo[2] = {o, o};
#pragma unroll 1
      for (; jj + 1 < cnt; jj += 2) {
        const double* rp0 = tile + jj * RS;
        const double* rp1 = rp0 + RS;
        const double2 rz0 = *reinterpret_cast<const double2*>(rp0);
        const double2 rz1 = *reinterpret_cast<const double2*>(rp1);
        const double2 ax0 = *reinterpret_cast<const double2*>(rp0 + 2);
        const double2 ax1 = *reinterpret_cast<const double2*>(rp1 + 2);
        const double rn[2] = {rz0.x, rz1.x}, zn[2] = {rz0.y, rz1.y};
        const double rn2[2] = {ax0.x, ax1.x}, rcpr[2] = {ax0.y, ax1.y};
        const double rnx[2] = {rz0.x + rz0.x, rz1.x + rz1.x};
        T5 t[2];
        double txx2[2];  // (unused: the general path has no swapped pair)
        unsigned nser_unused = 0;
        pair_tensor_sym_x<2>(oo, rn, zn, rn2, rnx, rcpr, a.gthr, logt, t, txx2, nser_unused);
        accumulate(t[0], rp0);
        accumulate(t[1], rp1);
      }
    }
#pragma unroll 1
    for (; jj < cnt; ++jj) {
      const double* rp = tile + jj * RS;
      const double2 rz = *reinterpret_cast<const double2*>(rp);
      const double2 aux = *reinterpret_cast<const double2*>(rp + 2);
      accumulate(pair_tensor(o, rz.x, rz.y, aux.x, aux.y, a.gthr, logt), rp);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // this warp is done with stage s
  }
  if (cur >= 0) flush();
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
