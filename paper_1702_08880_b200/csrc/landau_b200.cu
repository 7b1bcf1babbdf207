// landau_b200.cu -- host side and the C ABI of include/landau_b200.h.
//
// Kernels (all sm_100a, all FP64) live in the headers:
//   landau_pair.cuh    per-pair arithmetic of the axisymmetric Landau tensor
//   landau_common.cuh  constants, record layout, species coupling, PTX helpers
//   landau_sweep.cuh   K0 record pack, K1 general pair sweep (any outer points,
//                      4-stage TMA ring, per-warp mbarrier release), K1b combine
//   landau_sym.cuh     K1s symmetric all-points sweep (unordered tile pairs,
//                      rotated j-side accumulators) and its fixed-order reduce
//   landau_aux.cuh     Morton ordering, K2 element contraction, K3 CSR gather,
//                      K4 state sampling, per-pair entry, FP64 peak probe
// This file owns the context (stream, events, grow-only device scratch), the
// device mesh handle, the launch logic and every extern "C" entry point.
//
// Determinism: every reduction runs in a fixed order that is a function of
// the problem size (and the Morton order of the points); no atomics.
#include <cub/device/device_radix_sort.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/landau_b200.h"
#include "landau_common.cuh"
#include "landau_sweep.cuh"
#include "landau_sym.cuh"
#include "landau_aux.cuh"

namespace lb {

// ------------------------------------------------------------------ host side
thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
#define LB_CUDA(call)                                                                     \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(e_ == cudaErrorMemoryAllocation ? LB_ENOMEM : LB_ECUDA,                 \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                    \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
};

}  // namespace lb

struct lb_ctx {
  int device = 0;
  int num_sms = 0;
  cudaStream_t stream = nullptr;
  int last_launches = 0;
  cudaEvent_t ev[4] = {};
  // grow-only scratch
  lb::DevBuf in, rec, partial, out, elem, outer, aux, order;
  // symmetric all-points sweep state (lb_sym_*): sorted records, order, partials
  lb::DevBuf symord, symrec, syminv, symi, symj, symtot, symctr;
  int sym_n = -1, sym_S = 0, sym_Se = 0, sym_nt = 0;
  // CUDA graph of the state-level operator's device work (lb_assemble_state):
  // captured on the second call with an unchanged key, replayed after
  cudaGraphExec_t state_graph = nullptr;
  struct StateKey {
    const lb_mesh* m = nullptr;
    uint64_t mesh_uid = 0;
    int S = 0;
    double eps = 0.0;
    uint64_t gen = 0;
    lb::Coupling cp;
  } state_key;
  bool state_key_valid = false;
  int state_sym[4] = {-1, 0, 0, 0};  // sym_n, sym_S, sym_Se, sym_nt the graph leaves behind
};

struct lb_mesh {
  int device = 0;
  int ncell = 0, nslots = 0, ncontrib = 0;
  double* sizes = nullptr;    // (ncell, 2)
  double* basis = nullptr;    // B (81) then dB (162)
  int* slot_ptr = nullptr;    // (nslots + 1)
  int* gidx = nullptr;        // (ncontrib)
  double* gw = nullptr;       // (ncontrib)
  // sampling geometry (lb_mesh_set_geometry)
  int n_nodes = 0, n_free = 0, nnzP = 0;
  double* origins = nullptr;  // (ncell, 2)
  double* qgeo = nullptr;     // qpts (9, 2) then qwts (9)
  int* cell_nodes = nullptr;  // (ncell, 9)
  int* P_ptr = nullptr;       // (n_nodes + 1)
  int* P_idx = nullptr;       // (nnzP)
  double* P_w = nullptr;      // (nnzP)
  uint64_t uid = 0;           // fresh per create / set_geometry (keys captured graphs)
};

namespace lb {

// Bumped whenever any scratch buffer is (re)allocated: captured CUDA graphs
// bake device addresses in, so a graph is only replayed if no buffer moved.
std::atomic<uint64_t> g_buf_gen{0};

int ensure(DevBuf& b, size_t bytes) {
  if (bytes <= b.cap) return LB_OK;
  ++g_buf_gen;
  if (b.p) {  // grow: earlier asynchronous work (any stream) may still read it
    cudaDeviceSynchronize();
    cudaFree(b.p);
  }
  b.p = nullptr;
  b.cap = 0;
  size_t want = std::max(bytes, size_t(1) << 20);
  cudaError_t e = cudaMalloc(&b.p, want);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(LB_ENOMEM, std::string("cudaMalloc(") + std::to_string(want) + "): " +
                               cudaGetErrorString(e));
  }
  b.cap = want;
  return LB_OK;
}

int use_ctx(lb_ctx* ctx) {
  if (!ctx) return fail(LB_EINVAL, "null lb_ctx");
  LB_CUDA(cudaSetDevice(ctx->device));
  return LB_OK;
}

int chunk_len(int n) {
  int per = (n + kMaxChunks - 1) / kMaxChunks;
  per = ((per + kChunkAlign - 1) / kChunkAlign) * kChunkAlign;
  return std::max(per, kChunkAlign);
}

long long mask_threshold(double eps_d) {
  const double eps2 = eps_d * eps_d;
  long long bits;
  std::memcpy(&bits, &eps2, sizeof(bits));
  return std::max(bits, 1LL);
}

int make_coupling(int S, const double* coK, const double* coD, Coupling& cp) {
  cp = Coupling();
  cp.S = S;
  cp.Se = S;
  for (int t = 0; t < S * S; ++t) {
    cp.coK4[t] = 4.0 * coK[t];
    cp.coD4[t] = 4.0 * coD[t];
  }
  if (S < 2) return LB_OK;
  // rank-one test (to ~4 ulp): coK_ab = k_a k_b, coD_ab = al_a be_b
  const double tol = 1e-15;
  double k[LB_MAX_SPECIES], al[LB_MAX_SPECIES], be[LB_MAX_SPECIES];
  if (!(coD[0] != 0.0)) return LB_OK;
  for (int a = 0; a < S; ++a) {
    if (!(coK[a * S + a] > 0.0)) return LB_OK;
    k[a] = std::sqrt(coK[a * S + a]);
    al[a] = coD[a * S + 0];
    be[a] = coD[0 * S + a] / coD[0];
  }
  for (int a = 0; a < S; ++a)
    for (int b = 0; b < S; ++b) {
      const double kk = k[a] * k[b], cK = coK[a * S + b];
      const double dd = al[a] * be[b], cD = coD[a * S + b];
      if (std::fabs(kk - cK) > tol * std::fabs(cK) || std::fabs(dd - cD) > tol * std::fabs(cD))
        return LB_OK;
    }
  cp.collapsed = 1;
  cp.Se = 1;
  for (int a = 0; a < S; ++a) {
    cp.kw[a] = k[a];
    cp.dw[a] = be[a];
    cp.kout[a] = 4.0 * k[a];
    cp.dout[a] = 4.0 * al[a];
  }
  return LB_OK;
}

int record_stride(const Coupling& cp) { return rec_stride(cp.Se); }

constexpr int kOrderMin = 4096;  // outer sets at least this large are Morton-ordered

// Morton order of n points (r, z at the given stride): perm (sorted ->
// original index) in `buf`; when rs/zs are requested the reordered
// coordinates too.  Returns pointers into `buf`.
int morton_order(DevBuf& buf, int nout, const double* ro, const double* zo, int stride,
                 cudaStream_t st, const int** perm, const double** rs, const double** zs) {
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  size_t temp = 0;
  LB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                          (int*)nullptr, (int*)nullptr, nout, 0, 32, st));
  const size_t bk = al(sizeof(uint32_t) * nout), bi = al(sizeof(int) * nout),
               bd = al(sizeof(double) * nout);
  constexpr int kBoxBlocks = 64;
  const size_t total = 2 * bk + 2 * bi + 2 * bd + al(4 * (kBoxBlocks + 1) * sizeof(double)) + al(temp);
  int rc = ensure(buf, total);
  if (rc) return rc;
  char* p = static_cast<char*>(buf.p);
  uint32_t* k0 = reinterpret_cast<uint32_t*>(p);
  uint32_t* k1 = reinterpret_cast<uint32_t*>(p + bk);
  int* i0 = reinterpret_cast<int*>(p + 2 * bk);
  int* i1 = reinterpret_cast<int*>(p + 2 * bk + bi);
  double* r1 = reinterpret_cast<double*>(p + 2 * bk + 2 * bi);
  double* z1 = reinterpret_cast<double*>(p + 2 * bk + 2 * bi + bd);
  double* box = reinterpret_cast<double*>(p + 2 * bk + 2 * bi + 2 * bd);
  double* part = box + 4;
  void* tmp = p + 2 * bk + 2 * bi + 2 * bd + al(4 * (kBoxBlocks + 1) * sizeof(double));
  lb_bbox_kernel<<<kBoxBlocks, 256, 0, st>>>(nout, ro, zo, stride, part);
  lb_bbox_kernel<<<1, 64, 0, st>>>(kBoxBlocks, part, nullptr, 0, box);
  lb_morton_kernel<<<(nout + 255) / 256, 256, 0, st>>>(nout, ro, zo, stride, box, k0, i0);
  LB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, temp, k0, k1, i0, i1, nout, 0, 32, st));
  if (rs) {
    lb_gather_kernel<<<(nout + 255) / 256, 256, 0, st>>>(nout, i1, ro, zo, r1, z1);
    *rs = r1;
    *zs = z1;
  }
  LB_CUDA(cudaGetLastError());
  *perm = i1;
  return LB_OK;
}

template <int S>
int launch_sweep(lb_ctx* ctx, int nout, const double* ro, const double* zo, int n,
                 const double* rec, const Coupling& cp, long long gthr, double* K, double* D,
                 cudaStream_t st) {
  const size_t smem = sweep_smem_bytes<S>();
  static bool attr_done[64] = {};
  if (!attr_done[ctx->device & 63]) {
    LB_CUDA(cudaFuncSetAttribute(lb_sweep_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    attr_done[ctx->device & 63] = true;
  }
  int per_sm = 0;
  LB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lb_sweep_kernel<S>, kTI, smem));
  per_sm = std::max(per_sm, 1);
  int launches = 0;
  const int* perm = nullptr;
  if (nout >= kOrderMin) {
    int rc = morton_order(ctx->order, nout, ro, zo, 1, st, &perm, &ro, &zo);
    if (rc) return rc;
    launches += 4;  // own kernels: bbox (2), morton, gather (+ CUB radix sort)
  }
  const int jc = chunk_len(n);
  const int nchunk = (n + jc - 1) / jc;
  // outer batches bounded by the partial-buffer budget
  const size_t per_outer = size_t(nchunk) * 5 * S * sizeof(double);
  int batch = (int)std::min<size_t>((size_t)nout, std::max<size_t>(kTI, partial_budget() / per_outer));
  batch = std::max(kTI, (batch / kTI) * kTI);
  for (int o0 = 0; o0 < nout; o0 += batch) {
    const int nb = std::min(batch, nout - o0);
    const int nout_pad = ((nb + kTI - 1) / kTI) * kTI;
    int rc = ensure(ctx->partial, size_t(nchunk) * 5 * S * nout_pad * sizeof(double));
    if (rc) return rc;
    SweepArgs a;
    a.ro = ro + o0;
    a.zo = zo + o0;
    a.rec = rec;
    a.partial = static_cast<double*>(ctx->partial.p);
    a.nout = nb;
    a.nout_pad = nout_pad;
    a.n = n;
    a.jc = jc;
    a.nchunk = nchunk;
    a.gthr = gthr;
    const long long nitems = (long long)(nout_pad / kTI) * nchunk;
    const int grid = (int)std::min<long long>(nitems, (long long)ctx->num_sms * per_sm);
    lb_sweep_kernel<S><<<grid, kTI, smem, st>>>(a);
    LB_CUDA(cudaGetLastError());
    lb_combine_kernel<S><<<(nb + 127) / 128, 128, 0, st>>>(
        a.partial, nchunk, nb, nout_pad, cp, perm ? perm + o0 : nullptr,
        perm ? K : K + (size_t)o0 * cp.S * 2, perm ? D : D + (size_t)o0 * cp.S * 4);
    LB_CUDA(cudaGetLastError());
    launches += 2;
  }
  ctx->last_launches = launches;
  return LB_OK;
}

int sweep_dispatch(lb_ctx* ctx, int nout, const double* ro, const double* zo, int n, int S,
                   const double* rec, const Coupling& cp, long long gthr, double* K, double* D,
                   cudaStream_t st) {
  switch (cp.Se) {  // template = accumulator species sets
    case 1: return launch_sweep<1>(ctx, nout, ro, zo, n, rec, cp, gthr, K, D, st);
    case 2: return launch_sweep<2>(ctx, nout, ro, zo, n, rec, cp, gthr, K, D, st);
    case 3: return launch_sweep<3>(ctx, nout, ro, zo, n, rec, cp, gthr, K, D, st);
    case 4: return launch_sweep<4>(ctx, nout, ro, zo, n, rec, cp, gthr, K, D, st);
    case 5: return launch_sweep<5>(ctx, nout, ro, zo, n, rec, cp, gthr, K, D, st);
    case 6: return launch_sweep<6>(ctx, nout, ro, zo, n, rec, cp, gthr, K, D, st);
    case 7: return launch_sweep<7>(ctx, nout, ro, zo, n, rec, cp, gthr, K, D, st);
    case 8: return launch_sweep<8>(ctx, nout, ro, zo, n, rec, cp, gthr, K, D, st);
    default: return fail(LB_EINVAL, "species count must be in [1, 8]");
  }
}

int check_species(int S) {
  if (S < 1 || S > LB_MAX_SPECIES)
    return fail(LB_EINVAL, "species count " + std::to_string(S) + " outside [1, " +
                               std::to_string(LB_MAX_SPECIES) + "]");
  return LB_OK;
}


// ------------------------------------------------------------------ symmetric path (host)

int sym_prepare(lb_ctx* ctx, int n, const Coupling& cp, const double* rec, cudaStream_t st) {
  const int RS = record_stride(cp);
  const int nt = (n + kSymTile - 1) / kSymTile;
  const int npad = nt * kSymTile;
  const int* perm = nullptr;
  int rc = morton_order(ctx->symord, n, rec, rec + 1, RS, st, &perm, nullptr, nullptr);
  if (rc) return rc;
  if ((rc = ensure(ctx->symrec, (size_t)npad * RS * sizeof(double)))) return rc;
  if ((rc = ensure(ctx->syminv, (size_t)n * sizeof(int)))) return rc;
  lb_sym_gather_kernel<<<(npad + 255) / 256, 256, 0, st>>>(n, npad, RS, perm, rec,
                                                          static_cast<double*>(ctx->symrec.p));
  lb_invert_perm_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, perm, static_cast<int*>(ctx->syminv.p));
  LB_CUDA(cudaGetLastError());
  ctx->sym_n = n;
  ctx->sym_S = cp.S;
  ctx->sym_Se = cp.Se;
  ctx->sym_nt = nt;
  ctx->last_launches = 5;  // own kernels: bbox (2), morton, records gather, invert (+ CUB sort)
  return LB_OK;
}

template <int S>
int sym_partial(lb_ctx* ctx, long long gthr, int rank, int world, double* tot, cudaStream_t st) {
  const int nt = ctx->sym_nt;
  const int npad = nt * kSymTile;
  const int R0 = (int)((long long)nt * rank / world), R1 = (int)((long long)nt * (rank + 1) / world);
  const int nseg = sym_nseg(nt), hmax = sym_hmax(nt);
  int launches = 0;
  if (R0 >= R1) {
    LB_CUDA(cudaMemsetAsync(tot, 0, sizeof(double) * 5 * S * npad, st));
    ctx->last_launches = 0;
    return LB_OK;
  }
  const size_t smem = sym_smem_bytes<S>();
  static bool attr_done[64] = {};
  if (!attr_done[ctx->device & 63]) {
    LB_CUDA(cudaFuncSetAttribute(lb_symsweep_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    attr_done[ctx->device & 63] = true;
  }
  int per_sm = 0;
  LB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lb_symsweep_kernel<S>, kSymTile, smem));
  per_sm = std::max(per_sm, 1);
  const size_t row_i = (size_t)nseg * 5 * S * kSymTile * sizeof(double);
  const size_t row_j = (size_t)std::max(hmax, 1) * 5 * S * kSymTile * sizeof(double);
  const int RB = (int)std::max<size_t>(1, std::min<size_t>(R1 - R0, partial_budget() / (row_i + row_j)));
  int rc;
  if ((rc = ensure(ctx->symi, row_i * RB))) return rc;
  if ((rc = ensure(ctx->symj, row_j * RB))) return rc;
  const int nbatch = (R1 - R0 + RB - 1) / RB;
  if ((rc = ensure(ctx->symctr, sizeof(int) * nbatch))) return rc;
  int* ctr = static_cast<int*>(ctx->symctr.p);
  LB_CUDA(cudaMemsetAsync(ctr, 0, sizeof(int) * nbatch, st));
  for (int b0 = R0; b0 < R1; b0 += RB) {
    const int b1 = std::min(R1, b0 + RB);
    SymArgs a;
    a.rec = static_cast<const double*>(ctx->symrec.p);
    a.iside = static_cast<double*>(ctx->symi.p);
    a.jside = static_cast<double*>(ctx->symj.p);
    a.next_item = ctr + (b0 - R0) / RB;
    a.nt = nt;
    a.row0 = b0;
    a.row1 = b1;
    a.nseg = nseg;
    a.hmax = hmax;
    a.gthr = gthr;
    const long long nitems = (long long)(b1 - b0) * nseg;
    const int grid = (int)std::min<long long>(nitems, (long long)ctx->num_sms * per_sm);
    lb_symsweep_kernel<S><<<grid, kSymTile, smem, st>>>(a);
    LB_CUDA(cudaGetLastError());
    lb_symreduce_kernel<S><<<(npad + 127) / 128, 128, 0, st>>>(a.iside, a.jside, nt, b0, b1, nseg,
                                                               hmax, b0 == R0 ? 1 : 0, tot);
    LB_CUDA(cudaGetLastError());
    launches += 2;
  }
  ctx->last_launches = launches;
  return LB_OK;
}

template <int S>
int sym_combine(lb_ctx* ctx, const double* tot, const Coupling& cp, int q0, int q1, double* K,
                double* D, cudaStream_t st) {
  if (q1 <= q0) return LB_OK;
  const int npad = ctx->sym_nt * kSymTile;
  lb_sym_combine_kernel<S><<<(q1 - q0 + 127) / 128, 128, 0, st>>>(
      tot, npad, static_cast<const int*>(ctx->syminv.p), q0, q1, cp, K, D);
  LB_CUDA(cudaGetLastError());
  ctx->last_launches = 1;
  return LB_OK;
}

int sym_partial_dispatch(lb_ctx* ctx, int S, long long gthr, int rank, int world, double* tot,
                         cudaStream_t st) {
  switch (S) {
    case 1: return sym_partial<1>(ctx, gthr, rank, world, tot, st);
    case 2: return sym_partial<2>(ctx, gthr, rank, world, tot, st);
#if LB_SYM_MAXS >= 3
    case 3: return sym_partial<3>(ctx, gthr, rank, world, tot, st);
#endif
    default: return fail(LB_EINVAL, "symmetric sweep supports S <= " + std::to_string(kSymMaxS));
  }
}

int sym_combine_dispatch(lb_ctx* ctx, int S, const double* tot, const Coupling& cp, int q0, int q1,
                         double* K, double* D, cudaStream_t st) {
  switch (S) {
    case 1: return sym_combine<1>(ctx, tot, cp, q0, q1, K, D, st);
    case 2: return sym_combine<2>(ctx, tot, cp, q0, q1, K, D, st);
#if LB_SYM_MAXS >= 3
    case 3: return sym_combine<3>(ctx, tot, cp, q0, q1, K, D, st);
#endif
    default: return fail(LB_EINVAL, "symmetric sweep supports S <= " + std::to_string(kSymMaxS));
  }
}

// All-points sweep (outer == inner == the n packed records) on one device:
// symmetric path when S <= kSymMaxS, else the general sweep.
int all_points_sweep(lb_ctx* ctx, int n, const double* rec, const double* r, const double* z,
                     const Coupling& cp, long long gthr, double* K, double* D, cudaStream_t st) {
  if (cp.Se > kSymMaxS || n < kSymTile)
    return sweep_dispatch(ctx, n, r, z, n, cp.S, rec, cp, gthr, K, D, st);
  int rc = sym_prepare(ctx, n, cp, rec, st);
  if (rc) return rc;
  const int npad = ctx->sym_nt * kSymTile;
  if ((rc = ensure(ctx->symtot, (size_t)5 * cp.Se * npad * sizeof(double)))) return rc;
  double* tot = static_cast<double*>(ctx->symtot.p);
  if ((rc = sym_partial_dispatch(ctx, cp.Se, gthr, 0, 1, tot, st))) return rc;
  const int l = ctx->last_launches;  // sweep + reduce launches
  rc = sym_combine_dispatch(ctx, cp.Se, tot, cp, 0, n, K, D, st);
  ctx->last_launches += l + 5;        // + combine (set above) + 5 ordering kernels
  return rc;
}

int launch_pack(lb_ctx* ctx, int n, int S, const double* r, const double* z, const double* w,
                const double* f, const double* dfr, const double* dfz, const Coupling& cp,
                double* rec, cudaStream_t st) {
  if (n == 0) return LB_OK;
  PackW pw;
  pw.collapsed = cp.collapsed;
  for (int b = 0; b < LB_MAX_SPECIES; ++b) {
    pw.kw[b] = cp.kw[b];
    pw.dw[b] = cp.dw[b];
  }
  const int threads = 256;
  const int blocks = std::min((n + threads - 1) / threads, ctx->num_sms * 8);
  lb_pack_kernel<<<blocks, threads, 0, st>>>(n, S, record_stride(cp), r, z, w, f, dfr, dfz, pw, rec);
  LB_CUDA(cudaGetLastError());
  return LB_OK;
}

int launch_elements(lb_ctx* ctx, int ncell, int S, const double* sizes, const double* w,
                    const double* K, const double* D, const double* B, const double* dB,
                    double* elem, cudaStream_t st, int ncell_out = -1, int c_out = 0) {
  if (ncell_out < 0) ncell_out = ncell;
  if (ncell == 0) return LB_OK;
  const long long nwork = (long long)ncell * S;
  const int blocks =
      (int)std::min<long long>((nwork + kElemWarps - 1) / kElemWarps, (long long)ctx->num_sms * 16);
  lb_elements_kernel<<<blocks, 32 * kElemWarps, 0, st>>>(ncell, S, sizes, w, K, D, B, dB, elem,
                                                         ncell_out, c_out);
  LB_CUDA(cudaGetLastError());
  return LB_OK;
}

}  // namespace lb

using namespace lb;

// ====================================================================== C ABI
extern "C" {

int lb_version(void) { return 100; }

const char* lb_last_error(void) { return g_err.c_str(); }

int lb_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int lb_ctx_create(int device, lb_ctx** out) {
  if (!out) return fail(LB_EINVAL, "null output pointer");
  *out = nullptr;
  int ndev = lb_device_count();
  if (ndev <= 0) return fail(LB_ENODEV, "no CUDA device visible (the B200 path has no CPU fallback)");
  if (device < 0 || device >= ndev)
    return fail(LB_EINVAL, "device " + std::to_string(device) + " not in [0, " +
                               std::to_string(ndev) + ")");
  LB_CUDA(cudaSetDevice(device));
  lb_ctx* c = new lb_ctx();
  c->device = device;
  cudaDeviceProp prop;
  cudaError_t e = cudaGetDeviceProperties(&prop, device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete c;
    return fail(LB_ECUDA, std::string("context setup: ") + cudaGetErrorString(e));
  }
  if (prop.major < 10) {
    cudaStreamDestroy(c->stream);
    delete c;
    return fail(LB_ENODEV, std::string("device ") + prop.name + " is sm_" +
                               std::to_string(prop.major * 10 + prop.minor) +
                               "; this library is built for sm_100a (B200) only");
  }
  c->num_sms = prop.multiProcessorCount;
  for (auto& ev : c->ev) cudaEventCreate(&ev);
  *out = c;
  return LB_OK;
}

int lb_ctx_destroy(lb_ctx* ctx) {
  if (!ctx) return LB_OK;
  cudaSetDevice(ctx->device);
  for (DevBuf* b : {&ctx->in, &ctx->rec, &ctx->partial, &ctx->out, &ctx->elem, &ctx->outer, &ctx->aux,
                    &ctx->order, &ctx->symord, &ctx->symrec, &ctx->syminv, &ctx->symi, &ctx->symj,
                    &ctx->symtot, &ctx->symctr})
    if (b->p) cudaFree(b->p);
  for (auto& ev : ctx->ev)
    if (ev) cudaEventDestroy(ev);
  if (ctx->state_graph) cudaGraphExecDestroy(ctx->state_graph);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return LB_OK;
}

int lb_record_stride(int S, const double* coK, const double* coD) {
  if (check_species(S)) return -1;
  if (!coK || !coD) return rec_stride(S);
  Coupling cp;
  make_coupling(S, coK, coD, cp);
  return record_stride(cp);
}

int lb_accumulator_sets(int S, const double* coK, const double* coD) {
  if (check_species(S)) return -1;
  if (!coK || !coD) return S;
  Coupling cp;
  make_coupling(S, coK, coD, cp);
  return cp.Se;
}

int lb_chunk_len(int n) { return chunk_len(std::max(n, 0)); }

int lb_last_launch_count(lb_ctx* ctx) { return ctx ? ctx->last_launches : 0; }

int lb_pack_records_dev(lb_ctx* ctx, int n, int S, const double* r, const double* z,
                        const double* w, const double* f, const double* df_r,
                        const double* df_z, const double* coK, const double* coD, double* rec,
                        void* stream) {
  int rc = use_ctx(ctx);
  if (rc) return rc;
  if ((rc = check_species(S))) return rc;
  if (n < 0) return fail(LB_EINVAL, "negative point count");
  if (!coK || !coD) return fail(LB_EINVAL, "null coupling table");
  Coupling cp;
  make_coupling(S, coK, coD, cp);
  cudaStream_t st = (cudaStream_t)stream;  // NULL = legacy default stream
  rc = launch_pack(ctx, n, S, r, z, w, f, df_r, df_z, cp, rec, st);
  ctx->last_launches = n > 0 ? 1 : 0;
  return rc;
}

int lb_sweep_dev(lb_ctx* ctx, int nout, const double* outer_r, const double* outer_z, int n,
                 int S, const double* rec, const double* coK, const double* coD, double eps_d,
                 double* K_out, double* D_out, void* stream) {
  int rc = use_ctx(ctx);
  if (rc) return rc;
  if ((rc = check_species(S))) return rc;
  if (nout < 0 || n < 0) return fail(LB_EINVAL, "negative point count");
  if (!coK || !coD) return fail(LB_EINVAL, "null coupling table");
  cudaStream_t st = (cudaStream_t)stream;  // NULL = legacy default stream
  ctx->last_launches = 0;
  if (nout == 0) return LB_OK;
  if (n == 0) {  // empty inner set: all sums are +0
    LB_CUDA(cudaMemsetAsync(K_out, 0, sizeof(double) * nout * S * 2, st));
    LB_CUDA(cudaMemsetAsync(D_out, 0, sizeof(double) * nout * S * 4, st));
    return LB_OK;
  }
  Coupling cp;
  make_coupling(S, coK, coD, cp);
  return sweep_dispatch(ctx, nout, outer_r, outer_z, n, S, rec, cp, mask_threshold(eps_d), K_out,
                        D_out, st);
}

int lb_elements_dev(lb_ctx* ctx, int ncell, int S, const double* cell_sizes, const double* w,
                    const double* K, const double* D, const double* B, const double* dB,
                    double* elem_out, void* stream) {
  int rc = use_ctx(ctx);
  if (rc) return rc;
  if ((rc = check_species(S))) return rc;
  if (ncell < 0) return fail(LB_EINVAL, "negative cell count");
  cudaStream_t st = (cudaStream_t)stream;  // NULL = legacy default stream
  rc = launch_elements(ctx, ncell, S, cell_sizes, w, K, D, B, dB, elem_out, st);
  ctx->last_launches = ncell > 0 ? 1 : 0;
  return rc;
}

int lb_fused_sweep(lb_ctx* ctx, int nout, const double* outer_r, const double* outer_z, int n,
                   int S, const double* r, const double* z, const double* w, const double* f,
                   const double* df_r, const double* df_z, const double* coK, const double* coD,
                   double eps_d, double* K_out, double* D_out) {
  int rc = use_ctx(ctx);
  if (rc) return rc;
  if ((rc = check_species(S))) return rc;
  if (nout < 0 || n < 0) return fail(LB_EINVAL, "negative point count");
  if (nout == 0) return LB_OK;
  if (!outer_r || !outer_z || !K_out || !D_out || !coK || !coD)
    return fail(LB_EINVAL, "null argument");
  if (n > 0 && (!r || !z || !w || !f || !df_r || !df_z)) return fail(LB_EINVAL, "null inner field");
  Coupling cp;
  make_coupling(S, coK, coD, cp);
  cudaStream_t st = ctx->stream;
  const size_t nin = (size_t)(3 + 3 * S) * n;
  if ((rc = ensure(ctx->in, std::max<size_t>(nin, 1) * sizeof(double)))) return rc;
  if ((rc = ensure(ctx->rec, std::max<size_t>((size_t)n * record_stride(cp), 1) * sizeof(double)))) return rc;
  if ((rc = ensure(ctx->outer, (size_t)2 * nout * sizeof(double)))) return rc;
  if ((rc = ensure(ctx->out, (size_t)6 * S * nout * sizeof(double)))) return rc;
  double* din = static_cast<double*>(ctx->in.p);
  double *dr = din, *dz = dr + n, *dw = dz + n, *df = dw + n, *dfr = df + (size_t)S * n,
         *dfz = dfr + (size_t)S * n;
  double* dro = static_cast<double*>(ctx->outer.p);
  double* dzo = dro + nout;
  double* dK = static_cast<double*>(ctx->out.p);
  double* dD = dK + (size_t)2 * S * nout;
  const size_t bn = sizeof(double) * n, bsn = sizeof(double) * S * n;
  if (n > 0) {
    LB_CUDA(cudaMemcpyAsync(dr, r, bn, cudaMemcpyHostToDevice, st));
    LB_CUDA(cudaMemcpyAsync(dz, z, bn, cudaMemcpyHostToDevice, st));
    LB_CUDA(cudaMemcpyAsync(dw, w, bn, cudaMemcpyHostToDevice, st));
    LB_CUDA(cudaMemcpyAsync(df, f, bsn, cudaMemcpyHostToDevice, st));
    LB_CUDA(cudaMemcpyAsync(dfr, df_r, bsn, cudaMemcpyHostToDevice, st));
    LB_CUDA(cudaMemcpyAsync(dfz, df_z, bsn, cudaMemcpyHostToDevice, st));
  }
  LB_CUDA(cudaMemcpyAsync(dro, outer_r, sizeof(double) * nout, cudaMemcpyHostToDevice, st));
  LB_CUDA(cudaMemcpyAsync(dzo, outer_z, sizeof(double) * nout, cudaMemcpyHostToDevice, st));
  double* drec = static_cast<double*>(ctx->rec.p);
  if ((rc = launch_pack(ctx, n, S, dr, dz, dw, df, dfr, dfz, cp, drec, st))) return rc;
  if ((rc = lb_sweep_dev(ctx, nout, dro, dzo, n, S, drec, coK, coD, eps_d, dK, dD, st))) return rc;
  LB_CUDA(cudaMemcpyAsync(K_out, dK, sizeof(double) * 2 * S * nout, cudaMemcpyDeviceToHost, st));
  LB_CUDA(cudaMemcpyAsync(D_out, dD, sizeof(double) * 4 * S * nout, cudaMemcpyDeviceToHost, st));
  LB_CUDA(cudaStreamSynchronize(st));
  return LB_OK;
}

int lb_assemble_elements(lb_ctx* ctx, int ncell, const double* cell_sizes, int S, const double* r,
                         const double* z, const double* w, const double* f, const double* df_r,
                         const double* df_z, const double* coK, const double* coD, double eps_d,
                         const double* B, const double* dB, double* K_out, double* D_out,
                         double* elem_out, double* phase_ms) {
  int rc = use_ctx(ctx);
  if (rc) return rc;
  if ((rc = check_species(S))) return rc;
  if (ncell < 0) return fail(LB_EINVAL, "negative cell count");
  if (ncell == 0) return LB_OK;
  if (!cell_sizes || !r || !z || !w || !f || !df_r || !df_z || !coK || !coD || !B || !dB ||
      !elem_out)
    return fail(LB_EINVAL, "null argument");
  Coupling cp;
  make_coupling(S, coK, coD, cp);
  const int n = 9 * ncell;
  cudaStream_t st = ctx->stream;
  const size_t nin = (size_t)(3 + 3 * S) * n;
  if ((rc = ensure(ctx->in, nin * sizeof(double)))) return rc;
  if ((rc = ensure(ctx->rec, (size_t)n * record_stride(cp) * sizeof(double)))) return rc;
  if ((rc = ensure(ctx->out, (size_t)6 * S * n * sizeof(double)))) return rc;
  if ((rc = ensure(ctx->elem, (size_t)81 * S * ncell * sizeof(double)))) return rc;
  if ((rc = ensure(ctx->aux, (size_t)(2 * ncell + 81 + 162) * sizeof(double)))) return rc;
  double* din = static_cast<double*>(ctx->in.p);
  double *dr = din, *dz = dr + n, *dw = dz + n, *df = dw + n, *dfr = df + (size_t)S * n,
         *dfz = dfr + (size_t)S * n;
  double* dK = static_cast<double*>(ctx->out.p);
  double* dD = dK + (size_t)2 * S * n;
  double* dsz = static_cast<double*>(ctx->aux.p);
  double* dB_ = dsz + 2 * ncell;
  double* ddB = dB_ + 81;
  double* delem = static_cast<double*>(ctx->elem.p);
  const size_t bn = sizeof(double) * n, bsn = sizeof(double) * S * n;
  LB_CUDA(cudaEventRecord(ctx->ev[0], st));
  LB_CUDA(cudaMemcpyAsync(dr, r, bn, cudaMemcpyHostToDevice, st));
  LB_CUDA(cudaMemcpyAsync(dz, z, bn, cudaMemcpyHostToDevice, st));
  LB_CUDA(cudaMemcpyAsync(dw, w, bn, cudaMemcpyHostToDevice, st));
  LB_CUDA(cudaMemcpyAsync(df, f, bsn, cudaMemcpyHostToDevice, st));
  LB_CUDA(cudaMemcpyAsync(dfr, df_r, bsn, cudaMemcpyHostToDevice, st));
  LB_CUDA(cudaMemcpyAsync(dfz, df_z, bsn, cudaMemcpyHostToDevice, st));
  LB_CUDA(cudaMemcpyAsync(dsz, cell_sizes, sizeof(double) * 2 * ncell, cudaMemcpyHostToDevice, st));
  LB_CUDA(cudaMemcpyAsync(dB_, B, sizeof(double) * 81, cudaMemcpyHostToDevice, st));
  LB_CUDA(cudaMemcpyAsync(ddB, dB, sizeof(double) * 162, cudaMemcpyHostToDevice, st));
  double* drec = static_cast<double*>(ctx->rec.p);
  if ((rc = launch_pack(ctx, n, S, dr, dz, dw, df, dfr, dfz, cp, drec, st))) return rc;
  LB_CUDA(cudaEventRecord(ctx->ev[1], st));
  if ((rc = all_points_sweep(ctx, n, drec, dr, dz, cp, mask_threshold(eps_d), dK, dD, st)))
    return rc;
  LB_CUDA(cudaEventRecord(ctx->ev[2], st));
  if ((rc = launch_elements(ctx, ncell, S, dsz, dw, dK, dD, dB_, ddB, delem, st))) return rc;
  if (K_out) LB_CUDA(cudaMemcpyAsync(K_out, dK, sizeof(double) * 2 * S * n, cudaMemcpyDeviceToHost, st));
  if (D_out) LB_CUDA(cudaMemcpyAsync(D_out, dD, sizeof(double) * 4 * S * n, cudaMemcpyDeviceToHost, st));
  LB_CUDA(cudaMemcpyAsync(elem_out, delem, sizeof(double) * 81 * S * ncell, cudaMemcpyDeviceToHost, st));
  LB_CUDA(cudaEventRecord(ctx->ev[3], st));
  LB_CUDA(cudaStreamSynchronize(st));
  if (phase_ms) {
    float t = 0.f;
    for (int p = 0; p < 3; ++p) {
      LB_CUDA(cudaEventElapsedTime(&t, ctx->ev[p], ctx->ev[p + 1]));
      phase_ms[p] = t;
    }
  }
  return LB_OK;
}

int lb_fused_sweep_all(lb_ctx* ctx, int n, int S, const double* r, const double* z, const double* w,
                       const double* f, const double* df_r, const double* df_z, const double* coK,
                       const double* coD, double eps_d, double* K_out, double* D_out) {
  int rc = use_ctx(ctx);
  if (rc) return rc;
  if ((rc = check_species(S))) return rc;
  if (n < 0) return fail(LB_EINVAL, "negative point count");
  if (n == 0) return LB_OK;
  if (!r || !z || !w || !f || !df_r || !df_z || !coK || !coD || !K_out || !D_out)
    return fail(LB_EINVAL, "null argument");
  Coupling cp;
  make_coupling(S, coK, coD, cp);
  cudaStream_t st = ctx->stream;
  const size_t nin = (size_t)(3 + 3 * S) * n;
  if ((rc = ensure(ctx->in, nin * sizeof(double)))) return rc;
  if ((rc = ensure(ctx->rec, (size_t)n * record_stride(cp) * sizeof(double)))) return rc;
  if ((rc = ensure(ctx->out, (size_t)6 * S * n * sizeof(double)))) return rc;
  double* din = static_cast<double*>(ctx->in.p);
  double *dr = din, *dz = dr + n, *dw = dz + n, *df = dw + n, *dfr = df + (size_t)S * n,
         *dfz = dfr + (size_t)S * n;
  double* dK = static_cast<double*>(ctx->out.p);
  double* dD = dK + (size_t)2 * S * n;
  const size_t bn = sizeof(double) * n, bsn = sizeof(double) * S * n;
  LB_CUDA(cudaMemcpyAsync(dr, r, bn, cudaMemcpyHostToDevice, st));
  LB_CUDA(cudaMemcpyAsync(dz, z, bn, cudaMemcpyHostToDevice, st));
  LB_CUDA(cudaMemcpyAsync(dw, w, bn, cudaMemcpyHostToDevice, st));
  LB_CUDA(cudaMemcpyAsync(df, f, bsn, cudaMemcpyHostToDevice, st));
  LB_CUDA(cudaMemcpyAsync(dfr, df_r, bsn, cudaMemcpyHostToDevice, st));
  LB_CUDA(cudaMemcpyAsync(dfz, df_z, bsn, cudaMemcpyHostToDevice, st));
  double* drec = static_cast<double*>(ctx->rec.p);
  if ((rc = launch_pack(ctx, n, S, dr, dz, dw, df, dfr, dfz, cp, drec, st))) return rc;
  if ((rc = all_points_sweep(ctx, n, drec, dr, dz, cp, mask_threshold(eps_d), dK, dD, st)))
    return rc;
  LB_CUDA(cudaMemcpyAsync(K_out, dK, sizeof(double) * 2 * S * n, cudaMemcpyDeviceToHost, st));
  LB_CUDA(cudaMemcpyAsync(D_out, dD, sizeof(double) * 4 * S * n, cudaMemcpyDeviceToHost, st));
  LB_CUDA(cudaStreamSynchronize(st));
  return LB_OK;
}

int lb_sym_supported(int S, const double* coK, const double* coD) {
  if (S < 1 || S > LB_MAX_SPECIES) return 0;
  if (!coK || !coD) return S <= kSymMaxS ? 1 : 0;
  Coupling cp;
  make_coupling(S, coK, coD, cp);
  return cp.Se <= kSymMaxS ? 1 : 0;
}

int lb_sym_npad(int n) { return ((std::max(n, 0) + kSymTile - 1) / kSymTile) * kSymTile; }

int lb_sym_prepare_dev(lb_ctx* ctx, int n, int S, const double* coK, const double* coD,
                       const double* rec, void* stream) {
  int rc = use_ctx(ctx);
  if (rc) return rc;
  if ((rc = check_species(S))) return rc;
  if (n < 1) return fail(LB_EINVAL, "symmetric sweep needs n >= 1");
  if (!coK || !coD) return fail(LB_EINVAL, "null coupling table");
  Coupling cp;
  make_coupling(S, coK, coD, cp);
  if (cp.Se > kSymMaxS)
    return fail(LB_EINVAL, "symmetric sweep supports at most " + std::to_string(kSymMaxS) +
                               " accumulator species sets");
  return sym_prepare(ctx, n, cp, rec, (cudaStream_t)stream);
}

int lb_sym_partial_dev(lb_ctx* ctx, int S, double eps_d, int rank, int world, double* tot,
                       void* stream) {
  int rc = use_ctx(ctx);
  if (rc) return rc;
  if (ctx->sym_n < 0 || ctx->sym_S != S) return fail(LB_EINVAL, "lb_sym_prepare_dev not called for this S");
  if (world < 1 || rank < 0 || rank >= world) return fail(LB_EINVAL, "bad rank / world");
  return sym_partial_dispatch(ctx, ctx->sym_Se, mask_threshold(eps_d), rank, world, tot,
                              (cudaStream_t)stream);
}

int lb_sym_combine_dev(lb_ctx* ctx, int S, const double* tot, const double* coK, const double* coD,
                       int q0, int q1, double* K_out, double* D_out, void* stream) {
  int rc = use_ctx(ctx);
  if (rc) return rc;
  if (ctx->sym_n < 0 || ctx->sym_S != S) return fail(LB_EINVAL, "lb_sym_prepare_dev not called for this S");
  if (q0 < 0 || q1 > ctx->sym_n || q0 > q1) return fail(LB_EINVAL, "bad point range");
  if (!coK || !coD) return fail(LB_EINVAL, "null coupling table");
  Coupling cp;
  make_coupling(S, coK, coD, cp);
  if (cp.Se != ctx->sym_Se) return fail(LB_EINVAL, "coupling differs from lb_sym_prepare_dev's");
  return sym_combine_dispatch(ctx, cp.Se, tot, cp, q0, q1, K_out, D_out, (cudaStream_t)stream);
}

int lb_mesh_create(lb_ctx* ctx, int ncell, const double* cell_sizes, const double* B,
                   const double* dB, int nslots, const int* slot_ptr, int ncontrib,
                   const int* gather_idx, const double* gather_w, lb_mesh** out) {
  int rc = use_ctx(ctx);
  if (rc) return rc;
  if (!out) return fail(LB_EINVAL, "null output pointer");
  *out = nullptr;
  if (ncell < 0 || nslots < 0 || ncontrib < 0) return fail(LB_EINVAL, "negative size");
  if (!cell_sizes || !B || !dB || !slot_ptr || (ncontrib && (!gather_idx || !gather_w)))
    return fail(LB_EINVAL, "null argument");
  lb_mesh* m = new lb_mesh();
  m->device = ctx->device;
  m->ncell = ncell;
  m->uid = ++g_buf_gen;
  m->nslots = nslots;
  m->ncontrib = ncontrib;
  cudaError_t e = cudaSuccess;
  auto alloc = [&](void** p, size_t b) {
    if (e == cudaSuccess) e = cudaMalloc(p, std::max<size_t>(b, 8));
  };
  alloc((void**)&m->sizes, sizeof(double) * 2 * ncell);
  alloc((void**)&m->basis, sizeof(double) * 243);
  alloc((void**)&m->slot_ptr, sizeof(int) * (nslots + 1));
  alloc((void**)&m->gidx, sizeof(int) * ncontrib);
  alloc((void**)&m->gw, sizeof(double) * ncontrib);
  if (e == cudaSuccess) e = cudaMemcpy(m->sizes, cell_sizes, sizeof(double) * 2 * ncell, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(m->basis, B, sizeof(double) * 81, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(m->basis + 81, dB, sizeof(double) * 162, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(m->slot_ptr, slot_ptr, sizeof(int) * (nslots + 1), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && ncontrib) e = cudaMemcpy(m->gidx, gather_idx, sizeof(int) * ncontrib, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && ncontrib) e = cudaMemcpy(m->gw, gather_w, sizeof(double) * ncontrib, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    lb_mesh_destroy(m);
    cudaGetLastError();
    return fail(e == cudaErrorMemoryAllocation ? LB_ENOMEM : LB_ECUDA,
                std::string("lb_mesh_create: ") + cudaGetErrorString(e));
  }
  *out = m;
  return LB_OK;
}

int lb_mesh_destroy(lb_mesh* m) {
  if (!m) return LB_OK;
  cudaSetDevice(m->device);
  for (void* p : {(void*)m->sizes, (void*)m->basis, (void*)m->slot_ptr, (void*)m->gidx, (void*)m->gw,
                  (void*)m->origins, (void*)m->qgeo, (void*)m->cell_nodes, (void*)m->P_ptr,
                  (void*)m->P_idx, (void*)m->P_w})
    if (p) cudaFree(p);
  delete m;
  return LB_OK;
}

int lb_assemble_csr(lb_ctx* ctx, const lb_mesh* mesh, int S, const double* r, const double* z,
                    const double* w, const double* f, const double* df_r, const double* df_z,
                    const double* coK, const double* coD, double eps_d, double* csr_out,
                    double* K_out, double* D_out, double* phase_ms) {
  int rc = use_ctx(ctx);
  if (rc) return rc;
  if ((rc = check_species(S))) return rc;
  if (!mesh || mesh->device != ctx->device) return fail(LB_EINVAL, "mesh handle missing or on another device");
  const int ncell = mesh->ncell, n = 9 * ncell;
  if (ncell == 0) return LB_OK;
  if (!r || !z || !w || !f || !df_r || !df_z || !coK || !coD || !csr_out)
    return fail(LB_EINVAL, "null argument");
  Coupling cp;
  make_coupling(S, coK, coD, cp);
  cudaStream_t st = ctx->stream;
  const size_t nin = (size_t)(3 + 3 * S) * n;
  if ((rc = ensure(ctx->in, nin * sizeof(double)))) return rc;
  if ((rc = ensure(ctx->rec, (size_t)n * record_stride(cp) * sizeof(double)))) return rc;
  if ((rc = ensure(ctx->out, (size_t)6 * S * n * sizeof(double)))) return rc;
  if ((rc = ensure(ctx->elem, ((size_t)81 * S * ncell + (size_t)S * mesh->nslots) * sizeof(double))))
    return rc;
  double* din = static_cast<double*>(ctx->in.p);
  double *dr = din, *dz = dr + n, *dw = dz + n, *df = dw + n, *dfr = df + (size_t)S * n,
         *dfz = dfr + (size_t)S * n;
  double* dK = static_cast<double*>(ctx->out.p);
  double* dD = dK + (size_t)2 * S * n;
  double* delem = static_cast<double*>(ctx->elem.p);
  double* dcsr = delem + (size_t)81 * S * ncell;
  const size_t bn = sizeof(double) * n, bsn = sizeof(double) * S * n;
  LB_CUDA(cudaEventRecord(ctx->ev[0], st));
  LB_CUDA(cudaMemcpyAsync(dr, r, bn, cudaMemcpyHostToDevice, st));
  LB_CUDA(cudaMemcpyAsync(dz, z, bn, cudaMemcpyHostToDevice, st));
  LB_CUDA(cudaMemcpyAsync(dw, w, bn, cudaMemcpyHostToDevice, st));
  LB_CUDA(cudaMemcpyAsync(df, f, bsn, cudaMemcpyHostToDevice, st));
  LB_CUDA(cudaMemcpyAsync(dfr, df_r, bsn, cudaMemcpyHostToDevice, st));
  LB_CUDA(cudaMemcpyAsync(dfz, df_z, bsn, cudaMemcpyHostToDevice, st));
  double* drec = static_cast<double*>(ctx->rec.p);
  if ((rc = launch_pack(ctx, n, S, dr, dz, dw, df, dfr, dfz, cp, drec, st))) return rc;
  LB_CUDA(cudaEventRecord(ctx->ev[1], st));
  if ((rc = all_points_sweep(ctx, n, drec, dr, dz, cp, mask_threshold(eps_d), dK, dD, st)))
    return rc;
  LB_CUDA(cudaEventRecord(ctx->ev[2], st));
  if ((rc = launch_elements(ctx, ncell, S, mesh->sizes, dw, dK, dD, mesh->basis, mesh->basis + 81,
                            delem, st)))
    return rc;
  if (mesh->nslots) {
    lb_csr_gather_kernel<<<(mesh->nslots + 255) / 256, 256, 0, st>>>(
        mesh->nslots, 81 * ncell, S, mesh->slot_ptr, mesh->gidx, mesh->gw, delem, dcsr);
    LB_CUDA(cudaGetLastError());
  }
  LB_CUDA(cudaMemcpyAsync(csr_out, dcsr, sizeof(double) * S * mesh->nslots, cudaMemcpyDeviceToHost, st));
  if (K_out) LB_CUDA(cudaMemcpyAsync(K_out, dK, sizeof(double) * 2 * S * n, cudaMemcpyDeviceToHost, st));
  if (D_out) LB_CUDA(cudaMemcpyAsync(D_out, dD, sizeof(double) * 4 * S * n, cudaMemcpyDeviceToHost, st));
  LB_CUDA(cudaEventRecord(ctx->ev[3], st));
  LB_CUDA(cudaStreamSynchronize(st));
  if (phase_ms) {
    float t = 0.f;
    for (int p = 0; p < 3; ++p) {
      LB_CUDA(cudaEventElapsedTime(&t, ctx->ev[p], ctx->ev[p + 1]));
      phase_ms[p] = t;
    }
  }
  return LB_OK;
}

int lb_mesh_set_geometry(lb_mesh* m, const double* origins, const double* qpts, const double* qwts,
                         const int* cell_nodes, int n_nodes, int n_free, const int* P_ptr,
                         const int* P_idx, const double* P_w) {
  if (!m) return fail(LB_EINVAL, "null mesh");
  if (!origins || !qpts || !qwts || !cell_nodes || !P_ptr || n_nodes < 0 || n_free < 0)
    return fail(LB_EINVAL, "bad geometry argument");
  LB_CUDA(cudaSetDevice(m->device));
  int nnzP = 0;
  std::memcpy(&nnzP, P_ptr + n_nodes, sizeof(int));
  if (nnzP < 0 || (nnzP && (!P_idx || !P_w))) return fail(LB_EINVAL, "bad prolongation");
  for (void* p : {(void*)m->origins, (void*)m->qgeo, (void*)m->cell_nodes, (void*)m->P_ptr,
                  (void*)m->P_idx, (void*)m->P_w})
    if (p) cudaFree(p);
  m->origins = m->qgeo = m->P_w = nullptr;
  m->cell_nodes = m->P_ptr = m->P_idx = nullptr;
  cudaError_t e = cudaSuccess;
  auto up = [&](void** dst, const void* src, size_t b) {
    if (e == cudaSuccess) e = cudaMalloc(dst, std::max<size_t>(b, 8));
    if (e == cudaSuccess && b) e = cudaMemcpy(*dst, src, b, cudaMemcpyHostToDevice);
  };
  up((void**)&m->origins, origins, sizeof(double) * 2 * m->ncell);
  if (e == cudaSuccess) e = cudaMalloc((void**)&m->qgeo, sizeof(double) * 27);
  if (e == cudaSuccess) e = cudaMemcpy(m->qgeo, qpts, sizeof(double) * 18, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(m->qgeo + 18, qwts, sizeof(double) * 9, cudaMemcpyHostToDevice);
  up((void**)&m->cell_nodes, cell_nodes, sizeof(int) * 9 * m->ncell);
  up((void**)&m->P_ptr, P_ptr, sizeof(int) * (n_nodes + 1));
  up((void**)&m->P_idx, P_idx, sizeof(int) * nnzP);
  up((void**)&m->P_w, P_w, sizeof(double) * nnzP);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(e == cudaErrorMemoryAllocation ? LB_ENOMEM : LB_ECUDA,
                std::string("lb_mesh_set_geometry: ") + cudaGetErrorString(e));
  }
  m->n_nodes = n_nodes;
  m->n_free = n_free;
  m->nnzP = nnzP;
  m->uid = ++g_buf_gen;
  return LB_OK;
}

int lb_sample_state_dev(lb_ctx* ctx, const lb_mesh* m, int S, int c0, int c1, const double* coeffs,
                        double* r, double* z, double* w, double* f, double* df_r, double* df_z,
                        void* stream) {
  int rc = use_ctx(ctx);
  if (rc) return rc;
  if ((rc = check_species(S))) return rc;
  if (!m || !m->cell_nodes) return fail(LB_EINVAL, "mesh has no sampling geometry (lb_mesh_set_geometry)");
  if (c0 < 0 || c1 > m->ncell || c0 > c1) return fail(LB_EINVAL, "bad cell range");
  const int nloc = 9 * (c1 - c0);
  ctx->last_launches = 0;
  if (nloc == 0) return LB_OK;
  lb_sample_kernel<<<(nloc + 127) / 128, 128, 0, (cudaStream_t)stream>>>(
      c0, c1, S, m->n_free, m->origins, m->sizes, m->qgeo, m->basis, m->cell_nodes, m->P_ptr,
      m->P_idx, m->P_w, coeffs, r, z, w, f, df_r, df_z);
  LB_CUDA(cudaGetLastError());
  ctx->last_launches = 1;
  return LB_OK;
}

// Field-wise (padding- and unused-entry-blind) equality of graph keys.
static bool same_state_key(const lb_ctx::StateKey& a, const lb_ctx::StateKey& b) {
  if (a.m != b.m || a.mesh_uid != b.mesh_uid || a.S != b.S || a.eps != b.eps || a.gen != b.gen)
    return false;
  const Coupling &x = a.cp, &y = b.cp;
  if (x.S != y.S || x.Se != y.Se || x.collapsed != y.collapsed) return false;
  for (int i = 0; i < x.S * x.S; ++i)
    if (x.coK4[i] != y.coK4[i] || x.coD4[i] != y.coD4[i]) return false;
  for (int i = 0; i < x.S; ++i)
    if (x.kw[i] != y.kw[i] || x.dw[i] != y.dw[i] || x.kout[i] != y.kout[i] || x.dout[i] != y.dout[i])
      return false;
  return true;
}

int lb_assemble_state(lb_ctx* ctx, const lb_mesh* m, int S, const double* coeffs, const double* coK,
                      const double* coD, double eps_d, double* csr_out, double* data_out,
                      double* phase_ms) {
  int rc = use_ctx(ctx);
  if (rc) return rc;
  if ((rc = check_species(S))) return rc;
  if (!m || !m->cell_nodes || m->device != ctx->device)
    return fail(LB_EINVAL, "mesh handle missing, on another device, or without geometry");
  if (!coeffs || !coK || !coD || !csr_out) return fail(LB_EINVAL, "null argument");
  const int ncell = m->ncell, n = 9 * ncell;
  if (ncell == 0) return LB_OK;
  Coupling cp;
  make_coupling(S, coK, coD, cp);
  cudaStream_t st = ctx->stream;
  const size_t nin = (size_t)(3 + 3 * S) * n + (size_t)S * m->n_free;
  if ((rc = ensure(ctx->in, nin * sizeof(double)))) return rc;
  if ((rc = ensure(ctx->rec, (size_t)n * record_stride(cp) * sizeof(double)))) return rc;
  if ((rc = ensure(ctx->out, (size_t)6 * S * n * sizeof(double)))) return rc;
  if ((rc = ensure(ctx->elem, ((size_t)81 * S * ncell + (size_t)S * m->nslots) * sizeof(double))))
    return rc;
  double* din = static_cast<double*>(ctx->in.p);
  double *dr = din, *dz = dr + n, *dw = dz + n, *df = dw + n, *dfr = df + (size_t)S * n,
         *dfz = dfr + (size_t)S * n, *dco = dfz + (size_t)S * n;
  double* dK = static_cast<double*>(ctx->out.p);
  double* dD = dK + (size_t)2 * S * n;
  double* delem = static_cast<double*>(ctx->elem.p);
  double* dcsr = delem + (size_t)81 * S * ncell;
  double* drec = static_cast<double*>(ctx->rec.p);
  const long long gthr = mask_threshold(eps_d);
  // device work: sample -> pack -> symmetric sweep -> elements -> CSR gather
  auto issue = [&]() -> int {
    lb_sample_kernel<<<(n + 127) / 128, 128, 0, st>>>(0, ncell, S, m->n_free, m->origins, m->sizes,
                                                      m->qgeo, m->basis, m->cell_nodes, m->P_ptr,
                                                      m->P_idx, m->P_w, dco, dr, dz, dw, df, dfr, dfz);
    LB_CUDA(cudaGetLastError());
    int r = launch_pack(ctx, n, S, dr, dz, dw, df, dfr, dfz, cp, drec, st);
    if (r) return r;
    if ((r = all_points_sweep(ctx, n, drec, dr, dz, cp, gthr, dK, dD, st))) return r;
    if ((r = launch_elements(ctx, ncell, S, m->sizes, dw, dK, dD, m->basis, m->basis + 81, delem, st)))
      return r;
    if (m->nslots) {
      lb_csr_gather_kernel<<<(m->nslots + 255) / 256, 256, 0, st>>>(m->nslots, 81 * ncell, S,
                                                                     m->slot_ptr, m->gidx, m->gw,
                                                                     delem, dcsr);
      LB_CUDA(cudaGetLastError());
    }
    return LB_OK;
  };
  LB_CUDA(cudaEventRecord(ctx->ev[0], st));
  LB_CUDA(cudaMemcpyAsync(dco, coeffs, sizeof(double) * S * m->n_free, cudaMemcpyHostToDevice, st));
  LB_CUDA(cudaEventRecord(ctx->ev[1], st));
  lb_ctx::StateKey key;
  key.m = m;
  key.mesh_uid = m->uid;
  key.S = S;
  key.eps = eps_d;
  key.gen = g_buf_gen;
  key.cp = cp;
  const bool same = ctx->state_key_valid && same_state_key(key, ctx->state_key);
  static const bool no_graph = std::getenv("LB_NO_GRAPH") != nullptr;
  if (same && ctx->state_graph && !no_graph) {
    LB_CUDA(cudaGraphLaunch(ctx->state_graph, st));  // replay (launch-bound small meshes)
    // the replay rewrote the symmetric-sweep scratch: keep the host view in step
    ctx->sym_n = ctx->state_sym[0];
    ctx->sym_S = ctx->state_sym[1];
    ctx->sym_Se = ctx->state_sym[2];
    ctx->sym_nt = ctx->state_sym[3];
  } else if (same && !no_graph) {
    // second call with an unchanged key: every buffer is sized, capture once
    cudaGraph_t graph = nullptr;
    LB_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    const int rc_issue = issue();
    const cudaError_t ce = cudaStreamEndCapture(st, &graph);
    cudaGraphExec_t exec = nullptr;
    if (rc_issue == LB_OK && ce == cudaSuccess && g_buf_gen == key.gen &&
        cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess) {
      ctx->state_graph = exec;
      ctx->state_sym[0] = ctx->sym_n;
      ctx->state_sym[1] = ctx->sym_S;
      ctx->state_sym[2] = ctx->sym_Se;
      ctx->state_sym[3] = ctx->sym_nt;
      LB_CUDA(cudaGraphLaunch(exec, st));
    } else {  // capture not possible: run eagerly
      cudaGetLastError();
      if ((rc = issue())) return rc;
    }
    if (graph) cudaGraphDestroy(graph);
  } else {
    if (ctx->state_graph) {
      cudaGraphExecDestroy(ctx->state_graph);
      ctx->state_graph = nullptr;
    }
    if ((rc = issue())) return rc;
    key.gen = g_buf_gen;  // buffers may have grown during this first call
    ctx->state_key = key;
    ctx->state_key_valid = true;
  }
  LB_CUDA(cudaEventRecord(ctx->ev[2], st));
  LB_CUDA(cudaMemcpyAsync(csr_out, dcsr, sizeof(double) * S * m->nslots, cudaMemcpyDeviceToHost, st));
  if (data_out)  // r, z, w, f, df_r, df_z as one (3 + 3S) x n block
    LB_CUDA(cudaMemcpyAsync(data_out, din, sizeof(double) * (3 + 3 * S) * n, cudaMemcpyDeviceToHost, st));
  LB_CUDA(cudaEventRecord(ctx->ev[3], st));
  LB_CUDA(cudaStreamSynchronize(st));
  if (phase_ms) {
    float t = 0.f;
    for (int p = 0; p < 3; ++p) {
      LB_CUDA(cudaEventElapsedTime(&t, ctx->ev[p], ctx->ev[p + 1]));
      phase_ms[p] = t;
    }
  }
  return LB_OK;
}

int lb_elements_csr(lb_ctx* ctx, const lb_mesh* m, int S, const double* w, const double* K,
                    const double* D, double* csr_out) {
  int rc = use_ctx(ctx);
  if (rc) return rc;
  if ((rc = check_species(S))) return rc;
  if (!m || m->device != ctx->device) return fail(LB_EINVAL, "mesh handle missing or on another device");
  if (!w || !K || !D || !csr_out) return fail(LB_EINVAL, "null argument");
  const int ncell = m->ncell, n = 9 * ncell;
  if (ncell == 0) return LB_OK;
  cudaStream_t st = ctx->stream;
  if ((rc = ensure(ctx->in, (size_t)(1 + 6 * S) * n * sizeof(double)))) return rc;
  if ((rc = ensure(ctx->elem, ((size_t)81 * S * ncell + (size_t)S * m->nslots) * sizeof(double))))
    return rc;
  double* dw = static_cast<double*>(ctx->in.p);
  double* dK = dw + n;
  double* dD = dK + (size_t)2 * S * n;
  double* delem = static_cast<double*>(ctx->elem.p);
  double* dcsr = delem + (size_t)81 * S * ncell;
  LB_CUDA(cudaMemcpyAsync(dw, w, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  LB_CUDA(cudaMemcpyAsync(dK, K, sizeof(double) * 2 * S * n, cudaMemcpyHostToDevice, st));
  LB_CUDA(cudaMemcpyAsync(dD, D, sizeof(double) * 4 * S * n, cudaMemcpyHostToDevice, st));
  if ((rc = launch_elements(ctx, ncell, S, m->sizes, dw, dK, dD, m->basis, m->basis + 81, delem, st)))
    return rc;
  if (m->nslots) {
    lb_csr_gather_kernel<<<(m->nslots + 255) / 256, 256, 0, st>>>(m->nslots, 81 * ncell, S, m->slot_ptr,
                                                                   m->gidx, m->gw, delem, dcsr);
    LB_CUDA(cudaGetLastError());
  }
  LB_CUDA(cudaMemcpyAsync(csr_out, dcsr, sizeof(double) * S * m->nslots, cudaMemcpyDeviceToHost, st));
  LB_CUDA(cudaStreamSynchronize(st));
  return LB_OK;
}

int lb_operator_partial_dev(lb_ctx* ctx, const lb_mesh* m, int S, int c0, int c1, const double* w,
                            const double* K, const double* D, double* csr_out, void* stream) {
  int rc = use_ctx(ctx);
  if (rc) return rc;
  if ((rc = check_species(S))) return rc;
  if (!m || m->device != ctx->device) return fail(LB_EINVAL, "mesh handle missing or on another device");
  if (c0 < 0 || c1 > m->ncell || c0 > c1) return fail(LB_EINVAL, "bad cell range");
  cudaStream_t st = (cudaStream_t)stream;
  const size_t nel = (size_t)81 * S * m->ncell;
  if ((rc = ensure(ctx->elem, std::max<size_t>(nel, 1) * sizeof(double)))) return rc;
  double* delem = static_cast<double*>(ctx->elem.p);
  LB_CUDA(cudaMemsetAsync(delem, 0, nel * sizeof(double), st));
  int launches = 0;
  if (c1 > c0) {
    if ((rc = launch_elements(ctx, c1 - c0, S, m->sizes + 2 * (size_t)c0, w, K, D, m->basis,
                              m->basis + 81, delem, st, m->ncell, c0)))
      return rc;
    ++launches;
  }
  if (m->nslots) {
    lb_csr_gather_kernel<<<(m->nslots + 255) / 256, 256, 0, st>>>(m->nslots, 81 * m->ncell, S,
                                                                   m->slot_ptr, m->gidx, m->gw, delem,
                                                                   csr_out);
    LB_CUDA(cudaGetLastError());
    ++launches;
  }
  ctx->last_launches = launches;
  return LB_OK;
}

int lb_tensor_pairs(lb_ctx* ctx, int npair, const double* r, const double* z, const double* rbar,
                    const double* zbar, double* UK, double* UD) {
  int rc = use_ctx(ctx);
  if (rc) return rc;
  if (npair < 0) return fail(LB_EINVAL, "negative pair count");
  if (npair == 0) return LB_OK;
  if (!r || !z || !rbar || !zbar || !UK || !UD) return fail(LB_EINVAL, "null argument");
  cudaStream_t st = ctx->stream;
  if ((rc = ensure(ctx->aux, sizeof(double) * 12 * (size_t)npair))) return rc;
  double* d = static_cast<double*>(ctx->aux.p);
  const size_t b = sizeof(double) * npair;
  LB_CUDA(cudaMemcpyAsync(d, r, b, cudaMemcpyHostToDevice, st));
  LB_CUDA(cudaMemcpyAsync(d + npair, z, b, cudaMemcpyHostToDevice, st));
  LB_CUDA(cudaMemcpyAsync(d + 2 * (size_t)npair, rbar, b, cudaMemcpyHostToDevice, st));
  LB_CUDA(cudaMemcpyAsync(d + 3 * (size_t)npair, zbar, b, cudaMemcpyHostToDevice, st));
  double* dUK = d + 4 * (size_t)npair;
  double* dUD = dUK + 4 * (size_t)npair;
  lb_pairs_kernel<<<(npair + 127) / 128, 128, 0, st>>>(npair, d, d + npair, d + 2 * (size_t)npair,
                                                       d + 3 * (size_t)npair, dUK, dUD);
  LB_CUDA(cudaGetLastError());
  LB_CUDA(cudaMemcpyAsync(UK, dUK, 4 * b, cudaMemcpyDeviceToHost, st));
  LB_CUDA(cudaMemcpyAsync(UD, dUD, 4 * b, cudaMemcpyDeviceToHost, st));
  LB_CUDA(cudaStreamSynchronize(st));
  return LB_OK;
}

int lb_fp64_peak(lb_ctx* ctx, double* tflops, double* ms) {
  int rc = use_ctx(ctx);
  if (rc) return rc;
  if (!tflops || !ms) return fail(LB_EINVAL, "null output");
  cudaStream_t st = ctx->stream;
  if ((rc = ensure(ctx->aux, 256 * sizeof(double)))) return rc;
  int per_sm = 0;
  LB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lb_dfma_kernel, 256, 0));
  const int blocks = ctx->num_sms * std::max(per_sm, 1) * 4;
  cudaEvent_t e0, e1;
  LB_CUDA(cudaEventCreate(&e0));
  LB_CUDA(cudaEventCreate(&e1));
  double best = 1e30;
  for (int rep = 0; rep < 6; ++rep) {  // first rep is warm-up
    LB_CUDA(cudaEventRecord(e0, st));
    lb_dfma_kernel<<<blocks, 256, 0, st>>>(1.0 + rep, static_cast<double*>(ctx->aux.p));
    LB_CUDA(cudaGetLastError());
    LB_CUDA(cudaEventRecord(e1, st));
    LB_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    LB_CUDA(cudaEventElapsedTime(&t, e0, e1));
    if (rep > 0) best = std::min(best, (double)t);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const double flops = 2.0 * kDfmaChains * (double)kDfmaIters * 256.0 * blocks;
  *ms = best;
  *tflops = flops / (best * 1e-3) / 1e12;
  return LB_OK;
}

}  // extern "C"
