// Does the FP64 tensor-core path (mma.sync m8n8k4 f64, SASS DMMA) run on a
// pipe separate from DFMA on sm_100a (B200)?  Three kernels over the same
// grid: DFMA-only warps, DMMA-only warps, and CTAs whose warps are split
// half/half.  If the mixed kernel's combined FLOP rate exceeds the larger
// of the two pure rates, DMMA adds FP64 throughput next to the CUDA cores.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// per warp: `iters` x 8 x ILP DFMA (thread) or `iters` x 8 x ILP DMMA (warp,
// 8*8*4 = 256 FMA each)
template <int ILP>
__device__ void do_dfma(double* out, int iters) {
  double v[ILP];
#pragma unroll
  for (int c = 0; c < ILP; ++c) v[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int c = 0; c < ILP; ++c) v[c] = fma(v[c], 0.999999, 1e-7);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < ILP; ++c) s += v[c];
  if (s == 1234.5) out[0] = s;
}

template <int ILP>
__device__ void do_dmma(double* out, int iters) {
  double d[ILP][2];
#pragma unroll
  for (int c = 0; c < ILP; ++c) d[c][0] = d[c][1] = threadIdx.x * 1e-9 + c;
  const double a = 0.999999 + threadIdx.x * 1e-12, b = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int c = 0; c < ILP; ++c) dmma(d[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < ILP; ++c) s += d[c][0] + d[c][1];
  if (s == 1234.5) out[0] = s;
}

// mode 0: all DFMA, 1: all DMMA, 2: even warps DFMA / odd warps DMMA
template <int ILP>
__global__ void mixed(double* out, int mode, int it_fma, int it_mma) {
  const int w = threadIdx.x >> 5;
  const bool is_mma = mode == 1 || (mode == 2 && (w & 1));
  if (is_mma)
    do_dmma<ILP>(out, it_mma);
  else
    do_dfma<ILP>(out, it_fma);
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int dev = 0, nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int warps = 8, blocks = nsm * 2;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int it_mma : {250, 500, 1000, 2000}) {
    const int it_fma = 2000;
    double tf[3];
    for (int mode = 0; mode < 3; ++mode) {
      mixed<4><<<blocks, 32 * warps>>>(out, mode, it_fma, it_mma);
      cudaEventRecord(e0);
      mixed<4><<<blocks, 32 * warps>>>(out, mode, it_fma, it_mma);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double nw = (double)warps * blocks;
      const double fma_warps = mode == 0 ? nw : mode == 1 ? 0 : nw / 2;
      const double mma_warps = nw - fma_warps;
      const double flops = 2.0 * (fma_warps * it_fma * 8 * 4 * 32 + mma_warps * it_mma * 8 * 4 * 256.0);
      tf[mode] = flops / (ms * 1e-3) / 1e12;
      printf("it_mma=%5d mode=%d (%s): %.3f ms, %.2f TFLOP/s\n", it_mma, mode,
             mode == 0 ? "DFMA" : mode == 1 ? "DMMA" : "half/half", ms, tf[mode]);
    }
    printf("  mixed / max(pure) = %.3f\n", tf[2] / (tf[0] > tf[1] ? tf[0] : tf[1]));
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
