// Dependent-latency and throughput microbenchmarks for the FP64 pipe on
// sm_100a (B200): DFMA chains at ILP 1/2/4/8 with 1..16 warps per SMSP.
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void chain(double* out, double a, double b, int iters, long long* cyc) {
  double v[ILP];
#pragma unroll
  for (int c = 0; c < ILP; ++c) v[c] = threadIdx.x * 1e-9 + c;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int c = 0; c < ILP; ++c) v[c] = fma(v[c], a, b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < ILP; ++c) s += v[c];
  if (s == 1234.5) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int ILP>
void run(int warps, int blocks) {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, 8);
  const int iters = 2000;
  chain<ILP><<<blocks, 32 * warps>>>(out, 0.999999, 1e-7, iters, cyc);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  chain<ILP><<<blocks, 32 * warps>>>(out, 0.999999, 1e-7, iters, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double per_warp_dfma = (double)iters * 8 * ILP;
  const double total = per_warp_dfma * warps * blocks * 32;
  printf("ILP=%d warps/CTA=%2d blocks=%4d: cycles per dependent DFMA (thread 0) %.2f, "
         "chip %.2f TFLOP/s\n",
         ILP, warps, blocks, (double)c / (iters * 8), 2 * total / (ms * 1e-3) / 1e12);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<1>(1, 1);
  run<2>(1, 1);
  run<4>(1, 1);
  run<8>(1, 1);
  // one SM, increasing warps (4 SMSPs)
  for (int w : {4, 8, 16, 32}) run<1>(w, 1);
  for (int w : {4, 8, 16}) run<2>(w, 1);
  for (int w : {4, 8, 16}) run<4>(w, 1);
  // full chip
  run<1>(16, 148 * 4);
  run<2>(16, 148 * 4);
  run<4>(16, 148 * 4);
  run<8>(8, 148 * 4);
  return 0;
}
