// Dependent latencies of the synchronisation primitives the block-LU panel
// chains per column (redux.sync, shfl, LDS, STS + bar.sync + LDS at 64 /
// 288 / 384 threads, an IEEE double division).  Measured on B200: 27 / 30 /
// 38 / 46-66 / 80 cycles.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a lat_sync.cu -o lat_sync
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_redux(unsigned* out, int iters, long long* cyc) {
  unsigned x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __reduce_max_sync(0xffffffffu, x + i) ^ threadIdx.x;
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_shfl(unsigned* out, int iters, long long* cyc) {
  unsigned x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __shfl_xor_sync(0xffffffffu, x + i, 1);
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_lds(unsigned* out, int iters, long long* cyc) {
  __shared__ unsigned s[64];
  s[threadIdx.x] = threadIdx.x; __syncwarp();
  unsigned x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = s[(x + i) & 31];
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_bar(unsigned* out, int iters, long long* cyc) {
  __shared__ unsigned s[1024];
  unsigned x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { s[threadIdx.x] = x + i; __syncthreads(); x = s[(threadIdx.x + 32) % blockDim.x]; }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_div(double* out, int iters, long long* cyc) {
  double x = 1.5 + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = 1.0 / x + 1.0;
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  unsigned* o; double* od; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&od, 8192); cudaMalloc(&c, 8);
  const int it = 10000; long long h;
  k_redux<<<1, 32>>>(o, it, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("redux.max dependent: %.1f cyc\n", (double)h / it);
  k_shfl<<<1, 32>>>(o, it, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("shfl dependent: %.1f cyc\n", (double)h / it);
  k_lds<<<1, 32>>>(o, it, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("lds dependent: %.1f cyc\n", (double)h / it);
  for (int nt : {64, 288, 384}) { k_bar<<<1, nt>>>(o, it, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("sts+bar+lds (%d thr): %.1f cyc\n", nt, (double)h / it); }
  k_div<<<1, 32>>>(od, it, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("ddiv+dadd dependent: %.1f cyc\n", (double)h / it);
  return 0;
}
