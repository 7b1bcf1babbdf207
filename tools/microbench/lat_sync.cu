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
__global__ void k_dmma(double* out, int iters, long long* cyc, int chains) {
  double d[8][2];
  for (int c = 0; c < 8; ++c) d[c][0] = d[c][1] = threadIdx.x * 1e-3 + c;
  const double a = 0.999, b = 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (chains == 1) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d[0][0]), "+d"(d[0][1]) : "d"(a), "d"(b));
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
    }
  }
  long long t1 = clock64();
  double s = 0; for (int c = 0; c < 8; ++c) s += d[c][0] + d[c][1];
  if (s == 1234.5) out[0] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  unsigned* o; double* od; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&od, 8192); cudaMalloc(&c, 8);
  const int it = 10000; long long h;
  k_redux<<<1, 32>>>(o, it, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("redux.max dependent: %.1f cyc\n", (double)h / it);
  k_shfl<<<1, 32>>>(o, it, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("shfl dependent: %.1f cyc\n", (double)h / it);
  k_lds<<<1, 32>>>(o, it, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("lds dependent: %.1f cyc\n", (double)h / it);
  for (int nt : {64, 288, 384}) { k_bar<<<1, nt>>>(o, it, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("sts+bar+lds (%d thr): %.1f cyc\n", nt, (double)h / it); }
  k_dmma<<<1, 32>>>(od, it, c, 1); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("dmma m8n8k4 dependent: %.1f cyc\n", (double)h / it);
  k_dmma<<<1, 32>>>(od, it, c, 8); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("dmma m8n8k4, 8 chains, 1 warp: %.1f cyc per mma\n", (double)h / it / 8);
  k_dmma<<<1, 128>>>(od, it, c, 8); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("dmma m8n8k4, 8 chains, 4 warps: %.1f cyc per mma per warp\n", (double)h / it / 8);
  k_div<<<1, 32>>>(od, it, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("ddiv+dadd dependent: %.1f cyc\n", (double)h / it);
  return 0;
}
