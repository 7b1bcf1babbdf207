// Dense LU timing on the device: cuBLAS batched getrf vs cuSOLVER getrf,
// to size the block-tridiagonal solver's diagonal blocks.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a lu_bench.cu -lcublas -lcusolver -o lu_bench
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <cstdio>
#include <vector>

int main() {
  cublasHandle_t bl;
  cusolverDnHandle_t so;
  cublasCreate(&bl);
  cusolverDnCreate(&so);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int n : {64, 128, 260, 354, 520, 1040, 2080, 3807, 8385}) {
    const int batch = 4;
    size_t nn = (size_t)n * n;
    std::vector<double> h(nn * batch);
    for (size_t i = 0; i < h.size(); ++i) h[i] = ((i * 2654435761u) % 1000) / 1000.0;
    for (int b = 0; b < batch; ++b)
      for (int i = 0; i < n; ++i) h[b * nn + (size_t)i * n + i] += n;
    double *A, *A0;
    cudaMalloc(&A, nn * batch * 8);
    cudaMalloc(&A0, nn * batch * 8);
    cudaMemcpy(A0, h.data(), nn * batch * 8, cudaMemcpyHostToDevice);
    int *piv, *info;
    cudaMalloc(&piv, sizeof(int) * n * batch);
    cudaMalloc(&info, sizeof(int) * batch);
    std::vector<double*> ptr(batch);
    for (int b = 0; b < batch; ++b) ptr[b] = A + b * nn;
    double** dptr;
    cudaMalloc(&dptr, sizeof(double*) * batch);
    cudaMemcpy(dptr, ptr.data(), sizeof(double*) * batch, cudaMemcpyHostToDevice);
    float tb = -1, ts = -1;
    if (n <= 1040) {
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemcpy(A, A0, nn * batch * 8, cudaMemcpyDeviceToDevice);
        cudaEventRecord(e0);
        cublasDgetrfBatched(bl, n, dptr, n, piv, info, batch);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&tb, e0, e1);
      }
    }
    int lw = 0;
    cusolverDnDgetrf_bufferSize(so, n, n, A, n, &lw);
    double* work;
    cudaMalloc(&work, sizeof(double) * lw);
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemcpy(A, A0, nn * batch * 8, cudaMemcpyDeviceToDevice);
      cudaEventRecord(e0);
      for (int b = 0; b < batch; ++b) cusolverDnDgetrf(so, n, n, A + b * nn, n, work, piv + b * n, info + b);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ts, e0, e1);
    }
    // getrs with n right-hand sides (X = D^-1 U) after cusolver getrf
    float tr = -1;
    double* B;
    cudaMalloc(&B, nn * batch * 8);
    cudaMemcpy(B, A0, nn * batch * 8, cudaMemcpyDeviceToDevice);
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      for (int b = 0; b < batch; ++b)
        cusolverDnDgetrs(so, CUBLAS_OP_N, n, n, A + b * nn, n, piv + b * n, B + b * nn, n, info + b);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&tr, e0, e1);
    }
    printf("n=%5d x%d: cublas getrfBatched %8.3f ms   cusolver getrf %8.3f ms (%.1f TF)   getrs(nrhs=n) %8.3f ms\n",
           n, batch, tb, ts, batch * 2.0 / 3 * n * (double)n * n / (ts * 1e-3) / 1e12, tr);
    cudaFree(A); cudaFree(A0); cudaFree(piv); cudaFree(info); cudaFree(dptr); cudaFree(work); cudaFree(B);
  }
  return 0;
}
