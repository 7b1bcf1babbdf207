// cuBLAS batched LU / inverse / triangular-solve timings at the block sizes
// of the Crank-Nicolson solver (nb 68..354) and batch counts of the cyclic
// reduction levels.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a lu_bench2.cu -lcublas -o lu_bench2
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

int main() {
  cublasHandle_t bl;
  cublasCreate(&bl);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int n : {68, 260, 354}) {
    for (int batch : {4, 64, 256}) {
      size_t nn = (size_t)n * n;
      std::vector<double> h(nn * batch);
      for (size_t i = 0; i < h.size(); ++i) h[i] = ((i * 2654435761u) % 1000) / 1000.0;
      for (int b = 0; b < batch; ++b)
        for (int i = 0; i < n; ++i) h[b * nn + (size_t)i * n + i] += n;
      double *A, *A0, *C, *B;
      cudaMalloc(&A, nn * batch * 8);
      cudaMalloc(&A0, nn * batch * 8);
      cudaMalloc(&C, nn * batch * 8);
      cudaMalloc(&B, nn * batch * 8);
      cudaMemcpy(A0, h.data(), nn * batch * 8, cudaMemcpyHostToDevice);
      int *piv, *info;
      cudaMalloc(&piv, sizeof(int) * n * batch);
      cudaMalloc(&info, sizeof(int) * batch);
      std::vector<double*> pa(batch), pc(batch), pb(batch);
      for (int b = 0; b < batch; ++b) {
        pa[b] = A + b * nn;
        pc[b] = C + b * nn;
        pb[b] = B + b * nn;
      }
      double **dA, **dC, **dB;
      cudaMalloc(&dA, sizeof(double*) * batch);
      cudaMalloc(&dC, sizeof(double*) * batch);
      cudaMalloc(&dB, sizeof(double*) * batch);
      cudaMemcpy(dA, pa.data(), sizeof(double*) * batch, cudaMemcpyHostToDevice);
      cudaMemcpy(dC, pc.data(), sizeof(double*) * batch, cudaMemcpyHostToDevice);
      cudaMemcpy(dB, pb.data(), sizeof(double*) * batch, cudaMemcpyHostToDevice);
      float tf = 0, ti = 0, ts = 0, tg = 0, tv = 0;
      int hinfo = 0;
      const double one = 1.0, zero = 0.0;
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemcpy(A, A0, nn * batch * 8, cudaMemcpyDeviceToDevice);
        cudaMemcpy(B, A0, nn * batch * 8, cudaMemcpyDeviceToDevice);
        cudaEventRecord(e0);
        cublasDgetrfBatched(bl, n, dA, n, piv, info, batch);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&tf, e0, e1);
        cudaEventRecord(e0);
        cublasDgetriBatched(bl, n, dA, n, piv, dC, n, info, batch);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ti, e0, e1);
        cudaEventRecord(e0);
        cublasDgetrsBatched(bl, CUBLAS_OP_N, n, n, dA, n, piv, dB, n, &hinfo, batch);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ts, e0, e1);
        cudaEventRecord(e0);
        cublasDgemmBatched(bl, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, dC, n, dA, n, &zero, dB, n, batch);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&tg, e0, e1);
        cudaEventRecord(e0);
        cublasDgemvBatched(bl, CUBLAS_OP_N, n, n, &one, dC, n, dA, 1, &zero, dB, 1, batch);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&tv, e0, e1);
      }
      // no pivoting: getrf with a null pivot array + two triangular solves
      float tfn = 0, tt = 0;
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemcpy(A, A0, nn * batch * 8, cudaMemcpyDeviceToDevice);
        cudaMemcpy(B, A0, nn * batch * 8, cudaMemcpyDeviceToDevice);
        cudaEventRecord(e0);
        cublasDgetrfBatched(bl, n, dA, n, nullptr, info, batch);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&tfn, e0, e1);
        cudaEventRecord(e0);
        cublasDtrsmBatched(bl, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_UNIT, n, n,
                           &one, dA, n, dB, n, batch);
        cublasDtrsmBatched(bl, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, n,
                           n, &one, dA, n, dB, n, batch);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&tt, e0, e1);
      }
      printf("n=%4d batch=%4d: getrf %7.3f  getri %7.3f  getrs(nrhs=n) %7.3f  gemm %7.3f  gemv %7.3f ms"
             "  | no-pivot getrf %7.3f  2x trsm(nrhs=n) %7.3f ms\n", n, batch, tf, ti, ts, tg, tv, tfn, tt);
      cudaFree(A); cudaFree(A0); cudaFree(C); cudaFree(B); cudaFree(piv); cudaFree(info);
      cudaFree(dA); cudaFree(dC); cudaFree(dB);
    }
  }
  return 0;
}
