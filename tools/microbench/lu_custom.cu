// Custom batched LU (lb_getrf_kernel) and slab solve (lb_getrs_slab_kernel)
// of csrc/landau_lu.cuh against cuBLAS getrfBatched / getrsBatched at the
// Crank-Nicolson solver's block sizes: residuals and timings.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I../../paper_1702_08880_b200/csrc \
//        lu_custom.cu -lcublas -o lu_custom
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#ifndef LU_W
#define LU_W 32
#endif
#ifndef LU_KB
#define LU_KB 32
#endif
#ifndef LU_NT
#define LU_NT 256  // slab-solve threads
#endif
#ifndef LU_MWT
#define LU_MWT 0  // slab-solve warp tiles per warp (0: sized for 383 rows)
#endif
#include "landau_lu.cuh"

using namespace lb;
constexpr int KB = LU_KB, W = LU_W;

static double urand(unsigned long long& s) {
  s = s * 6364136223846793005ULL + 1442695040888963407ULL;
  return ((s >> 11) * (1.0 / 9007199254740992.0)) * 2.0 - 1.0;
}

int main(int argc, char** argv) {
  cublasHandle_t bl;
  cublasCreate(&bl);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  bool ok = true;
#ifdef LB_LU_PROF
  for (int n : {68, 260, 354}) {
    const size_t nn = (size_t)n * n;
    std::vector<double> hA(nn);
    unsigned long long seed = 99;
    for (auto& v : hA) v = urand(seed);
    double *A, *inv;
    int *piv, *perm, *info;
    cudaMalloc(&A, nn * 8);
    cudaMalloc(&inv, (size_t)lu_inv_stride<KB>(n) * 8);
    cudaMalloc(&piv, sizeof(int) * n);
    cudaMalloc(&perm, sizeof(int) * n);
    cudaMalloc(&info, sizeof(int));
    double** dA;
    cudaMalloc(&dA, sizeof(double*));
    cudaMemcpy(dA, &A, sizeof(double*), cudaMemcpyHostToDevice);
    const size_t sf = getrf_smem_bytes<KB>(n);
    cudaFuncSetAttribute(lb_getrf_kernel<KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sf);
    for (int i = 0; i < n; ++i) hA[(size_t)i * n + i] += 4.0;  // (unpivoted rep stays stable)
    for (int rep = 0; rep < 4; ++rep) {
      const int pv = rep < 2;  // reps 0, 1 pivoted; 2, 3 unpivoted
      if (rep == 2) printf("(unpivoted)\n");
      cudaMemcpy(A, hA.data(), nn * 8, cudaMemcpyHostToDevice);
      long long z[8] = {};
      cudaMemcpyToSymbol(lu_prof, z, sizeof(z));
      cudaMemcpyToSymbol(lu_prof2, z, 4 * sizeof(long long));
      lb_getrf_kernel<KB><<<1, kGetrfThreads, sf>>>(n, dA, piv, perm, info, inv, pv);
      cudaDeviceSynchronize();
      long long h[8], h2[4];
      cudaMemcpyFromSymbol(h, lu_prof, sizeof(h));
      cudaMemcpyFromSymbol(h2, lu_prof2, sizeof(h2));
      printf("  column loop (thread 0): candidates+publish %lld, barrier issue %lld, winner+loads %lld, update %lld cycles\n", h2[1], h2[3], h2[0], h2[2]);
      long long tot = 0;
      for (int k = 0; k < 5; ++k) tot += h[k];
      tot += h[5] + h[6];
      printf("prof n=%d: load %lld factor %lld store+inv %lld gather %lld U12 %lld U12-store %lld update %lld cycles (total %lld = %.1f us at 1.9 GHz)\n",
             n, h[0], h[1], h[2], h[5], h[6], h[3], h[4], tot, tot / 1.9e3);
      // the slab solve of 2n right-hand sides with these factors
      double* B;
      cudaMalloc(&B, (size_t)n * 2 * n * 8);
      cudaMemset(B, 0, (size_t)n * 2 * n * 8);
      double** dB;
      cudaMalloc(&dB, sizeof(double*));
      cudaMemcpy(dB, &B, sizeof(double*), cudaMemcpyHostToDevice);
      const size_t ss = getrs_smem_bytes<KB, W>(n);
      cudaFuncSetAttribute(lb_getrs_slab_kernel<KB, W, LU_NT, LU_MWT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ss);
      cudaMemcpyToSymbol(lu_prof, z, sizeof(z));
      lb_getrs_slab_kernel<KB, W, LU_NT, LU_MWT><<<dim3(1, (2 * n + W - 1) / W), LU_NT, ss>>>(n, 2 * n, dA, perm, inv, dB);
      cudaDeviceSynchronize();
      cudaMemcpyFromSymbol(h, lu_prof, sizeof(h));
      printf("prof getrs n=%d: wait+sync %lld DiX %lld update %lld writeback %lld sync+issue %lld cycles (%.1f us)\n", n,
             h[1], h[2], h[3], h[4], h[5], (h[1] + h[2] + h[3] + h[4] + h[5]) / 1.9e3);
      cudaFree(B);
      cudaFree(dB);
    }
  }
  return 0;
#endif
  std::vector<int> sizes = {5, 17, 32, 33, 67, 68, 131, 260, 354, 383};
  if (argc > 1) {  // explicit sizes: lu_custom n1 n2 ...
    sizes.clear();
    for (int a = 1; a < argc; ++a) sizes.push_back(std::atoi(argv[a]));
  }
  for (int n : sizes) {
    if (getrs_smem_bytes<KB, W>(n) > 232448) {
      printf("n=%3d: W=%d slab needs %zu B of shared memory, skipped\n", n, W, getrs_smem_bytes<KB, W>(n));
      continue;
    }
    std::vector<int> batches = {4, 64, 256};
    if (const char* e = std::getenv("LU_BATCHES")) {  // e.g. LU_BATCHES=8,16,32
      batches.clear();
      for (const char* q = e; *q;) {
        batches.push_back(std::atoi(q));
        while (*q && *q != ',') ++q;
        if (*q == ',') ++q;
      }
    }
    for (int batch : batches) {
      for (int kind = 0; kind < 2; ++kind) {  // 0: random (pivoting matters), 1: diagonally weighted
        const int m = 2 * n;
        const size_t nn = (size_t)n * n, nm = (size_t)n * m;
        std::vector<double> hA(nn * batch), hB(nm * batch);
        unsigned long long seed = 12345 + n * 7 + batch * 13 + kind;
        for (auto& v : hA) v = urand(seed);
        for (auto& v : hB) v = urand(seed);
        if (kind == 1)
          for (int b = 0; b < batch; ++b)
            for (int i = 0; i < n; ++i) hA[b * nn + (size_t)i * n + i] += 4.0;
        double *A, *A0, *B, *B0, *inv;
        int *piv, *perm, *info;
        cudaMalloc(&A, nn * batch * 8);
        cudaMalloc(&A0, nn * batch * 8);
        cudaMalloc(&B, nm * batch * 8);
        cudaMalloc(&B0, nm * batch * 8);
        cudaMalloc(&inv, (size_t)lu_inv_stride<KB>(n) * batch * 8);
        cudaMalloc(&piv, sizeof(int) * n * batch);
        cudaMalloc(&perm, sizeof(int) * n * batch);
        cudaMalloc(&info, sizeof(int) * batch);
        cudaMemcpy(A0, hA.data(), nn * batch * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(B0, hB.data(), nm * batch * 8, cudaMemcpyHostToDevice);
        std::vector<double*> pa(batch), pb(batch);
        for (int b = 0; b < batch; ++b) {
          pa[b] = A + b * nn;
          pb[b] = B + b * nm;
        }
        double **dA, **dB;
        cudaMalloc(&dA, sizeof(double*) * batch);
        cudaMalloc(&dB, sizeof(double*) * batch);
        cudaMemcpy(dA, pa.data(), sizeof(double*) * batch, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, pb.data(), sizeof(double*) * batch, cudaMemcpyHostToDevice);
        const size_t sf = getrf_smem_bytes<KB>(n), ss = getrs_smem_bytes<KB, W>(n);
        cudaFuncSetAttribute(lb_getrf_kernel<KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sf);
        cudaFuncSetAttribute(lb_getrs_slab_kernel<KB, W, LU_NT, LU_MWT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ss);
        const dim3 gs(batch, (m + W - 1) / W);
        float tc_f = 0, tc_s = 0, tb_f = 0, tb_s = 0;
        int hinfo = 0;
        for (int rep = 0; rep < 3; ++rep) {
          // custom
          cudaMemcpy(A, A0, nn * batch * 8, cudaMemcpyDeviceToDevice);
          cudaMemcpy(B, B0, nm * batch * 8, cudaMemcpyDeviceToDevice);
          cudaEventRecord(e0);
          lb_getrf_kernel<KB><<<batch, kGetrfThreads, sf>>>(n, dA, piv, perm, info, inv, 1);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          cudaEventElapsedTime(&tc_f, e0, e1);
          cudaEventRecord(e0);
          lb_getrs_slab_kernel<KB, W, LU_NT, LU_MWT><<<gs, LU_NT, ss>>>(n, m, dA, perm, inv, dB);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          cudaEventElapsedTime(&tc_s, e0, e1);
        }
        cudaError_t err = cudaGetLastError();
        if (err != cudaSuccess) {
          printf("CUDA error %s\n", cudaGetErrorString(err));
          return 1;
        }
        // residuals on the host: |P A - L U| / |A| and |A X - B| / (|A| |X|) for a few matrices
        std::vector<double> hF(nn * batch), hX(nm * batch);
        std::vector<int> hp(n * batch), hi(batch);
        cudaMemcpy(hF.data(), A, nn * batch * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(hX.data(), B, nm * batch * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(hp.data(), perm, sizeof(int) * n * batch, cudaMemcpyDeviceToHost);
        cudaMemcpy(hi.data(), info, sizeof(int) * batch, cudaMemcpyDeviceToHost);
        double elu = 0, esol = 0;
        for (int b : {0, batch - 1}) {
          const double* a = &hA[b * nn];
          const double* f = &hF[b * nn];
          const int* pr = &hp[b * n];
          double amax = 0;
          for (size_t t = 0; t < nn; ++t) amax = fmax(amax, fabs(a[t]));
          for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) {
              double s = 0;
              for (int k = 0; k <= std::min(i, j); ++k) s += (k == i ? 1.0 : f[(size_t)k * n + i]) * f[(size_t)j * n + k];
              elu = fmax(elu, fabs(s - a[(size_t)j * n + pr[i]]) / amax);
            }
          const double* x = &hX[b * nm];
          const double* bb = &hB[b * nm];
          double xmax = 0;
          for (size_t t = 0; t < nm; ++t) xmax = fmax(xmax, fabs(x[t]));
          for (int c = 0; c < m; c += 7)
            for (int i = 0; i < n; ++i) {
              double s = 0;
              for (int k = 0; k < n; ++k) s += a[(size_t)k * n + i] * x[(size_t)c * n + k];
              esol = fmax(esol, fabs(s - bb[(size_t)c * n + i]) / (amax * xmax * n));
            }
        }
        // cuBLAS
        for (int rep = 0; rep < 3; ++rep) {
          cudaMemcpy(A, A0, nn * batch * 8, cudaMemcpyDeviceToDevice);
          cudaMemcpy(B, B0, nm * batch * 8, cudaMemcpyDeviceToDevice);
          cudaEventRecord(e0);
          cublasDgetrfBatched(bl, n, dA, n, piv, info, batch);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          cudaEventElapsedTime(&tb_f, e0, e1);
          cudaEventRecord(e0);
          cublasDgetrsBatched(bl, CUBLAS_OP_N, n, m, dA, n, piv, dB, n, &hinfo, batch);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          cudaEventElapsedTime(&tb_s, e0, e1);
        }
        const bool good = elu < 1e-13 && esol < 1e-14 && hi[0] == 0;
        ok = ok && good;
        printf("n=%3d batch=%3d %s: custom getrf %7.3f getrs(2n) %7.3f ms | cuBLAS %7.3f %7.3f ms | "
               "|PA-LU|/|A| %.1e  |AX-B| %.1e %s\n",
               n, batch, kind ? "diag" : "rand", tc_f, tc_s, tb_f, tb_s, elu, esol, good ? "ok" : "FAIL");
        cudaFree(A); cudaFree(A0); cudaFree(B); cudaFree(B0); cudaFree(inv);
        cudaFree(piv); cudaFree(perm); cudaFree(info); cudaFree(dA); cudaFree(dB);
      }
    }
  }
  printf(ok ? "ALL OK\n" : "FAILURES\n");
  return ok ? 0 : 1;
}
