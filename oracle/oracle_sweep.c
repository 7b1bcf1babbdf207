/* oracle_sweep.c -- restatement of the reference's fused sweep driver,
 * accumulation and coupling (axlandau/kernel.py:392-493), the scalar
 * closed form (kernel.py:179-235) and elliptic_KE (kernel.py:93-128).
 * TEST INFRASTRUCTURE ONLY (see landau_oracle.h).  Compiled WITHOUT
 * fast-math: the accumulation runs in strict inner-index order exactly as
 * `_accumulate_block` / `_combine` do; OpenMP over outer points plays the
 * role of numba's prange (each outer point owns its accumulators). */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "../paper_1702_08880_b200/csrc/landau_coefs.h"
#include "landau_oracle.h"

static const double PK[11] = LB_PK, QK[11] = LB_QK, PE[11] = LB_PE, QEX[11] = LB_QEX;
static const double S2C[10] = LB_S2C, S3C[10] = LB_S3C;

int orc_version(void) { return 100; }

int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

static void elliptic_scalar(double x, double *K, double *E) { /* kernel.py:116-128 */
  const double lx = log(x);
  double pk = PK[10], qk = QK[10], pe = PE[10], qe = QEX[10];
  for (int t = 9; t >= 0; --t) {
    pk = pk * x + PK[t];
    qk = qk * x + QK[t];
    pe = pe * x + PE[t];
    qe = qe * x + QEX[t];
  }
  *K = pk - lx * qk;
  *E = pe - lx * qe;
}

void orc_elliptic_ke(int n, const double *m, double *K, double *E) {
  for (int i = 0; i < n; ++i) elliptic_scalar(1.0 - m[i], &K[i], &E[i]);
}

int orc_tensor_pair(double r, double z, double rbar, double zbar, double *UK, double *UD) {
  if (r < 0.0 || rbar < 0.0) return -1; /* kernel.py:219-220 */
  const double dz = z - zbar;           /* _base_integrals, kernel.py:179-203 */
  const double q = (r - rbar) * (r - rbar) + dz * dz;
  const double p = q + 4.0 * r * rbar;
  if (q == 0.0) return -2;
  const double x = q / p;
  const double m = 4.0 * r * rbar / p;
  double K, E;
  elliptic_scalar(x, &K, &E);
  const double em1 = E * p / q;
  double s2, s3;
  if (m < LB_M_SWITCH) {
    s2 = 0.0;
    s3 = S3C[9];
    for (int t = 8; t >= 1; --t) {
      s2 = (s2 + S2C[t + 1]) * m;
      s3 = s3 * m + S3C[t];
    }
    s2 = (s2 + S2C[1]) * m;
    s3 = s3 * m + S3C[0];
  } else {
    s2 = 2.0 * (em1 - K) / m - em1;
    s3 = 4.0 * (em1 + E - 2.0 * K) / (m * m) - 4.0 * (em1 - K) / m + em1;
  }
  const double c3 = 4.0 * pow(p, -1.5);
  const double b1 = 4.0 * K / sqrt(p);
  const double b3 = em1 * c3, b4 = s2 * c3, b5 = s3 * c3;
  const double dz2 = dz * dz; /* axisym_tensor_pair, kernel.py:224-234 */
  const double xz = -dz * (r * b3 - rbar * b4);
  const double zz = b1 - dz2 * b3;
  UD[0] = b1 - r * r * b3 + 2.0 * r * rbar * b4 - rbar * rbar * b5;
  UD[1] = xz;
  UD[2] = xz;
  UD[3] = zz;
  UK[0] = dz2 * b4 + r * rbar * (b3 - b5);
  UK[1] = xz;
  UK[2] = dz * (rbar * b3 - r * b4);
  UK[3] = zz;
  return 0;
}

void orc_sweep(int nout, const double *ro, const double *zo, int n, int S, const double *r,
               const double *z, const double *w, const double *f, const double *dfr,
               const double *dfz, const double *coK, const double *coD, double eps2, int blk,
               double *Kout, double *Dout, int nthreads) {
  if (blk <= 0) blk = 256;
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel num_threads(nthreads)
#endif
  {
    double *scratch = (double *)malloc(sizeof(double) * (7 * (size_t)blk + 5 * (size_t)S));
    double *xb = scratch, *lb = xb + blk, *txx = lb + blk, *tzz = txx + blk, *txz = tzz + blk,
           *tkr = txz + blk, *tzr = tkr + blk, *A = tzr + blk;
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 8)
#endif
    for (int i = 0; i < nout; ++i) {
      const double ri = ro[i], zi = zo[i];
      memset(A, 0, sizeof(double) * 5 * S);
      for (int n0 = 0; n0 < n; n0 += blk) {
        const int nb = n - n0 < blk ? n - n0 : blk;
        orc_lanes(ri, zi, r, z, n0, nb, eps2, txx, tzz, txz, tkr, tzr, xb, lb);
        /* _accumulate_block (kernel.py:393-415): strict inner-index order */
        for (int k = 0; k < nb; ++k) {
          const int nn = n0 + k;
          const double wn = w[nn];
          const double vkr = tkr[k], vzr = tzr[k], vxx = txx[k], vzz = tzz[k], vxz = txz[k];
          for (int b = 0; b < S; ++b) {
            const double gr = dfr[(size_t)b * n + nn] * wn;
            const double gz = dfz[(size_t)b * n + nn] * wn;
            const double fb = f[(size_t)b * n + nn] * wn;
            double *Ab = A + 5 * b;
            Ab[0] += vkr * gr + vxz * gz;
            Ab[1] += vzr * gr + vzz * gz;
            Ab[2] += fb * vxx;
            Ab[3] += fb * vxz;
            Ab[4] += fb * vzz;
          }
        }
      }
      /* _combine (kernel.py:419-440) */
      for (int a = 0; a < S; ++a) {
        double k0 = 0.0, k1 = 0.0, d0 = 0.0, d1 = 0.0, d2 = 0.0;
        for (int b = 0; b < S; ++b) {
          const double ck = coK[a * S + b], cd = coD[a * S + b];
          k0 += ck * A[5 * b + 0];
          k1 += ck * A[5 * b + 1];
          d0 += cd * A[5 * b + 2];
          d1 += cd * A[5 * b + 3];
          d2 += cd * A[5 * b + 4];
        }
        double *Ko = Kout + ((size_t)i * S + a) * 2;
        double *Do = Dout + ((size_t)i * S + a) * 4;
        Ko[0] = k0;
        Ko[1] = k1;
        Do[0] = d0;
        Do[1] = d1;
        Do[2] = d1;
        Do[3] = d2;
      }
    }
    free(scratch);
  }
}
