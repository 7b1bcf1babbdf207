/* oracle_lanes.c -- restatement of `_lanes` (axlandau/kernel.py:306-389).
 * TEST INFRASTRUCTURE ONLY (see landau_oracle.h).  Compiled like numba's
 * `fastmath=True` lanes (-O3 -ffast-math) so the four lane passes vectorize;
 * the same lane formulation as the reference: exact divides, the
 * exponent/mantissa-split logarithm, both S2/S3 branches evaluated and
 * selected. */
#include <stdint.h>
#include <string.h>

#include "../paper_1702_08880_b200/csrc/landau_coefs.h"
#include "landau_oracle.h"

static const double PK[11] = LB_PK, QK[11] = LB_QK, PE[11] = LB_PE, QEX[11] = LB_QEX;
static const double S2C[10] = LB_S2C, S3C[10] = LB_S3C;

#if defined(__x86_64__) && !defined(ORC_NO_CLONES)
#define ORC_CLONES __attribute__((target_clones("arch=x86-64-v4", "arch=x86-64-v3", "default")))
#else
#define ORC_CLONES
#endif

ORC_CLONES
void orc_lanes(double ri, double zi, const double *r, const double *z, int n0, int nb,
               double eps2, double *txx, double *tzz, double *txz, double *tkr, double *tzr,
               double *xb, double *lb) {
  /* pass 1: x = d2/(d2 + 4 ri rn)  (kernel.py:310-316) */
  for (int k = 0; k < nb; ++k) {
    const double rn = r[n0 + k];
    const double dz = zi - z[n0 + k];
    const double dist2 = (ri - rn) * (ri - rn) + dz * dz;
    const double d2 = dist2 > 1e-300 ? dist2 : 1.0;
    xb[k] = d2 / (d2 + 4.0 * ri * rn);
  }
  /* passes 2-3: ln x by exponent/mantissa split + atanh series (317-337) */
  for (int k = 0; k < nb; ++k) {
    int64_t bits, lbits;
    memcpy(&bits, &xb[k], 8);
    lbits = (bits & (int64_t)0xFFFFFFFFFFFFFLL) | (int64_t)0x3FF0000000000000LL;
    double mant;
    memcpy(&mant, &lbits, 8);
    const double e = (double)((bits >> 52) - 1023);
    const double big = mant > LB_SQRT2 ? 1.0 : 0.0;
    mant = mant * (1.0 - 0.5 * big);
    const double s = (mant - 1.0) / (mant + 1.0);
    const double u = s * s;
    double p = 2.0 / 17.0;
    p = p * u + 2.0 / 15.0;
    p = p * u + 2.0 / 13.0;
    p = p * u + 2.0 / 11.0;
    p = p * u + 2.0 / 9.0;
    p = p * u + 2.0 / 7.0;
    p = p * u + 0.4;
    p = p * u + 2.0 / 3.0;
    p = p * u + 2.0;
    lb[k] = (e + big) * LB_LN2 + s * p;
  }
  /* pass 4: elliptic polynomials, S2/S3, tensor components (338-389) */
  for (int k = 0; k < nb; ++k) {
    const double rn = r[n0 + k];
    const double dz = zi - z[n0 + k];
    const double dz2 = dz * dz;
    const double dist2 = (ri - rn) * (ri - rn) + dz2;
    const double g = (dist2 >= eps2 && dist2 > 0.0) ? 1.0 : 0.0;
    const double d2 = dist2 > 1e-300 ? dist2 : 1.0;
    const double P = d2 + 4.0 * ri * rn;
    const double invP = 1.0 / P;
    const double m = 4.0 * ri * rn * invP;
    const double x = d2 * invP;
    const double lx = lb[k];
    double pk = PK[10], qk = QK[10], pe = PE[10], qe = QEX[10];
    for (int t = 9; t >= 0; --t) {
      pk = pk * x + PK[t];
      qk = qk * x + QK[t];
      pe = pe * x + PE[t];
      qe = qe * x + QEX[t];
    }
    const double EK = pk - lx * qk;
    const double EE = pe - lx * qe;
    const double isP = 1.0 / __builtin_sqrt(P);
    const double Em1 = EE * P / d2;
    const double mg = m > 1e-300 ? m : 1.0;
    const double invm = 1.0 / mg;
    const double S2c = 2.0 * (Em1 - EK) * invm - Em1;
    const double S3c = 4.0 * (Em1 + EE - 2.0 * EK) * invm * invm - 4.0 * (Em1 - EK) * invm + Em1;
    double s2s = S2C[9], s3s = S3C[9];
    for (int t = 8; t >= 1; --t) {
      s2s = s2s * m + S2C[t];
      s3s = s3s * m + S3C[t];
    }
    s2s = s2s * m;
    s3s = s3s * m + S3C[0];
    const int small = m < LB_M_SWITCH;
    const double S2 = small ? s2s : S2c;
    const double S3 = small ? s3s : S3c;
    const double c3 = 4.0 * isP * invP;
    const double B1 = 4.0 * EK * isP;
    const double B3 = Em1 * c3;
    const double B4 = S2 * c3;
    const double B5 = S3 * c3;
    const double rr = ri * rn;
    txx[k] = g * (B1 - ri * ri * B3 + 2.0 * rr * B4 - rn * rn * B5);
    tzz[k] = g * (B1 - dz2 * B3);
    txz[k] = g * (-dz * (ri * B3 - rn * B4));
    tkr[k] = g * (dz2 * B4 + rr * (B3 - B5));
    tzr[k] = g * (dz * (rn * B3 - ri * B4));
  }
}
