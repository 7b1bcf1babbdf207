// landau_pair.cuh -- per-pair FP64 arithmetic of the axisymmetric Landau
// tensor, restructured for the sm_100a FP64 pipe.
//
// Mathematically this is the reference's `_lanes` (axlandau/kernel.py:306-389)
// and scalar `_base_integrals`/`axisym_tensor_pair` (kernel.py:179-235):
//
//   d^2 = (ri-rn)^2 + dz^2, P = d^2 + 4 ri rn, x = d^2/P, m = 4 ri rn/P
//   K = PK(x) - ln x QK(x), E = PE(x) - ln x QEx(x)          (kernel.py:351-361)
//   Em1 = E P/d^2; S2, S3 closed form (m >= 0.01) or series  (kernel.py:363-378)
//   B1 = 4K/sqrt(P), B3 = Em1 c3, B4 = S2 c3, B5 = S3 c3, c3 = 4 P^-3/2
//   5 tensor components masked by g = [d^2 >= eps^2 and d^2 > 0]  (kernel.py:384-389)
//
// What differs (the arithmetic, not the math):
//  * no IEEE divides: 1/sqrt(P) is MUFU.RSQ64H + one cubic Newton step,
//    1/P = (1/sqrt P)^2, 1/d^2 is MUFU.RCP64H + one cubic step, 2/m = P * (1/(2 ri)) * (1/rn) from per-point reciprocals;
//  * the common factor 4 of B1..B5 is pulled out (an exact power-of-two
//    scaling) and folded into the species coupling coefficients;
//  * the m < 0.01 series and the closed form are a real branch instead of
//    computing both and selecting (kernel.py:366-378 always computes both);
//  * the log is table-driven (no divide) instead of the reference's
//    exponent/mantissa split + atanh series (kernel.py:317-337); both are
//    accurate to ~1 ulp;
//  * the mask and the d^2 guard are 64-bit integer compares on the bit
//    pattern (d^2 >= 0, so IEEE order == integer order);
//  * the tensor components are formed from B1, B3, B4 and the two
//    DIFFERENCES c34 = B3 - B4 = c3 (Em1 - S2) and c35 = B3 - B5 =
//    c3 (Em1 - S3), which have closed forms free of the 1/x terms (using
//    Em1 (1 - m) = E):  Em1 - S2 = (2/m)(K - E),  Em1 - S3 =
//    (4/m^2)((2 - m) K - 2 E)  (m >= 0.01; below, the series' S2/S3 are
//    subtracted directly).  With dr = ri - rn (kernel.py:384-389 rearranged):
//      UD_xx = B1 - dr^2 B3 - 2 ri rn c34 + rn^2 c35
//      UD_zz = B1 - dz^2 B3,  UD_xz = -dz (dr B3 + rn c34)
//      UK_rr = dz^2 B4 + ri rn c35,  UK_zr = dz (rn c34 - dr B4)
//    The reference's forms (e.g. ri rn (B3 - B5)) subtract two O(1/x)
//    terms: for near-coincident pairs (x = d^2/P -> 0) they lose
//    ~log10(1/x) digits, which at config 4's per-species meshes (tungsten
//    mesh, points ~1e-5 apart) put the reference itself ~1e-10 from exact
//    arithmetic (tools/diag/hp_point.py); these forms do not, and cost one
//    FP64 operation less per pair.
// Every change is a re-association or a <= 1-ulp reciprocal; the parity
// tests bound the end-to-end effect (<= 1e-10 scaled, measured ~1e-14).
#pragma once
#include <cstdint>
#include "landau_coefs.h"

#ifndef LB_SERIES_MODE
#define LB_SERIES_MODE 1  // 1: one series branch per lockstep group (selected per pair); 0: one per pair
#endif

#ifndef LB_KD_I2F
#define LB_KD_I2F 1  // exponent to double by I2F.F64 (off the FP64 pipe); 0: magic-number DADD
#endif

#ifndef LB_ESTRIN
#define LB_ESTRIN 0  // 1: Estrin-form polynomials (shorter dependency chains)
#endif

namespace lb {

// Coefficient tables live in the constant bank so DFMA reads them as
// c[0x3][..] operands (64-bit literals would cost a UMOV/IMAD.MOV pair each).
__constant__ double c_pk[11] = LB_PK;
__constant__ double c_qk[11] = LB_QK;
__constant__ double c_pe[11] = LB_PE;
__constant__ double c_qe[11] = LB_QEX;
__constant__ double c_s2[10] = LB_S2C;
__constant__ double c_s3[10] = LB_S3C;
// log1p tail coefficients (-1/8, 1/7, -1/6, 1/5, 1/3), spare, spare, spare,
// spare, ln2, the series switch 0.01, the 2^52 + 2^31 magic
__constant__ double c_misc[12] = {-1.0 / 8.0, 1.0 / 7.0, -1.0 / 6.0, 1.0 / 5.0, 1.0 / 3.0,
                                  0.0,        0.0,       0.0,        0.0,       LB_LN2,
                                  LB_M_SWITCH, 4503601774854144.0};
// (invc, logc) table of log_table(), copied to shared memory by the kernels
__constant__ double c_logt[2 << LB_LOGT_BITS] = LB_LOGT;

// bit pattern of 1e-300 (the reference's d^2 guard, kernel.py:315,345)
constexpr long long kTinyBits = 0x01A56E1FC2F8F359LL;
// bit pattern of sqrt(2) (mantissa fold threshold, kernel.py:324)
constexpr long long kSqrt2Bits = 0x3FF6A09E667F3BCDLL;
// bit pattern of 0.99 = 1 - 0.01, the series / closed-form switch
// (kernel.py:151) expressed on x = 1 - m
constexpr long long kXSwitchBits = 0x3FEFAE147AE147AELL;

__device__ __forceinline__ double rcp_approx(double a) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
  return r;
}
__device__ __forceinline__ double rsqrt_approx(double a) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
  return r;
}

// 1/a for normal positive a: ~2^-23 seed, one cubic step -> ~1 ulp.
__device__ __forceinline__ double rcp_nr(double a) {
  double r = rcp_approx(a);
  double e = fma(-a, r, 1.0);
  e = fma(e, e, e);
  return fma(r, e, r);
}

// 1/sqrt(a) for normal positive a: seed + one cubic step (1 + e/2 + 3e^2/8).
__device__ __forceinline__ double rsqrt_nr(double a) {
  double y = rsqrt_approx(a);
  double h = a * y;
  double e = fma(-h, y, 1.0);
  double c = fma(0.375, e, 0.5);
  double ye = y * e;
  return fma(ye, c, y);
}

constexpr long long kLogOff = 0x3FE6000000000000LL;

// Stage 1 of the log: table lookup and argument reduction.  Returns r with
// |r| < 2^-(LB_LOGT_BITS); logc and the exponent (as a double) are written to the refs.
__device__ __forceinline__ double log_reduce(double x, const double2* __restrict__ tab,
                                             double& logc, double& kd) {
  const long long ix = __double_as_longlong(x);
  const long long tmp = ix - kLogOff;
  const int i = (int)((tmp >> (52 - LB_LOGT_BITS)) & ((1 << LB_LOGT_BITS) - 1));
  const int k = (int)(tmp >> 52);
  const double z = __longlong_as_double(ix - (tmp & (long long)0xFFF0000000000000ULL));
  const double2 t = tab[i];  // (invc, logc)
  logc = t.y;
  // exact int -> double: 2^52 + 2^31 + k, minus the same magic
#if LB_KD_I2F
  kd = (double)k;  // I2F.F64 (conversion unit) instead of a DADD on the FP64 pipe
#else
  kd = __longlong_as_double(0x4330000080000000LL + (long long)k) - c_misc[11];
#endif
  return fma(z, t.x, -1.0);
}

// Stage 2 of the log: ln x = k ln2 + logc + ln(1 + r).
__device__ __forceinline__ double log_finish(double r, double logc, double kd) {
#if LB_ESTRIN
  // q(r) = -1/2 + r/3 - r^2/4 + r^3/5 - r^4/6 + r^5/7 - r^6/8, depth 3
  const double r2 = r * r;
  const double q = fma(fma(-0.125, r2, fma(r, c_misc[1], c_misc[2])), r2 * r2,
                       fma(fma(r, c_misc[3], -0.25), r2, fma(r, c_misc[4], -0.5)));
  const double l1p = fma(r2, q, r);
#elif LB_LOGT_BITS >= 9
  // |r| < 2^-9: q(r) = -1/2 + r/3 - r^2/4 + r^3/5 - r^4/6 (terms to r^6)
  double q = fma(r, c_misc[2], c_misc[3]);  // -1/6 r + 1/5
  q = fma(q, r, -0.25);
  q = fma(q, r, c_misc[4]);                 //  1/3
  q = fma(q, r, -0.5);
  const double l1p = fma(r * r, q, r);
#else
  double q = fma(r, c_misc[0], c_misc[1]);  // -1/8 r + 1/7
  q = fma(q, r, c_misc[2]);                 // -1/6
  q = fma(q, r, c_misc[3]);                 //  1/5
  q = fma(q, r, -0.25);
  q = fma(q, r, c_misc[4]);                 //  1/3
  q = fma(q, r, -0.5);
  const double l1p = fma(r * r, q, r);
#endif
  return fma(kd, c_misc[9], logc + l1p);
}

// ln(x) for normal positive x (the reference uses an exponent/mantissa split
// + atanh series, kernel.py:317-337; any log accurate to ~1 ulp agrees to
// 1e-16).  Here: table-driven reduction, no divide.  The mantissa is folded
// around 1 (z in [0.6875, 1.375)), a 2^LB_LOGT_BITS-entry table gives invc ~ 1/z and
// logc = -ln(invc) (invc == 1 exactly on the two bins touching 1.0, so ln x
// keeps full relative accuracy as x -> 1), r = z*invc - 1 (|r| < 2^-9 with
// the 512-entry table, one FMA), ln(1+r) = r + r^2 q(r), q the degree-4 Taylor tail.
// Measured max relative error 2.2e-16 (tools/gen_coefs.py table).
__device__ __forceinline__ double log_table(double x, const double2* __restrict__ tab) {
  double logc, kd;
  const double r = log_reduce(x, tab, logc, kd);
  return log_finish(r, logc, kd);
}

// Per-outer-point invariants (hoisted out of the pair loop).  Scaled by
// exact powers of two (see "Scaled pair quantities" below).
struct Outer {
  double ri, zi;
  double ri2;   // 4 ri^2
  double rtri;  // 1/(4 ri), 0 when ri == 0 (then m == 0 and the series runs)
  double ri4;   // 4 ri
};

__device__ __forceinline__ Outer make_outer(double ri, double zi) {
  Outer o;
  o.ri = ri;
  o.zi = zi;
  o.ri2 = 4.0 * (ri * ri);
  o.rtri = ri > 0.0 ? 1.0 / (4.0 * ri) : 0.0;
  o.ri4 = 4.0 * ri;
  return o;
}

// Scaled pair quantities.  Every factor below is an exact power of two, so
// each rounded value is the unscaled one times that power and the tensor
// components are bitwise those of the unscaled formulas; the scalings only
// let the products meet without extra multiplications:
//   rq = 4 ri rn (P = rq + d^2, m = rq / P),
//   c34' = c34 / 2 and c35' = c35 / 4 (from 1/(4 ri rn) instead of 1/(2 ri rn)),
//   records carry 4 rn^2 and 2 rn, outer points 4 ri^2:
//   2 ri rn c34 = rq c34',  ri rn c35 = rq c35',  rn^2 c35 = (4 rn^2) c35',
//   rn c34 = (2 rn) c34',  ri^2 c35 = (4 ri^2) c35',  B4 = B3 - 2 c34'.
// The five distinct tensor components, each scaled by 1/4:
//   xx = UD_xx, zz = UD_zz = UK_zz, xz = UD_xz = UD_zx = UK_rz,
//   kr = UK_rr, zr = UK_zr                                   (kernel.py:384-389)
struct T5 {
  double xx, zz, xz, kr, zr;
};

// The symmetric part of one pair (each / 4; all zero for masked pairs):
// B1, B3, B4 and the differences c34 = B3 - B4, c35 = B3 - B5 in their
// well-conditioned closed forms; dz, dz^2, dr = ri - rn and ri rn.
struct PairB {
  double B1, B3, B4, c34, c35;  // c34 = (B3 - B4) / 2, c35 = (B3 - B5) / 4 (scaled)
  double dz, dz2, dr, rr;       // rr = 4 ri rn
};

// gthr = max(bits(eps^2), 1): the pair contributes iff bits(d^2) >= gthr,
// i.e. d^2 >= eps^2 and d^2 > 0 (kernel.py:344).
// Stage 1 of a pair: geometry, mask, 1/sqrt(P), x and the log's table
// lookup -- the long-latency front (MUFU, shared-memory table) that the
// symmetric sweep issues one step ahead of the rest.
struct PairS1 {
  double dz, dz2, dr, d2, P, rr, isPm, invP, x, lr, logc, kd;
};


// MG ("merged guard"): when the mask threshold is above the d^2 guard
// (eps_d^2 > 1e-300, e.g. assemble_collision's 1e-14 L), every pair the
// guard would touch is masked anyway, so one compare serves both; the host
// picks the variant (sym_partial), the general form keeps the reference's
// semantics for eps_d ~ 0 (kernel.py:315,344-345).
template <bool MG = false>
__device__ __forceinline__ PairS1 pair_stage1(const Outer& o, double rn, double zn, long long gthr,
                                              const double2* __restrict__ logt) {
  PairS1 s;
  s.dr = o.ri - rn;
  s.dz = o.zi - zn;
  s.dz2 = s.dz * s.dz;
  const double dist2 = fma(s.dr, s.dr, s.dz2);
  const long long di = __double_as_longlong(dist2);
  const bool g = di >= gthr;  // d^2 >= eps^2 and d^2 > 0 (kernel.py:344)
  const double d2 = (MG ? g : di > kTinyBits) ? dist2 : 1.0;
  s.d2 = d2;
  // ri rn; 4 ri rn and 2 ri rn below are exact scalings of it, so P, m and
  // u round exactly as with (4 ri) rn and (2 ri) rn
  s.rr = o.ri4 * rn;  // 4 ri rn (exactly 4 (ri rn))
  s.P = s.rr + d2;
  const double isP = rsqrt_nr(s.P);
  s.invP = isP * isP;
  s.x = d2 * s.invP;
  // mask (kernel.py:344) applied once: with isP := 0 every B, hence every
  // tensor component of both orientations, is an exact (signed) zero
  s.isPm = g ? isP : 0.0;
  s.lr = log_reduce(s.x, logt, s.logc, s.kd);
  return s;
}

// Stage 2: ln x, K(m), E(m), then B1, B3, B4 and the differences c34, c35
// (each / 4; closed form or, for m < 0.01, the series).
__device__ __forceinline__ PairB pair_stage2(const Outer& o, double rn, double rcpr, const PairS1& s) {
  const double x = s.x, P = s.P, invP = s.invP;
  const double lx = log_finish(s.lr, s.logc, s.kd);


#if LB_ESTRIN
  // the reference's four degree-10 polynomials (kernel.py:351-359; QK[10] =
  // QEx[10] = QEx[0] = 0) in Estrin form: depth 4 instead of 10, sharing
  // x^2, x^4, x^8 -- same coefficients, re-associated evaluation
  const double x2 = x * x, x4 = x2 * x2, x8 = x4 * x4;
  const double pk = fma(fma(c_pk[10], x2, fma(c_pk[9], x, c_pk[8])), x8,
                        fma(fma(fma(c_pk[7], x, c_pk[6]), x2, fma(c_pk[5], x, c_pk[4])), x4,
                            fma(fma(c_pk[3], x, c_pk[2]), x2, fma(c_pk[1], x, c_pk[0]))));
  const double pe = fma(fma(c_pe[10], x2, fma(c_pe[9], x, c_pe[8])), x8,
                        fma(fma(fma(c_pe[7], x, c_pe[6]), x2, fma(c_pe[5], x, c_pe[4])), x4,
                            fma(fma(c_pe[3], x, c_pe[2]), x2, fma(c_pe[1], x, c_pe[0]))));
  const double qk = fma(fma(c_qk[9], x, c_qk[8]), x8,
                        fma(fma(fma(c_qk[7], x, c_qk[6]), x2, fma(c_qk[5], x, c_qk[4])), x4,
                            fma(fma(c_qk[3], x, c_qk[2]), x2, fma(c_qk[1], x, c_qk[0]))));
  const double qe = x * fma(c_qe[9], x8,
                            fma(fma(fma(c_qe[8], x, c_qe[7]), x2, fma(c_qe[6], x, c_qe[5])), x4,
                                fma(fma(c_qe[4], x, c_qe[3]), x2, fma(c_qe[2], x, c_qe[1]))));
#else
  // four Horner chains in x (kernel.py:351-359); QK[10] = QEx[10] = QEx[0] = 0
  double pk = fma(c_pk[10], x, c_pk[9]);
  double qk = c_qk[9];
  double pe = fma(c_pe[10], x, c_pe[9]);
  double qe = c_qe[9];
  pk = fma(pk, x, c_pk[8]);  qk = fma(qk, x, c_qk[8]);  pe = fma(pe, x, c_pe[8]);  qe = fma(qe, x, c_qe[8]);
  pk = fma(pk, x, c_pk[7]);  qk = fma(qk, x, c_qk[7]);  pe = fma(pe, x, c_pe[7]);  qe = fma(qe, x, c_qe[7]);
  pk = fma(pk, x, c_pk[6]);  qk = fma(qk, x, c_qk[6]);  pe = fma(pe, x, c_pe[6]);  qe = fma(qe, x, c_qe[6]);
  pk = fma(pk, x, c_pk[5]);  qk = fma(qk, x, c_qk[5]);  pe = fma(pe, x, c_pe[5]);  qe = fma(qe, x, c_qe[5]);
  pk = fma(pk, x, c_pk[4]);  qk = fma(qk, x, c_qk[4]);  pe = fma(pe, x, c_pe[4]);  qe = fma(qe, x, c_qe[4]);
  pk = fma(pk, x, c_pk[3]);  qk = fma(qk, x, c_qk[3]);  pe = fma(pe, x, c_pe[3]);  qe = fma(qe, x, c_qe[3]);
  pk = fma(pk, x, c_pk[2]);  qk = fma(qk, x, c_qk[2]);  pe = fma(pe, x, c_pe[2]);  qe = fma(qe, x, c_qe[2]);
  pk = fma(pk, x, c_pk[1]);  qk = fma(qk, x, c_qk[1]);  pe = fma(pe, x, c_pe[1]);  qe = fma(qe, x, c_qe[1]);
  pk = fma(pk, x, c_pk[0]);  qk = fma(qk, x, c_qk[0]);  pe = fma(pe, x, c_pe[0]);  qe = qe * x;
#endif
  const double EK = fma(-lx, qk, pk);
  const double EE = fma(-lx, qe, pe);
  const double isPm = s.isPm;
  PairB p;
  p.B1 = EK * isPm;
  // B3 = Em1 c3 = E (P/d^2) P^-3/2 = E P^-1/2 / d^2: one reciprocal of d^2
  // instead of 1/x and P^-3/2 (c3 is only needed by the rare series branch)
  p.B3 = EE * (isPm * rcp_nr(s.d2));
  // m < 0.01 (kernel.py:376) tested as x = 1 - m > 0.99 on the bit pattern;
  // m itself is only needed by the series
  if (__double_as_longlong(x) > kXSwitchBits) {
    // hypergeometric series (kernel.py:369-375)
    const double m = s.rr * invP;
    double s2 = c_s2[9], s3 = c_s3[9];
    s2 = fma(s2, m, c_s2[8]);  s3 = fma(s3, m, c_s3[8]);
    s2 = fma(s2, m, c_s2[7]);  s3 = fma(s3, m, c_s3[7]);
    s2 = fma(s2, m, c_s2[6]);  s3 = fma(s3, m, c_s3[6]);
    s2 = fma(s2, m, c_s2[5]);  s3 = fma(s3, m, c_s3[5]);
    s2 = fma(s2, m, c_s2[4]);  s3 = fma(s3, m, c_s3[4]);
    s2 = fma(s2, m, c_s2[3]);  s3 = fma(s3, m, c_s3[3]);
    s2 = fma(s2, m, c_s2[2]);  s3 = fma(s3, m, c_s3[2]);
    s2 = fma(s2, m, c_s2[1]);  s3 = fma(s3, m, c_s3[1]);
    const double S2 = s2 * m;
    const double S3 = fma(s3, m, c_s3[0]);
    const double c3 = isPm * invP;  // P^-3/2 (the 4 is folded into the coupling)
    p.B4 = S2 * c3;
    p.c34 = 0.5 * fma(-S2, c3, p.B3);   // (Em1 - S2) c3 / 2
    p.c35 = 0.25 * fma(-S3, c3, p.B3);  // (Em1 - S3) c3 / 4
  } else {
    // closed form (kernel.py:366-367) as the differences from Em1, in
    // 2/m = P/(2 ri rn) (m >= 0.01, so rn > 0):
    //   Em1 - S2 = (2/m)(K - E),  Em1 - S3 = (2/m)^2 ((1 + x) K - 2 E)
    // with c3 (2/m) = P^-1/2 / (2 ri rn); scaled: a = 1/(4 ri rn)
    const double a = o.rtri * rcpr;  // 1/(4 ri rn)
    const double cq = isPm * a;      // c3 (2/m) / 2
    p.c34 = cq * (EK - EE);
    p.c35 = (cq * (P * a)) * fma(x, EK, fma(-2.0, EE, EK));  // ((1 + x) K - 2 E) / 4
    p.B4 = fma(-2.0, p.c34, p.B3);
  }
  p.dz = s.dz;
  p.dz2 = s.dz2;
  p.dr = s.dr;
  p.rr = s.rr;
  return p;
}

// The symmetric part of one pair (stage 1 + stage 2).
__device__ __forceinline__ PairB pair_core(const Outer& o, double rn, double zn, double rcpr,
                                           long long gthr, const double2* __restrict__ logt) {
  return pair_stage2(o, rn, rcpr, pair_stage1(o, rn, zn, gthr, logt));
}

// Direct-pair tensor components from the symmetric part (kernel.py:384-389
// rearranged, see the header): w2 = B1 - dr^2 B3 - 2 ri rn c34 is shared by
// UD_xx of both orientations.
__device__ __forceinline__ double pair_w2(const PairB& p) {
  return fma(-p.rr, p.c34, fma(-(p.dr * p.dr), p.B3, p.B1));  // 2 ri rn c34 = rq c34'

}
#ifndef LB_SHARED_U
#define LB_SHARED_U 1  // UD_xz and UK_zr share rn c34 (one FP64 operation fewer per pair)
#endif
// rnx = 2 rn, rn2 = 4 rn^2 (the record's scaled fields)
__device__ __forceinline__ T5 pair_tensors(double rnx, double rn2, const PairB& p, double w2) {
  T5 t;
  t.xx = fma(rn2, p.c35, w2);
  t.zz = fma(-p.dz2, p.B3, p.B1);
#if LB_SHARED_U
  const double u = rnx * p.c34;  // rn c34
  t.xz = -p.dz * fma(p.dr, p.B3, u);
  t.zr = p.dz * fma(-p.dr, p.B4, u);
#else
  t.xz = -p.dz * fma(p.dr, p.B3, rnx * p.c34);
  t.zr = p.dz * fma(rnx, p.c34, -(p.dr * p.B4));
#endif
  t.kr = fma(p.rr, p.c35, p.dz2 * p.B4);
  return t;  // masked pairs: all B and c are zero (pair_core), so is every component
}

// One (outer, inner) pair: the five tensor components / 4.
__device__ __forceinline__ T5 pair_tensor(const Outer& o, double rn, double zn, double rn2,
                                          double rcpr, long long gthr,
                                          const double2* __restrict__ logt) {
  const PairB p = pair_core(o, rn, zn, rcpr, gthr, logt);
  return pair_tensors(rn + rn, rn2, p, pair_w2(p));  // rn2: the record's 4 rn^2
}

// One unordered pair: the direct components in `t` and, returned, the one
// new component of the swapped pair, UD_xx(j,i) / 4 = (B1 - dr^2 B3 -
// 2 ri rn c34 + ri^2 c35) / 4; the others are permutations of `t`.
__device__ __forceinline__ double pair_tensor_sym(const Outer& o, double rn, double zn, double rn2,
                                                  double rcpr, long long gthr,
                                                  const double2* __restrict__ logt, T5& t) {
  const PairB p = pair_core(o, rn, zn, rcpr, gthr, logt);
  const double w2 = pair_w2(p);
  t = pair_tensors(rn + rn, rn2, p, w2);  // rn2: the record's 4 rn^2
  return fma(o.ri2, p.c35, w2);
}

// U unordered pairs (outer point oo[u], inner point u) evaluated in lockstep:
// the same arithmetic as pair_tensor_sym, interleaved so every polynomial
// coefficient is loaded once for U fused multiply-adds and the U dependency
// chains overlap.  The closed form for S2/S3 is evaluated for every pair and
// replaced by the series where m < 0.01 (kernel.py:366-378 likewise computes
// both and selects).  `nser` counts the calls that took the series branch
// (the benchmark's executed-instruction count; callers may ignore it).
template <int U, bool MG = false>
__device__ __forceinline__ void pair_tensor_sym_x(const Outer (&oo)[U], const double (&rn)[U],
                                                  const double (&zn)[U], const double (&rn2)[U],
                                                  const double (&rnx)[U],
                                                  const double (&rcpr)[U], long long gthr,
                                                  const double2* __restrict__ logt, T5 (&t)[U],
                                                  double (&txx2)[U], unsigned& nser) {
  PairS1 s[U];
  double lx[U], x[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    s[u] = pair_stage1<MG>(oo[u], rn[u], zn[u], gthr, logt);
    x[u] = s[u].x;
  }
#pragma unroll
  for (int u = 0; u < U; ++u) lx[u] = log_finish(s[u].lr, s[u].logc, s[u].kd);
  // four Horner chains in x per pair (kernel.py:351-359); QK[10] = QEx[10] = QEx[0] = 0
  double pk[U], qk[U], pe[U], qe[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    pk[u] = fma(c_pk[10], x[u], c_pk[9]);
    qk[u] = c_qk[9];
    pe[u] = fma(c_pe[10], x[u], c_pe[9]);
    qe[u] = c_qe[9];
  }
#pragma unroll
  for (int k = 8; k >= 1; --k) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      pk[u] = fma(pk[u], x[u], c_pk[k]);
      qk[u] = fma(qk[u], x[u], c_qk[k]);
      pe[u] = fma(pe[u], x[u], c_pe[k]);
      qe[u] = fma(qe[u], x[u], c_qe[k]);
    }
  }
  PairB p[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    pk[u] = fma(pk[u], x[u], c_pk[0]);
    qk[u] = fma(qk[u], x[u], c_qk[0]);
    pe[u] = fma(pe[u], x[u], c_pe[0]);
    qe[u] = qe[u] * x[u];
    const double EK = fma(-lx[u], qk[u], pk[u]);
    const double EE = fma(-lx[u], qe[u], pe[u]);
    const double isPm = s[u].isPm;
    p[u].B1 = EK * isPm;
    p[u].B3 = EE * (isPm * rcp_nr(s[u].d2));  // E P^-1/2 / d^2 = Em1 c3
    // closed form (kernel.py:366-367) as the differences from Em1 (header):
    // Em1 - S2 = (2/m)(K - E), Em1 - S3 = (2/m)^2 ((1 + x) K - 2 E);
    // c3 (2/m) = P^-1/2 / (2 ri rn); scaled (header): a = 1/(4 ri rn), c34 / 2, c35 / 4
    const double a = oo[u].rtri * rcpr[u];  // 1/(4 ri rn)
    const double cq = isPm * a;
    p[u].c34 = cq * (EK - EE);
    p[u].c35 = (cq * (s[u].P * a)) * fma(x[u], EK, fma(-2.0, EE, EK));  // ((1 + x) K - 2 E) / 4
    p[u].B4 = fma(-2.0, p[u].c34, p[u].B3);
    p[u].dz = s[u].dz;
    p[u].dz2 = s[u].dz2;
    p[u].dr = s[u].dr;
    p[u].rr = s[u].rr;
  }
#if LB_SERIES_MODE == 0
#pragma unroll
  for (int u = 0; u < U; ++u) {
    // m < 0.01 (kernel.py:376), tested as x = 1 - m > 0.99 on the bit pattern
    if (__double_as_longlong(x[u]) > kXSwitchBits) {
      ++nser;
      const double m = s[u].rr * s[u].invP;
      double s2 = c_s2[9], s3 = c_s3[9];
#pragma unroll
      for (int k = 8; k >= 1; --k) {
        s2 = fma(s2, m, c_s2[k]);
        s3 = fma(s3, m, c_s3[k]);
      }
      const double c3 = s[u].isPm * s[u].invP;
      const double S2 = s2 * m, S3 = fma(s3, m, c_s3[0]);
      p[u].B4 = S2 * c3;
      p[u].c34 = 0.5 * fma(-S2, c3, p[u].B3);   // (Em1 - S2) c3 / 2
      p[u].c35 = 0.25 * fma(-S3, c3, p[u].B3);  // (Em1 - S3) c3 / 4
    }
  }
#else
  // one branch for the U pairs: the series (rare: m < 0.01 needs a point
  // near the axis) runs for all U in lockstep and is selected per pair
  bool ser[U], any = false;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    ser[u] = __double_as_longlong(x[u]) > kXSwitchBits;  // m < 0.01 (kernel.py:376)
    any |= ser[u];
  }
  if (any) {
    ++nser;
    double m[U], s2[U], s3[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      m[u] = s[u].rr * s[u].invP;
      s2[u] = c_s2[9];
      s3[u] = c_s3[9];
    }
#pragma unroll
    for (int k = 8; k >= 1; --k)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        s2[u] = fma(s2[u], m[u], c_s2[k]);
        s3[u] = fma(s3[u], m[u], c_s3[k]);
      }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double c3 = s[u].isPm * s[u].invP;
      const double S2 = s2[u] * m[u], S3 = fma(s3[u], m[u], c_s3[0]);
      const double b4 = S2 * c3, d34 = 0.5 * fma(-S2, c3, p[u].B3),
                   d35 = 0.25 * fma(-S3, c3, p[u].B3);  // (Em1 - S2) c3 / 2, (Em1 - S3) c3 / 4
      p[u].B4 = ser[u] ? b4 : p[u].B4;
      p[u].c34 = ser[u] ? d34 : p[u].c34;
      p[u].c35 = ser[u] ? d35 : p[u].c35;
    }
  }
#endif
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const double w2 = pair_w2(p[u]);
    t[u] = pair_tensors(rnx[u], rn2[u], p[u], w2);
    txx2[u] = fma(oo[u].ri2, p[u].c35, w2);
  }
}

}  // namespace lb
