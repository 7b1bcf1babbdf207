/*
 * landau_oracle.h -- CPU restatement of the reference algorithm for the
 * Landau pair-integration path.  TEST INFRASTRUCTURE ONLY: used by tests/,
 * __graft_entry__.smoke() and bench.py's CPU-baseline / reference arm as the
 * checker and the CPU timing; never by the product path.
 *
 * Follows pkg/src/axlandau/kernel.py of the reference:
 *   orc_elliptic_ke   kernel.py:93-128  (elliptic_KE / _elliptic_scalar)
 *   orc_tensor_pair   kernel.py:179-235 (_base_integrals / axisym_tensor_pair)
 *   orc_lanes         kernel.py:306-389 (_lanes, blocked lane passes)
 *   orc_sweep         kernel.py:392-493 (_accumulate_block, _combine,
 *                                        _sweep_serial / _sweep_parallel)
 */
#ifndef LANDAU_ORACLE_H
#define LANDAU_ORACLE_H
#ifdef __cplusplus
extern "C" {
#endif

int orc_version(void);
int orc_max_threads(void);

void orc_elliptic_ke(int n, const double *m, double *K, double *E);

/* returns 0, or -1 for r < 0 / rbar < 0, -2 for coincident points */
int orc_tensor_pair(double r, double z, double rbar, double zbar, double *UK, double *UD);

void orc_lanes(double ri, double zi, const double *r, const double *z, int n0, int nb,
               double eps2, double *txx, double *tzz, double *txz, double *tkr, double *tzr,
               double *xb, double *lb);

/* K (nout,S,2), D (nout,S,2,2); coK/coD (S,S) from _coupling; eps2 = eps_d^2;
 * blk = lane block (256 in the reference); nthreads <= 0 -> all cores. */
void orc_sweep(int nout, const double *ro, const double *zo, int n, int S, const double *r,
               const double *z, const double *w, const double *f, const double *dfr,
               const double *dfz, const double *coK, const double *coD, double eps2, int blk,
               double *K, double *D, int nthreads);

#ifdef __cplusplus
}
#endif
#endif
