"""High-precision D/K of selected outer points (golden generation only; run
in the build container by make_golden.py).

The reference's own arithmetic (kernel.py:306-440: its frozen K/E fits, the
m < 0.01 series, the closed forms of S2/S3, B1..B5, the five tensor
components, _accumulate_block and _combine) evaluated in mpmath at 40
digits for the inner points within `rnear` of the outer point -- the pairs
whose tensors cancel O(r^2/d^2) terms -- plus the oracle's double-precision
sweep (oracle/, pinned to the reference) for the well-conditioned rest.
This is the value the reference's formulas give in exact arithmetic: the
yardstick for outer points that own the closest pairs, where two
double-precision implementations legitimately differ by ~1e-10
(DESIGN.md section 4).
"""

from __future__ import annotations

import mpmath as mp
import numpy as np

mp.mp.dps = 40


def _tables():
    from axlandau import kernel as K_

    cv = lambda t: [mp.mpf(float(c)) for c in t]  # noqa: E731
    return cv(K_._PK), cv(K_._QK), cv(K_._PE), cv(K_._QEx), cv(K_._S2C), cv(K_._S3C)


def _poly(c, x):
    acc = mp.mpf(0)
    for t in reversed(c):
        acc = acc * x + t
    return acc


def pair_hp(ri, zi, rn, zn, tab):
    """(UK_rr, UK_zr, UD_xx, UD_xz, UD_zz) at 40 digits (kernel.py:306-389)."""
    PK, QK, PE, QE, S2C, S3C = tab
    ri, zi, rn, zn = (mp.mpf(float(v)) for v in (ri, zi, rn, zn))
    dz = zi - zn
    d2 = (ri - rn) ** 2 + dz * dz
    P = d2 + 4 * ri * rn
    x = d2 / P
    m = 4 * ri * rn / P
    lx = mp.log(x)
    Kk = _poly(PK, x) - lx * _poly(QK, x)
    Ee = _poly(PE, x) - lx * _poly(QE, x)
    Em1 = Ee * P / d2
    if m >= mp.mpf("0.01"):
        S2 = 2 * (Em1 - Kk) / m - Em1
        S3 = 4 * (Em1 + Ee - 2 * Kk) / m ** 2 - 4 * (Em1 - Kk) / m + Em1
    else:
        S2 = _poly(S2C, m)
        S3 = _poly(S3C, m)
    isP = 1 / mp.sqrt(P)
    c3 = 4 * isP / P
    B1, B3, B4, B5 = 4 * Kk * isP, Em1 * c3, S2 * c3, S3 * c3
    return (dz * dz * B4 + ri * rn * (B3 - B5), dz * (rn * B3 - ri * B4),
            B1 - ri * ri * B3 + 2 * ri * rn * B4 - rn * rn * B5, -dz * (ri * B3 - rn * B4),
            B1 - dz * dz * B3)


def hp_kd(points, r, z, w, f, dfr, dfz, nu_hat, mass_ratio_o, eps_d, rnear, oracle):
    """K (len, S, 2), D (len, S, 2, 2) of the outer points `points` (indices
    into the inner set) against all inner points."""
    tab = _tables()
    S = f.shape[0]
    coK, coD = oracle.coupling(nu_hat, mass_ratio_o)
    Ks, Ds = [], []
    for p in points:
        d2 = (r - r[p]) ** 2 + (z - z[p]) ** 2
        near = np.nonzero(d2 < rnear * rnear)[0]
        far = np.nonzero(d2 >= rnear * rnear)[0]
        A = [[mp.mpf(0)] * 5 for _ in range(S)]
        for j in near:
            if d2[j] == 0.0 or d2[j] < eps_d * eps_d:  # the mask (kernel.py:344)
                continue
            tkr, tzr, txx, txz, tzz = pair_hp(r[p], z[p], r[j], z[j], tab)
            wj = mp.mpf(float(w[j]))
            for b in range(S):
                gr = mp.mpf(float(dfr[b, j])) * wj
                gz = mp.mpf(float(dfz[b, j])) * wj
                fw = mp.mpf(float(f[b, j])) * wj
                A[b][0] += tkr * gr + txz * gz
                A[b][1] += tzr * gr + tzz * gz
                A[b][2] += fw * txx
                A[b][3] += fw * txz
                A[b][4] += fw * tzz
        Kf, Df = oracle.fused_sweep(r[p:p + 1], z[p:p + 1], r[far], z[far], w[far],
                                    np.ascontiguousarray(f[:, far]), np.ascontiguousarray(dfr[:, far]),
                                    np.ascontiguousarray(dfz[:, far]), nu_hat, mass_ratio_o,
                                    eps_d=eps_d)
        K = np.zeros((S, 2))
        D = np.zeros((S, 2, 2))
        for a in range(S):
            for c in range(2):
                K[a, c] = float(sum(mp.mpf(float(coK[a, b])) * A[b][c] for b in range(S))
                                + mp.mpf(float(Kf[0, a, c])))
            for (c, d), q in (((0, 0), 2), ((0, 1), 3), ((1, 1), 4)):
                D[a, c, d] = float(sum(mp.mpf(float(coD[a, b])) * A[b][q] for b in range(S))
                                   + mp.mpf(float(Df[0, a, c, d])))
            D[a, 1, 0] = D[a, 0, 1]
        Ks.append(K)
        Ds.append(D)
    return np.array(Ks), np.array(Ds)
