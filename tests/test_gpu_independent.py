"""The device pair arithmetic against INDEPENDENT oracles (no polynomial
fits, no series, no reduction identities), mirroring the reference's own
independent checks (test_kernel.py:39-46, 94-146; the reference's oracles
are tests/_oracles.py): the arithmetic-geometric mean for K(m), E(m), and a
periodic trapezoid rule for the azimuthal integrals of the 3V Landau tensor.
The oracles below are written from the textbook definitions."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def agm_elliptic(m: float):
    """K(m) = pi / (2 M(1, sqrt(1-m))); E(m) = K (1 - sum_k 2^(k-1) c_k^2),
    c_0 = sqrt(m), c_{k+1} = (a_k - b_k)/2 (Gauss / Legendre)."""
    a, b = 1.0, math.sqrt(1.0 - m)
    acc, w = 0.5 * m, 0.5
    for _ in range(60):
        c = 0.5 * (a - b)
        if abs(c) <= 2e-16 * a:
            break
        a, b = 0.5 * (a + b), math.sqrt(a * b)
        w *= 2.0
        acc += w * c * c
    K = math.pi / (2.0 * a)
    return K, K * (1.0 - acc)


def azimuthal_tensors(r, z, rb, zb, rtol=1e-13):
    """UK, UD (2x2 in (r, z)) of the pair by the periodic trapezoid rule over
    the inner point's azimuth phi, with grid doubling to convergence.  With
    v = (r, 0, z), vb = (rb cos phi, rb sin phi, zb), d = v - vb and
    U = (|d|^2 I - d d^T)/|d|^3:  UD_ab = int U_ab,  UK_a1 = int U_a . e_r(phi),
    UK_a2 = int U_az, for a, b in {x, z}."""

    def integrals(n):
        phi = 2.0 * np.pi * np.arange(n) / n
        c, s = np.cos(phi), np.sin(phi)
        d = np.stack([r - rb * c, -rb * s, np.full(n, z - zb)], axis=1)  # (n, 3)
        n2 = np.einsum("ij,ij->i", d, d)
        U = (n2[:, None, None] * np.eye(3) - d[:, :, None] * d[:, None, :]) / n2[:, None, None] ** 1.5
        er = np.stack([c, s, np.zeros(n)], axis=1)
        rows = [0, 2]  # x, z
        UD = U[:, rows][:, :, rows].mean(axis=0) * 2.0 * np.pi
        Ur = np.einsum("iab,ib->ia", U, er)[:, rows].mean(axis=0) * 2.0 * np.pi
        UK = np.stack([Ur, UD[:, 1]], axis=1)
        return UK, UD

    n = 128
    UK, UD = integrals(n)
    while n < (1 << 22):
        n *= 2
        UK2, UD2 = integrals(n)
        scale = max(np.abs(UK2).max(), np.abs(UD2).max())
        done = max(np.abs(UK2 - UK).max(), np.abs(UD2 - UD).max()) <= rtol * scale
        UK, UD = UK2, UD2
        if done:
            return UK, UD
    raise RuntimeError("trapezoid rule did not converge")


def test_elliptic_against_agm(gpu):
    """test_kernel.py:39-46: 500 samples including m -> 1 - 1e-12, rel 1e-10."""
    rng = np.random.default_rng(4046)
    m = np.concatenate([rng.random(496), [0.0, 0.5, 1.0 - 1e-6, 1.0 - 1e-12]])
    K, E = gpu.elliptic_KE(m)
    ref = np.array([agm_elliptic(x) for x in m])
    assert np.max(np.abs(K - ref[:, 0]) / ref[:, 0]) < 1e-10
    assert np.max(np.abs(E - ref[:, 1]) / ref[:, 1]) < 1e-10


def test_pairs_against_azimuthal_quadrature(gpu):
    """test_kernel.py:94-108: 60 pairs with separation >= 0.1, rel 1e-8."""
    rng = np.random.default_rng(9408)
    P = []
    while len(P) < 60:
        r, rb = rng.uniform(0.01, 2.0, 2)
        z, zb = rng.uniform(-2.0, 2.0, 2)
        if (r - rb) ** 2 + (z - zb) ** 2 >= 0.1**2:
            P.append((r, z, rb, zb))
    P = np.array(P)
    UK, UD = gpu.axisym_tensor_pairs(P[:, 0], P[:, 1], P[:, 2], P[:, 3])
    worst = 0.0
    for k, (r, z, rb, zb) in enumerate(P):
        UKq, UDq = azimuthal_tensors(r, z, rb, zb)
        scale = max(np.abs(UKq).max(), np.abs(UDq).max())
        worst = max(worst, max(np.abs(UK[k] - UKq).max(), np.abs(UD[k] - UDq).max()) / scale)
    print("device tensors vs azimuthal quadrature", worst)
    assert worst < 1e-8


def test_pair_symmetries(gpu):
    """test_kernel.py:111-124: UD symmetric, UK's z-column = UD's z-column,
    mirror symmetry z -> -z (200 pairs)."""
    rng = np.random.default_rng(11124)
    r, rb = rng.uniform(0.05, 2.0, (2, 200))
    z, zb = rng.uniform(-2.0, 2.0, (2, 200))
    keep = (r - rb) ** 2 + (z - zb) ** 2 >= 1e-4
    r, rb, z, zb = r[keep], rb[keep], z[keep], zb[keep]
    UK, UD = gpu.axisym_tensor_pairs(r, z, rb, zb)
    UKm, UDm = gpu.axisym_tensor_pairs(r, -z, rb, -zb)
    assert np.array_equal(UD[:, 0, 1], UD[:, 1, 0])
    assert np.allclose(UK[:, :, 1], UD[:, :, 1], rtol=1e-13)
    flip = np.diag([1.0, -1.0])
    assert np.allclose(UDm, flip @ UD @ flip, rtol=1e-12, atol=1e-13)


def test_series_switch_continuity(gpu):
    """test_kernel.py:127-137: pairs either side of m = 0.01 agree."""
    r = rb = 0.05
    dz = math.sqrt(4 * r * rb * (1 - 0.01) / 0.01)
    lo = gpu.axisym_tensor_pair(r, 0.0, rb, dz * (1 + 1e-6))
    hi = gpu.axisym_tensor_pair(r, 0.0, rb, dz * (1 - 1e-6))
    scale = np.abs(lo.UD).max()
    assert np.abs(lo.UD - hi.UD).max() / scale < 1e-5
    assert np.abs(lo.UK - hi.UK).max() / scale < 1e-5


def test_on_axis_inner_point_against_quadrature(gpu):
    """test_kernel.py:140-146: rbar = 0 (m = 0, pure series) vs quadrature."""
    t = gpu.axisym_tensor_pair(0.5, 0.3, 0.0, -0.2)
    assert np.all(np.isfinite(t.UK)) and np.all(np.isfinite(t.UD))
    UKq, UDq = azimuthal_tensors(0.5, 0.3, 1e-9, -0.2)
    assert np.abs(t.UD - UDq).max() / np.abs(UDq).max() < 1e-7
