"""Parity of the sm_100a pair sweep (through the C ABI) with the reference
goldens and the CPU oracle.  Bar: per species / component scaled error
max|dX|/max|X_ref| <= 1e-10 (BASELINE.json north_star); measured values are
printed (-s) and sit near 1e-14."""

import numpy as np
import pytest

from conftest import data_from, golden, params_from, scaled, worst_component

pytestmark = pytest.mark.gpu

TOL = 1e-10


def _rel_pairs(UK, UD, UKr, UDr):
    s = np.maximum(np.abs(UKr).reshape(len(UKr), -1).max(1), np.abs(UDr).reshape(len(UDr), -1).max(1))
    e = np.maximum(np.abs(UK - UKr).reshape(len(UK), -1).max(1), np.abs(UD - UDr).reshape(len(UD), -1).max(1))
    return e / s


def test_tensor_pairs_match_reference(gpu):
    g = golden("pairs")
    P = g["pairs"]
    UK, UD = gpu.axisym_tensor_pairs(P[:, 0], P[:, 1], P[:, 2], P[:, 3])
    err = _rel_pairs(UK, UD, g["UK"], g["UD"])
    # Conditioning of the closed form (both implementations round differently):
    #  * UD_xx / UK_rr cancel terms of size (r/|d|)^2 for near-coincident pairs;
    #  * S3 = 4(Em1+E-2K)/m^2 - ... cancels O(1) terms to O(m^2) just above the
    #    series switch m = 0.01, amplifying rounding by ~1/m^2 (kernel.py:366-367).
    d2 = (P[:, 0] - P[:, 2]) ** 2 + (P[:, 1] - P[:, 3]) ** 2
    m = 4 * P[:, 0] * P[:, 2] / (d2 + 4 * P[:, 0] * P[:, 2])
    with np.errstate(divide="ignore"):
        amp = 1.0 + np.maximum(P[:, 0], P[:, 2]) ** 2 / d2 + np.where(m >= 0.01, 1.0 / m**2, 0.0)
    tol = 64 * np.finfo(float).eps * amp
    benign = amp < 10
    print("pairs worst (benign)", err[benign].max(), "worst err/tol", (err / tol).max())
    assert err[benign].max() < 1e-13
    assert np.all(err <= tol)


def test_pairs_against_exact_arithmetic(gpu):
    """The 1000 pairs against the reference's formulas in 40-digit arithmetic
    (tests/golden/pairs_hp.npz): the device's cancellation-free tensor forms
    (landau_pair.cuh) are accurate to ~1e-15 of each pair's scale even for
    near-coincident pairs, where the reference's own double-precision result
    is off by up to 1 % (UD_xx / UK_rr cancel O(r^2/d^2) terms at d = 1e-7);
    the only amplification left is the closed form's 1/m^2 just above the
    series switch m = 0.01, which the reference shares (kernel.py:366-367)."""
    g, h = golden("pairs"), golden("pairs_hp")
    P = g["pairs"]
    UK, UD = gpu.axisym_tensor_pairs(P[:, 0], P[:, 1], P[:, 2], P[:, 3])
    err = _rel_pairs(UK, UD, h["UK"], h["UD"])
    ref_err = _rel_pairs(g["UK"], g["UD"], h["UK"], h["UD"])
    d2 = (P[:, 0] - P[:, 2]) ** 2 + (P[:, 1] - P[:, 3]) ** 2
    m = 4 * P[:, 0] * P[:, 2] / (d2 + 4 * P[:, 0] * P[:, 2])
    with np.errstate(divide="ignore"):
        tol = 64 * np.finfo(float).eps * (1.0 + np.where(m >= 0.01, 1.0 / m**2, 0.0))
    print("pairs vs 40-digit: device worst", err.max(), "worst err/tol", (err / tol).max(),
          "| reference worst", ref_err.max())
    assert np.all(err <= tol)


def test_elliptic_KE_device(gpu):
    """elliptic_KE (kernel.py:93-113, test_kernel.py:30-46): known values,
    the reference's own outputs on the 1000-pair fixture to 1e-15 relative
    (table log and fused Horner vs numpy), scalar/array forms."""
    K, E = gpu.elliptic_KE(0.5)
    assert isinstance(K, float)
    assert abs(K - 1.854074677301369) <= 1e-14 * K and abs(E - 1.350643881047669) <= 1e-14 * E
    K0, E0 = gpu.elliptic_KE(0.0)
    # the fits reproduce pi/2 at m = 0 to their accuracy (rtol 1e-14, test_kernel.py:30-36)
    assert abs(K0 - np.pi / 2) <= 1e-14 * np.pi / 2 and abs(E0 - np.pi / 2) <= 1e-14 * np.pi / 2
    g = golden("pairs")
    K, E = gpu.elliptic_KE(g["m"])
    assert K.shape == g["m"].shape
    assert np.max(np.abs(K - g["K"]) / np.abs(g["K"])) <= 1e-15
    assert np.max(np.abs(E - g["E"]) / np.abs(g["E"])) <= 1e-15


def test_tensor_pair_structure(gpu):
    g = golden("pairs")
    P = g["pairs"][:600]
    UK, UD = gpu.axisym_tensor_pairs(P[:, 0], P[:, 1], P[:, 2], P[:, 3])
    assert np.array_equal(UD[:, 0, 1], UD[:, 1, 0])            # UD symmetric
    assert np.array_equal(UK[:, :, 1], UD[:, :, 1])            # UK z-column == UD z-column
    t = gpu.axisym_tensor_pair(0.5, 0.3, 0.0, -0.2)            # on-axis inner point
    assert np.all(np.isfinite(t.UK)) and np.all(np.isfinite(t.UD))


def test_sweep_small_all_outer(gpu):
    g = golden("sweep_small")
    K, D = gpu.fused_sweep(g["r"], g["z"], data_from(g), params_from(g))
    err = worst_component(K, D, g["K"], g["D"])
    print("sweep_small", err)
    assert err < TOL
    assert np.array_equal(D[..., 0, 1], D[..., 1, 0])


def test_proximity_mask(gpu):
    g = golden("sweep_small")
    data = data_from(g, "1")
    params = params_from(g, "nu1", "mro1")
    ro, zo = np.array([g["prox_outer"][0]]), np.array([g["prox_outer"][1]])
    Kw, Dw = gpu.fused_sweep(ro, zo, data, params)
    Km, Dm = gpu.fused_sweep(ro, zo, data, params, eps_d=1e-6)
    assert scaled(Km, g["K_masked"]) < TOL and scaled(Dm, g["D_masked"]) < TOL
    # with the partner 1e-9 away, UK_rr = dz^2 B4 + ri rn (B3 - B5) and UD_xx
    # cancel terms of size ~1/d^2 = 1e18: that pair's contribution is rounding
    # noise in any implementation; the reference test only asks for finite
    # values that differ from the masked sums (test_kernel.py:223-231).
    assert np.all(np.isfinite(Kw)) and np.all(np.isfinite(Dw))
    assert not np.allclose(Kw, Km, rtol=1e-8)


def test_fused_inner_loop_single_point(gpu):
    g = golden("sweep_small")
    data, params = data_from(g, "1"), params_from(g, "nu1", "mro1")
    acc = gpu.fused_inner_loop((data.r[5], data.z[5], data.w[5]), data, params)
    K, D = gpu.fused_sweep(data.r[5:6], data.z[5:6], data, params)
    assert np.array_equal(acc.K, K[0]) and np.array_equal(acc.D, D[0])


@pytest.mark.parametrize("case", ["cfg1", "cfg2", "hanging", "cfg3"])
def test_mesh_sweeps(gpu, case):
    g = golden(case)
    eps = float(g["eps_d"]) if "eps_d" in g else 1e-14 * float(g["mesh_L"])
    if "idx" in g:  # subset fixtures: compare the all-points (symmetric) rows
        K, D = gpu.fused_sweep(g["r"], g["z"], data_from(g), params_from(g), eps_d=eps)
        K, D = K[g["idx"]], D[g["idx"]]
    else:
        K, D = gpu.fused_sweep(g["r"], g["z"], data_from(g), params_from(g), eps_d=eps)
    err = worst_component(K, D, g["K"], g["D"])
    print(case, err)
    assert err < TOL


def test_cfg3_q3_point_set(gpu):
    """BASELINE config 3 as worded: Q3 elements / 4x4 Gauss points on the
    refined mesh (950 cells, N = 15,200, two species, bi-Maxwellian
    electrons).  The all-points device call on the committed point set vs
    the reference's fused_sweep (2048 points + the 64 closest-pair owners).
    The Q3 element contraction has no reference (parity unpinned, not built)."""
    from paper_1702_08880_b200 import QuadPointData, synthetic

    g = golden("cfg3q3")
    r, z, w = synthetic.q3_points(g["origins"], g["sizes"])
    idx = g["idx"]
    assert np.array_equal(r[idx], g["r_idx"]) and np.array_equal(w[idx], g["w_idx"])
    f, dfr, dfz, nu, mro = synthetic.cfg3_state_values(r, z)
    data = QuadPointData(N=r.size, r=r, z=z, w=w, f=f, df_r=dfr, df_z=dfz)
    K, D = gpu.fused_sweep(r, z, data, params_from(g), eps_d=float(g["eps_d"]))
    err = worst_component(K[idx], D[idx], g["K"], g["D"])
    print("cfg3 Q3 / 4x4 point set (N=%d)" % r.size, err)
    assert err < TOL


def test_four_species(gpu):
    g = golden("cfg4s")
    idx = g["idx"]
    K, D = gpu.fused_sweep(g["r"][idx], g["z"][idx], data_from(g), params_from(g),
                           eps_d=float(g["eps_d"]))
    err = worst_component(K, D, g["K"], g["D"])
    print("cfg4 species S=4", err)
    assert err < TOL


def _cfg5(N):
    from paper_1702_08880_b200 import synthetic

    wl = synthetic.cfg5(N)
    data = pytest.importorskip("paper_1702_08880_b200").QuadPointData(
        N=N, r=wl.r, z=wl.z, w=wl.w, f=wl.f, df_r=wl.df_r, df_z=wl.df_z)
    params = pytest.importorskip("paper_1702_08880_b200").CollisionParams(
        nu_hat=wl.nu_hat, mass_ratio_o=wl.mass_ratio_o)
    return wl, data, params


def test_cfg5_4096_full(gpu):
    g = golden("cfg5_4096")
    wl, data, params = _cfg5(4096)
    assert wl.checksum() == float(g["checksum"])
    K, D = gpu.fused_sweep(wl.r, wl.z, data, params, eps_d=wl.eps_d)
    err = worst_component(K, D, g["K"], g["D"])
    print("cfg5 N=4096", err)
    assert err < TOL


def test_cfg5_headline_subset_with_closest_pairs(gpu):
    """N = 2^16, the benchmarked configuration: the all-points call (the
    symmetric, species-collapsed path bench.py times) indexed at 192 evenly
    spaced points + the 64 closest-pair owners, against the reference's
    fused_sweep rows; the general (ordered-pair) path on the same outer
    subset as well."""
    g = golden("cfg5_65536")
    wl, data, params = _cfg5(65536)
    assert wl.checksum() == float(g["checksum"])
    idx = g["idx"]
    K, D = gpu.fused_sweep(wl.r, wl.z, data, params, eps_d=wl.eps_d)
    err = worst_component(K[idx], D[idx], g["K"], g["D"])
    Kg, Dg = gpu.fused_sweep(wl.r[idx], wl.z[idx], data, params, eps_d=wl.eps_d)
    err_g = worst_component(Kg, Dg, g["K"], g["D"])
    print("cfg5 N=65536 subset: symmetric (benchmarked) path", err, "general path", err_g)
    assert err < TOL and err_g < TOL


def test_cfg5_headline_full_properties(gpu):
    """Full N = 2^16 all-points evaluation (symmetric path): run-to-run
    determinism (bitwise), finiteness, agreement with the general path on
    outer subsets; general-path outer-split invariance (bitwise)."""
    wl, data, params = _cfg5(65536)
    K, D = gpu.fused_sweep(wl.r, wl.z, data, params, eps_d=wl.eps_d)
    assert np.all(np.isfinite(K)) and np.all(np.isfinite(D))
    K2, D2 = gpu.fused_sweep(wl.r, wl.z, data, params, eps_d=wl.eps_d)
    assert np.array_equal(K, K2) and np.array_equal(D, D2)
    Kw, Dw = gpu.fused_sweep(wl.r[:16384], wl.z[:16384], data, params, eps_d=wl.eps_d)
    err = worst_component(K[:16384], D[:16384], Kw, Dw)
    print("cfg5 N=65536 symmetric vs general", err)
    assert err < 1e-12
    for lo, hi in ((0, 8192), (8192 + 17, 8192 * 2 - 5)):
        Ks, Ds = gpu.fused_sweep(wl.r[lo:hi], wl.z[lo:hi], data, params, eps_d=wl.eps_d)
        assert np.array_equal(Ks, Kw[lo:hi]) and np.array_equal(Ds, Dw[lo:hi])


def test_cfg5_max_size(gpu, oracle):
    """BASELINE config 5 at its largest size, N = 2^20 (1.1e12 ordered pairs,
    scratch-bounded row batches on the symmetric path): finite, D symmetric;
    32 evenly spaced outer points agree with the oracle to 1e-10, and the 16
    owners of the globally closest pairs agree to 1e-10 with the reference's
    formulas evaluated in 40-digit arithmetic (tests/golden/hp_sweep.py) --
    there the reference's own double-precision arithmetic (the oracle) is
    2.1e-10 off, the cancellation of its O(r^2/d^2) tensor terms (DESIGN.md
    section 4)."""
    N = 1 << 20
    wl, data, params = _cfg5(N)
    hp = golden("cfg5hp")
    assert wl.checksum() == float(hp["checksum"])
    K, D = gpu.fused_sweep(wl.r, wl.z, data, params, eps_d=wl.eps_d)
    assert np.all(np.isfinite(K)) and np.all(np.isfinite(D))
    assert np.array_equal(D[..., 0, 1], D[..., 1, 0])
    idx = np.linspace(0, N - 1, 32).astype(np.int64)
    Kr, Dr = oracle.fused_sweep(wl.r[idx], wl.z[idx], wl.r, wl.z, wl.w, wl.f, wl.df_r, wl.df_z,
                                wl.nu_hat, wl.mass_ratio_o, eps_d=wl.eps_d)
    err = worst_component(K[idx], D[idx], Kr, Dr)
    close = hp["idx"]
    err_hp = worst_component(K[close], D[close], hp["K"], hp["D"])
    Ko, Do = oracle.fused_sweep(wl.r[close], wl.z[close], wl.r, wl.z, wl.w, wl.f, wl.df_r,
                                wl.df_z, wl.nu_hat, wl.mass_ratio_o, eps_d=wl.eps_d)
    print("cfg5 N=2^20: evenly spaced vs oracle", err, "| closest-pair owners vs exact", err_hp,
          "(oracle vs exact", worst_component(Ko, Do, hp["K"], hp["D"]), ")")
    assert err < TOL and err_hp < TOL


@pytest.mark.parametrize("S", [1, 3, 5, 8])
def test_species_counts_vs_oracle(gpu, oracle, S):
    rng = np.random.default_rng(100 + S)
    n = 1000 + 37 * S  # ragged (not a multiple of the 128-point tile)
    r = rng.uniform(0.0, 3.0, n)
    z = rng.uniform(-3.0, 3.0, n)
    w = rng.uniform(0.1, 1.0, n)
    f, dfr, dfz = (rng.standard_normal((S, n)) for _ in range(3))
    nu = rng.uniform(0.5, 2.0, (S, S))
    nu = nu + nu.T
    mro = rng.uniform(0.01, 1.0, S)
    import paper_1702_08880_b200 as pkg

    data = pkg.QuadPointData(N=n, r=r, z=z, w=w, f=f, df_r=dfr, df_z=dfz)
    params = pkg.CollisionParams(nu_hat=nu, mass_ratio_o=mro)
    ro, zo = r[::7], z[::7]
    K, D = gpu.fused_sweep(ro, zo, data, params, eps_d=1e-13)
    Kr, Dr = oracle.fused_sweep(ro, zo, r, z, w, f, dfr, dfz, nu, mro, eps_d=1e-13)
    err = worst_component(K, D, Kr, Dr)
    print(f"S={S} random", err)
    assert err < TOL


def test_edge_sizes(gpu, oracle):
    import paper_1702_08880_b200 as pkg

    g = golden("cfg1")
    data, params = data_from(g), params_from(g)
    # empty outer set
    K, D = gpu.fused_sweep(np.zeros(0), np.zeros(0), data, params)
    assert K.shape == (0, 1, 2) and D.shape == (0, 1, 2, 2)
    # one outer point, 129 outer points (tile + 1), arbitrary off-grid points
    for m in (1, 129):
        ro = np.linspace(0.01, 4.9, m)
        zo = np.linspace(-4.9, 4.9, m)
        K, D = gpu.fused_sweep(ro, zo, data, params, eps_d=5e-14)
        Kr, Dr = oracle.fused_sweep(ro, zo, g["r"], g["z"], g["w"], g["f"], g["df_r"],
                                    g["df_z"], g["nu_hat"], g["mass_ratio_o"], eps_d=5e-14)
        assert worst_component(K, D, Kr, Dr) < TOL
    # empty inner set: all sums zero
    empty = pkg.QuadPointData(N=0, r=np.zeros(0), z=np.zeros(0), w=np.zeros(0),
                              f=np.zeros((1, 0)), df_r=np.zeros((1, 0)), df_z=np.zeros((1, 0)))
    K, D = gpu.fused_sweep(np.ones(3), np.zeros(3), empty, params)
    assert not K.any() and not D.any()
    # outer point on the axis (r = 0) and coincident with an inner point
    ro = np.array([0.0, g["r"][3]])
    zo = np.array([0.7, g["z"][3]])
    K, D = gpu.fused_sweep(ro, zo, data, params, eps_d=5e-14)
    Kr, Dr = oracle.fused_sweep(ro, zo, g["r"], g["z"], g["w"], g["f"], g["df_r"], g["df_z"],
                                g["nu_hat"], g["mass_ratio_o"], eps_d=5e-14)
    assert np.all(np.isfinite(K)) and worst_component(K, D, Kr, Dr) < TOL


def test_workers_and_block_size_do_not_change_results(gpu):
    # test_kernel.py:197-212 asserts bitwise invariance to both
    g = golden("sweep_small")
    data, params = data_from(g), params_from(g)
    base = gpu.fused_sweep(g["r"], g["z"], data, params)
    for kw in ({"workers": 4}, {"block_size": 16}, {"block_size": 1000}):
        other = gpu.fused_sweep(g["r"], g["z"], data, params, **kw)
        assert np.array_equal(base[0], other[0]) and np.array_equal(base[1], other[1])


def test_species_mismatch_raises(gpu):
    g = golden("sweep_small")
    with pytest.raises(ValueError):
        gpu.fused_sweep(g["r"], g["z"], data_from(g), params_from(g, "nu1", "mro1"))


@pytest.mark.parametrize("S,rank1", [(2, False), (3, False), (2, True), (4, True), (6, True)])
def test_all_points_coupling_layouts(gpu, oracle, S, rank1):
    """All-points sweep (symmetric path) for per-species accumulation (a
    coupling that is not rank one) and for the species-collapsed layout (rank
    one, the reference's own collision_params structure), vs the oracle."""
    import paper_1702_08880_b200 as pkg

    rng = np.random.default_rng(300 + S)
    n = 3000 + 11 * S
    r = rng.uniform(0.0, 3.0, n)
    z = rng.uniform(-3.0, 3.0, n)
    w = rng.uniform(0.1, 1.0, n)
    f, dfr, dfz = (rng.standard_normal((S, n)) for _ in range(3))
    if rank1:
        e = rng.uniform(0.5, 3.0, S)
        nu = np.outer(e**2, e**2)
        nu = nu / nu[0, 0]
    else:
        nu = rng.uniform(0.5, 2.0, (S, S))
    mro = rng.uniform(0.01, 1.0, S)
    data = pkg.QuadPointData(N=n, r=r, z=z, w=w, f=f, df_r=dfr, df_z=dfz)
    params = pkg.CollisionParams(nu_hat=nu, mass_ratio_o=mro)
    K, D = gpu.fused_sweep(r, z, data, params, eps_d=1e-13)
    Kr, Dr = oracle.fused_sweep(r, z, r, z, w, f, dfr, dfz, nu, mro, eps_d=1e-13)
    err = worst_component(K, D, Kr, Dr)
    print(f"all-points S={S} rank1={rank1}", err)
    assert err < 1e-10
    assert np.array_equal(D[..., 0, 1], D[..., 1, 0])


@pytest.mark.parametrize("n", [128, 129, 255, 256, 300, 383])
@pytest.mark.parametrize("rank1", [True, False])
def test_all_points_tile_boundaries(gpu, oracle, n, rank1):
    """All-points (symmetric) sweep at tile-count edges: one tile (only the
    diagonal tile pair), one tile + 1 point (padding), an even tile count
    (the opposite tile is shared by half the rows), odd counts -- for the
    collapsed (two points x two partners per thread) and the per-species
    kernels, vs the oracle."""
    import paper_1702_08880_b200 as pkg

    S = 2
    rng = np.random.default_rng(900 + n)
    r = rng.uniform(0.0, 3.0, n)
    z = rng.uniform(-3.0, 3.0, n)
    w = rng.uniform(0.1, 1.0, n)
    f, dfr, dfz = (rng.standard_normal((S, n)) for _ in range(3))
    e = np.array([1.0, 2.0])
    nu = np.outer(e**2, e**2) if rank1 else np.array([[1.0, 0.7], [0.7, 2.0]])
    mro = np.array([1.0, 0.3])
    data = pkg.QuadPointData(N=n, r=r, z=z, w=w, f=f, df_r=dfr, df_z=dfz)
    params = pkg.CollisionParams(nu_hat=nu, mass_ratio_o=mro)
    K, D = gpu.fused_sweep(r, z, data, params, eps_d=1e-13)
    Kr, Dr = oracle.fused_sweep(r, z, r, z, w, f, dfr, dfz, nu, mro, eps_d=1e-13)
    err = worst_component(K, D, Kr, Dr)
    assert err < TOL, (n, rank1, err)


def test_multibatch_runs_match(gpu, oracle):
    """Scratch-bounded batching (outer batches on the general path, row
    batches on the symmetric path) at N = 2^15, forced with a 1 MiB budget in
    a subprocess, agrees with the single-batch run and the oracle."""
    import json
    import os
    import subprocess
    import sys

    code = r"""
import json, sys, numpy as np
sys.path.insert(0, '.')
import paper_1702_08880_b200 as pkg
from paper_1702_08880_b200 import synthetic
wl = synthetic.cfg5(32768)
d = pkg.QuadPointData(N=wl.N, r=wl.r, z=wl.z, w=wl.w, f=wl.f, df_r=wl.df_r, df_z=wl.df_z)
p = pkg.CollisionParams(nu_hat=wl.nu_hat, mass_ratio_o=wl.mass_ratio_o)
K, D = pkg.fused_sweep(wl.r, wl.z, d, p, eps_d=wl.eps_d)
Kg, Dg = pkg.fused_sweep(wl.r[:-1], wl.z[:-1], d, p, eps_d=wl.eps_d)
np.savez(sys.argv[1], K=K, D=D, Kg=Kg, Dg=Dg)
"""
    import tempfile

    outs = []
    for budget in (None, "1"):
        env = dict(os.environ)
        if budget:
            env["LB_PARTIAL_BUDGET_MB"] = budget
        with tempfile.NamedTemporaryFile(suffix=".npz", delete=False) as fh:
            path = fh.name
        subprocess.run([sys.executable, "-c", code, path], check=True, env=env,
                       cwd=str(__import__("conftest").ROOT))
        outs.append(np.load(path))
    a, b = outs
    e_sym = worst_component(b["K"], b["D"], a["K"], a["D"])
    e_gen = worst_component(b["Kg"], b["Dg"], a["Kg"], a["Dg"])
    print("multi-batch vs single: symmetric", e_sym, "general", e_gen)
    assert e_sym < 1e-13 and e_gen < 1e-13
    from paper_1702_08880_b200 import synthetic

    wl = synthetic.cfg5(32768)
    idx = np.arange(0, 32768, 97)
    Kr, Dr = oracle.fused_sweep(wl.r[idx], wl.z[idx], wl.r, wl.z, wl.w, wl.f, wl.df_r, wl.df_z,
                                wl.nu_hat, wl.mass_ratio_o, eps_d=wl.eps_d)
    assert worst_component(b["K"][idx], b["D"][idx], Kr, Dr) < 1e-10


@pytest.mark.parametrize("eps_d", [0.0, 5e-14, 0.05])
def test_all_points_duplicates_axis_and_mask(gpu, oracle, eps_d):
    """All-points (symmetric) sweep on a point set with exact duplicates
    (coincident pairs: masked, d^2 == 0), points on the axis (r = 0: m = 0,
    the series branch) and near-coincident pairs, for eps_d = 0 (the
    reference's separate d^2 <= 1e-300 guard: the two-compare kernel
    variant), the default-size exclusion radius and a large one that masks
    many pairs (the merged-compare variant), vs the oracle (kernel.py:344-345)."""
    import paper_1702_08880_b200 as pkg

    S, n = 2, 1500
    rng = np.random.default_rng(31)
    r = rng.uniform(0.0, 3.0, n)
    z = rng.uniform(-3.0, 3.0, n)
    r[:40] = 0.0                                # on the axis
    r[40:80], z[40:80] = r[80:120], z[80:120]   # exact duplicates
    r[120:160] = r[160:200] + 1e-9              # near-coincident pairs
    z[120:160] = z[160:200]
    w = rng.uniform(0.1, 1.0, n)
    f, dfr, dfz = (rng.standard_normal((S, n)) for _ in range(3))
    e = np.array([1.0, 2.0])
    nu, mro = np.outer(e**2, e**2), np.array([1.0, 0.3])
    data = pkg.QuadPointData(N=n, r=r, z=z, w=w, f=f, df_r=dfr, df_z=dfz)
    params = pkg.CollisionParams(nu_hat=nu, mass_ratio_o=mro)
    K, D = gpu.fused_sweep(r, z, data, params, eps_d=eps_d)
    Kr, Dr = oracle.fused_sweep(r, z, r, z, w, f, dfr, dfz, nu, mro, eps_d=eps_d)
    assert np.all(np.isfinite(K)) and np.all(np.isfinite(D))
    # the near-coincident pairs (d = 1e-9) are where two double formulations
    # of the reference's tensors legitimately part; the
    # rest of the set is held to the north_star bar
    far = np.ones(n, bool)
    if eps_d < 1e-9:
        far[120:200] = False
    err = worst_component(K[far], D[far], Kr[far], Dr[far])
    print("eps_d", eps_d, "worst", err)
    assert err < TOL
