"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container (where the read-only reference tree exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

It imports `axlandau` from /root/reference/pkg/src, evaluates the reference's
own public functions (`axisym_tensor_pair`, `elliptic_KE`, `fused_sweep`
with workers=1, `assemble_collision`, `assemble_naive`, `mass_matrix`,
`linear_cn_step`, `moments`) on seeded inputs, and writes compressed .npz
fixtures next to this script.  Nothing at test / bench time reads the
reference tree; the tests compare the oracle and the CUDA path against these
files.  Case recipes mirror the reference tests they are named after.
"""

from __future__ import annotations

import math
import os
import sys
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = Path(__file__).resolve().parent
sys.path.insert(0, REF_SRC)
sys.path.insert(0, str(HERE.parents[1]))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import axlandau as ax  # noqa: E402
from axlandau import kernel as axk  # noqa: E402
from axlandau.solver import linear_cn_step  # noqa: E402
import scipy.sparse as sp  # noqa: E402
import scipy.sparse.linalg as spla  # noqa: E402

from paper_1702_08880_b200 import synthetic  # noqa: E402


def csr_parts(prefix, m):
    m = sp.csr_matrix(m)
    m.sort_indices()
    return {f"{prefix}_data": m.data, f"{prefix}_indices": m.indices.astype(np.int64),
            f"{prefix}_indptr": m.indptr.astype(np.int64),
            f"{prefix}_shape": np.array(m.shape, dtype=np.int64)}


def mesh_parts(mesh, ref):
    out = {"mesh_sizes": mesh.sizes, "mesh_cell_nodes": mesh.cell_nodes.astype(np.int64),
           "mesh_n_nodes": np.int64(mesh.n_nodes), "mesh_L": np.float64(mesh.domain.L),
           "mesh_free_r": mesh.nodes[mesh.free_nodes, 0],
           "mesh_free_z": mesh.nodes[mesh.free_nodes, 1],
           "mesh_origins": mesh.origins, "ref_qpts": ref.qpts, "ref_qwts": ref.qwts,
           "ref_B": ref.B, "ref_dB": ref.dB}
    out.update(csr_parts("mesh_P", mesh.prolongation))
    return out


def data_parts(data):
    return {"r": data.r, "z": data.z, "w": data.w, "f": data.f, "df_r": data.df_r,
            "df_z": data.df_z}


def params_parts(params):
    return {"nu_hat": params.nu_hat, "mass_ratio_o": params.mass_ratio_o}


def blocks_parts(prefix, cm):
    out = {}
    for a, b in enumerate(cm.blocks):
        out.update(csr_parts(f"{prefix}{a}", b))
    out[f"{prefix}_count"] = np.int64(len(cm.blocks))
    return out


def moment_matrix(mesh, ref):
    """Rows (n, z, v^2/2, v^2 z/2) x free dofs with 2 pi restored, so that
    moments(species a) = mass_a-scaled rows @ coeffs[a] (physics.py:130-146)."""
    eye = ax.StateVector(np.eye(mesh.n_free))
    d = ax.sample_state(mesh, ref, eye)
    wf = d.f * d.w[None, :] * (2.0 * np.pi)
    v2 = d.r ** 2 + d.z ** 2
    return np.stack([wf.sum(axis=1), wf @ d.z, 0.5 * (wf @ v2), 0.5 * (wf @ (v2 * d.z))])


def save(name, **arrays):
    path = HERE / f"{name}.npz"
    np.savez_compressed(path, **arrays)
    print(f"{path.name}: {path.stat().st_size / 1024:.0f} KiB")


def case_pairs():
    """Known-answer pairs for axisym_tensor_pair (test_kernel.py:94-146) and
    elliptic_KE (test_kernel.py:30-46)."""
    rng = np.random.default_rng(20260814)
    rows = []
    # generic, like test_pair_matches_azimuthal_quadrature / symmetries
    n = 600
    r = rng.uniform(0.01, 2.0, n); rb = rng.uniform(0.01, 2.0, n)
    z = rng.uniform(-2.0, 2.0, n); zb = rng.uniform(-2.0, 2.0, n)
    rows.append(np.stack([r, z, rb, zb], 1))
    # straddling the series switch m = 0.01 (test_pair_series_branch_continuous)
    rr = rng.uniform(0.02, 0.5, 100)
    mt = 0.01 * (1.0 + rng.uniform(-0.05, 0.05, 100))
    dz = np.sqrt(4 * rr * rr * (1 - mt) / mt)
    rows.append(np.stack([rr, np.zeros(100), rr, dz], 1))
    # on-axis inner / outer points (test_pair_on_axis_inner_point)
    k = 50
    rows.append(np.stack([rng.uniform(0.05, 2, k), rng.uniform(-2, 2, k), np.zeros(k),
                          rng.uniform(-2, 2, k)], 1))
    rows.append(np.stack([np.zeros(k), rng.uniform(-2, 2, k), rng.uniform(0.05, 2, k),
                          rng.uniform(-2, 2, k)], 1))
    # near-coincident pairs (x -> 0, K log-singular)
    k = 100
    r0 = rng.uniform(0.1, 2.0, k); z0 = rng.uniform(-2, 2, k)
    eps = 10.0 ** rng.uniform(-7, -2, k)
    ang = rng.uniform(0, 2 * np.pi, k)
    rows.append(np.stack([r0, z0, r0 + eps * np.cos(ang), z0 + eps * np.sin(ang)], 1))
    # far apart (small m via separation)
    k = 100
    rows.append(np.stack([rng.uniform(0.01, 0.3, k), rng.uniform(-5, -4, k),
                          rng.uniform(0.01, 0.3, k), rng.uniform(4, 5, k)], 1))
    P = np.concatenate(rows)
    UK = np.empty((len(P), 2, 2)); UD = np.empty((len(P), 2, 2))
    for t, (a, b, c, d) in enumerate(P):
        pr = ax.axisym_tensor_pair(a, b, c, d)
        UK[t] = pr.UK; UD[t] = pr.UD
    ms = np.concatenate([np.linspace(0.0, 0.98, 400), 1.0 - np.geomspace(1e-12, 0.02, 100)])
    K, E = ax.elliptic_KE(ms)
    save("pairs", pairs=P, UK=UK, UD=UD, m=ms, K=K, E=E)


def case_sweep_small():
    """test_kernel.py:161-231: 2x4 mesh on DomainSpec() (L=2), e/i species."""
    domain = ax.DomainSpec()
    ref = ax.build_reference_element()
    mesh = ax.cartesian_mesh(domain, 2, 4)
    sp_ = [ax.Species("e", 1.0, -1.0, 0.2, shift=-0.5), ax.Species("i", 4.0, 1.0, 0.1)]
    state = ax.maxwellian_init(mesh, ref, sp_, neutralize=True)
    data = ax.sample_state(mesh, ref, state)
    params = ax.collision_params(sp_)
    K, D = ax.fused_sweep(data.r, data.z, data, params, workers=1)
    # single species + proximity mask (test_kernel.py:223-231)
    state1 = ax.maxwellian_init(mesh, ref, sp_[:1], neutralize=False)
    data1 = ax.sample_state(mesh, ref, state1)
    params1 = ax.collision_params(sp_[:1])
    r0, z0 = data1.r[10] + 1e-9, data1.z[10]
    Kw, Dw = ax.fused_sweep(np.array([r0]), np.array([z0]), data1, params1)
    Km, Dm = ax.fused_sweep(np.array([r0]), np.array([z0]), data1, params1, eps_d=1e-6)
    # scalar reduction pin for 4 outer points (test_kernel.py:173-194)
    save("sweep_small", **data_parts(data), **params_parts(params), K=K, D=D,
         r1=data1.r, z1=data1.z, w1=data1.w, f1=data1.f, df_r1=data1.df_r, df_z1=data1.df_z,
         nu1=params1.nu_hat, mro1=params1.mass_ratio_o, prox_outer=np.array([r0, z0]),
         K_with=Kw, D_with=Dw, K_masked=Km, D_masked=Dm)


def case_cfg1():
    """BASELINE config 1: L=5, 8x16 Q2 mesh (N=1152), drifting Maxwellian
    electrons (n=1 -> 2x maxwellian_init, whose prefactor is 1/2), eps_d=5e-14;
    full D/K, the assembled operator, and one CN step / composed BE step."""
    domain = ax.DomainSpec(L=5.0)
    ref = ax.build_reference_element()
    mesh = ax.cartesian_mesh(domain, 8, 16)
    sp_ = [ax.Species("e", 1.0, -1.0, 0.5, shift=0.5)]
    state = ax.maxwellian_init(mesh, ref, sp_, neutralize=False)
    state.coeffs *= 2.0
    data = ax.sample_state(mesh, ref, state)
    params = ax.collision_params(sp_)
    eps_d = ax.assembly.default_eps_d(mesh)
    K, D = ax.fused_sweep(data.r, data.z, data, params, eps_d=eps_d, workers=1)
    cm = ax.assemble_collision(mesh, ref, data, params)
    M = ax.mass_matrix(mesh, ref)
    dt = 0.1
    cn = linear_cn_step(M, cm, dt, state)
    be = spla.splu((M - dt * cm.blocks[0]).tocsc()).solve(M @ state.coeffs[0])
    moms0 = ax.moments(mesh, ref, state, sp_)
    moms_cn = ax.moments(mesh, ref, cn, sp_)
    save("cfg1", **mesh_parts(mesh, ref), **data_parts(data), **params_parts(params),
         eps_d=np.float64(eps_d), K=K, D=D, **blocks_parts("C", cm), **csr_parts("M", M),
         coeffs=state.coeffs, dt=np.float64(dt), cn_coeffs=cn.coeffs, be_coeffs=be[None, :],
         Wm=moment_matrix(mesh, ref), masses=np.array([s.mass for s in sp_]),
         moms0=np.stack([moms0.n, moms0.p_z, moms0.E, moms0.q_z]),
         moms_cn=np.stack([moms_cn.n, moms_cn.p_z, moms_cn.E, moms_cn.q_z]))


def case_hanging():
    """test_assembly.py:43-51: hanging-node mesh, two species, random state;
    fused and naive reference assemblies."""
    domain = ax.DomainSpec()
    ref = ax.build_reference_element()
    mesh = ax.refine(ax.cartesian_mesh(domain, 2, 2), [3])
    sp_ = [ax.Species("e", mass=1.0, charge=-1.0, temperature=0.2, shift=-1.0),
           ax.Species("i", mass=4.0, charge=1.0, temperature=0.02)]
    params = ax.collision_params(sp_)
    rng = np.random.default_rng(20260814)
    state = ax.StateVector(rng.standard_normal((2, mesh.n_free)))
    data = ax.sample_state(mesh, ref, state)
    fused = ax.assemble_collision(mesh, ref, data, params)
    naive = ax.assemble_naive(mesh, ref, state, params)
    K, D = ax.fused_sweep(data.r, data.z, data, params, eps_d=ax.assembly.default_eps_d(mesh))
    save("hanging", **mesh_parts(mesh, ref), **data_parts(data), **params_parts(params),
         coeffs=state.coeffs, K=K, D=D, **blocks_parts("C", fused),
         **blocks_parts("N", naive))


def case_cons():
    """test_assembly.py:79-97: perturbed two-species Maxwellian on 8x16 (L=2)."""
    domain = ax.DomainSpec()
    ref = ax.build_reference_element()
    mesh = ax.cartesian_mesh(domain, 8, 16)
    sp_ = [ax.Species("e", mass=1.0, charge=-1.0, temperature=0.2, shift=-1.0),
           ax.Species("i", mass=4.0, charge=1.0, temperature=0.02)]
    r = mesh.nodes[mesh.free_nodes, 0]
    z = mesh.nodes[mesh.free_nodes, 1]
    state = ax.maxwellian_init(mesh, ref, sp_)
    state.coeffs[:] *= 1.0 + 0.1 * np.sin(3 * z) * np.cos(2 * r)
    data = ax.sample_state(mesh, ref, state)
    params = ax.collision_params(sp_)
    cm = ax.assemble_collision(mesh, ref, data, params)
    save("cons", **mesh_parts(mesh, ref), **data_parts(data), **params_parts(params),
         coeffs=state.coeffs, masses=np.array([s.mass for s in sp_]),
         **blocks_parts("C", cm))


def case_cfg2():
    """BASELINE config 2 (reference-native reading): electrons + deuterium
    (m=3670), T_e = 2 T_i, one shared 16x32 mesh on L=5, S=2."""
    domain = ax.DomainSpec(L=5.0)
    ref = ax.build_reference_element()
    mesh = ax.cartesian_mesh(domain, 16, 32)
    sp_ = [ax.Species("e", 1.0, -1.0, 0.5), ax.Species("D", 3670.0, 1.0, 0.25)]
    state = ax.maxwellian_init(mesh, ref, sp_)
    data = ax.sample_state(mesh, ref, state)
    params = ax.collision_params(sp_)
    eps_d = ax.assembly.default_eps_d(mesh)
    K, D = ax.fused_sweep(data.r, data.z, data, params, eps_d=eps_d, workers=1)
    cm = ax.assemble_collision(mesh, ref, data, params)
    save("cfg2", **mesh_parts(mesh, ref), **data_parts(data), **params_parts(params),
         eps_d=np.float64(eps_d), K=K, D=D, coeffs=state.coeffs,
         masses=np.array([s.mass for s in sp_]), **blocks_parts("C", cm))


def case_cfg1_advance():
    """BASELINE config 1 time integration: the reference's own advance()
    (solver.py:153-200) on the 8x16 mesh with the drifting Maxwellian of
    case_cfg1, 10 steps of dt = 0.1, Newton to 1e-12 (at most 4 frozen-
    coefficient iterations per step); per-step states, moments and residual
    histories.  (Config 2's deuterium, sigma = 0.012 on an h = 0.3 mesh, makes
    the reference's iteration diverge, so it is no parity target.)"""
    from axlandau.solver import StepConfig, advance

    domain = ax.DomainSpec(L=5.0)
    ref = ax.build_reference_element()
    mesh = ax.cartesian_mesh(domain, 8, 16)
    sp_ = [ax.Species("e", 1.0, -1.0, 0.5, shift=0.5)]
    state = ax.maxwellian_init(mesh, ref, sp_, neutralize=False)
    state.coeffs *= 2.0
    params = ax.collision_params(sp_)
    cfg = StepConfig(dt=0.1, newton_tol=1e-12, max_newton=4)
    hist = []

    def record(step, t, st, moms, info):
        hist.append(info["residuals"] + [np.nan] * (cfg.max_newton - len(info["residuals"])))

    traj = advance(mesh, ref, sp_, state, 1.0, cfg, params=params, callback=record)
    states = np.stack([s.coeffs for _, s, _ in traj])
    moms = np.stack([np.stack([m.n, m.p_z, m.E, m.q_z]) for _, _, m in traj])
    M = ax.mass_matrix(mesh, ref)
    save("cfg1adv", **mesh_parts(mesh, ref), **params_parts(params), **csr_parts("M", M),
         states=states, moms=moms, residuals=np.array(hist), dt=np.float64(cfg.dt),
         newton_tol=np.float64(cfg.newton_tol), max_newton=np.int64(cfg.max_newton),
         masses=np.array([s.mass for s in sp_]), Wm=moment_matrix(mesh, ref))


def _cfg3_setup():
    """Config 3's refined mesh and bi-Maxwellian state (see case_cfg3)."""
    domain = ax.DomainSpec(L=5.0)
    ref = ax.build_reference_element()
    mesh = ax.cartesian_mesh(domain, 8, 16)
    for _ in range(3):
        o, sz = mesh.origins, mesh.sizes
        rmin, rmax = o[:, 0], o[:, 0] + sz[:, 0]
        zlo, zhi = o[:, 1], o[:, 1] + sz[:, 1]
        zn = np.where((zlo <= 0) & (zhi >= 0), 0.0, np.minimum(abs(zlo), abs(zhi)))
        vmin = np.hypot(rmin, zn)
        vmax = np.hypot(rmax, np.maximum(abs(zlo), abs(zhi)))
        mesh = ax.refine(mesh, np.where((vmin <= 0.7) | ((vmax >= 0.6) & (vmin <= 1.6)))[0])
    sp_ = [ax.Species("e", 1.0, -1.0, 0.4), ax.Species("i", 4.0, 1.0, 0.2)]
    r = mesh.nodes[mesh.free_nodes, 0]
    z = mesh.nodes[mesh.free_nodes, 1]
    s_perp, s_par = 2.0 * 0.4, 2.0 * 0.6  # sigma^2 = 2T/m, T_par = 1.5 T_perp
    fe = 0.5 * (math.pi ** 1.5 * s_perp * math.sqrt(s_par)) ** -1 * np.exp(-r * r / s_perp - z * z / s_par)
    fi = ax.physics.maxwellian_values(sp_[1], r, z)
    state = ax.StateVector(np.stack([fe, fi]))
    return mesh, ref, sp_, state


def case_cfg3():
    """BASELINE config 3, reference-native reading: Q2 on an
    8x16 base (L=5) refined 3 rounds toward the origin and the thermal shell
    |v| ~ 1 (hanging nodes), bi-Maxwellian electrons (T_par = 1.5 T_perp)
    plus Maxwellian ions built directly as a StateVector; D/K, the operator,
    and one frozen-coefficient Newton step (solver.py:103-134)."""
    from axlandau.solver import StepConfig, newton_step

    mesh, ref, sp_, state = _cfg3_setup()
    data = ax.sample_state(mesh, ref, state)
    params = ax.collision_params(sp_)
    eps_d = ax.assembly.default_eps_d(mesh)
    idx = np.unique(np.linspace(0, data.N - 1, 1024).astype(np.int64))
    K, D = ax.fused_sweep(data.r[idx], data.z[idx], data, params, eps_d=eps_d, workers=1)
    cm = ax.assemble_collision(mesh, ref, data, params)
    cfg = StepConfig(dt=0.1, max_newton=1)
    M = ax.mass_matrix(mesh, ref)
    nxt, rnorm = newton_step(state, state, mesh, ref, params, cfg, M=M)
    moms0 = ax.moments(mesh, ref, state, sp_)
    moms1 = ax.moments(mesh, ref, nxt, sp_)
    save("cfg3", **mesh_parts(mesh, ref), **data_parts(data), **params_parts(params),
         eps_d=np.float64(eps_d), idx=idx, K=K, D=D, coeffs=state.coeffs,
         masses=np.array([s.mass for s in sp_]), **blocks_parts("C", cm), **csr_parts("M", M),
         dt=np.float64(cfg.dt), newton_coeffs=nxt.coeffs, newton_rnorm=np.float64(rnorm),
         Wm=moment_matrix(mesh, ref),
         moms0=np.stack([moms0.n, moms0.p_z, moms0.E, moms0.q_z]),
         moms1=np.stack([moms1.n, moms1.p_z, moms1.E, moms1.q_z]))


def case_cfg3_advance():
    """Config 3 time integration (hanging nodes, two species): the reference's
    advance() for 3 steps of dt = 0.1, Newton to 1e-12 (at most 3 iterations);
    per-step states, moments and residual histories."""
    from axlandau.solver import StepConfig, advance

    mesh, ref, sp_, state = _cfg3_setup()
    params = ax.collision_params(sp_)
    cfg = StepConfig(dt=0.1, newton_tol=1e-12, max_newton=3)
    hist = []

    def record(step, t, st, moms, info):
        hist.append(info["residuals"] + [np.nan] * (cfg.max_newton - len(info["residuals"])))

    traj = advance(mesh, ref, sp_, state, 0.3, cfg, params=params, callback=record)
    states = np.stack([s.coeffs for _, s, _ in traj])
    moms = np.stack([np.stack([m.n, m.p_z, m.E, m.q_z]) for _, _, m in traj])
    M = ax.mass_matrix(mesh, ref)
    save("cfg3adv", **mesh_parts(mesh, ref), **params_parts(params), **csr_parts("M", M),
         states=states, moms=moms, residuals=np.array(hist), dt=np.float64(cfg.dt),
         newton_tol=np.float64(cfg.newton_tol), max_newton=np.int64(cfg.max_newton),
         masses=np.array([s.mass for s in sp_]), Wm=moment_matrix(mesh, ref))


def case_cfg4_species():
    """BASELINE config 4 species set (e, D, C6+, W10+; n = 1/0.8/0.02/0.001,
    T = 1/1/0.5/0.5; non-neutral, so the state is built directly with a
    seeded 1% perturbation) on a 16x32 mesh, S = 4, 512 outer points."""
    domain = ax.DomainSpec(L=5.0)
    ref = ax.build_reference_element()
    mesh = ax.cartesian_mesh(domain, 16, 32)
    spec = [("e", 1.0, -1.0, 1.0, 1.0), ("D", 3670.0, 1.0, 0.8, 1.0),
            ("C", 21900.0, 6.0, 0.02, 0.5), ("W", 335000.0, 10.0, 0.001, 0.5)]
    sp_ = [ax.Species(nm, m, q, T) for nm, m, q, _, T in spec]
    r = mesh.nodes[mesh.free_nodes, 0]
    z = mesh.nodes[mesh.free_nodes, 1]
    rng = np.random.default_rng(4)
    coeffs = []
    for (nm, m, q, dens, T), s in zip(spec, sp_):
        s2 = s.sigma2
        vals = dens * (math.pi * s2) ** -1.5 * np.exp(-(r * r + z * z) / s2)
        coeffs.append(vals * (1.0 + 0.01 * rng.standard_normal(vals.shape)))
    state = ax.StateVector(np.stack(coeffs))
    data = ax.sample_state(mesh, ref, state)
    params = ax.collision_params(sp_)
    eps_d = ax.assembly.default_eps_d(mesh)
    idx = np.unique(np.linspace(0, data.N - 1, 512).astype(np.int64))
    K, D = ax.fused_sweep(data.r[idx], data.z[idx], data, params, eps_d=eps_d, workers=1)
    save("cfg4s", **data_parts(data), **params_parts(params), eps_d=np.float64(eps_d),
         idx=idx, K=K, D=D)


def _species_meshes_case(name, spec, grid, seed=None):
    """Per-species meshes (PAPER.md 3.0.2; BASELINE configs 2 / 4 as
    worded): species a on its own uniform grid over L_a = 5 sigma_a.  The
    composed reference oracle: one reference fused_sweep
    over the species-tagged union point set (f_b = 0 off mesh b; exact), then
    each species' transform + contraction + condensation on its own mesh
    (assembly.py:151-169 restated in oracle/oracle.py, pinned against the
    reference by tests/test_oracle.py)."""
    sys.path.insert(0, str(HERE.parents[1]))
    from oracle import oracle as O

    ref = ax.build_reference_element()
    sp_ = [ax.Species(nm, m, q, T) for nm, m, q, _, T in spec]
    params = ax.collision_params(sp_)
    rng = np.random.default_rng(seed) if seed is not None else None
    meshes, datas, coeffs = [], [], []
    for (nm, m, q, dens, T), s in zip(spec, sp_):
        mesh = ax.cartesian_mesh(ax.DomainSpec(L=5.0 * math.sqrt(s.sigma2)), *grid)
        st = ax.maxwellian_init(mesh, ref, [s], neutralize=False)
        st.coeffs *= 2.0 * dens  # the reference prefactor is 1/2 (physics.py:97-100)
        if rng is not None:
            st.coeffs *= 1.0 + 0.01 * rng.standard_normal(st.coeffs.shape)
        meshes.append(mesh)
        coeffs.append(st.coeffs[0])
        datas.append(ax.sample_state(mesh, ref, st))
    S = len(spec)
    ns = [d.N for d in datas]
    off = np.concatenate([[0], np.cumsum(ns)])
    n = int(off[-1])
    f = np.zeros((S, n)); dfr = np.zeros((S, n)); dfz = np.zeros((S, n))
    for a, d in enumerate(datas):
        f[a, off[a]:off[a + 1]] = d.f[0]
        dfr[a, off[a]:off[a + 1]] = d.df_r[0]
        dfz[a, off[a]:off[a + 1]] = d.df_z[0]
    union = ax.QuadPointData(N=n, r=np.concatenate([d.r for d in datas]),
                             z=np.concatenate([d.z for d in datas]),
                             w=np.concatenate([d.w for d in datas]), f=f, df_r=dfr, df_z=dfz)
    eps_d = min(ax.assembly.default_eps_d(m) for m in meshes)
    K, D = ax.fused_sweep(union.r, union.z, union, params, eps_d=eps_d, workers=1)
    out = {"S": np.int64(S), "eps_d": np.float64(eps_d), "offsets": off, "K": K, "D": D,
           **params_parts(params), "masses": np.array([s.mass for s in sp_])}
    for a, (mesh, d) in enumerate(zip(meshes, datas)):
        sl = slice(off[a], off[a + 1])
        elem = O.element_matrices(K[sl, a:a + 1], D[sl, a:a + 1], d.w, mesh.sizes, ref.B, ref.dB)
        blk = O.condense(elem, mesh.cell_nodes, mesh.n_nodes, mesh.prolongation)[0]
        for k, v in mesh_parts(mesh, ref).items():
            out[f"s{a}_{k}"] = v
        for k, v in data_parts(d).items():
            out[f"s{a}_{k}"] = v
        out.update(csr_parts(f"s{a}_C", blk))
        out[f"s{a}_coeffs"] = coeffs[a]
    save(name, **out)


def case_cfg2_meshes():
    """Config 2 as worded: e and D (m = 3670), T_e = 2 T_i, each on its own
    16x32 mesh scaled to its thermal speed (9216 union points)."""
    _species_meshes_case("cfg2m", [("e", 1.0, -1.0, 1.0, 0.5), ("D", 3670.0, 1.0, 1.0, 0.25)],
                         (16, 32))


def case_cfg2_meshes_be(steps=10, dt=0.5):
    """Config 2 as worded, time integration: e and D (m = 3670), T_e = 2 T_i,
    each on its own 16x32 mesh scaled to its thermal speed; `steps`
    backward-Euler steps of temperature relaxation, (M_a - dt C_a[f]) f_a+ =
    M_a f_a with C_a at the old state (the reference has Crank-Nicolson
    only: SURVEY 8(c)(iii) composes backward Euler from its pieces).  Each
    step is the composed reference oracle of case_cfg2_meshes (reference
    sample_state per mesh, ONE reference fused_sweep over the species-tagged
    union, the pinned per-mesh contraction + condensation) and scipy splu.
    Records every step's states and per-species moments."""
    sys.path.insert(0, str(HERE.parents[1]))
    from oracle import oracle as O

    spec = [("e", 1.0, -1.0, 1.0, 0.5), ("D", 3670.0, 1.0, 1.0, 0.25)]
    ref = ax.build_reference_element()
    sp_ = [ax.Species(nm, m, q, T) for nm, m, q, _, T in spec]
    params = ax.collision_params(sp_)
    meshes, coeffs, Ms = [], [], []
    for (nm, m, q, dens, T), s in zip(spec, sp_):
        mesh = ax.cartesian_mesh(ax.DomainSpec(L=5.0 * math.sqrt(s.sigma2)), 16, 32)
        st = ax.maxwellian_init(mesh, ref, [s], neutralize=False)
        st.coeffs *= 2.0 * dens  # the reference prefactor is 1/2 (physics.py:97-100)
        meshes.append(mesh)
        coeffs.append(st.coeffs[0].copy())
        Ms.append(ax.mass_matrix(mesh, ref))
    S = len(spec)
    eps_d = min(ax.assembly.default_eps_d(m) for m in meshes)
    traj = [[c.copy() for c in coeffs]]
    for _ in range(steps):
        datas = [ax.sample_state(mesh, ref, ax.StateVector(c[None, :])) for mesh, c in zip(meshes, coeffs)]
        ns = [d.N for d in datas]
        off = np.concatenate([[0], np.cumsum(ns)])
        n = int(off[-1])
        f = np.zeros((S, n)); dfr = np.zeros((S, n)); dfz = np.zeros((S, n))
        for a, d in enumerate(datas):
            f[a, off[a]:off[a + 1]] = d.f[0]
            dfr[a, off[a]:off[a + 1]] = d.df_r[0]
            dfz[a, off[a]:off[a + 1]] = d.df_z[0]
        union = ax.QuadPointData(N=n, r=np.concatenate([d.r for d in datas]),
                                 z=np.concatenate([d.z for d in datas]),
                                 w=np.concatenate([d.w for d in datas]), f=f, df_r=dfr, df_z=dfz)
        K, D = ax.fused_sweep(union.r, union.z, union, params, eps_d=eps_d, workers=1)
        new = []
        for a, (mesh, d) in enumerate(zip(meshes, datas)):
            sl = slice(off[a], off[a + 1])
            elem = O.element_matrices(K[sl, a:a + 1], D[sl, a:a + 1], d.w, mesh.sizes, ref.B, ref.dB)
            C = O.condense(elem, mesh.cell_nodes, mesh.n_nodes, mesh.prolongation)[0]
            new.append(spla.splu((Ms[a] - dt * C).tocsc()).solve(Ms[a] @ coeffs[a]))
        coeffs = new
        traj.append([c.copy() for c in coeffs])
    out = {"S": np.int64(S), "eps_d": np.float64(eps_d), "dt": np.float64(dt),
           "steps": np.int64(steps), **params_parts(params),
           "masses": np.array([s.mass for s in sp_])}
    for a, mesh in enumerate(meshes):
        for k, v in mesh_parts(mesh, ref).items():
            out[f"s{a}_{k}"] = v
        out.update(csr_parts(f"s{a}_M", Ms[a]))
        out[f"s{a}_Wm"] = moment_matrix(mesh, ref)
        out[f"s{a}_states"] = np.stack([t[a] for t in traj])
    save("cfg2be", **out)


def case_cfg4_meshes():
    """Config 4 as worded but on 8x16 meshes (the 64x128 union of 294,912
    points is beyond the reference's CPU budget): e, D, C6+, W10+ each on its
    own mesh, densities 1/0.8/0.02/0.001, T 1/1/0.5/0.5, 1 % seeded noise."""
    _species_meshes_case("cfg4m", [("e", 1.0, -1.0, 1.0, 1.0), ("D", 3670.0, 1.0, 0.8, 1.0),
                                   ("C", 21900.0, 6.0, 0.02, 0.5),
                                   ("W", 335000.0, 10.0, 0.001, 0.5)], (8, 16), seed=4)


def _closest_owners(r, z, k=64):
    from scipy.spatial import cKDTree

    pts = np.stack([r, z], 1)
    dist, _ = cKDTree(pts).query(pts, k=2)
    return np.argsort(dist[:, 1], kind="stable")[:k]


def _cfg4_species():
    spec = [("e", 1.0, -1.0, 1.0, 1.0), ("D", 3670.0, 1.0, 0.8, 1.0),
            ("C", 21900.0, 6.0, 0.02, 0.5), ("W", 335000.0, 10.0, 0.001, 0.5)]
    return spec, [ax.Species(nm, m, q, T) for nm, m, q, _, T in spec]


def case_cfg4_full():
    """BASELINE config 4 at its stated size, shared mesh (reference-native):
    cartesian_mesh(L=5, 64, 128), N = 73,728, S = 4 (e, D, C6+, W10+,
    n = 1/0.8/0.02/0.001, T = 1/1/0.5/0.5, non-neutral, seeded 1 % noise --
    the state of case_cfg4_species on the full mesh).  The FULL reference
    assemble_collision (fused_sweep workers=1 over all 5.4e9 ordered pairs,
    then the reference's transform + scatter), with the sweep's K/D captured:
    stored are K/D at 128 evenly spaced whole cells + the 64 closest-pair
    owners, those cells' element matrices (pinned restatement, oracle/), 256
    evenly spaced rows of every species' C and each block's max |C|."""
    import time

    sys.path.insert(0, str(HERE.parents[1]))
    from oracle import oracle as O

    domain = ax.DomainSpec(L=5.0)
    ref = ax.build_reference_element()
    mesh = ax.cartesian_mesh(domain, 64, 128)
    spec, sp_ = _cfg4_species()
    r = mesh.nodes[mesh.free_nodes, 0]
    z = mesh.nodes[mesh.free_nodes, 1]
    rng = np.random.default_rng(4)
    coeffs = []
    for (nm, m, q, dens, T), s in zip(spec, sp_):
        s2 = s.sigma2
        vals = dens * (math.pi * s2) ** -1.5 * np.exp(-(r * r + z * z) / s2)
        coeffs.append(vals * (1.0 + 0.01 * rng.standard_normal(vals.shape)))
    state = ax.StateVector(np.stack(coeffs))
    data = ax.sample_state(mesh, ref, state)
    params = ax.collision_params(sp_)
    eps_d = ax.assembly.default_eps_d(mesh)
    seen = {}
    sweep = ax.assembly.fused_sweep

    def capture(*a, **k):  # assembly.py imports fused_sweep by value (assembly.py:38-43)
        k["workers"] = 1
        seen["KD"] = sweep(*a, **k)
        return seen["KD"]

    ax.assembly.fused_sweep = capture
    t0 = time.time()
    try:
        cm = ax.assemble_collision(mesh, ref, data, params, eps_d=eps_d)
    finally:
        ax.assembly.fused_sweep = sweep
    print(f"cfg4full: reference assemble_collision {time.time() - t0:.0f} s")
    K, D = seen["KD"]
    cells = np.unique(np.linspace(0, mesh.n_cells - 1, 128).astype(np.int64))
    pts = (9 * cells[:, None] + np.arange(9)[None, :]).ravel()
    idx = np.unique(np.concatenate([pts, _closest_owners(data.r, data.z)]))
    elem = O.element_matrices(K[pts], D[pts], data.w[pts], mesh.sizes[cells], ref.B, ref.dB)
    rows = np.unique(np.linspace(0, mesh.n_free - 1, 256).astype(np.int64))
    out = {**mesh_parts(mesh, ref), **params_parts(params), "eps_d": np.float64(eps_d),
           "coeffs": state.coeffs, "masses": np.array([s.mass for s in sp_]),
           "idx": idx, "K": K[idx], "D": D[idx], "r_idx": data.r[idx], "z_idx": data.z[idx],
           "w_idx": data.w[idx], "cells": cells, "elem": elem, "rows": rows,
           "C_max": np.array([np.abs(b.data).max() for b in cm.blocks]),
           "timings": np.array([cm.timings[k] for k in ("kernel", "fe_transform", "scatter")])}
    for a, b in enumerate(cm.blocks):
        out.update(csr_parts(f"R{a}", b[rows]))
    save("cfg4full", **out)


def case_cfg4_meshes_full():
    """BASELINE config 4 as worded at its stated size: e, D, C6+, W10+ each
    on its OWN 64x128 mesh over L_a = 5 sigma_a (294,912 union points, 8.7e10
    ordered pairs), densities 1/0.8/0.02/0.001, T 1/1/0.5/0.5, 1 % seeded
    noise.  Composed reference oracle on patches: per
    species four 4x4-cell patches; the reference fused_sweep (workers=1) of
    their points + the 64 closest-pair owners of the union against ALL union
    points; each patch's element matrices (pinned restatement) condensed on
    the species' mesh, keeping the rows of the 49 nodes interior to each
    patch (those rows see only patch cells, so they are the full operator's
    rows)."""
    import time

    sys.path.insert(0, str(HERE.parents[1]))
    from oracle import oracle as O

    spec, sp_ = _cfg4_species()
    ref = ax.build_reference_element()
    params = ax.collision_params(sp_)
    rng = np.random.default_rng(4)
    nr, nz = 64, 128
    meshes, datas, coeffs = [], [], []
    for (nm, m, q, dens, T), s in zip(spec, sp_):
        mesh = ax.cartesian_mesh(ax.DomainSpec(L=5.0 * math.sqrt(s.sigma2)), nr, nz)
        st = ax.maxwellian_init(mesh, ref, [s], neutralize=False)
        st.coeffs *= 2.0 * dens  # the reference prefactor is 1/2 (physics.py:97-100)
        st.coeffs *= 1.0 + 0.01 * rng.standard_normal(st.coeffs.shape)
        meshes.append(mesh)
        coeffs.append(st.coeffs[0])
        datas.append(ax.sample_state(mesh, ref, st))
    S = len(spec)
    off = np.concatenate([[0], np.cumsum([d.N for d in datas])])
    n = int(off[-1])
    f = np.zeros((S, n)); dfr = np.zeros((S, n)); dfz = np.zeros((S, n))
    for a, d in enumerate(datas):
        f[a, off[a]:off[a + 1]] = d.f[0]
        dfr[a, off[a]:off[a + 1]] = d.df_r[0]
        dfz[a, off[a]:off[a + 1]] = d.df_z[0]
    union = ax.QuadPointData(N=n, r=np.concatenate([d.r for d in datas]),
                             z=np.concatenate([d.z for d in datas]),
                             w=np.concatenate([d.w for d in datas]), f=f, df_r=dfr, df_z=dfz)
    eps_d = min(ax.assembly.default_eps_d(m) for m in meshes)
    # four 4x4-cell patches per species mesh (cells are z-major: cell = j nr + i)
    corners = [(3, 10), (20, 60), (40, 100), (58, 120)]
    patch_cells = np.array(sorted(j * nr + i for (i0, j0) in corners
                                  for j in range(j0, j0 + 4) for i in range(i0, i0 + 4)))
    pts_local = (9 * patch_cells[:, None] + np.arange(9)[None, :]).ravel()
    pts = np.concatenate([off[a] + pts_local for a in range(S)])
    idx = np.unique(np.concatenate([pts, _closest_owners(union.r, union.z)]))
    t0 = time.time()
    K, D = ax.fused_sweep(union.r[idx], union.z[idx], union, params, eps_d=eps_d, workers=1)
    print(f"cfg4mfull: reference fused_sweep {idx.size} x {n} in {time.time() - t0:.0f} s")
    pos = {int(p): k for k, p in enumerate(idx)}
    out = {"S": np.int64(S), "eps_d": np.float64(eps_d), "offsets": off, "idx": idx, "K": K,
           "D": D, **params_parts(params), "masses": np.array([s.mass for s in sp_]),
           "patch_cells": patch_cells}
    for a, (mesh, d) in enumerate(zip(meshes, datas)):
        sel = np.array([pos[int(off[a] + p)] for p in pts_local])
        elem = np.zeros((1, mesh.n_cells, 9, 9))
        elem[:, patch_cells] = O.element_matrices(K[sel, a:a + 1], D[sel, a:a + 1], d.w[pts_local],
                                                  mesh.sizes[patch_cells], ref.B, ref.dB)
        blk = O.condense(elem, mesh.cell_nodes, mesh.n_nodes, mesh.prolongation)[0]
        # nodes interior to a patch: on no cell outside the patch
        outside = np.setdiff1d(np.arange(mesh.n_cells), patch_cells)
        inner_nodes = np.setdiff1d(np.unique(mesh.cell_nodes[patch_cells]),
                                   np.unique(mesh.cell_nodes[outside]))
        free_pos = {int(v): k for k, v in enumerate(mesh.free_nodes)}
        rows = np.array(sorted(free_pos[int(v)] for v in inner_nodes if int(v) in free_pos))
        assert rows.size == 4 * 49, rows.size
        for k, v in mesh_parts(mesh, ref).items():
            # the meshes differ only in scale: the topology (cell_nodes,
            # prolongation) and reference tables are stored once, with s0
            if a and (k.startswith("mesh_P") or k in ("mesh_cell_nodes", "ref_B", "ref_dB",
                                                      "ref_qpts", "ref_qwts")):
                assert np.array_equal(v, out[f"s0_{k}"])
                continue
            out[f"s{a}_{k}"] = v
        out[f"s{a}_coeffs"] = coeffs[a]
        out[f"s{a}_rows"] = rows
        out[f"s{a}_r_idx"] = d.r[pts_local]
        out[f"s{a}_w_idx"] = d.w[pts_local]
        out.update(csr_parts(f"s{a}_R", blk[rows]))
    save("cfg4mfull", **out)


def case_cfg3_q3():
    """BASELINE config 3 as worded, D/K parity: the 4x4
    Gauss points of Q3 elements on the config-3 refined mesh (8x16 base, 3
    refinement rounds toward the origin and the thermal shell: 950 cells,
    N = 15,200 points) with the config-3 state evaluated analytically there
    (synthetic.q3_points / cfg3_state_values, pinned here against the
    reference's element_geometry operation order and maxwellian_values).
    The reference's point-set-agnostic fused_sweep (workers=1) gives D/K of
    2048 evenly spaced points + the 64 closest-pair owners against all N.
    The Q3 Jacobian has no reference ("parity unpinned")."""
    mesh, ref, sp_, state = _cfg3_setup()
    r, z, w = synthetic.q3_points(mesh.origins, mesh.sizes)
    f, dfr, dfz, nu, mro = synthetic.cfg3_state_values(r, z)
    params = ax.collision_params(sp_)
    assert np.array_equal(params.nu_hat, nu) and np.array_equal(params.mass_ratio_o, mro)
    assert np.array_equal(f[1], ax.physics.maxwellian_values(sp_[1], r, z))
    # the geometry restatement reproduces the reference's own Q2 points bitwise
    r2, z2, w2 = synthetic.gauss_points(mesh.origins, mesh.sizes, ref.qpts, ref.qwts)
    g2 = ax.fem.element_geometry(mesh, ref)
    assert np.array_equal(r2, g2.coords[:, :, 0].ravel()) and np.array_equal(w2, g2.weights.ravel())
    data = ax.QuadPointData(N=r.size, r=r, z=z, w=w, f=f, df_r=dfr, df_z=dfz)
    eps_d = ax.assembly.default_eps_d(mesh)
    idx = np.unique(np.concatenate([np.linspace(0, r.size - 1, 2048).astype(np.int64),
                                    _closest_owners(r, z)]))
    K, D = ax.fused_sweep(r[idx], z[idx], data, params, eps_d=eps_d, workers=1)
    save("cfg3q3", origins=mesh.origins, sizes=mesh.sizes, eps_d=np.float64(eps_d), idx=idx,
         K=K, D=D, r_idx=r[idx], z_idx=z[idx], w_idx=w[idx], **params_parts(params))


def case_cfg5_hp():
    """High-precision yardstick (tests/golden/hp_sweep.py) for the outer
    points that own the globally closest pairs: config 5 at N = 2^20 (16
    owners, the test_cfg5_max_size set) and config 4 as worded at full size
    (the 64 owners in the 294,912-point union of cfg4mfull)."""
    import time

    sys.path.insert(0, str(HERE.parents[1]))
    sys.path.insert(0, str(HERE))
    from oracle import oracle as O
    import hp_sweep

    t0 = time.time()
    N = 1 << 20
    wl = synthetic.cfg5(N)
    close = _closest_owners(wl.r, wl.z, 16)
    K5, D5 = hp_sweep.hp_kd(close, wl.r, wl.z, wl.w, wl.f, wl.df_r, wl.df_z, wl.nu_hat,
                            wl.mass_ratio_o, wl.eps_d, 0.3, O)
    print(f"cfg5hp: N=2^20 owners {time.time() - t0:.0f} s")
    # config 4 as worded: the union's 64 closest-pair owners (sampled by the
    # pinned restatement of sample_state, bitwise the reference's)
    g = np.load(HERE / "cfg4mfull.npz")
    S = int(g["S"])
    off = g["offsets"]
    n = int(off[-1])
    r = np.empty(n); z = np.empty(n); w = np.empty(n)
    f, dfr, dfz = np.zeros((S, n)), np.zeros((S, n)), np.zeros((S, n))
    for a in range(S):
        key = lambda k: f"s{a}_{k}" if f"s{a}_{k}" in g else f"s0_{k}"  # noqa: E731
        P = sp.csr_matrix((g[key("mesh_P_data")], g[key("mesh_P_indices")], g[key("mesh_P_indptr")]),
                          shape=tuple(g[key("mesh_P_shape")]))
        ra, za, wa, fa, dra, dza = O.sample_state(g[key("mesh_origins")], g[key("mesh_sizes")],
                                                  g[key("mesh_cell_nodes")], P, g[key("ref_qpts")],
                                                  g[key("ref_qwts")], g[key("ref_B")], g[key("ref_dB")],
                                                  g[f"s{a}_coeffs"])
        sl = slice(off[a], off[a + 1])
        r[sl], z[sl], w[sl] = ra, za, wa
        f[a, sl], dfr[a, sl], dfz[a, sl] = fa[0], dra[0], dza[0]
    own = _closest_owners(r, z, 64)
    t0 = time.time()
    K4, D4 = hp_sweep.hp_kd(own, r, z, w, f, dfr, dfz, g["nu_hat"], g["mass_ratio_o"],
                            float(g["eps_d"]), 2e-3, O)
    print(f"cfg5hp: config-4-as-worded owners {time.time() - t0:.0f} s")
    save("cfg5hp", idx=close, K=K5, D=D5, checksum=np.float64(wl.checksum()),
         cfg4m_idx=own, cfg4m_K=K4, cfg4m_D=D4)


def case_pairs_hp():
    """The 1000 tensor-pair inputs of pairs.npz evaluated with the
    reference's formulas (kernel.py:306-389) in 40-digit arithmetic
    (hp_sweep.pair_hp): the yardstick for pairs whose double-precision
    closed form is ill-conditioned (near-coincident points, where UD_xx /
    UK_rr cancel O(r^2/d^2) terms)."""
    sys.path.insert(0, str(HERE))
    import hp_sweep

    P = np.load(HERE / "pairs.npz")["pairs"]
    tab = hp_sweep._tables()
    UK = np.empty((P.shape[0], 2, 2))
    UD = np.empty((P.shape[0], 2, 2))
    for k, (r, z, rb, zb) in enumerate(P):
        tkr, tzr, txx, txz, tzz = (float(v) for v in hp_sweep.pair_hp(r, z, rb, zb, tab))
        UK[k] = [[tkr, txz], [tzr, tzz]]
        UD[k] = [[txx, txz], [txz, tzz]]
    save("pairs_hp", UK=UK, UD=UD)


def case_cfg5(N, n_sub=None):
    """BASELINE config 5 recipe (paper_1702_08880_b200/synthetic.py).  Full
    N^2 when n_sub is None, else n_sub evenly spaced outer points plus the 64
    owners of the globally closest pairs."""
    wl = synthetic.cfg5(N)
    params = axk.CollisionParams(nu_hat=wl.nu_hat, mass_ratio_o=wl.mass_ratio_o)
    data = ax.QuadPointData(N=N, r=wl.r, z=wl.z, w=wl.w, f=wl.f, df_r=wl.df_r, df_z=wl.df_z)
    if n_sub is None:
        idx = np.arange(N)
    else:
        from scipy.spatial import cKDTree
        dist, _ = cKDTree(np.stack([wl.r, wl.z], 1)).query(np.stack([wl.r, wl.z], 1), k=2)
        close = np.argsort(dist[:, 1])[:64]
        idx = np.unique(np.concatenate([np.linspace(0, N - 1, n_sub).astype(np.int64), close]))
    K, D = ax.fused_sweep(wl.r[idx], wl.z[idx], data, params, eps_d=wl.eps_d, workers=1)
    extra = {} if n_sub is not None else {"r": wl.r, "z": wl.z}
    save(f"cfg5_{N}", idx=idx, K=K, D=D, checksum=np.float64(wl.checksum()), **extra)


def main():
    which = set(sys.argv[1:])
    cases = {"pairs": case_pairs, "sweep_small": case_sweep_small, "cfg1": case_cfg1,
             "hanging": case_hanging, "cons": case_cons, "cfg2": case_cfg2,
             "cfg3": case_cfg3, "cfg1adv": case_cfg1_advance, "cfg3adv": case_cfg3_advance, "cfg4s": case_cfg4_species, "cfg2m": case_cfg2_meshes,
             "cfg4m": case_cfg4_meshes, "cfg2be": case_cfg2_meshes_be,
             "cfg4full": case_cfg4_full, "cfg3q3": case_cfg3_q3, "cfg5hp": case_cfg5_hp, "pairshp": case_pairs_hp, "cfg4mfull": case_cfg4_meshes_full,
             "cfg5_4096": lambda: case_cfg5(4096),
             "cfg5_65536": lambda: case_cfg5(65536, n_sub=192)}
    for name, fn in cases.items():
        if not which or name in which:
            fn()


if __name__ == "__main__":
    main()
