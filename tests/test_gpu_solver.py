"""Device Crank-Nicolson step: newton_step and
linear_cn_step (solver.py:103-150) with the operator assembled and the
per-species systems (M - dt/2 C_a) solved on the B200 (block-tridiagonal
LU of the banded matrix), against the reference's SuperLU results.
Bar: post-step state max|df|/max|f_ref| <= 1e-10, moments relative <= 1e-10."""

from types import SimpleNamespace

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from conftest import blocks_from, csr_from, golden, mesh_from, params_from, ref_from

pytestmark = pytest.mark.gpu

TOL = 1e-10


def _scaled(x, ref):
    return float(np.abs(x - ref).max() / np.abs(ref).max())


def test_newton_step_cfg3(gpu):
    """BASELINE config 3 (refined mesh, 168 hanging nodes, two species): one
    newton_step(state, state, ..., M=M) with max_newton=1 (the fixture's
    reference call) reproduces the reference's next state and residual."""
    g = golden("cfg3")
    cfg = SimpleNamespace(dt=float(g["dt"]), eps_d=None)
    M = csr_from(g, "M")
    f0 = g["coeffs"]
    nxt, rnorm = gpu.newton_step(f0, f0, mesh_from(g), ref_from(g), params_from(g), cfg, M=M)
    err = _scaled(nxt, g["newton_coeffs"])
    print("cfg3 device newton step", err, "rnorm", rnorm, float(g["newton_rnorm"]))
    assert err <= TOL
    assert abs(rnorm - float(g["newton_rnorm"])) <= 1e-8 * float(g["newton_rnorm"])
    m = g["masses"]
    moms = np.stack([g["Wm"] @ nxt[a] * np.array([1.0, m[a], m[a], m[a]]) for a in range(2)], 1)
    ref = g["moms1"]
    assert np.all(np.abs(moms - ref)[[0, 2]] <= 1e-10 * np.abs(ref[[0, 2]]))
    assert np.all(np.abs(moms - ref)[[1, 3]] <= 1e-10 * np.abs(ref[[0, 2]]))


def test_newton_step_c_old_and_device_mass(gpu):
    """C_old passed in (as advance() does) and M assembled on the device give
    the same step as the defaults."""
    g = golden("cfg3")
    mesh, ref, params = mesh_from(g), ref_from(g), params_from(g)
    cfg = SimpleNamespace(dt=float(g["dt"]), eps_d=None)
    M = csr_from(g, "M")
    f0 = g["coeffs"]
    C_old = gpu.assemble_at(mesh, ref, f0, params)
    a, ra = gpu.newton_step(f0, f0, mesh, ref, params, cfg, M=M, C_old=C_old)
    b, rb = gpu.newton_step(f0, f0, mesh, ref, params, cfg, M=None)
    assert _scaled(a, g["newton_coeffs"]) <= TOL
    assert _scaled(b, g["newton_coeffs"]) <= TOL
    assert abs(ra - rb) <= 1e-12 * abs(ra)


@pytest.mark.parametrize("case", ["cfg1", "cfg3"])
def test_device_mass_matrix(gpu, case):
    """Device mass matrix (fem.py:152-167: r-weighted 3x3 Gauss, P^T M P)
    against the reference's mass_matrix."""
    g = golden(case)
    mesh, ref = mesh_from(g), ref_from(g)
    from paper_1702_08880_b200.solver import _mesh_solver, pattern_values

    s = _mesh_solver(mesh, ref, 1)
    s.set_mass(None)
    got = s.mass_values()
    want = pattern_values(csr_from(g, "M"), s.indptr, s.indices, s.n)
    err = _scaled(got, want)
    print(case, "device mass matrix", err, "bandwidth", s.bandwidth)
    assert err <= 1e-14


def test_linear_cn_step_cfg1(gpu):
    """linear_cn_step (solver.py:137-150) with the reference's own C and M
    gives the reference's CN state (the fixture's cn_coeffs)."""
    g = golden("cfg1")
    C = SimpleNamespace(blocks=blocks_from(g, "C"))
    out = gpu.linear_cn_step(csr_from(g, "M"), C, float(g["dt"]), g["coeffs"])
    err = _scaled(out[0], g["cn_coeffs"][0])
    print("cfg1 device linear CN", err)
    assert err <= TOL


def test_linear_cn_matches_splu_multi_species(gpu):
    """Banded block LU vs SuperLU on the two-species hanging-node operator,
    both signs of dt (time reversibility of the frozen-C map)."""
    g = golden("cfg3")
    M = csr_from(g, "M")
    blocks = blocks_from(g, "C")
    C = SimpleNamespace(blocks=blocks)
    f0 = g["coeffs"]
    for dt in (0.1, 1.0, -0.1):
        out = gpu.linear_cn_step(M, C, dt, f0)
        for a in range(2):
            want = spla.splu((M - 0.5 * dt * blocks[a]).tocsc()).solve((M + 0.5 * dt * blocks[a]) @ f0[a])
            assert _scaled(out[a], want) <= TOL, (dt, a)
    # test_solver.py:85-91 (reversible to 1e-10) and 73-82 (frozen residual)
    fwd = gpu.linear_cn_step(M, C, 0.1, f0)
    back = gpu.linear_cn_step(M, C, -0.1, fwd)
    assert _scaled(back, f0) < 1e-10
    R = np.stack([M @ (fwd[a] - f0[a]) - 0.05 * (blocks[a] @ fwd[a] + blocks[a] @ f0[a])
                  for a in range(2)])
    assert np.linalg.norm(R) < 1e-10 * np.linalg.norm(M @ f0.T)


def test_singular_system_raises_step_failure(gpu):
    """A singular system (zero matrix) raises StepFailure, as splu's
    RuntimeError does in the reference (solver.py:127-129)."""
    g = golden("cfg1")
    M = csr_from(g, "M")
    Z = sp.csr_matrix(M.shape)
    C = SimpleNamespace(blocks=[Z])
    with pytest.raises(gpu.StepFailure):
        gpu.linear_cn_step(Z, C, 0.1, g["coeffs"])


def test_newton_iterations_contract(gpu):
    """advance()'s inner loop (solver.py:171-185): repeated device Newton
    iterations at a fixed old state contract (test_solver.py:94-108: ratios
    < 0.6), track the same iteration done on the host with SuperLU to 1e-10,
    and conserve density to the reference's digits at every iterate."""
    g = golden("cfg3")
    mesh, ref, params = mesh_from(g), ref_from(g), params_from(g)
    dt = float(g["dt"])
    cfg = SimpleNamespace(dt=dt, eps_d=None)
    M = csr_from(g, "M")
    f0 = g["coeffs"]
    C_old = gpu.assemble_at(mesh, ref, f0, params)
    guess, host, res = f0, f0.copy(), []
    n0 = g["Wm"][0] @ f0.T
    for _ in range(5):
        guess, r = gpu.newton_step(guess, f0, mesh, ref, params, cfg, M=M, C_old=C_old)
        res.append(r)
        Cg = gpu.assemble_at(mesh, ref, host, params)
        nxt = np.empty_like(host)
        for a in range(2):
            R = M @ (host[a] - f0[a]) - 0.5 * dt * (Cg.blocks[a] @ host[a] + C_old.blocks[a] @ f0[a])
            nxt[a] = host[a] + spla.splu((M - 0.5 * dt * Cg.blocks[a]).tocsc()).solve(-R)
        host = nxt
        assert _scaled(guess, host) <= TOL
        n1 = g["Wm"][0] @ guess.T
        assert np.all(np.abs(n1 - n0) <= 1e-11 * np.abs(n0))
    print("newton residuals", res)
    assert np.all(np.array(res[1:]) / np.array(res[:-1]) < 0.6)


@pytest.mark.parametrize("nr,nz", [(16, 32), (32, 64)])
def test_config4_mesh_newton_step_matches_splu(gpu, nr, nz):
    """Uniform Q2 meshes with BASELINE config 4's four species -- 16x32
    (2145 free nodes, 68-row blocks) and 32x64 (8385 free nodes, 132-row
    blocks in 64 block rows, six reduction levels), both through the
    package's block-LU kernels (landau_lu.cuh): the device Newton step
    equals the host step done with SuperLU
    on the same device operator, and the device mass matrix integrates r
    over the domain."""
    from paper_1702_08880_b200 import synthetic
    from paper_1702_08880_b200.solver import _mesh_solver

    mesh, nodes = synthetic.uniform_q2_mesh(5.0, nr, nz)
    ref = synthetic.q2_reference()
    f0, nu, mro = synthetic.cfg4_state(nodes)
    params = gpu.CollisionParams(nu_hat=nu, mass_ratio_o=mro)
    s = _mesh_solver(mesh, ref, 4)
    s.set_mass(None)
    M = sp.csr_matrix((s.mass_values(), s.indices, s.indptr), shape=(s.n, s.n))
    # sum_ij M_ij = int r dr dz over [0,L] x [-L,L] = L^2/2 * 2L
    assert abs(M.sum() - 5.0**3) <= 1e-12 * 5.0**3
    dt = 0.1
    cfg = SimpleNamespace(dt=dt, eps_d=None)
    C_old = gpu.assemble_at(mesh, ref, f0, params)
    nxt, rnorm = gpu.newton_step(f0, f0, mesh, ref, params, cfg, M=M, C_old=C_old)
    host = np.empty_like(f0)
    for a in range(4):
        R = -0.5 * dt * (C_old.blocks[a] @ f0[a] + C_old.blocks[a] @ f0[a])
        host[a] = f0[a] + spla.splu((M - 0.5 * dt * C_old.blocks[a]).tocsc()).solve(-R)
    for a in range(4):
        err = _scaled(nxt[a], host[a])
        print("config-4 mesh species", a, "device vs splu", err)
        assert err <= TOL


@pytest.mark.parametrize("case", ["cfg1adv", "cfg3adv"])
def test_advance_trajectory(gpu, case):
    """BASELINE config 1 (10 steps) and config 3 (3 steps; hanging nodes, two
    species) time integration: the reference's advance() loop (solver.py:
    153-200: C_old at each step, up to max_newton frozen-coefficient
    iterations, early exit below newton_tol) run with the device operator and
    device Newton step reproduces the reference trajectory -- every step's
    state to 1e-10 scaled, density / momentum / energy to 1e-10 relative, and
    the residual histories."""
    g = golden(case)
    mesh, ref, params = mesh_from(g), ref_from(g), params_from(g)
    M = csr_from(g, "M")
    cfg = SimpleNamespace(dt=float(g["dt"]), eps_d=None)
    tol, max_newton = float(g["newton_tol"]), int(g["max_newton"])
    states, moms_ref, res_ref = g["states"], g["moms"], g["residuals"]
    Wm, masses = g["Wm"], g["masses"]
    state = states[0]
    worst = 0.0
    for step in range(1, states.shape[0]):
        C_old = gpu.assemble_at(mesh, ref, state, params)
        guess, res = state, []
        for _ in range(max_newton):
            guess, r = gpu.newton_step(guess, state, mesh, ref, params, cfg, M=M, C_old=C_old)
            res.append(r)
            if r < tol:
                break
        state = guess
        worst = max(worst, _scaled(state, states[step]))
        want = res_ref[step - 1][~np.isnan(res_ref[step - 1])]
        assert len(res) == len(want)
        assert np.allclose(res, want, rtol=1e-6, atol=0.0)
        for a, m in enumerate(masses):
            moms = Wm @ state[a] * np.array([1.0, m, m, m])
            ref_m = moms_ref[step][:, a]
            # density and energy relative; momentum relative to the density scale
            assert np.all(np.abs(moms - ref_m)[[0, 2]] <= 1e-10 * np.abs(ref_m[[0, 2]]))
            assert abs(moms[1] - ref_m[1]) <= 1e-10 * abs(ref_m[0])
    print(case, "trajectory: worst state error", worst)
    assert worst <= TOL


def test_unpivoted_lu_falls_back_to_pivoting(gpu):
    """The solver factorises without pivoting first and accepts the result
    only after a backward-error check; a system whose first diagonal entry
    is exactly zero (nonsingular, but not factorable without pivoting) must
    fall back to the pivoted block LU and still equal SuperLU."""
    from paper_1702_08880_b200 import solver as S

    g = golden("cfg1")
    M = csr_from(g, "M")
    C0 = blocks_from(g, "C")[0]
    dt = float(g["dt"])
    # the first row of the first eliminated (odd) diagonal block in band
    # order: its pivot is the raw matrix entry, so zero it
    pat = (abs(M) + abs(C0)).tocsr()
    pat.sort_indices()
    perm, bw = S.band_order(pat.indptr, pat.indices, pat.shape[0])
    node = int(perm[max(bw, 1)])
    M = M.tolil()
    M[node, node] = 0.5 * dt * C0[node, node]  # (M - dt/2 C)[node, node] == 0
    M = M.tocsr()
    C = SimpleNamespace(blocks=[C0])
    f0 = g["coeffs"]
    out = gpu.linear_cn_step(M, C, dt, f0)
    A = (M - 0.5 * dt * C0).tocsc()
    assert A[node, node] == 0.0
    want = spla.splu(A).solve((M + 0.5 * dt * C0) @ f0[0])
    assert _scaled(out[0], want) <= TOL
    stats = [s.stats() for s in S._LINEAR.values()]
    assert any(st["fallbacks"] >= 1 and st["pivoting"] for st in stats), stats
    assert min(st["rel_residual"] for st in stats) < 1e-12


_CUBLAS_LU_SCRIPT = r"""
import sys, numpy as np
from types import SimpleNamespace
sys.path.insert(0, sys.argv[1])
import paper_1702_08880_b200 as gpu
from paper_1702_08880_b200 import synthetic
from paper_1702_08880_b200.solver import _mesh_solver
import scipy.sparse as sp
mesh, nodes = synthetic.uniform_q2_mesh(5.0, 32, 64)
ref = synthetic.q2_reference()
f0, nu, mro = synthetic.cfg4_state(nodes)
params = gpu.CollisionParams(nu_hat=nu, mass_ratio_o=mro)
s = _mesh_solver(mesh, ref, 4)
s.set_mass(None)
M = sp.csr_matrix((s.mass_values(), s.indices, s.indptr), shape=(s.n, s.n))
cfg = SimpleNamespace(dt=0.1, eps_d=None)
C_old = gpu.assemble_at(mesh, ref, f0, params)
nxt, rnorm = gpu.newton_step(f0, f0, mesh, ref, params, cfg, M=M, C_old=C_old)
np.save(sys.argv[2], nxt)
"""


_CUBLAS_LU_CFG3_SCRIPT = r"""
import sys, numpy as np
from types import SimpleNamespace
sys.path.insert(0, sys.argv[1])
sys.path.insert(0, sys.argv[1] + "/tests")
import paper_1702_08880_b200 as gpu
from conftest import csr_from, golden, mesh_from, params_from, ref_from
g = golden("cfg3")
cfg = SimpleNamespace(dt=float(g["dt"]), eps_d=None)
nxt, rnorm = gpu.newton_step(g["coeffs"], g["coeffs"], mesh_from(g), ref_from(g), params_from(g), cfg,
                             M=csr_from(g, "M"))
np.save(sys.argv[2], nxt)
"""


def test_custom_block_lu_matches_cublas_path_cfg3(gpu, tmp_path):
    """Config 3 (hanging nodes, 354-row blocks, the unpivoted path): the
    shared-memory block-LU kernels and the global-memory LU path
    (LB_CN_GM_LU=1, in a subprocess; the path blocks over 384 rows take)
    give the same Newton step, and both the reference's."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    outs = {}
    for name, extra in (("custom", {}), ("cublas", {"LB_CN_GM_LU": "1"})):
        out = tmp_path / f"{name}.npy"
        subprocess.run([sys.executable, "-c", _CUBLAS_LU_CFG3_SCRIPT, str(root), str(out)],
                       env=dict(os.environ, **extra), check=True, timeout=600)
        outs[name] = np.load(out)
    g = golden("cfg3")
    err = _scaled(outs["custom"], outs["cublas"])
    print("cfg3 shared-memory LU vs global-memory LU", err)
    assert err <= 1e-12
    for v in outs.values():
        assert _scaled(v, g["newton_coeffs"]) <= TOL


def test_custom_block_lu_matches_cublas_path(gpu, tmp_path):
    """The shared-memory block LU + [L U] slab-solve kernels and the
    global-memory LU + substitution (LB_CN_GM_LU=1, read once per process,
    so it runs in a subprocess) give the same Newton step on the 32x64
    config-4 mesh (132-row blocks, four species): within the suite's 1e-10
    bar (the electron system is the ill-conditioned one that needs
    pivoting; both differ from SuperLU by ~3e-11 there, the other species
    agree to ~1e-16)."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    outs = {}
    for name, extra in (("custom", {}), ("cublas", {"LB_CN_GM_LU": "1"})):
        env = dict(os.environ, **extra)
        out = tmp_path / f"{name}.npy"
        subprocess.run([sys.executable, "-c", _CUBLAS_LU_SCRIPT, str(root), str(out)], env=env,
                       check=True, timeout=600)
        outs[name] = np.load(out)
    for a in range(4):
        err = _scaled(outs["custom"][a], outs["cublas"][a])
        print("species", a, "shared-memory LU vs global-memory LU", err)
        assert err <= TOL


def test_species_meshes_backward_euler_trajectory(gpu):
    """BASELINE config 2 as worded, time integration: electrons and deuterium
    (m = 3670, T_e = 2 T_i) each on its own 16x32 mesh scaled to its thermal
    speed, 10 backward-Euler steps of temperature relaxation.  The device
    path (device sampling per mesh, one union sweep, per-mesh assembly,
    lb_cn_theta_step with theta = 1) reproduces the composed reference
    trajectory (tests/golden/make_golden.py case_cfg2_meshes_be: reference
    sample_state + fused_sweep + pinned contraction, scipy splu): every
    step's states to 1e-10 scaled, per-species density / momentum / energy
    to 1e-10; each species' density is conserved (1e-13 relative) and the
    energy moves from the electrons to the ions."""
    from conftest import Prefixed

    g = golden("cfg2be")
    S, dt, steps = int(g["S"]), float(g["dt"]), int(g["steps"])
    meshes = [mesh_from(Prefixed(g, f"s{a}_")) for a in range(S)]
    ref = ref_from(Prefixed(g, "s0_"))
    params = params_from(g)
    Ms = [csr_from(g, f"s{a}_M") for a in range(S)]
    masses = g["masses"]
    states = [g[f"s{a}_states"][0].copy() for a in range(S)]
    worst, worst_mom = 0.0, 0.0
    for step in range(1, steps + 1):
        states = gpu.species_meshes_step(meshes, ref, states, params, dt, Ms)
        for a in range(S):
            want = g[f"s{a}_states"][step]
            worst = max(worst, _scaled(states[a], want))
            scale = np.array([1.0, masses[a], masses[a], masses[a]])
            mom = (g[f"s{a}_Wm"] @ states[a]) * scale
            ref_mom = (g[f"s{a}_Wm"] @ want) * scale
            worst_mom = max(worst_mom, abs(mom[0] - ref_mom[0]) / abs(ref_mom[0]),
                            abs(mom[2] - ref_mom[2]) / abs(ref_mom[2]),
                            abs(mom[1] - ref_mom[1]) / abs(ref_mom[0]))
            n0 = (g[f"s{a}_Wm"] @ g[f"s{a}_states"][0])[0]
            assert abs(mom[0] - n0) <= 1e-13 * abs(n0)
    print("cfg2 per-species meshes, 10 BE steps: worst state", worst, "worst moment", worst_mom)
    assert worst <= TOL and worst_mom <= TOL
    E0 = [(g[f"s{a}_Wm"] @ g[f"s{a}_states"][0])[2] * masses[a] for a in range(S)]
    E1 = [(g[f"s{a}_Wm"] @ states[a])[2] * masses[a] for a in range(S)]
    assert E1[0] < E0[0] and E1[1] > E0[1]  # electrons cool, ions heat


def test_theta_step_is_backward_euler_and_cn(gpu):
    """lb_cn_theta_step: theta = 1 solves (M - dt C) f+ = M f and theta = 1/2
    is linear_cn_step, both against scipy on the cfg1 fixture."""
    g = golden("cfg1")
    M = csr_from(g, "M")
    C = SimpleNamespace(blocks=blocks_from(g, "C"))
    f = np.atleast_2d(g["coeffs"])
    dt = 0.1
    be = gpu.backward_euler_step(M, C, dt, f)
    cn = gpu.theta_step(M, C, dt, f, 0.5)
    cn_ref = gpu.linear_cn_step(M, C, dt, f)
    for a in range(f.shape[0]):
        A = (M - dt * C.blocks[a]).tocsc()
        want = spla.splu(A).solve(M @ f[a])
        assert _scaled(be[a], want) <= 1e-12
        want_cn = spla.splu((M - 0.5 * dt * C.blocks[a]).tocsc()).solve((M + 0.5 * dt * C.blocks[a]) @ f[a])
        assert _scaled(cn[a], want_cn) <= 1e-12
    assert np.array_equal(cn, cn_ref)
    with pytest.raises(ValueError):
        gpu.theta_step(M, C, dt, f, 0.0)


@pytest.mark.parametrize("dominant", [True, False])
def test_wide_band_blocks_above_384_rows(gpu, dominant):
    """A banded system whose bandwidth (420) exceeds the shared-memory LU's
    384-row blocks: the solver takes the global-memory block LU (no library
    fallback) and matches scipy's splu -- diagonally dominant (unpivoted LU
    accepted) and not (the pivoted refactorisation)."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    from types import SimpleNamespace

    from paper_1702_08880_b200.solver import linear_cn_step

    n, b = 2100, 420
    rng = np.random.default_rng(7 if dominant else 8)
    offs = np.arange(-b, b + 1)
    diags = [rng.uniform(-1, 1, n - abs(k)) for k in offs]
    C = sp.diags(diags, offs, shape=(n, n), format="csr")
    M = sp.identity(n, format="csr") * (3.0 * b if dominant else 0.5)
    dt = 0.2
    f = rng.uniform(-1, 1, (1, n))
    out = linear_cn_step(M, SimpleNamespace(blocks=[C]), dt, f)
    ref = spla.splu((M - 0.5 * dt * C).tocsc()).solve((M + 0.5 * dt * C) @ f[0])
    err = np.abs(np.asarray(out)[0] - ref).max() / np.abs(ref).max()
    print("bandwidth 420 (global-memory block LU), dominant" if dominant else "not dominant", err)
    assert err < 1e-10
