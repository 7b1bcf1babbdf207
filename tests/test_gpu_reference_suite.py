"""The drop-in proven by execution: the reference's OWN test suites run with
the B200 path installed (`paper_1702_08880_b200.install(axlandau)`), on the
GPU.

The reference (pure Python + numba) is installed unmodified into
baseline/_ref with its tests (tools/install_reference.sh; git-ignored, it
travels to the GPU box with the repository snapshot).  Each suite runs in a
subprocess under the plugin tools/ref_install_plugin.py, which patches every
by-value import of the hot path (kernel.fused_sweep / fused_inner_loop,
assembly.assemble_collision, solver._assemble_at / newton_step /
linear_cn_step, cli) before the test modules import them, and counts the
calls that reach this package.  Suites: test_kernel.py,
test_assembly.py, test_solver.py, test_cli.py, and acceptance criteria 3-4
(test_acceptance.py:108-192); plus the reference's own advance() loop.
"""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _reference():
    """(import root, tests dir) of the reference: baseline/_ref on the GPU
    box, else the read-only tree of the build container."""
    inst = ROOT / "baseline" / "_ref"
    if (inst / "axlandau").is_dir() and (inst / "axlandau_tests").is_dir():
        return inst, inst / "axlandau_tests"
    src = Path("/root/reference/pkg")
    if (src / "src" / "axlandau").is_dir():
        return src / "src", src / "tests"
    return None, None


def _run_suite(tmp_path, files, kexpr=None, timeout=1500):
    pytest.importorskip("numba")
    pkg_root, tests = _reference()
    if pkg_root is None:
        pytest.fail("reference not installed: run tools/install_reference.sh (baseline/_ref)")
    calls = tmp_path / "calls.json"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT / "tools"), str(ROOT), str(pkg_root), str(tests)])
    env["NUMBA_CACHE_DIR"] = str(tmp_path / "numba")
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    env["LB_REF_CALLS"] = str(calls)
    cmd = [sys.executable, "-m", "pytest", "-p", "ref_install_plugin", "-p", "no:cacheprovider",
           "--rootdir", str(tmp_path), "-q", "-rfEs", *[str(tests / f) for f in files]]
    if kexpr:
        cmd += ["-k", kexpr]
    out = subprocess.run(cmd, cwd=str(tmp_path), env=env, capture_output=True, text=True,
                         timeout=timeout)
    tail = out.stdout[-4000:] + out.stderr[-2000:]
    print(tail)
    assert out.returncode == 0, tail
    counts = json.loads(calls.read_text())
    return counts, out.stdout


def test_reference_kernel_suite(gpu, tmp_path):
    counts, log = _run_suite(tmp_path, ["test_kernel.py"])
    assert counts["axlandau.kernel.fused_sweep"] > 0 or counts["axlandau.fused_sweep"] > 0
    assert " passed" in log


def test_reference_assembly_suite(gpu, tmp_path):
    counts, log = _run_suite(tmp_path, ["test_assembly.py"])
    assert counts["axlandau.assembly.assemble_collision"] + counts["axlandau.assemble_collision"] > 0


def test_reference_solver_suite(gpu, tmp_path):
    counts, log = _run_suite(tmp_path, ["test_solver.py"])
    assert counts["axlandau.solver.newton_step"] + counts["axlandau.solver._assemble_at"] > 0


def test_reference_cli_suite(gpu, tmp_path):
    """test_cli.py: the reference's command layer (run / converge / bench /
    mesh, exit codes) over the installed B200 path -- cli.py imports
    assemble_collision and fused_sweep by value (cli.py:27-29)."""
    counts, log = _run_suite(tmp_path, ["test_cli.py"])
    assert sum(counts.values()) > 0


def test_reference_acceptance_criteria_3_4(gpu, tmp_path):
    counts, log = _run_suite(tmp_path, ["test_acceptance.py"],
                             kexpr="criterion_3 or criterion_4")
    assert "2 passed" in log
    assert sum(counts.values()) > 0


def _import_reference():
    pkg_root, tests = _reference()
    if pkg_root is None:
        pytest.fail("reference not installed: run tools/install_reference.sh (baseline/_ref)")
    pytest.importorskip("numba")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/lb_numba_cache")
    if str(pkg_root) not in sys.path:
        sys.path.insert(0, str(pkg_root))
    import axlandau

    return axlandau


def _cfg3_reference_setup(ax):
    """make_golden.py _cfg3_setup: 8x16 base refined 3 rounds toward the origin
    and the thermal shell, bi-Maxwellian electrons + Maxwellian ions."""
    import math

    import numpy as np

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
    s_perp, s_par = 2.0 * 0.4, 2.0 * 0.6
    fe = 0.5 * (math.pi ** 1.5 * s_perp * math.sqrt(s_par)) ** -1 * np.exp(-r * r / s_perp - z * z / s_par)
    fi = ax.physics.maxwellian_values(sp_[1], r, z)
    return mesh, ref, sp_, ax.StateVector(np.stack([fe, fi]))


@pytest.mark.parametrize("case", ["cfg1adv", "cfg3adv"])
def test_reference_advance_runs_on_device(gpu, case):
    """The reference's OWN time loop, `axlandau.solver.advance`
    (solver.py:153-199), with the B200 path installed: every Newton
    iteration's operator assembly (`_assemble_at`) and linear solve
    (`newton_step`) run on the device, the loop itself is the reference's.
    BASELINE config 1 (10 CN steps) and config 3 (3 steps, hanging nodes, two
    species) reproduce the reference's trajectories (tests/golden,
    generated with the reference alone) to 1e-10 scaled per step, with the
    same Newton residual histories."""
    import numpy as np

    from conftest import golden

    ax = _import_reference()
    from axlandau.solver import StepConfig

    import paper_1702_08880_b200 as lb

    g = golden(case)
    if case == "cfg1adv":
        mesh = ax.cartesian_mesh(ax.DomainSpec(L=5.0), 8, 16)
        ref = ax.build_reference_element()
        sp_ = [ax.Species("e", 1.0, -1.0, 0.5, shift=0.5)]
        state = ax.maxwellian_init(mesh, ref, sp_, neutralize=False)
        state.coeffs *= 2.0
        t_end = 1.0
    else:
        mesh, ref, sp_, state = _cfg3_reference_setup(ax)
        t_end = 0.3
    assert np.array_equal(state.coeffs, g["states"][0])
    cfg = StepConfig(dt=float(g["dt"]), newton_tol=float(g["newton_tol"]),
                     max_newton=int(g["max_newton"]))
    hist, calls = [], {"newton": 0}
    saved = lb.install(ax)
    try:
        dev_newton = ax.solver.newton_step

        def counted(*a, **k):
            calls["newton"] += 1
            return dev_newton(*a, **k)

        ax.solver.newton_step = counted
        traj = ax.solver.advance(mesh, ref, sp_, state, t_end, cfg, params=ax.collision_params(sp_),
                                 callback=lambda step, t, st, moms, info: hist.append(info["residuals"]))
    finally:
        lb.uninstall(ax, saved)
    states = np.stack([s.coeffs for _, s, _ in traj])
    assert states.shape == g["states"].shape and calls["newton"] >= len(traj) - 1
    worst = max(np.abs(states[k] - g["states"][k]).max() / np.abs(g["states"][k]).max()
                for k in range(states.shape[0]))
    for k, res in enumerate(hist):
        want = g["residuals"][k][~np.isnan(g["residuals"][k])]
        assert len(res) == len(want) and np.allclose(res, want, rtol=1e-6, atol=0.0)
    print(case, "reference advance() on the device: worst step state error", worst,
          "newton iterations", calls["newton"])
    assert worst <= 1e-10
