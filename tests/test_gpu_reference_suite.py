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
test_assembly.py, test_solver.py, and acceptance criteria 3-4
(test_acceptance.py:108-192).
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


def test_reference_acceptance_criteria_3_4(gpu, tmp_path):
    counts, log = _run_suite(tmp_path, ["test_acceptance.py"],
                             kexpr="criterion_3 or criterion_4")
    assert "2 passed" in log
    assert sum(counts.values()) > 0
