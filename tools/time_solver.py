"""Time one Crank-Nicolson Newton iteration (solver.newton_step,
solver.py:103-134) on the device against the reference's host path (the
same device operator assembly, then scipy `splu` per species as the
reference does), for the fixture meshes (cfg1, cfg3) and the BASELINE
config 4 shared 64x128 Q2 mesh with four species.

    python tools/time_solver.py [cfg1 cfg3 cfg4]
"""
import hashlib
import sys
import time
from pathlib import Path
from types import SimpleNamespace

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, str(ROOT / "tools"))

import numpy as np  # noqa: E402
import scipy.sparse as sp  # noqa: E402
import scipy.sparse.linalg as spla  # noqa: E402

import paper_1702_08880_b200 as pkg  # noqa: E402
from paper_1702_08880_b200.solver import _mesh_solver  # noqa: E402


def fixture_case(name):
    from conftest import csr_from, golden, mesh_from, params_from, ref_from

    g = golden(name)
    return mesh_from(g), ref_from(g), params_from(g), g["coeffs"], csr_from(g, "M"), float(g["dt"])


def config4_case():
    from paper_1702_08880_b200.synthetic import cfg4_state, q2_reference, uniform_q2_mesh

    mesh, nodes = uniform_q2_mesh(5.0, 64, 128)
    ref = q2_reference()
    coeffs, nu_hat, mro = cfg4_state(nodes)
    params = pkg.CollisionParams(nu_hat=nu_hat, mass_ratio_o=mro)
    s = _mesh_solver(mesh, ref, 4)
    s.set_mass(None)  # device mass matrix (the uniform mesh has no reference fixture)
    M = sp.csr_matrix((s.mass_values(), s.indices, s.indptr), shape=(s.n, s.n))
    return mesh, ref, params, coeffs, M, 0.1


def host_newton(mesh, ref, params, f, M, dt, C_old):
    """The reference's newton_step with the device operator: assemble C at
    the guess, residual, splu per species (solver.py:116-133)."""
    Cg = pkg.assemble_at(mesh, ref, f, params)
    out = np.empty_like(f)
    for a in range(f.shape[0]):
        R = M @ (f[a] - f[a]) - 0.5 * dt * (Cg.blocks[a] @ f[a] + C_old.blocks[a] @ f[a])
        A = (M - 0.5 * dt * Cg.blocks[a]).tocsc()
        out[a] = f[a] + spla.splu(A).solve(-R)
    return out


def main():
    for name in sys.argv[1:] or ["cfg1", "cfg3", "cfg4"]:
        mesh, ref, params, f, M, dt = config4_case() if name == "cfg4" else fixture_case(name)
        cfg = SimpleNamespace(dt=dt, eps_d=None)
        C_old = pkg.assemble_at(mesh, ref, f, params)
        dev, _ = pkg.newton_step(f, f, mesh, ref, params, cfg, M=M, C_old=C_old)  # warm
        td = []
        for _ in range(5):
            t0 = time.perf_counter()
            dev, rnorm = pkg.newton_step(f, f, mesh, ref, params, cfg, M=M, C_old=C_old)
            td.append(time.perf_counter() - t0)
        th = []
        for _ in range(2 if name == "cfg4" else 5):
            t0 = time.perf_counter()
            host = host_newton(mesh, ref, params, f, M, dt, C_old)
            th.append(time.perf_counter() - t0)
        s = _mesh_solver(mesh, ref, f.shape[0])
        from paper_1702_08880_b200.solver import LAST_PHASES_MS as ph
        err = np.abs(dev - host).max() / np.abs(host).max()
        print(f"{name}: n_free={s.n} S={f.shape[0]} bandwidth={s.bandwidth} blocks={-(-s.n // s.nb)}  "
              f"device newton_step {min(td) * 1e3:.2f} ms  host (device assembly + splu) "
              f"{min(th) * 1e3:.2f} ms  x{min(th) / min(td):.1f}  rel diff {err:.1e}  rnorm {rnorm:.3e}"
              f"  device phases (assemble, residual+fill, LU, solve) {np.round(ph, 2).tolist()} ms"
              f"  solver {s.stats()}  sha1(f_next) {hashlib.sha1(np.ascontiguousarray(dev).tobytes()).hexdigest()[:12]}")


if __name__ == "__main__":
    main()
