"""Diagnostic: per-point D/K errors of the per-species config-4 union sweep
vs the reference fixture; saves the device K, D at the fixture points."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np  # noqa: E402

import paper_1702_08880_b200 as pkg  # noqa: E402
from conftest import golden, mesh_from, params_from, ref_from  # noqa: E402
from test_gpu_cfg4_full import _Species  # noqa: E402

g = golden("cfg4mfull")
S = int(g["S"])
views = [_Species(g, a) for a in range(S)]
meshes = [mesh_from(v) for v in views]
ref = ref_from(views[0])
datas = [pkg.sample_state(m, ref, g[f"s{a}_coeffs"][None, :]) for a, m in enumerate(meshes)]
blocks, (K, D) = pkg.assemble_species_meshes(meshes, ref, datas, params_from(g), eps_d=float(g["eps_d"]))
idx = g["idx"]
Kd, Dd = K[idx], D[idx]
np.savez(ROOT / "gpurun_out" / "cfg4m_points.npz", K=Kd, D=Dd, idx=idx)
for a in range(S):
    for nm, X, Xr in (("Drr", Dd[:, a, 0, 0], g["D"][:, a, 0, 0]), ("Drz", Dd[:, a, 0, 1], g["D"][:, a, 0, 1]),
                      ("Dzz", Dd[:, a, 1, 1], g["D"][:, a, 1, 1]), ("Kr", Kd[:, a, 0], g["K"][:, a, 0]),
                      ("Kz", Kd[:, a, 1], g["K"][:, a, 1])):
        e = np.abs(X - Xr) / np.abs(Xr).max()
        top = np.argsort(e)[-3:][::-1]
        print(a, nm, " ".join(f"p={idx[t]} err={e[t]:.2e} dev={X[t]:.17e} ref={Xr[t]:.17e}" for t in top))
