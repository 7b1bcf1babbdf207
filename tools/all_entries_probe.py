"""Small end-to-end run of the device entries (general and symmetric sweeps,
collapsed and per-species; the state-level operator; a device Newton step)
with finiteness checks -- a quick probe to run under a memory checker where
one is available (compute-sanitizer is closed on this GPU pool)."""
import sys
from pathlib import Path
from types import SimpleNamespace

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402

import paper_1702_08880_b200 as pkg  # noqa: E402
from conftest import csr_from, golden, mesh_from, params_from, ref_from  # noqa: E402

rng = np.random.default_rng(1)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 400
for S, rank1 in ((2, True), (2, False), (3, False)):
    r, z, w = rng.uniform(0, 3, n), rng.uniform(-3, 3, n), rng.uniform(0.1, 1, n)
    f, dfr, dfz = (rng.standard_normal((S, n)) for _ in range(3))
    e = rng.uniform(0.5, 2, S)
    nu = np.outer(e**2, e**2) if rank1 else rng.uniform(0.5, 2, (S, S))
    data = pkg.QuadPointData(N=n, r=r, z=z, w=w, f=f, df_r=dfr, df_z=dfz)
    params = pkg.CollisionParams(nu_hat=nu, mass_ratio_o=rng.uniform(0.1, 1, S))
    K, D = pkg.fused_sweep(r, z, data, params, eps_d=1e-13)          # symmetric
    K2, D2 = pkg.fused_sweep(r[:n // 3], z[:n // 3], data, params)   # general
    assert np.isfinite(K).all() and np.isfinite(K2).all()
g = golden("cfg1")
mesh, ref, params = mesh_from(g), ref_from(g), params_from(g)
cm = pkg.assemble_at(mesh, ref, g["coeffs"], params)
nxt, rn = pkg.newton_step(g["coeffs"], g["coeffs"], mesh, ref, params,
                          SimpleNamespace(dt=0.1, eps_d=None), M=csr_from(g, "M"))
print("sanitize probe ok", float(np.abs(nxt).max()), rn)
