"""Bitwise A/B of two library builds on the same inputs (tools/ab_variants.sh
companion): D/K of the all-points and general sweeps, the per-pair entry
and an element contraction, compared with array_equal.
    python tools/bitwise_ab.py LIB_A LIB_B"""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def run(lib, out):
    code = r'''
import sys, numpy as np
sys.path.insert(0, %r)
import paper_1702_08880_b200 as pkg
from paper_1702_08880_b200 import synthetic
res = {}
for n in (1000, 4096, 65536):
    wl = synthetic.cfg5(n, seed=3)
    data = pkg.QuadPointData(N=wl.N, r=wl.r, z=wl.z, w=wl.w, f=wl.f, df_r=wl.df_r, df_z=wl.df_z)
    params = pkg.CollisionParams(nu_hat=wl.nu_hat, mass_ratio_o=wl.mass_ratio_o)
    K, D = pkg.fused_sweep(wl.r, wl.z, data, params, eps_d=wl.eps_d)
    res[f"K{n}"], res[f"D{n}"] = K, D
    if n <= 4096:
        K2, D2 = pkg.fused_sweep(wl.r[::3].copy(), wl.z[::3].copy(), data, params, eps_d=wl.eps_d)
        res[f"Kg{n}"], res[f"Dg{n}"] = K2, D2
rng = np.random.default_rng(5)
P = np.abs(rng.normal(size=(2000, 4)))
UK, UD = pkg.axisym_tensor_pairs(P[:, 0], P[:, 1], P[:, 2], P[:, 3])
res["UK"], res["UD"] = UK, UD
np.savez(%r, **res)
''' % (str(ROOT), out)
    env = dict(os.environ, LB_LIB=lib)
    subprocess.run([sys.executable, "-c", code], check=True, env=env)


if __name__ == "__main__":
    a, b = sys.argv[1], sys.argv[2]
    run(a, "/tmp/ab_a.npz")
    run(b, "/tmp/ab_b.npz")
    import numpy as np
    A, B = np.load("/tmp/ab_a.npz"), np.load("/tmp/ab_b.npz")
    bad = [k for k in A.files if not np.array_equal(A[k], B[k])]
    for k in A.files:
        d = np.abs(A[k] - B[k]).max() / max(np.abs(A[k]).max(), 1e-300)
        print(k, "bitwise" if k not in bad else f"DIFFERS (scaled {d:.2e})")
    print("ALL BITWISE EQUAL" if not bad else f"{len(bad)} arrays differ")
