"""Diagnostic (build container: needs the reference for the 40-digit
evaluation): for the config-4-as-worded points where the device and the
reference differ most, the distance of each from the reference's formulas
in 40-digit arithmetic (tests/golden/hp_sweep.py).  Device values come from
tools/diag/cfg4m_points.py (run on the GPU, gpurun_out/cfg4m_points.npz).

    python tools/diag/cfg4m_vs_exact.py [point ...]
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path[:0] = [str(ROOT), str(ROOT / "tests"), str(ROOT / "tests" / "golden"),
                str(ROOT / "baseline" / "_ref")]
import numpy as np  # noqa: E402

import hp_sweep  # noqa: E402
from conftest import golden  # noqa: E402
from oracle import oracle as O  # noqa: E402
from test_oracle import _sample  # noqa: E402


def main():
    g = golden("cfg4mfull")
    S = int(g["S"])

    class V:
        def __init__(self, a):
            self.a = a

        def __getitem__(self, k):
            key = f"s{self.a}_{k}"
            return g[key] if key in g else g[f"s0_{k}"]

    parts = [_sample(O, V(a), g[f"s{a}_coeffs"]) for a in range(S)]
    off = g["offsets"]
    n = int(off[-1])
    r, z, w = (np.concatenate([p[i] for p in parts]) for i in range(3))
    f, dfr, dfz = np.zeros((S, n)), np.zeros((S, n)), np.zeros((S, n))
    for a, p in enumerate(parts):
        sl = slice(off[a], off[a + 1])
        f[a, sl], dfr[a, sl], dfz[a, sl] = p[3][0], p[4][0], p[5][0]
    dev = np.load(ROOT / "gpurun_out" / "cfg4m_points.npz")
    idx = list(dev["idx"])
    pts = [int(a) for a in sys.argv[1:]] or [272677, 243301, 246968, 269426]
    Kh, Dh = hp_sweep.hp_kd(pts, r, z, w, f, dfr, dfz, g["nu_hat"], g["mass_ratio_o"],
                            float(g["eps_d"]), 2e-3, O)
    sK = np.abs(g["K"][:, :, 0]).max(axis=0)
    sD = np.abs(g["D"][:, :, 0, 0]).max(axis=0)
    for m, p in enumerate(pts):
        k = idx.index(p)
        for a in range(S):
            print(f"point {p} species {a}: K_r dev-exact {(dev['K'][k, a, 0] - Kh[m, a, 0]) / sK[a]:+.2e} "
                  f"ref-exact {(g['K'][k, a, 0] - Kh[m, a, 0]) / sK[a]:+.2e} | D_rr dev-exact "
                  f"{(dev['D'][k, a, 0, 0] - Dh[m, a, 0, 0]) / sD[a]:+.2e} "
                  f"ref-exact {(g['D'][k, a, 0, 0] - Dh[m, a, 0, 0]) / sD[a]:+.2e}")


if __name__ == "__main__":
    main()
