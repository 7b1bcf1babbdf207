"""Time the operator-level entries on the GPU for the reference fixtures:
assemble_collision (data in) and assemble_at (state in), per call, with
device phase timings."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))

import numpy as np  # noqa: E402

from conftest import data_from, golden, mesh_from, params_from, ref_from  # noqa: E402
import paper_1702_08880_b200 as pkg  # noqa: E402

for case in sys.argv[1:] or ["cfg1", "cfg3", "cfg2"]:
    g = golden(case)
    mesh, ref, data, params = mesh_from(g), ref_from(g), data_from(g), params_from(g)
    coeffs = np.array(g["coeffs"])  # the fixture is a lazy npz: read once, outside the timing
    for name, fn in (("assemble_collision", lambda: pkg.assemble_collision(mesh, ref, data, params)),
                     ("assemble_at", lambda: pkg.assemble_at(mesh, ref, coeffs, params))):
        fn()
        ts = []
        for _ in range(20):
            t0 = time.perf_counter()
            cm = fn()
            ts.append(time.perf_counter() - t0)
        t = np.median(ts)
        print(f"{case:6s} N={data.N:6d} S={data.f.shape[0]} {name:18s} {t*1e3:8.3f} ms/call  "
              f"device kernel {cm.timings['kernel']*1e3:.3f} fe {cm.timings['fe_transform']*1e3:.3f} "
              f"host scatter {cm.timings['scatter']*1e3:.3f} ms")
