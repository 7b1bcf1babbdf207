"""cProfile of one state-level operator call at BASELINE config 4 (shared
64x128 mesh, S = 4): where the host time beside the 21 ms of kernels goes."""
import cProfile
import io
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1702_08880_b200 as pkg  # noqa: E402
from paper_1702_08880_b200.synthetic import cfg4_state, q2_reference, uniform_q2_mesh  # noqa: E402

mesh, nodes = uniform_q2_mesh(5.0, 64, 128)
ref = q2_reference()
coeffs, nu_hat, mro = cfg4_state(nodes)
params = pkg.CollisionParams(nu_hat=nu_hat, mass_ratio_o=mro)
for _ in range(3):
    C = pkg.assemble_at(mesh, ref, coeffs, params)
pr = cProfile.Profile()
pr.enable()
C = pkg.assemble_at(mesh, ref, coeffs, params)
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(14)
print(s.getvalue()[:3500])
print(C.timings)
