"""End-to-end probe of the public fused_sweep at N = 2^16 (pinned inputs):
the API call vs the bare library call with pageable / page-locked outputs,
and the bench's call pattern (results held until the next call)."""
import sys, time
sys.path.insert(0, str(__import__('pathlib').Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1702_08880_b200 as pkg
from paper_1702_08880_b200 import _lib, synthetic
from paper_1702_08880_b200.kernel import coupling, _inner_fields
wl = synthetic.cfg5(65536)
params = pkg.CollisionParams(nu_hat=wl.nu_hat, mass_ratio_o=wl.mass_ratio_o)
host = [wl.r, wl.z, wl.w, wl.f, wl.df_r, wl.df_z]
pin = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in host]
hp = [t.numpy() for t in pin]
data = pkg.QuadPointData(N=65536, r=hp[0], z=hp[1], w=hp[2], f=hp[3], df_r=hp[4], df_z=hp[5])
S = 2; n = 65536
coK, coD = coupling(params)
ctx = _lib.context(); p = _lib.dptr; lib = _lib.load()
def run(K, D):
    _lib.check(lib.lb_fused_sweep_all(ctx.handle, n, S, p(hp[0]), p(hp[1]), p(hp[2]), p(hp[3]), p(hp[4]), p(hp[5]), p(coK), p(coD), float(wl.eps_d), p(K), p(D)))
Kp = torch.empty((n, S, 2), dtype=torch.float64).pin_memory().numpy()
Dp = torch.empty((n, S, 2, 2), dtype=torch.float64).pin_memory().numpy()
for name, f in [("api", lambda: pkg.fused_sweep(hp[0], hp[1], data, params, eps_d=wl.eps_d)),
                ("lib pageable", lambda: run(np.empty((n, S, 2)), np.empty((n, S, 2, 2)))),
                ("lib pinned", lambda: run(Kp, Dp))]:
    f(); ts = []
    for _ in range(8):
        t0 = time.perf_counter(); f(); ts.append(time.perf_counter() - t0)
    print(name, "%.3f ms" % (1e3 * min(ts)), "median %.3f" % (1e3 * sorted(ts)[4]))
# the bench's pattern: results kept until the next call returns
ts = []
K, D = pkg.fused_sweep(hp[0], hp[1], data, params, eps_d=wl.eps_d)
for _ in range(8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    K, D = pkg.fused_sweep(hp[0], hp[1], data, params, eps_d=wl.eps_d)
    ts.append(time.perf_counter() - t0)
print("bench pattern per step ms", [round(1e3 * t, 2) for t in ts])
