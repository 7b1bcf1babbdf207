"""Per-rank kernel time of a G-GPU split of the headline sweep, emulated on
one GPU: every rank's row groups (lb_sym_partial_dev, sweep + group
reduction) timed alone with CUDA events, for G = 1, 2, 4, 8.  The slowest
rank against 1/G of the single-GPU time is the share a G-GPU run can reach
before collectives (this pool gives one GPU per call).

    python tools/rank_shares.py [N] [reps]
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_1702_08880_b200 as pkg  # noqa: E402
from paper_1702_08880_b200 import _lib, synthetic  # noqa: E402
from paper_1702_08880_b200.shard import ShardedSweep, local_fields, sym_rank_groups  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    dev = torch.device("cuda", 0)
    wl = synthetic.cfg5(n)
    params = pkg.CollisionParams(nu_hat=wl.nu_hat, mass_ratio_o=wl.mass_ratio_o)
    sh = ShardedSweep(n, wl.S, params, wl.eps_d, dev, align=1)
    f = [torch.from_numpy(a).to(dev) for a in local_fields(wl, 0, n)]
    sh.pack_local(*f)
    sh.all_gather()
    sh.sym_prepare()
    lib, h = _lib.load(), sh._ctx.handle
    st = torch.cuda.current_stream().cuda_stream
    buf = torch.empty((8,) + tuple(sh.tot.shape[1:]), dtype=torch.float64, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = {"N": n, "reps": reps}
    single = None
    for G in (1, 2, 4, 8):
        times = []
        for r in range(G):
            best = float("inf")
            for _ in range(reps):
                e0.record()
                _lib.check(lib.lb_sym_partial_dev(h, wl.S, wl.eps_d, r, G, buf.data_ptr(), st))
                e1.record()
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1))
            times.append(best)
        if G == 1:
            single = times[0]
        slow = max(times)
        out[f"G{G}"] = {"rank_ms": times, "slowest_ms": slow, "ideal_ms": single / G,
                        "share": single / G / slow, "groups": [sym_rank_groups(r, G) for r in range(G)]}
        print(f"G={G}: slowest rank {slow:.3f} ms vs ideal {single / G:.3f} ms -> "
              f"{100 * single / G / slow:.1f} % ({', '.join(f'{t:.3f}' for t in times)})")
    try:
        print(json.dumps(out), flush=True)
    except BrokenPipeError:  # output piped into head
        pass


if __name__ == "__main__":
    main()
