"""Profiling driver: W warm-up + 1 measured D/K evaluation of the headline
workload (cfg5, N = 2^16, S = 2) through the device path, for ncu
(`-k regex:lb_sweep_kernel -s W -c 1`).  Prints the event-timed sweep."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_1702_08880_b200 as pkg  # noqa: E402
from paper_1702_08880_b200 import _lib, synthetic  # noqa: E402
from paper_1702_08880_b200.shard import ShardedSweep, local_fields  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    n = int(args[0]) if len(args) > 0 else 65536
    reps = int(args[1]) if len(args) > 1 else 4
    dev = torch.device("cuda", 0)
    S = int(next((a.split("=")[1] for a in sys.argv if a.startswith("--S=")), 2))
    sp = synthetic.CFG5_SPECIES if S == 2 else tuple(
        synthetic.SpeciesSpec(f"s{k}", m, q, T) for k, (m, q, T) in enumerate(
            [(1.0, -1.0, 1.0), (3670.0, 1.0, 1.0), (21900.0, 6.0, 0.5), (335000.0, 10.0, 0.5),
             (2.0, 1.0, 1.0), (3.0, 1.0, 1.0), (4.0, 1.0, 1.0), (5.0, 1.0, 1.0)][:S]))
    wl = synthetic.cfg5(n, species=sp)
    params = pkg.CollisionParams(nu_hat=wl.nu_hat, mass_ratio_o=wl.mass_ratio_o)
    sym = "--general" not in sys.argv
    world = int(next((a.split("=")[1] for a in sys.argv if a.startswith("--world=")), 1))
    rank = int(next((a.split("=")[1] for a in sys.argv if a.startswith("--rank=")), 0))
    sh = ShardedSweep(n, wl.S, params, wl.eps_d, dev, align=1, symmetric=sym)
    f = [torch.from_numpy(a).to(dev) for a in local_fields(wl, 0, n)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for k in range(reps):
        sh.pack_local(*f)
        sh.all_gather()
        if sh.symmetric:
            sh.sym_prepare()
            e0.record()
            if world > 1:  # one rank's row groups of a `world`-GPU split (per-rank kernel time)
                _lib.check(_lib.load().lb_sym_partial_dev(
                    sh._ctx.handle, wl.S, wl.eps_d, rank, world, sh.tot.data_ptr(),
                    torch.cuda.current_stream().cuda_stream))
            else:
                sh.sym_partial()
            e1.record()
            sh.sym_finish()
        else:
            e0.record()
            sh.sweep_local(f[0], f[1])
            e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if world > 1:
            print(f"rep {k}: rank {rank} of {world}: {ms:.3f} ms (x{world} = {ms * world:.2f} ms single-GPU equiv.)")
            continue
        print(f"rep {k}: sweep {ms:.3f} ms, {n * n / ms / 1e6:.3e} Gpairs/s... "
              f"model {pkg.flop_count(n, wl.S, n) / ms / 1e9:.2f} TFLOP/s, S={wl.S}, "
              f"{'symmetric' if sh.symmetric else 'general'}")


if __name__ == "__main__":
    t = time.time()
    main()
    print(f"wall {time.time() - t:.1f}s")
