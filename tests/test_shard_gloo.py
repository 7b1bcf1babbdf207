"""Multi-rank host logic of the sharded path on CPU: world_size 2 (and 3)
over `gloo`, with the device pack / sweep swapped for CPU stand-ins (the
record layout restated in numpy, the oracle sweep).  Checks that outer-point
sharding + the all-gather of packed inner records reproduce the
single-process result bitwise, including uneven (cell-aligned) shards."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _pack_cpu(r, z, w, f, dfr, dfz, out):
    S = f.shape[0]
    out.zero_()
    out[:, 0] = r
    out[:, 1] = z
    out[:, 2] = r * r
    out[:, 3] = torch.where(r > 0, 1.0 / torch.where(r > 0, r, torch.ones_like(r)),
                            torch.zeros_like(r))
    for b in range(S):
        out[:, 4 + 3 * b] = dfr[b] * w
        out[:, 5 + 3 * b] = dfz[b] * w
        out[:, 6 + 3 * b] = f[b] * w


def _make_sweep(nu, mro, eps_d):
    from oracle import oracle as O

    def sweep(ro, zo, rec, K, D):
        rec = rec.numpy()
        S = K.shape[1]
        n = rec.shape[0]
        f = np.ascontiguousarray(rec[:, 6:4 + 3 * S:3].T)
        dfr = np.ascontiguousarray(rec[:, 4:4 + 3 * S:3].T)
        dfz = np.ascontiguousarray(rec[:, 5:4 + 3 * S:3].T)
        Kn, Dn = O.fused_sweep(ro.numpy(), zo.numpy(), rec[:, 0], rec[:, 1], np.ones(n), f, dfr,
                               dfz, nu, mro, eps_d=eps_d, threads=1)
        K.copy_(torch.from_numpy(Kn))
        D.copy_(torch.from_numpy(Dn))

    return sweep


def _worker(rank, world, port, n, align, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1702_08880_b200 import synthetic
        from paper_1702_08880_b200.shard import ShardedSweep, local_fields

        wl = synthetic.cfg5(n, seed=77)
        params = type("P", (), {"nu_hat": wl.nu_hat, "mass_ratio_o": wl.mass_ratio_o})
        sh = ShardedSweep(n, wl.S, params, wl.eps_d, "cpu", align=align, pack_fn=_pack_cpu,
                          sweep_fn=_make_sweep(wl.nu_hat, wl.mass_ratio_o, wl.eps_d))
        fields = [torch.from_numpy(a) for a in local_fields(wl, sh.lo, sh.hi)]
        K, D = sh.step(*fields)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), K=K.numpy(), D=D.numpy(),
                 lo=sh.lo, hi=sh.hi)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,align", [(2, 1152, 9), (3, 1000, 9), (2, 1024, 1)])
def test_sharded_equals_single(tmp_path, world, n, align):
    from oracle import oracle as O
    from paper_1702_08880_b200 import synthetic

    O.build()
    mp.spawn(_worker, args=(world, _free_port(), n, align, str(tmp_path)), nprocs=world,
             join=True)
    wl = synthetic.cfg5(n, seed=77)
    Kf, Df = O.fused_sweep(wl.r, wl.z, wl.r, wl.z, wl.w, wl.f, wl.df_r, wl.df_z, wl.nu_hat,
                           wl.mass_ratio_o, eps_d=wl.eps_d, threads=1)
    covered = 0
    for rank in range(world):
        d = np.load(tmp_path / f"rank{rank}.npz")
        lo, hi = int(d["lo"]), int(d["hi"])
        if align > 1 and hi < n:
            assert hi % align == 0
        covered += hi - lo
        assert np.array_equal(d["K"], Kf[lo:hi])
        assert np.array_equal(d["D"], Df[lo:hi])
    assert covered == n
