"""Device-pointer path (lb_pack_records_dev / lb_sweep_dev on torch's
stream) used by the multi-GPU layer and the bench: equals the host entry
bitwise, and per-rank outer shards emulated one after another on one GPU
(no cross-rank waiting) reproduce the full result bitwise."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _setup(n):
    import torch

    import paper_1702_08880_b200 as pkg
    from paper_1702_08880_b200 import synthetic

    wl = synthetic.cfg5(n)
    params = pkg.CollisionParams(nu_hat=wl.nu_hat, mass_ratio_o=wl.mass_ratio_o)
    data = pkg.QuadPointData(N=n, r=wl.r, z=wl.z, w=wl.w, f=wl.f, df_r=wl.df_r, df_z=wl.df_z)
    return torch, pkg, wl, params, data


def test_dev_path_on_torch_stream_equals_host_entry(gpu):
    torch, pkg, wl, params, data = _setup(8192)
    from paper_1702_08880_b200.shard import ShardedSweep, local_fields

    K0, D0 = pkg.fused_sweep(wl.r, wl.z, data, params, eps_d=wl.eps_d)
    dev = torch.device("cuda", 0)
    sh = ShardedSweep(wl.N, wl.S, params, wl.eps_d, dev, align=1)
    f = [torch.from_numpy(a).to(dev) for a in local_fields(wl, 0, wl.N)]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):  # a non-default stream: results must be ordered on it
        K, D = sh.step(*f)
        Kh, Dh = K.cpu(), D.cpu()
    torch.cuda.synchronize()
    assert np.array_equal(Kh.numpy(), K0) and np.array_equal(Dh.numpy(), D0)
    assert sh.launches == 7  # pack + Morton ordering (4) + sweep + combine


@pytest.mark.parametrize("world", [2, 3, 8])
def test_emulated_ranks_reproduce_full_result(gpu, world):
    torch, pkg, wl, params, data = _setup(4608)
    from paper_1702_08880_b200.shard import ShardPlan

    K0, D0 = pkg.fused_sweep(wl.r, wl.z, data, params, eps_d=wl.eps_d)
    plan = ShardPlan(wl.N, world, 9)
    for r in range(world):
        lo, hi = plan.bounds(r)
        K, D = pkg.fused_sweep(wl.r[lo:hi], wl.z[lo:hi], data, params, eps_d=wl.eps_d)
        assert np.array_equal(K, K0[lo:hi]) and np.array_equal(D, D0[lo:hi])
