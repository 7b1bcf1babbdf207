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


# ---------------------------------------------------------------- symmetric path
def _sym_fns(wl):
    """numpy stand-ins for the symmetric path's three device steps: the sum of
    row group g (points [128 B(g), 128 B(g+1)) as inner points, B(g) =
    nt g / 8) is the oracle sweep of every point against that inner subset,
    stored as the 5S accumulators (K_r, K_z, D_rr, D_rz, D_zz per species);
    the combine adds the eight groups in group order."""
    from oracle import oracle as O
    from paper_1702_08880_b200.shard import SYM_GROUPS, sym_rank_groups

    n, S = wl.N, wl.S
    nt = -(-n // 128)

    def prepare(rec):
        pass

    def partial(tot):
        rank, world = dist.get_rank(), dist.get_world_size()
        g0, g1 = sym_rank_groups(rank, world)
        for g in range(g0, g1):
            lo, hi = 128 * (nt * g // SYM_GROUPS), min(n, 128 * (nt * (g + 1) // SYM_GROUPS))
            tot[g - g0].zero_()
            if lo >= hi:
                continue
            K, D = O.fused_sweep(wl.r, wl.z, wl.r[lo:hi], wl.z[lo:hi], wl.w[lo:hi],
                                 np.ascontiguousarray(wl.f[:, lo:hi]),
                                 np.ascontiguousarray(wl.df_r[:, lo:hi]),
                                 np.ascontiguousarray(wl.df_z[:, lo:hi]), wl.nu_hat,
                                 wl.mass_ratio_o, eps_d=wl.eps_d, threads=1)
            acc = np.concatenate([K, D.reshape(n, S, 4)[:, :, [0, 1, 3]]], axis=2)  # (n, S, 5)
            tot[g - g0, :, :n] = torch.from_numpy(acc.reshape(n, 5 * S).T.copy())

    def combine(groups, q0, q1, K, D):
        assert len(groups) == SYM_GROUPS
        v = groups[0].clone()
        for g in range(1, SYM_GROUPS):
            v = v + groups[g]
        a = v[:, q0:q1].T.reshape(q1 - q0, S, 5)
        K.copy_(a[:, :, 0:2])
        D[:, :, 0, 0] = a[:, :, 2]
        D[:, :, 0, 1] = a[:, :, 3]
        D[:, :, 1, 0] = a[:, :, 3]
        D[:, :, 1, 1] = a[:, :, 4]

    return prepare, partial, combine


def _sym_worker(rank, world, port, n, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1702_08880_b200 import synthetic
        from paper_1702_08880_b200.shard import ShardedSweep, local_fields

        wl = synthetic.cfg5(n, seed=78)
        params = type("P", (), {"nu_hat": wl.nu_hat, "mass_ratio_o": wl.mass_ratio_o})
        sh = ShardedSweep(n, wl.S, params, wl.eps_d, "cpu", align=9, pack_fn=_pack_cpu,
                          sweep_fn=_make_sweep(wl.nu_hat, wl.mass_ratio_o, wl.eps_d),
                          sym_fns=_sym_fns(wl))
        assert sh.symmetric
        fields = [torch.from_numpy(a) for a in local_fields(wl, sh.lo, sh.hi)]
        K, D = sh.step(*fields)
        np.savez(os.path.join(out_dir, f"w{world}_rank{rank}.npz"), K=K.numpy(), D=D.numpy(),
                 lo=sh.lo, hi=sh.hi, g0=sh.g0, g1=sh.g1)
    finally:
        dist.destroy_process_group()


def test_symmetric_host_logic_bitwise_over_world_sizes(tmp_path):
    """Symmetric path host logic over gloo (world 1, 2, 3): every rank owns
    whole row groups, the group sums are all-gathered and each owner adds the
    eight in group order -- so K and D are bitwise identical for every world
    size (kernel.py:508-511), and match the full oracle sweep."""
    from oracle import oracle as O
    from paper_1702_08880_b200 import synthetic

    O.build()
    n = 1161  # 10 tiles of 128 (ragged), 129 cells
    res = {}
    for world in (1, 2, 3):
        mp.spawn(_sym_worker, args=(world, _free_port(), n, str(tmp_path)), nprocs=world,
                 join=True)
        K = np.empty((n, 2, 2))
        D = np.empty((n, 2, 2, 2))
        groups = []
        for rank in range(world):
            d = np.load(tmp_path / f"w{world}_rank{rank}.npz")
            lo, hi = int(d["lo"]), int(d["hi"])
            K[lo:hi], D[lo:hi] = d["K"], d["D"]
            groups.append((int(d["g0"]), int(d["g1"])))
        assert groups[0][0] == 0 and groups[-1][1] == 8
        assert all(groups[k][1] == groups[k + 1][0] for k in range(world - 1))
        res[world] = (K, D)
    for world in (2, 3):
        assert np.array_equal(res[world][0], res[1][0]) and np.array_equal(res[world][1], res[1][1])
    wl = synthetic.cfg5(n, seed=78)
    Kf, Df = O.fused_sweep(wl.r, wl.z, wl.r, wl.z, wl.w, wl.f, wl.df_r, wl.df_z, wl.nu_hat,
                           wl.mass_ratio_o, eps_d=wl.eps_d, threads=1)
    assert O.per_component_scaled_error(res[1][0], res[1][1], Kf, Df) < 1e-12
