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

    K0, D0 = pkg.fused_sweep(wl.r[:-1], wl.z[:-1], data, params, eps_d=wl.eps_d)
    dev = torch.device("cuda", 0)
    sh = ShardedSweep(wl.N, wl.S, params, wl.eps_d, dev, align=1, symmetric=False)
    f = [torch.from_numpy(a).to(dev) for a in local_fields(wl, 0, wl.N)]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):  # a non-default stream: results must be ordered on it
        K, D = sh.step(*f)
        Kh, Dh = K.cpu(), D.cpu()
    torch.cuda.synchronize()
    assert np.array_equal(Kh.numpy()[:-1], K0) and np.array_equal(Dh.numpy()[:-1], D0)
    assert sh.launches == 7  # pack + Morton ordering (4 own + CUB sort) + sweep + combine


@pytest.mark.parametrize("world", [2, 3, 8])
def test_emulated_ranks_reproduce_full_result(gpu, world):
    """General path: per-rank outer shards, run one after another on one GPU
    (no cross-rank waiting), equal the single-call rows bitwise."""
    torch, pkg, wl, params, data = _setup(4608)
    from paper_1702_08880_b200.shard import ShardPlan

    half = wl.N - 1  # not the all-points call: the general (ordered-pair) path
    K0, D0 = pkg.fused_sweep(wl.r[:half], wl.z[:half], data, params, eps_d=wl.eps_d)
    plan = ShardPlan(half, world, 9)
    for r in range(world):
        lo, hi = plan.bounds(r)
        K, D = pkg.fused_sweep(wl.r[lo:hi], wl.z[lo:hi], data, params, eps_d=wl.eps_d)
        assert np.array_equal(K, K0[lo:hi]) and np.array_equal(D, D0[lo:hi])


def test_symmetric_dev_path_matches_general(gpu, oracle):
    """Symmetric all-points path (tile pairs, each unordered pair once) vs the
    general sweep and the oracle, on a ragged N (not a multiple of 128)."""
    torch, pkg, wl, params, data = _setup(5000)
    from paper_1702_08880_b200.shard import ShardedSweep, local_fields

    dev = torch.device("cuda", 0)
    f = [torch.from_numpy(a).to(dev) for a in local_fields(wl, 0, wl.N)]
    sym = ShardedSweep(wl.N, wl.S, params, wl.eps_d, dev, align=1)
    gen = ShardedSweep(wl.N, wl.S, params, wl.eps_d, dev, align=1, symmetric=False)
    assert sym.symmetric and not gen.symmetric
    Ks, Ds = (t.cpu().numpy() for t in sym.step(*f))
    Kg, Dg = (t.cpu().numpy() for t in gen.step(*f))
    Kr, Dr = oracle.fused_sweep(wl.r, wl.z, wl.r, wl.z, wl.w, wl.f, wl.df_r, wl.df_z,
                                wl.nu_hat, wl.mass_ratio_o, eps_d=wl.eps_d)
    from conftest import worst_component

    e_sg = worst_component(Ks, Ds, Kg, Dg)
    e_so = worst_component(Ks, Ds, Kr, Dr)
    print("sym vs general", e_sg, "sym vs oracle", e_so)
    assert e_sg < 1e-12 and e_so < 1e-10
    # deterministic run to run
    K2, D2 = (t.cpu().numpy() for t in sym.step(*f))
    assert np.array_equal(K2, Ks) and np.array_equal(D2, Ds)
    # host all-points entry == device symmetric path, bitwise
    Kh, Dh = pkg.fused_sweep(wl.r, wl.z, data, params, eps_d=wl.eps_d)
    assert np.array_equal(Kh, Ks) and np.array_equal(Dh, Ds)


@pytest.mark.parametrize("world", [2, 3, 5, 8])
def test_symmetric_ranks_bitwise_equal_single(gpu, world):
    """Emulate `world` ranks on one GPU one after another: each rank's row
    groups (lb_sym_groups) -> its group sums; the eight group sums combined in
    group order reproduce the single-rank K and D BITWISE, as the reference
    promises for `workers` (kernel.py:508-511, test_kernel.py:197-212)."""
    import ctypes

    torch, pkg, wl, params, data = _setup(4096 + 77)
    from paper_1702_08880_b200 import _lib
    from paper_1702_08880_b200.shard import SYM_GROUPS, ShardedSweep, local_fields, sym_rank_groups

    dev = torch.device("cuda", 0)
    f = [torch.from_numpy(a).to(dev) for a in local_fields(wl, 0, wl.N)]
    sh = ShardedSweep(wl.N, wl.S, params, wl.eps_d, dev, align=1)
    K0, D0 = (t.cpu().numpy() for t in sh.step(*f))
    lib, h = _lib.load(), sh._ctx.handle
    st = torch.cuda.current_stream().cuda_stream
    groups = torch.full((SYM_GROUPS,) + tuple(sh.tot.shape[1:]), float("nan"), dtype=torch.float64,
                        device=dev)
    for r in range(world):
        g0, g1 = sym_rank_groups(r, world)
        a, b = ctypes.c_int(-1), ctypes.c_int(-1)
        assert lib.lb_sym_groups(r, world, ctypes.byref(a), ctypes.byref(b)) == SYM_GROUPS
        assert (a.value, b.value) == (g0, g1)
        part = torch.full((max(g1 - g0, 1),) + tuple(sh.tot.shape[1:]), float("nan"),
                          dtype=torch.float64, device=dev)
        _lib.check(lib.lb_sym_partial_dev(h, wl.S, wl.eps_d, r, world, part.data_ptr(), st))
        groups[g0:g1] = part[:g1 - g0]
    K = torch.empty_like(sh.K)
    D = torch.empty_like(sh.D)
    p = _lib.dptr
    _lib.check(lib.lb_sym_combine_dev(h, wl.S, groups.data_ptr(), p(sh.coK), p(sh.coD), 0, wl.N,
                                      K.data_ptr(), D.data_ptr(), st))
    torch.cuda.synchronize()
    assert np.array_equal(K.cpu().numpy(), K0) and np.array_equal(D.cpu().numpy(), D0)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_multirank_bench_functional(gpu, world):
    """The multi-GPU bench path end to end with `world` ranks over gloo on
    one GPU (ranks time-share the device; no kernel waits on another rank):
    all-gather of packed records, symmetric row-group split, all-gather of
    the group sums, per-rank combine -- every rank's rows vs the oracle, and
    bitwise equal to the single-GPU all-points call."""
    import json
    import socket
    import subprocess
    import sys

    from conftest import ROOT

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1", f"--master-port={port}",
           "bench.py", "--gpus", str(world), "--backend", "gloo", "--check", "--steps", "3",
           "--warmup", "3", "--points", "12000", "--no-clocks", "--e2e-steps", "1"]
    out = subprocess.run(cmd, cwd=str(ROOT), capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == world
    print("multi-rank", world, "check", line["check_all_ranks_scaled_err_vs_oracle"])
    assert line["check_all_ranks_scaled_err_vs_oracle"] < 1e-10
    assert line["check_all_ranks_bitwise_equal_single"] is True


@pytest.mark.parametrize("world", [2, 3])
def test_multirank_bench_p2p(gpu, world):
    """The peer-memory reduction (CUDA IPC mappings of every rank's group
    sums, read by one fused reduce + combine kernel) with `world` ranks over
    gloo on one GPU (ordering by host barriers; no kernel waits on another
    rank): every rank's rows vs the oracle and bitwise equal to one GPU."""
    import json
    import socket
    import subprocess
    import sys

    from conftest import ROOT

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1", f"--master-port={port}",
           "bench.py", "--gpus", str(world), "--backend", "gloo", "--p2p", "--check", "--steps", "3",
           "--warmup", "3", "--points", "12000", "--no-clocks", "--e2e-steps", "2"]
    out = subprocess.run(cmd, cwd=str(ROOT), capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert "peer-memory" in line["config"]["parallelism"]
    print("p2p multi-rank", world, "check", line["check_all_ranks_scaled_err_vs_oracle"])
    assert line["check_all_ranks_scaled_err_vs_oracle"] < 1e-10
    assert line["check_all_ranks_bitwise_equal_single"] is True


@pytest.mark.parametrize("world,case", [(1, "cfg3"), (2, "cfg3"), (3, "hanging"), (2, "cfg2")])
def test_sharded_operator(gpu, tmp_path, world, case):
    """Multi-GPU state-level operator (cells sharded, device sampling,
    all-gather, symmetric row-group split, all-gather of (w, K, D), element
    contraction + CSR gather), `world` ranks over gloo on one GPU, vs the
    reference blocks -- and bitwise equal to the single-GPU operator."""
    import socket
    import subprocess
    import sys

    from conftest import ROOT, blocks_from, golden

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = tmp_path / "blocks.npz"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1", f"--master-port={port}",
           "tools/sharded_operator_check.py", case, str(out), "gloo"]
    res = subprocess.run(cmd, cwd=str(ROOT), capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    d = np.load(out)
    worst = 0.0
    for a, ref in enumerate(blocks_from(golden(case))):
        r = ref.toarray()
        worst = max(worst, np.abs(d[f"b{a}"] - r).max() / np.abs(r).max())
    print(f"sharded operator {case} world={world}", worst)
    assert worst < 1e-10
    assert bool(d["bitwise_single"])


def test_bench_json_contract(gpu):
    """bench.py prints one JSON line with the driver's keys (short run)."""
    import json
    import subprocess
    import sys

    from conftest import ROOT

    out = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3",
                          "--points", "8192", "--cpu-seconds", "1", "--e2e-steps", "1",
                          "--peak-seconds", "0.1"], cwd=str(ROOT), capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["steps"] == 3 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"]
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in d["cpu_baseline"]
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"]
    assert d["parity_scaled_err_vs_oracle"] < 1e-10
