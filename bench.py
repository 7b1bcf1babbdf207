#!/usr/bin/env python
"""Benchmark: Landau point-pair evaluations/s at N = 2^16 (BASELINE.json).

Workload: BASELINE config 5 ("pure kernel sweep") at N = 65536 points, S = 2
species, outer = inner, seeded synthetic recipe (paper_1702_08880_b200/
synthetic.py).  One step = one D/K evaluation of all N^2 ordered pairs:
each rank packs its shard of the inner field state, one all-gather
replicates it (N > 1), each rank sweeps its N/G outer points against all N
inner points.  `value` = N^2 * steps / (max over ranks of the summed
device-timed step durations).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`--impl reference` times the reference algorithm's CPU implementation (the
C restatement in oracle/, all host threads) on a bounded outer sample of the
same workload, rank 0 only: the reference's own numba fused_sweep when the
unmodified reference is installed in baseline/_ref
(tools/install_reference.sh), else the C restatement in oracle/.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

METRIC = "Landau point-pair evals/s at N=2^16"
UNIT = "pairs/s"
def flops_per_pair(S: int) -> int:
    """The reference's flop model per ordered pair (kernel.py:560-574)."""
    return 165 + 20 * S * S


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms while active."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.idx)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        return self.summary()

    def summary(self):
        rows = []
        for _, ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), float(parts[3]), parts[5:9]))
            except ValueError:
                continue
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k, v in enumerate(r[3]) if v == "Active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows),
                "sm_max_mhz": max(r[1] for r in rows),
                "power_w_max": max(r[2] for r in rows),
                "samples": len(rows), "reasons": reasons}


def physical_gpu(local_rank: int) -> int:
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        ids = [v for v in vis.split(",") if v.strip()]
        if local_rank < len(ids) and ids[local_rank].strip().isdigit():
            return int(ids[local_rank])
    return local_rank


# ----------------------------------------------------------------- CPU side
def cpu_sample(wl, seconds: float, threads: int, min_outer: int = 128):
    """Time the oracle (reference algorithm restated in C, OpenMP) on a
    bounded sample: k evenly spaced outer points x all N inner points."""
    from oracle import oracle as O

    N = wl.N

    def run(k):
        idx = np.linspace(0, N - 1, k).astype(np.int64)
        t0 = time.perf_counter()
        K, D = O.fused_sweep(wl.r[idx], wl.z[idx], wl.r, wl.z, wl.w, wl.f, wl.df_r, wl.df_z,
                             wl.nu_hat, wl.mass_ratio_o, eps_d=wl.eps_d, threads=threads)
        return time.perf_counter() - t0, idx, K, D

    t, *_ = run(min_outer)  # warm (page-in, thread pool)
    rate = min_outer * N / max(t, 1e-9)
    k = int(min(N, max(min_outer, rate * seconds / N)))
    return k, run


def _import_reference():
    """The unmodified reference (axlandau, numba) installed in baseline/_ref
    by tools/install_reference.sh, or None."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "axlandau").is_dir():
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/lb_numba_cache")
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    try:
        import axlandau
    except Exception:  # numba missing or incompatible
        return None
    return axlandau


def reference_arm(args):
    """The reference's own CPU implementation of the path on this host: its
    numba fused_sweep (kernel.py:504-536, all host threads) when the
    unmodified reference is installed in baseline/_ref, else the C
    restatement in oracle/ (OpenMP); a bounded sample of outer points x all
    N inner points per step, rank 0 only."""
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    from oracle import oracle as O
    from paper_1702_08880_b200 import synthetic

    O.build()
    wl = synthetic.cfg5(args.n)
    threads = O.max_threads()
    # each step is a bounded sample sized so the whole run stays ~2 minutes
    per_step = min(args.ref_step_seconds, 120.0 / max(args.steps + args.warmup, 1))
    ax = _import_reference()
    port = None
    if ax is not None:
        data = ax.QuadPointData(N=wl.N, r=wl.r, z=wl.z, w=wl.w, f=wl.f, df_r=wl.df_r, df_z=wl.df_z)
        params = ax.kernel.CollisionParams(nu_hat=wl.nu_hat, mass_ratio_o=wl.mass_ratio_o)

        def run(k):
            idx = np.linspace(0, wl.N - 1, k).astype(np.int64)
            t0 = time.perf_counter()
            ax.fused_sweep(wl.r[idx], wl.z[idx], data, params, eps_d=wl.eps_d, workers=threads)
            return time.perf_counter() - t0, idx, None, None

        run(16)  # JIT compile + thread pool
        t, *_ = run(64)
        k = int(min(wl.N, max(64, 64 * per_step / max(t, 1e-9))))
        kind = "reference"
        sample = (f"{{k}} evenly spaced outer points x all {wl.N} inner points per step "
                  f"(the reference's own numba fused_sweep, kernel.py:504-536, workers={threads}; "
                  f"unmodified install in baseline/_ref)")
        kp, runp = cpu_sample(wl, min(per_step, 4.0), threads, min_outer=16)
        tp, *_ = runp(kp)
        port = {"value": kp * wl.N / tp, "unit": UNIT, "cores": threads,
                "sample": f"{kp} outer points x all {wl.N} inner points (oracle/ C restatement)"}
    else:
        k, run = cpu_sample(wl, per_step, threads, min_outer=16)
        kind = "port"
        sample = (f"{{k}} evenly spaced outer points x all {wl.N} inner points per step "
                  f"(oracle/ C restatement of kernel.py:306-493, OpenMP {threads} threads; the "
                  f"reference itself is not installed in baseline/_ref)")
    for _ in range(args.warmup):
        run(k)
    times = [run(k)[0] for _ in range(args.steps)]
    pairs = k * wl.N
    value = pairs * len(times) / sum(times)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"cfg5 pure kernel sweep N={wl.N} S={wl.S} (BASELINE configs[4])",
                   "N": wl.N, "S": wl.S, "sample_outer_points": k},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": sample.format(k=k)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "model_gflops": value * flops_per_pair(wl.S) / 1e9,
    }
    if port:
        line["oracle_port"] = port
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------- GPU side
def ours_arm(args):
    import torch
    import torch.distributed as dist

    import paper_1702_08880_b200 as pkg
    from paper_1702_08880_b200 import _lib, synthetic
    from paper_1702_08880_b200.shard import ShardedSweep, local_fields

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local_rank = env_int("LOCAL_RANK", 0)
    if world != args.gpus and world > 1:
        print(f"warning: WORLD_SIZE={world} but --gpus={args.gpus}", file=sys.stderr)
    # one process per GPU; --backend gloo with more ranks than GPUs is a
    # functional check of the sharded path only (host collectives, ranks
    # time-share a GPU, no kernel waits on another rank) -- never a timing
    dev_index = local_rank % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.backend)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def allmax(vals):
        t = torch.tensor(vals, dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    wl = synthetic.cfg5(args.n)
    N, S = wl.N, wl.S
    params = pkg.CollisionParams(nu_hat=wl.nu_hat, mass_ratio_o=wl.mass_ratio_o)
    sh = ShardedSweep(N, S, params, wl.eps_d, dev, align=1, p2p=args.p2p)
    nloc = sh.hi - sh.lo
    nacc = sh.nacc  # accumulator species sets (1: rank-one species collapse)
    host = local_fields(wl, sh.lo, sh.hi)
    d_fields = [torch.from_numpy(a).to(dev) for a in host]
    lib = _lib.load()
    ctx = _lib.context(dev_index)

    # FP64 peak at this box's clocks (DFMA microbenchmark; MEASURED_PEAKS.json has none)
    tf, ms = _lib.C.c_double(), _lib.C.c_double()
    bursts = []
    t_end = time.time() + args.peak_seconds
    while time.time() < t_end or not bursts:
        _lib.check(lib.lb_fp64_peak(ctx.handle, _lib.C.byref(tf), _lib.C.byref(ms)))
        bursts.append(tf.value)
    fp64_burst = max(bursts)
    fp64_sustained = statistics.median(bursts[len(bursts) // 2:])

    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)  # 256 MiB > 126 MB L2
    st = torch.cuda.current_stream(dev)

    def step(ev=None):
        sh.pack_local(*d_fields)
        sh.all_gather()
        if sh.symmetric:  # each unordered pair once; tile pairs split over ranks
            sh.sym_prepare()
            if ev is not None:
                ev[0].record(st)
            sh.sym_partial()  # lb_symsweep_kernel + its fixed-order reduction
            if ev is not None:
                ev[1].record(st)
            sh.sym_reduce()
            sh.sym_finish()
        else:
            if ev is not None:
                ev[0].record(st)
            sh.sweep_local(d_fields[0], d_fields[1])
            if ev is not None:
                ev[1].record(st)

    for _ in range(args.warmup):
        step()
    barrier()

    sampler = ClockSampler(physical_gpu(dev_index)) if args.clocks else None
    if sampler:
        sampler.start()
    E = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    sh.launches = 0
    # execution counters of the symmetric sweep (thread-steps by kind) over
    # the timed steps: with the per-step FP64 counts of this library's SASS
    # they give the executed FP64 work (tools/sass_fp64.py)
    counting = sh.symmetric and nacc == 1
    if counting:
        _lib.check(lib.lb_sym_counters(sh._ctx.handle, 1, None))
    barrier()
    for k in range(args.steps):
        flush.fill_(float(k))  # evict L2 between timed steps (outside the step events)
        E[k][0].record(st)
        step(ev=(E[k][1], E[k][2]))
        E[k][3].record(st)
    barrier()
    clocks = sampler.stop() if sampler else None
    launches = sh.launches
    step_ms = [E[k][0].elapsed_time(E[k][3]) for k in range(args.steps)]
    sweep_ms = [E[k][1].elapsed_time(E[k][2]) for k in range(args.steps)]
    tot_ms, tot_sweep_ms = allmax([sum(step_ms), sum(sweep_ms)])
    pairs_step = N * N
    value = pairs_step * args.steps / (tot_ms * 1e-3)
    counts = None
    if counting:
        cbuf = (_lib.C.c_ulonglong * 3)()
        _lib.check(lib.lb_sym_counters(sh._ctx.handle, 0, cbuf))
        counts = [int(c) for c in cbuf]
    # roofline of the dominant kernel on this rank: executed FP64 flops per
    # launch / launch time (the hardware fraction), and the reference's flop
    # model per ordered pair delivered (model_frac, can exceed 1: the
    # symmetric path evaluates each unordered pair once and the species
    # collapse makes S = 2 cost what S = 1 costs)
    sweep_avg_s = sum(sweep_ms) / len(sweep_ms) * 1e-3
    # ordered pairs this rank's sweep delivers: its outer points x N (general
    # path) or its 1/world share of the tile pairs, each feeding both points
    flops_launch = pkg.flop_count(N, S, N / world if sh.symmetric else nloc)
    model_tf = flops_launch / sweep_avg_s / 1e12
    executed = None
    if counts is not None:
        from tools import sass_fp64

        try:
            # the kernel variant this eps_d selects (merged mask/guard compare
            # when eps_d^2 > 1e-300, landau_pair.cuh pair_stage1)
            sass = sass_fp64.analyse(Path(lib._name), sass_fp64.KERNELS[wl.eps_d ** 2 > 1e-300])
            ex = sass_fp64.executed(counts, sass)
            executed = {
                "flops_per_launch": ex["flops"] / args.steps,
                "fp64_instr_per_launch": ex["instr"] / args.steps,
                "pairs_per_launch": ex["pairs"] / args.steps,
                "thread_steps": {"off_diagonal": counts[0], "diagonal": counts[1],
                                 "series_branch": counts[2], "over_steps": args.steps},
                "sass_per_thread_step": {"instr": sass["instr"], "flops": sass["flops"],
                                         "pairs": sass["pairs_per_thread_step"]},
                "fp64_instr_per_unordered_pair": ex["instr"] / max(ex["pairs"], 1),
                "derivation": "kernel execution counters (lb_sym_counters) x FP64 "
                              "instructions per thread-step counted in this library's "
                              "SASS (tools/sass_fp64.py: DFMA = 2 flops, DMUL/DADD = 1); "
                              "FP64 work outside the pair loop (< 1 %) not counted",
            }
        except (RuntimeError, OSError, subprocess.CalledProcessError) as err:
            executed = {"error": str(err)}
    if executed and "flops_per_launch" in executed:
        achieved_tf = executed["flops_per_launch"] / sweep_avg_s / 1e12
        bound_note = "executed FP64 flops (in-run counters x SASS)"
    else:  # general path / uncollapsed kernels: the model figure only
        achieved_tf = model_tf
        bound_note = "model flops (no execution counters for this kernel)"

    # e2e through the public API with pinned host buffers (copies inside the timed region)
    e2e = None
    if world == 1:
        pin = [torch.from_numpy(a).pin_memory() for a in host]
        hp = [t.numpy() for t in pin]
        data = pkg.QuadPointData(N=N, r=hp[0], z=hp[1], w=hp[2], f=hp[3], df_r=hp[4], df_z=hp[5])
        # warm-up calls, results held as in the timed loop (the outputs come
        # from the caching pinned allocator, which needs two live sets)
        for _ in range(max(2, args.warmup)):
            K, D = pkg.fused_sweep(hp[0], hp[1], data, params, eps_d=wl.eps_d)
        ts = []
        for _ in range(args.e2e_steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            K, D = pkg.fused_sweep(hp[0], hp[1], data, params, eps_d=wl.eps_d)
            ts.append(time.perf_counter() - t0)
        # the all-points call (outer == inner) uploads r, z, w, f, df_r, df_z
        # once (kernel.py:504 called as in assembly.py:148); no outer copies
        h2d = 8 * (3 + 3 * S) * N
        d2h = 8 * 6 * S * N
        e2e = {"value": pairs_step * len(ts) / sum(ts), "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "api": "paper_1702_08880_b200.fused_sweep (numpy in/out, pinned host)"}
    else:
        pin = [torch.from_numpy(a).pin_memory() for a in host]
        Kh = torch.empty((nloc, S, 2), dtype=torch.float64).pin_memory()
        Dh = torch.empty((nloc, S, 2, 2), dtype=torch.float64).pin_memory()
        ts = []
        for it in range(args.e2e_steps + 1):
            barrier()
            t0 = time.perf_counter()
            for dst, src in zip(d_fields, pin):
                dst.copy_(src, non_blocking=True)
            K, D = sh.step(*d_fields)
            Kh.copy_(K, non_blocking=True)
            Dh.copy_(D, non_blocking=True)
            torch.cuda.synchronize()
            if it:
                ts.append(time.perf_counter() - t0)
        tmax = allmax([sum(ts)])[0]
        e2e = {"value": pairs_step * len(ts) / tmax, "unit": UNIT,
               "h2d_bytes_per_step": 8 * (3 + 3 * S) * nloc,
               "d2h_bytes_per_step": 8 * 6 * S * nloc,
               "api": "paper_1702_08880_b200.shard.ShardedSweep (pinned host in/out)"}

    # CPU baseline (rank 0, N=1): oracle on a bounded sample; doubles as a parity check
    cpu = None
    parity = None
    if world == 1 and rank == 0 and args.cpu_seconds > 0:
        from oracle import oracle as O

        O.build()
        threads = O.max_threads()
        k, run = cpu_sample(wl, args.cpu_seconds, threads)
        t, idx, Kr, Dr = run(k)
        cpu = {"value": k * N / t, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{k} evenly spaced outer points x all {N} inner points "
                         f"(oracle/ C restatement of kernel.py:306-493, OpenMP, {t:.1f} s)"}
        parity = O.per_component_scaled_error(K[idx], D[idx], Kr, Dr)
        # one core as well (the survey's per-core reference rate)
        k1, run1 = cpu_sample(wl, min(2.0, args.cpu_seconds / 5), 1, min_outer=16)
        t1, *_ = run1(k1)
        cpu["single_core_value"] = k1 * N / t1

    check = None
    bitwise = None
    if args.check:  # every rank's own rows vs the oracle on a sample (functional check)
        from oracle import oracle as O

        Kh_, Dh_ = sh.K.cpu().numpy(), sh.D.cpu().numpy()
        idx = np.arange(sh.lo, sh.hi, max(1, (sh.hi - sh.lo) // 64))
        Kr, Dr = O.fused_sweep(wl.r[idx], wl.z[idx], wl.r, wl.z, wl.w, wl.f, wl.df_r, wl.df_z,
                               wl.nu_hat, wl.mass_ratio_o, eps_d=wl.eps_d)
        err = O.per_component_scaled_error(Kh_[idx - sh.lo], Dh_[idx - sh.lo], Kr, Dr)
        check = allmax([err])[0]
        # this rank's rows vs the single-GPU all-points call on its device
        data1 = pkg.QuadPointData(N=N, r=wl.r, z=wl.z, w=wl.w, f=wl.f, df_r=wl.df_r,
                                  df_z=wl.df_z)
        K1, D1 = pkg.fused_sweep(wl.r, wl.z, data1, params, eps_d=wl.eps_d)
        same = (np.array_equal(Kh_, K1[sh.lo:sh.hi]) and np.array_equal(Dh_, D1[sh.lo:sh.hi]))
        bitwise = allmax([0.0 if same else 1.0])[0] == 0.0
    # DRAM traffic of the sweep launch: not measurable without a profiler;
    # taken from the committed ncu --set full capture, labelled with the
    # kernel version it was measured on
    traffic, traffic_src = None, None
    tf_file = ROOT / "profiles" / "sweep_traffic.json"
    if tf_file.exists() and sh.symmetric and nacc == 1:
        try:
            prof = json.loads(tf_file.read_text())
            traffic = prof.get("bytes_per_launch")
            traffic_src = {"source": prof.get("source"), "kernel_version": prof.get("version"),
                           "measured": "ncu --set full (dram__bytes_read.sum + "
                                       "dram__bytes_write.sum), one launch, committed profile"}
        except (OSError, ValueError):
            traffic = None

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (BASELINE config 5 recipe, seeded)",
            "config": {"workload": f"cfg5 pure kernel sweep N={N} S={S} (BASELINE configs[4])",
                       "N": N, "S": S, "outer_per_gpu": nloc, "pairs_per_step": pairs_step,
                       "parallelism": f"outer-point shards x{world}" + (
                           f" + {args.backend} all-gather of packed field state"
                           + ((" + row-group split, peer-memory (CUDA IPC) read of the group "
                               "sums fused with the combine" if sh.p2p else
                               " + row-group split, all-gather of the group sums")
                              if sh.symmetric else "")
                           if world > 1 else ""),
                       "l2": "flushed between timed steps (256 MiB write, outside step events)"},
            "roofline": {"bound": "fp64", "achieved": achieved_tf, "peak": fp64_sustained,
                         "unit": "TFLOP/s", "frac": achieved_tf / fp64_sustained,
                         "traffic": traffic, "traffic_source": traffic_src,
                         "achieved_is": bound_note,
                         "kernel": ((f"lb_symsweep_ib_kernel<1>" if nacc == 1 else f"lb_symsweep_kernel<{nacc}>")
                                    + " + lb_symreduce_kernel" if sh.symmetric
                                    else f"lb_sweep_kernel<{nacc}> (+ lb_combine_kernel, <1%)"),
                         "executed_fp64": executed,
                         "model_achieved": model_tf, "model_frac": model_tf / fp64_sustained,
                         "model_flops": "165+20*S^2 per ordered pair delivered (kernel.py:560-574)",
                         "species_collapsed": nacc == 1 and S > 1,
                         "peak_source": "measured DFMA microbenchmark on this GPU "
                                        "(lb_fp64_peak, median of the last half of the probe)",
                         "peak_burst": fp64_burst, "frac_of_nominal_37.2": achieved_tf / 37.2},
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
            "kernel_ms_per_step": tot_sweep_ms / args.steps,
            "path": "symmetric (unordered pairs)" if sh.symmetric else "general (ordered pairs)",
        }
        if cpu:
            line["cpu_baseline"] = cpu
            line["parity_scaled_err_vs_oracle"] = parity
        if check is not None:
            line["check_all_ranks_scaled_err_vs_oracle"] = check
            line["check_all_ranks_bitwise_equal_single"] = bitwise
        if args.backend != "nccl" and world > 1:
            line["note"] = f"functional run over {args.backend} (ranks may share a GPU): not a timing"

        print(json.dumps(line), flush=True)
    sh.close()  # peer-memory mode: unmap the peers' buffers (collective)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--points", dest="n", type=int, default=65536,
                    help="N (inner = outer points); the metric is quoted at 2^16")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-step-seconds", type=float, default=6.0)
    ap.add_argument("--no-clocks", dest="clocks", action="store_false")
    ap.add_argument("--peak-seconds", type=float, default=1.0,
                    help="duration of the FP64 DFMA peak probe (the roofline denominator)")
    ap.add_argument("--backend", choices=["nccl", "gloo"], default="nccl")
    ap.add_argument("--p2p", action="store_true",
                    help="symmetric path: peer-memory (CUDA IPC / NVLink) reduction fused with "
                         "the combine instead of the NCCL all-reduce")
    ap.add_argument("--check", action="store_true",
                    help="compare every rank's rows with the oracle on a sample")
    args = ap.parse_args()
    if args.warmup < 3:
        print("note: raising --warmup to the required minimum of 3", file=sys.stderr)
        args.warmup = 3
    return reference_arm(args) if args.impl == "reference" else ours_arm(args)


if __name__ == "__main__":
    sys.exit(main())
