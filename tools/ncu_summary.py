"""Summarise an ncu --set full report of the sweep kernel into a small JSON
(+ print), and a launch-list CSV into per-kernel shares.

    python tools/ncu_summary.py REPORT.ncu-rep [LAUNCHES.csv] > profiles/rNN_sweep.json
"""
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "smsp__inst_executed.sum",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "launch__shared_mem_per_block_dynamic",
]


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], check=True,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for vals in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, vals):
            d[h] = (v, u)
        kernels.append(d)
    return kernels


def summarise(report):
    res = []
    for d in raw(report):
        s = {"kernel": d.get("Kernel Name", ("?", ""))[0]}
        for k in KEYS:
            if k in d:
                v, u = d[k]
                try:
                    s[k] = [float(v.replace(",", "")), u]
                except ValueError:
                    s[k] = [v, u]
        stalls = {}
        for h, (v, u) in d.items():
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith(
                    "_per_issue_active.ratio"):
                try:
                    fv = float(v)
                except ValueError:
                    continue
                if fv > 0.01:
                    stalls[h[len("smsp__average_warps_issue_stalled_"):-len(
                        "_per_issue_active.ratio")]] = fv
        s["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
        # executed FP64 work: thread-level DFMA (2 flops) + DMUL + DADD per SMSP-cycle
        try:
            per = {op: float(d[f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed"][0])
                   for op in ("dfma", "dmul", "dadd")}
            clk = float(d["sm__cycles_elapsed.avg.per_second"][0]) * 1e9
            if d["sm__cycles_elapsed.avg.per_second"][1].lower().startswith("mhz"):
                clk = float(d["sm__cycles_elapsed.avg.per_second"][0]) * 1e6
            flops_per_cycle = 2 * per["dfma"] + per["dmul"] + per["dadd"]   # whole GPU
            insts_per_cycle = per["dfma"] + per["dmul"] + per["dadd"]
            nsm = 148
            s["executed_fp64"] = {
                "thread_ops_per_cycle_gpu": insts_per_cycle,
                "tflops": flops_per_cycle * clk / 1e12,
                "frac_of_issue_peak": insts_per_cycle / (64.0 * nsm),
                "frac_of_flop_peak": flops_per_cycle / (128.0 * nsm),
                "note": "DFMA counted as 2 flops; peak 64 DFMA/clk/SM (148 SMs)"}
        except (KeyError, ValueError):
            pass
        res.append(s)
    return res


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        agg[r[ki]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    return [{"kernel": k, "launches": len(v), "total_ms": sum(v) / 1e6,
             "share": sum(v) / tot} for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))]


if __name__ == "__main__":
    out = {"report": sys.argv[1], "kernels": summarise(sys.argv[1])}
    if len(sys.argv) > 2:
        out["launch_list"] = launches(sys.argv[2])
    print(json.dumps(out, indent=1))
