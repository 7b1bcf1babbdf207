"""FP64 instructions per step of the symmetric sweep, read from the SASS of
the built library (measurement infrastructure for bench.py's executed-FP64
roofline; not part of the product path).

The species-collapsed sweep `lb_symsweep_ib_kernel<1>` evaluates 4 pairs
(2 outer points x 2 partners) per thread-step in its innermost loop
(landau_sym.cuh).  That loop body holds two conditional regions: the
m < 0.01 series branch (`pair_tensor_sym_x`, taken per thread when one of
its 4 pairs needs it) and the j-side accumulation (skipped on diagonal
tiles).  This tool disassembles the kernel with cuobjdump, finds the leaf
loop holding the most FP64 instructions, splits its body at the forward
branches into the always-executed part and the two skippable regions, and
counts DFMA / DMUL / DADD in each.  With the kernel's own execution counters
(`lb_sym_counters`: off-diagonal, diagonal and series thread-steps) the
executed FP64 work of a launch is

    instr = n_off (body - series) + n_diag (body - series - jside) + n_ser series

(thread instructions; flops count DFMA twice).  FP64 work outside the loop
(the per-32-partner j-side gather and the partial-sum reduction) is not
counted: < 1 % of the launch, so the derived figure is a slight lower bound.

    python tools/sass_fp64.py [path/to/liblandau_b200.so]
"""

from __future__ import annotations

import json
import re
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_1702_08880_b200" / "liblandau_b200.so"
# lb_symsweep_ib_kernel<1, merged_guard>: the benchmark's eps_d takes the merged-guard variant
KERNELS = {True: "_ZN2lb21lb_symsweep_ib_kernelILi1ELb1EEEvNS_7SymArgsE",
           False: "_ZN2lb21lb_symsweep_ib_kernelILi1ELb0EEEvNS_7SymArgsE"}
KERNEL = KERNELS[True]
FP64 = ("DFMA", "DMUL", "DADD")
_LINE = re.compile(r"/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)\s*([^;]*);")


def cuobjdump() -> str:
    for cand in (shutil.which("cuobjdump"), "/usr/local/cuda/bin/cuobjdump"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("cuobjdump not found")


def disassemble(lib: Path = LIB, kernel: str = KERNEL):
    """[(address, predicate, opcode, operands)] of one kernel."""
    out = subprocess.run([cuobjdump(), "-sass", "-fun", kernel, str(lib)], check=True,
                         capture_output=True, text=True).stdout
    insts = []
    for m in _LINE.finditer(out):
        insts.append((int(m.group(1), 16), (m.group(2) or "").strip(), m.group(3), m.group(4)))
    if not insts:
        raise RuntimeError(f"no SASS for {kernel} in {lib}")
    return insts


def _target(ops: str):
    m = re.match(r"\s*(?:U?R\d+,\s*)?(0x[0-9a-f]+)", ops)
    return int(m.group(1), 16) if m else None


def _fp64(insts):
    c = {k: 0 for k in FP64}
    for _, _, op, _ in insts:
        base = op.split(".")[0]
        if base in c:
            c[base] += 1
    return c


def _flops(c):
    return c["DADD"] + c["DMUL"] + 2 * c["DFMA"]


def analyse(lib: Path = LIB, kernel: str = KERNEL) -> dict:
    insts = disassemble(lib, kernel)
    addr = [a for a, *_ in insts]
    loops = []
    for a, pred, op, ops in insts:
        if op.startswith("BRA"):
            t = _target(ops)
            if t is not None and t < a:
                loops.append((t, a))
    if not loops:
        raise RuntimeError("no loop found")

    def body(lo, hi):
        return [x for x in insts if lo <= x[0] <= hi]

    leaves = [(t, a) for (t, a) in loops
              if not any(t <= t2 and a2 <= a and (t2, a2) != (t, a) for (t2, a2) in loops)]
    t0, a0 = max(leaves, key=lambda L: sum(_fp64(body(*L)).values()))
    loop = body(t0, a0)
    # forward branches inside the loop -> skippable regions (start, end)
    regions = []
    for a, pred, op, ops in loop:
        if op.startswith("BRA") and not op.startswith("BRA.DIV"):
            t = _target(ops)
            if t is not None and a < t <= a0:
                regions.append((a + 16, t))
    regions = [r for r in regions if sum(_fp64(body(r[0], r[1] - 1)).values()) > 0]
    # nested regions: keep the outermost ones, in program order
    regions = sorted({r for r in regions
                      if not any(o[0] <= r[0] and r[1] <= o[1] and o != r for o in regions)})
    if len(regions) != 2:
        raise RuntimeError(f"expected 2 skippable FP64 regions in the loop, found {regions}")
    c_body = _fp64(loop)
    c_ser = _fp64(body(regions[0][0], regions[0][1] - 1))
    c_js = _fp64(body(regions[1][0], regions[1][1] - 1))
    sub = lambda a, b: {k: a[k] - b[k] for k in FP64}  # noqa: E731
    off = sub(c_body, c_ser)
    diag = sub(off, c_js)
    return {
        "kernel": kernel,
        "loop": [hex(t0), hex(a0)],
        "series_region": [hex(x) for x in regions[0]],
        "jside_region": [hex(x) for x in regions[1]],
        "pairs_per_thread_step": 4,
        "instr": {"off": sum(off.values()), "diag": sum(diag.values()),
                  "series": sum(c_ser.values())},
        "flops": {"off": _flops(off), "diag": _flops(diag), "series": _flops(c_ser)},
        "by_opcode": {"off": off, "diag": diag, "series": c_ser},
        "predicated_fp64_in_loop": sum(1 for _, p, op, _ in loop
                                       if p and op.split(".")[0] in FP64),
    }


def executed(counts, sass: dict) -> dict:
    """Executed FP64 thread instructions and flops of a launch from the
    kernel's counters (n_off, n_diag, n_ser) and the per-step SASS counts."""
    n_off, n_diag, n_ser = (int(x) for x in counts[:3])
    out = {}
    for key in ("instr", "flops"):
        c = sass[key]
        out[key] = n_off * c["off"] + n_diag * c["diag"] + n_ser * c["series"]
    out["pairs"] = sass["pairs_per_thread_step"] * (n_off + n_diag)
    return out


if __name__ == "__main__":
    print(json.dumps(analyse(Path(sys.argv[1]) if len(sys.argv) > 1 else LIB), indent=1))
