"""Build the in-tree CUDA library `liblandau_b200.so` for sm_100a.

The library is a plain `extern "C"` shared object (include/landau_b200.h);
Python reaches it through ctypes (`_lib.py`).  It is built in-tree so the
built file travels with the repository snapshot to the GPU box.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "liblandau_b200.so"
SOURCES = [CSRC / "landau_b200.cu"]
DEPS = SOURCES + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + [ROOT / "include" / "landau_b200.h"]

NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "--shared", "-Xcompiler", "-fPIC",
    "-cudart", "static",
    f"-I{ROOT / 'include'}",
]
# no libraries beyond the CUDA runtime: every kernel is this package's own
LINK_FLAGS: list = []


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the B200 library cannot be built")


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in DEPS)


def build(force: bool = False, verbose: bool = False, out: Path | None = None,
          defines: dict | None = None) -> Path:
    """Build the library (or, with `out`/`defines`, a tuning variant of it)."""
    target = Path(out) if out else LIB
    if out is None and not force and not needs_build():
        return LIB
    extra = [f"-D{k}={v}" for k, v in (defines or {}).items()]
    target.parent.mkdir(parents=True, exist_ok=True)
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-o", str(target), *map(str, SOURCES), *LINK_FLAGS]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return target


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
