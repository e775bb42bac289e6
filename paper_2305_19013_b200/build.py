"""Build the sm_100a kernel library in-tree: paper_2305_19013_b200/libekcg_b200.so.

Plain nvcc (no torch extension machinery): the library exports a C ABI
(include/ekcg_b200.h) that the Python driver binds with ctypes.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libekcg_b200.so"
SOURCES = ["sparse.cu", "stencil_march.cu", "stream.cu", "stream_wide.cu", "dense.cu", "small.cu", "fused.cu", "cluster_solve.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-warn-spills",
    f"-I{ROOT / 'include'}", f"-I{CSRC}",
]


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "ekcg_b200.h"]
    return any(p.stat().st_mtime > t for p in deps)


def needs_build() -> bool:
    """True when the library is missing, or stale and nvcc is available to rebuild it."""
    if not LIB.exists():
        return True
    return _stale() and Path(NVCC).exists()


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    cmd = [NVCC, *FLAGS, "-o", str(LIB), *[str(CSRC / s) for s in SOURCES]]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stdout}\n{res.stderr}")
    if verbose and res.stderr.strip():
        print(res.stderr, file=sys.stderr)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
