"""Build libqsv.so in-tree: hand-written sm_100a CUDA + C++ scheduler.

    python -m paper_2008_07140_b200.build_native [--force]

nvcc cross-compiles for sm_100a without a GPU; the .so lands next to this
file so it travels to the GPU box with the repo snapshot.  cudart is linked
statically (nvcc's default), which keeps the library independent of the
CUDA 12.8 runtime that torch bundles.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libqsv.so"
SOURCES = [CSRC / "qsv_api.cu", CSRC / "qsv_plan.cpp", CSRC / "qsv_jit.cpp"]
DEPS = SOURCES + [CSRC / "qsv_kernels.cuh", CSRC / "qsv_plan.h", CSRC / "qsv_jit.h", PKG.parent / "include" / "qsv.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def host_cxx() -> str:
    for cand in ("/usr/bin/g++", shutil.which("g++")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("g++ not found")


def command(out: Path = LIB, extra=()) -> list[str]:
    return [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++20", "-ccbin", host_cxx(),
            "-Xcompiler", "-fPIC,-O3", "-Xptxas", "-v", "--expt-relaxed-constexpr",
            "-shared", "-o", str(out), *map(str, SOURCES), "-ldl", *extra]


def stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in DEPS)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not stale():
        return LIB
    tmp = LIB.with_suffix(".so.tmp")
    proc = subprocess.run(command(tmp), capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError("libqsv build failed")
    (PKG / "build_ptxas.log").write_text(proc.stderr)
    if verbose:
        sys.stderr.write(proc.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
