"""In-tree build of the engine's C-ABI library for sm_100a.

    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -shared ...
      -> paper_2509_04377_b200/lib/libpe_b200.so

The .so is git-ignored but NOT gpurun-ignored, so the built library travels
to the GPU box with the repo snapshot. `load()` in _lib.py rebuilds when a
source is newer than the library (nvcc exists on the GPU image too).
"""
from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "lib"
LIB = LIB_DIR / "libpe_b200.so"
# C++ façade: the reference's pagedevict:: API over the C-ABI
FACADE_SRC = PKG / "cpp" / "pagedevict.cpp"
FACADE_HDR = ROOT / "include" / "pe" / "pagedevict.hpp"
FACADE_LIB = LIB_DIR / "libpagedevict_b200.so"
SOURCES = ["pe_engine.cu", "pe_decode.cu", "pe_prefill.cu", "pe_select.cu", "pe_attention.cu", "pe_table.cu"]
HEADERS = ["pe_internal.cuh", "pe_kernels.cuh", "pe_score.cuh", "pe_tma.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the PagedEviction engine needs the CUDA toolkit to build")


def inputs() -> list[Path]:
    return [CSRC / s for s in SOURCES] + [CSRC / h for h in HEADERS] + [ROOT / "include" / "pe.h",
                                                                        Path(__file__)]


def stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in inputs())


def build_facade(force: bool = False) -> Path:
    """g++ -std=c++20 the façade into libpagedevict_b200.so (links libpe_b200.so, rpath $ORIGIN)."""
    if (not force and FACADE_LIB.exists() and
            FACADE_LIB.stat().st_mtime >= max(p.stat().st_mtime for p in (FACADE_SRC, FACADE_HDR, LIB))):
        return FACADE_LIB
    tmp = FACADE_LIB.with_suffix(".so.tmp")
    cmd = ["g++", "-std=c++20", "-O2", "-g", "-fPIC", "-shared", "-Wall", "-Wextra",
           f"-I{ROOT / 'include'}", str(FACADE_SRC), f"-L{LIB_DIR}", "-lpe_b200",
           "-Wl,-rpath,$ORIGIN", "-o", str(tmp)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"g++ failed ({res.returncode}):\n{' '.join(cmd)}\n{res.stderr[-6000:]}")
    os.replace(tmp, FACADE_LIB)
    return FACADE_LIB


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not stale():
        build_facade()
        return LIB
    LIB_DIR.mkdir(parents=True, exist_ok=True)
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [
        nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
        "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v" if verbose else "-O3",
        f"-I{ROOT / 'include'}", f"-I{CSRC}",
        *os.environ.get("PE_NVCC_EXTRA", "").split(),  # e.g. -DPE_K0_TRACE for instrumented A/B builds
        *[str(CSRC / s) for s in SOURCES],
        "-o", str(tmp),
    ]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{' '.join(cmd)}\n{res.stderr[-6000:]}")
    if verbose:
        print(res.stderr)
    os.replace(tmp, LIB)
    build_facade(force=True)
    return LIB


if __name__ == "__main__":
    import sys

    print(build(force=True, verbose="-v" in sys.argv))
