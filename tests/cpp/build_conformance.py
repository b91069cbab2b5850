"""Builds the C++ façade conformance binaries (test infrastructure).

ref_conformance: the reference's OWN unit tests for the cache-manager API
(/root/reference/proj/tests/test_{paged_store,importance,policies,attention}.cpp),
compiled unchanged against the B200 façade headers (include/pagedevict/*.hpp
-> include/pe/pagedevict.hpp) with the doctest shim (tests/cpp/doctest.h)
and linked to libpagedevict_b200.so. The reference's test-only helpers
(tests/oracles.hpp, core/include/pagedevict/rng.hpp) are found through
include paths placed AFTER ours, so every hot-path header resolves to the
façade. The binary is built here (the reference tree is read at build time
only), is git-ignored and travels to the GPU box with the repo snapshot.

facade_tests: our own façade tests (tests/cpp/test_facade.cpp).
"""
from __future__ import annotations

import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
OUT = HERE / "_build"
LIB_DIR = ROOT / "paper_2509_04377_b200" / "lib"
REF = Path("/root/reference/proj")
REF_TESTS = ["test_paged_store.cpp", "test_importance.cpp", "test_policies.cpp", "test_attention.cpp"]


def _cxx(srcs: list[Path], out: Path, extra_inc: list[Path], shim_main: bool = True) -> Path:
    OUT.mkdir(parents=True, exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-g", f"-I{HERE}", f"-I{ROOT / 'include'}",
           *[f"-I{p}" for p in extra_inc], *map(str, srcs), *([str(HERE / "shim_main.cpp")] if shim_main else []),
           f"-L{LIB_DIR}", "-lpagedevict_b200", "-lpe_b200", f"-Wl,-rpath,{LIB_DIR}",
           "-Wl,-rpath,$ORIGIN/../../../paper_2509_04377_b200/lib", "-lpthread", "-o", str(out)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"g++ failed ({res.returncode}):\n{' '.join(cmd)}\n{res.stderr[-8000:]}")
    return out


def build_reference_conformance() -> Path | None:
    if not REF.exists():
        return None
    srcs = [REF / "tests" / t for t in REF_TESTS]
    return _cxx(srcs, OUT / "ref_conformance", [REF / "tests", REF / "core" / "include"])


def build_facade_tests() -> Path:
    OUT.mkdir(parents=True, exist_ok=True)
    obj = OUT / "pe_oracle.o"  # the C restatement, linked as the checker
    cmd = ["gcc", "-std=c11", "-O2", "-fno-fast-math", "-ffp-contract=off", "-c", str(ROOT / "oracle" / "pe_oracle.c"), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"gcc failed:\n{res.stderr[-4000:]}")
    return _cxx([HERE / "test_facade.cpp", obj], OUT / "facade_tests", [])


REF_CORE = ["page_pool.cpp", "block_table.cpp", "importance.cpp", "policy.cpp", "attention.cpp"]


def build_scenario() -> tuple[Path, Path | None]:
    """scenario_trace.cpp twice: against the façade (tests/cpp/_build/scenario_b200)
    and, where /root/reference exists, against the UNMODIFIED reference sources
    (oracle/_ref/scenario_ref — reference build outputs live under oracle/_ref)."""
    b200 = _cxx([HERE / "scenario_trace.cpp"], OUT / "scenario_b200", [], shim_main=False)
    ref_out = None
    if REF.exists():
        ref_dir = ROOT / "oracle" / "_ref"
        ref_dir.mkdir(parents=True, exist_ok=True)
        ref_out = ref_dir / "scenario_ref"
        cmd = ["g++", "-std=c++20", "-O2", f"-I{REF / 'core' / 'include'}", str(HERE / "scenario_trace.cpp"),
               *[str(REF / "core" / "src" / f) for f in REF_CORE], "-lpthread", "-o", str(ref_out)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"g++ failed ({res.returncode}):\n{' '.join(cmd)}\n{res.stderr[-8000:]}")
    return b200, ref_out


# the reference's JSON library (nlohmann/json, header-only; a pinned copy
# ships in this image under cudnn_frontend's third-party tree)
JSON_DIRS = [Path("/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann")]


def build_metrics_fmt() -> tuple[Path, Path | None]:
    """metrics_fmt.cpp against the façade (tests/cpp/_build/metrics_fmt_b200)
    and against the reference's metrics.cpp + JSON library
    (oracle/_ref/metrics_fmt_ref), for the byte-identical emitter test."""
    b200 = _cxx([HERE / "metrics_fmt.cpp"], OUT / "metrics_fmt_b200", [], shim_main=False)
    ref_out = None
    json_dir = next((d for d in JSON_DIRS if (d / "json.hpp").exists()), None)
    if REF.exists() and json_dir is not None:
        ref_dir = ROOT / "oracle" / "_ref"
        ref_dir.mkdir(parents=True, exist_ok=True)
        ref_out = ref_dir / "metrics_fmt_ref"
        cmd = ["g++", "-std=c++20", "-O2", f"-I{REF / 'core' / 'include'}", f"-I{json_dir}",
               str(HERE / "metrics_fmt.cpp"),
               *[str(REF / "core" / "src" / f) for f in REF_CORE + ["metrics.cpp"]], "-lpthread", "-o", str(ref_out)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"g++ failed ({res.returncode}):\n{' '.join(cmd)}\n{res.stderr[-8000:]}")
    return b200, ref_out


def build_acceptance() -> tuple[Path | None, Path | None]:
    """acceptance_device.cpp (criteria 1-3, 6, 8 of the reference's acceptance
    suite over the pagedevict:: API) against the façade
    (tests/cpp/_build/acceptance_b200) and against the UNMODIFIED reference
    sources (oracle/_ref/acceptance_ref). Needs the reference's test helpers
    (tests/oracles.hpp, rng.hpp) at build time, so it is built only here."""
    if not REF.exists():
        return None, None
    src = HERE / "acceptance_device.cpp"
    b200 = _cxx([src], OUT / "acceptance_b200", [REF / "tests", REF / "core" / "include"], shim_main=False)
    ref_dir = ROOT / "oracle" / "_ref"
    ref_dir.mkdir(parents=True, exist_ok=True)
    ref_out = ref_dir / "acceptance_ref"
    cmd = ["g++", "-std=c++20", "-O2", f"-I{REF / 'core' / 'include'}", f"-I{REF / 'tests'}", str(src),
           *[str(REF / "core" / "src" / f) for f in REF_CORE], "-lpthread", "-o", str(ref_out)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"g++ failed ({res.returncode}):\n{' '.join(cmd)}\n{res.stderr[-8000:]}")
    return b200, ref_out


def build_all() -> None:
    from paper_2509_04377_b200 import _build

    _build.build()
    build_facade_tests()
    build_reference_conformance()
    build_scenario()
    build_metrics_fmt()
    build_acceptance()
    build_examples()


if __name__ == "__main__":
    sys.path.insert(0, str(ROOT))
    build_all()
    print("built", sorted(p.name for p in OUT.iterdir()))


def build_examples() -> Path:
    """examples/decode_loop.cpp: the batched C-ABI driven from C++ host code."""
    OUT.mkdir(parents=True, exist_ok=True)
    out = OUT / "decode_loop"
    cmd = ["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}", "-I/usr/local/cuda/include",
           str(ROOT / "examples" / "decode_loop.cpp"), f"-L{LIB_DIR}", "-lpe_b200", "-L/usr/local/cuda/lib64",
           "-lcudart", f"-Wl,-rpath,{LIB_DIR}", "-Wl,-rpath,/usr/local/cuda/lib64", "-o", str(out)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"g++ failed ({res.returncode}):\n{' '.join(cmd)}\n{res.stderr[-4000:]}")
    return out
