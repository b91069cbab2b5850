"""compute-sanitizer over the engine's kernels (memcheck,
racecheck, synccheck; the reference itself has only -Wall -Wextra and a pool
thread test, proj/CMakeLists.txt:12-14, tests/test_paged_store.cpp:230-249).

The driver is examples/decode_loop (C++ host code over the C-ABI): prefill
prune+pack of every layer (K1 planner, score, select, copy), eviction cycles
(K0 appends with the two-level decoupled look-back across > 32 CTAs, K2 or
K2c with the last-CTA ticket push), GQA attention of every layer (K3 with
split merges) and the device invariant checker. The select / attention /
append variants are switched with the engine's environment knobs, so each
kernel family runs under each tool. Done = zero reported errors / hazards.

racecheck covers shared-memory hazards (including the cluster select's
DSMEM); global-memory ordering of the look-back is covered by the chain
parity tests (tests/test_engine_gpu.py::test_append_chain_parity*).
"""
from __future__ import annotations

import os
import re
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
BINARY = ROOT / "tests" / "cpp" / "_build" / "decode_loop"

# seqs layers kv_heads head_dim prompt budget cycles [score]: 40 x 8 x 8 =
# 2560 tables = 40 K0 CTAs (two look-back groups); 8192-token prompts with
# C=1024 take the sampled-window select (bitmap emit), 1024-token prompts
# with C=256 the full radix passes and position sweeps
SMALL = ["40", "8", "8", "128", "8192", "1024", "2"]
SHORT = ["40", "8", "8", "128", "1024", "256", "2"]

VARIANTS = {
    "default": ({}, SMALL),
    "short_prompts": ({}, SHORT),
    "cached_score": ({}, SMALL + ["1"]),
    "select_global": ({"PE_SELECT": "global"}, SMALL),
    "select_global_fallback": ({"PE_SELECT": "global_fallback", "PE_FB_GRID": "7"}, SMALL),
    "select_smem": ({"PE_SELECT": "smem"}, SMALL),
    "select_cluster": ({"PE_SELECT": "cluster"}, SMALL),
    "select_stream1024": ({"PE_SELECT": "stream"}, SMALL),
    "attn_splits4_cpasync": ({"PE_ATTN_SPLITS": "4", "PE_ATTN_TMA": "0"}, SMALL),
    "append_lookback_always": ({"PE_APPEND_FAST": "0"}, SMALL),
    "k2_chunked": ({"PE_K2_CTAS_PER_SM": "16"}, SMALL),
}

TOOL_VARIANTS = {
    "memcheck": list(VARIANTS),
    "racecheck": ["default", "short_prompts", "select_global", "select_global_fallback", "select_smem",
                  "select_stream1024", "select_cluster", "attn_splits4_cpasync"],
    "synccheck": ["default", "short_prompts", "select_global", "select_cluster", "attn_splits4_cpasync"],
}


def _sanitizer() -> str:
    for cand in ("/usr/local/cuda/bin/compute-sanitizer", shutil.which("compute-sanitizer")):
        if cand and Path(cand).exists():
            return cand
    pytest.skip("compute-sanitizer not found")


@pytest.mark.gpu
@pytest.mark.slow
@pytest.mark.parametrize("tool,variant", [(t, v) for t, vs in TOOL_VARIANTS.items() for v in vs])
def test_compute_sanitizer_clean(tool, variant):
    if not BINARY.exists():
        pytest.skip("decode_loop not built (tests/cpp/build_conformance.py)")
    env_extra, args = VARIANTS[variant]
    env = {**os.environ, **env_extra}
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "97", "--print-limit", "20"]
    if tool == "racecheck":
        cmd += ["--racecheck-report", "all"]
    res = subprocess.run(cmd + [str(BINARY), *args], capture_output=True, text=True, env=env, timeout=1200)
    out = res.stdout + res.stderr
    assert res.returncode == 0, out[-6000:]
    if tool == "racecheck":
        m = re.search(r"RACECHECK SUMMARY: (\d+) hazards? displayed \((\d+) errors?, (\d+) warnings?\)", out)
        assert m is None or m.groups() == ("0", "0", "0"), out[-6000:]
    else:
        assert "ERROR SUMMARY: 0 errors" in out, out[-6000:]
