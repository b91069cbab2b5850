#!/usr/bin/env python3
"""Regenerates tests/golden/metrics_fmt_ref.txt: the output of
tests/cpp/metrics_fmt.cpp built against the UNMODIFIED reference
(metrics.cpp + its JSON library; needs /root/reference, so it runs in the
dev container). tests/test_steplog.py compares the façade build and the
Python mirror (paper_2509_04377_b200/steplog.py) with it byte for byte."""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from tests.cpp import build_conformance  # noqa: E402

_, ref = build_conformance.build_metrics_fmt()
if ref is None:
    sys.exit("reference sources or JSON library not available")
out = subprocess.run([str(ref)], capture_output=True, text=True, check=True).stdout
(Path(__file__).resolve().parent / "metrics_fmt_ref.txt").write_text(out)
print(f"wrote {len(out.splitlines())} lines")
