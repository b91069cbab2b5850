#!/bin/bash
# Round re-entry check: GPU tests, smoke, default bench line.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv | tail -1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench_verify.txt 2>&1; tail -1 gpurun_out/bench_verify.txt
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_verify.txt 2>&1; tail -1 gpurun_out/bench_ref_verify.txt
