#!/usr/bin/env bash
# End-of-round evidence on one GPU box (run through gpurun from the repo root):
# pytest -m gpu, smoke(), the default bench line, the reference arm, the ncu
# launch list of a short bench run and bench_configs; outputs in gpurun_out/<tag>_*.
set -u
tag=${1:-final}
bash tools/gpu.sh tests $tag
bash tools/gpu.sh smoke $tag
bash tools/gpu.sh bench $tag
bash tools/gpu.sh ref $tag
bash tools/gpu.sh launches $tag --steps 2 --warmup 3
bash tools/gpu.sh configs $tag
