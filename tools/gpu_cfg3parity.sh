mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "cfg3_full_layer" 2>&1 | tail -5
