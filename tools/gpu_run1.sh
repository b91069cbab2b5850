set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 300 python __graft_entry__.py > gpurun_out/smoke.txt 2>&1; tail -5 gpurun_out/smoke.txt
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench1.txt 2>&1; tail -20 gpurun_out/bench1.txt
