mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench18.txt 2>&1; tail -1 gpurun_out/bench18.txt | cut -c1-2300
timeout 1500 python tools/bench_configs.py --configs cfg1,cfg2,cfg4,cfg5 > gpurun_out/configs18.jsonl 2> gpurun_out/configs18.err; tail -3 gpurun_out/configs18.err; cat gpurun_out/configs18.jsonl
