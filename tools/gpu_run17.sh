mkdir -p gpurun_out
timeout 1500 python tools/bench_configs.py --configs cfg1,cfg2,cfg4,cfg5 > gpurun_out/configs17.jsonl 2> gpurun_out/configs17.err; tail -3 gpurun_out/configs17.err; cat gpurun_out/configs17.jsonl
