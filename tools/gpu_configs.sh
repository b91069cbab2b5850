mkdir -p gpurun_out
timeout 1500 python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo rc=$?
cat gpurun_out/configs.jsonl | cut -c1-400
tail -3 gpurun_out/configs.err
