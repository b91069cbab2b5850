timeout 900 python tools/bench_configs.py --configs cfg4 > gpurun_out/c4.txt 2>gpurun_out/c4.err; echo rc=$?; tail -2 gpurun_out/c4.err; cat gpurun_out/c4.txt | cut -c1-300
