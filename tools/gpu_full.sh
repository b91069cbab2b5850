mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu > gpurun_out/bench_full.txt 2>&1; tail -3 gpurun_out/bench_full.txt | cut -c1-300; python -c "
import json; d=json.loads([x for x in open('gpurun_out/bench_full.txt') if x.startswith('{')][-1]); print(d['decode'])"
