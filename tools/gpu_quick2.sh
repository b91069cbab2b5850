mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench_q2.txt 2>&1; python -c "
import json; d=json.loads([x for x in open('gpurun_out/bench_q2.txt') if x.startswith('{')][-1])
print('value', d['value'], 'pct', d['pct_of_peak'], 'K2', d['roofline'], 'p50', d['p50_evict_step_us'], 'layer', d['p50_evict_layer_launch_us'])
print('prefill', d['prefill']); print('decode', d['decode']); print('e2e', d['e2e']); print('checks', d['checks']); print('cpu', d['cpu_baseline'])"
