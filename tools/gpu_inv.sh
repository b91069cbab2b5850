mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --no-cpu > gpurun_out/bench_inv.txt 2>&1; python -c "
import json; d=json.loads([x for x in open('gpurun_out/bench_inv.txt') if x.startswith('{')][-1]); print(d['checks']); print('value', d['value'], 'attn', d['decode'])"
