mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/tma_t.txt 2>&1; tail -2 gpurun_out/tma_t.txt
PE_ATTN_TMA=0 timeout 600 python -m pytest tests -m gpu -q -k "attention or cfg3" > gpurun_out/tma_t0.txt 2>&1; tail -1 gpurun_out/tma_t0.txt
for v in 0 1; do
  PE_ATTN_TMA=$v timeout 300 python bench.py --no-cpu --steps 3 > gpurun_out/tma.txt 2>&1
  python -c "
import json; d=json.loads([x for x in open('gpurun_out/tma.txt') if x.startswith('{')][-1]); print('tma $v attn', d['decode']['attention_us_per_layer_p50'], d['decode']['tokens_per_s'], 'full', d['decode']['full_cache']['attention_us_per_layer_p50'])"
done
timeout 900 python tools/bench_configs.py --configs cfg1,cfg2 > gpurun_out/cfg12.jsonl 2>/dev/null; python -c "
import json
for l in open('gpurun_out/cfg12.jsonl'):
    d=json.loads(l); print(d['config'], d['attention'], d['decode']['tokens_per_s'])"
