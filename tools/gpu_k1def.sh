mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "prefill or smoke or golden or cfg3 or facade" 2>&1 | tail -1
timeout 300 python bench.py --no-cpu --no-decode --steps 3 --warmup 3 > gpurun_out/k1.txt 2>&1; python -c "
import json; d=json.loads([x for x in open('gpurun_out/k1.txt') if x.startswith('{')][-1]); print('cfg3 prefill', d['prefill'])"
timeout 1500 python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; python - <<'PY'
import json
for l in open("gpurun_out/configs.jsonl"):
    d=json.loads(l); print(d["config"], "prefill", d["prefill"])
PY
