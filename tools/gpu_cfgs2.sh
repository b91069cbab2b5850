mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
timeout 600 python bench.py --no-cpu > gpurun_out/bq.txt 2>&1; python -c "
import json; d=json.loads([x for x in open('gpurun_out/bq.txt') if x.startswith('{')][-1]); print('value', d['value'], 'decode', d['decode'])"
timeout 1500 python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo rc=$?
python - <<'PY'
import json
for l in open("gpurun_out/configs.jsonl"):
    d=json.loads(l); print(d["config"], "prefill", d["prefill"]["frac"], "evict", d.get("evict_step_frac"), "attn", d["attention"], "tok/s", d["decode"]["tokens_per_s"])
PY
