mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py --no-cpu > gpurun_out/bench_quick.txt 2>&1
python - <<'PY'
import json
line=[l for l in open("gpurun_out/bench_quick.txt") if l.startswith("{")][-1]
d=json.loads(line)
print("value", d["value"], "K2", d["roofline"]["achieved"], "p50", d["p50_evict_step_us"], "prefill", d["prefill"]["ms_per_layer_p50"], d["prefill"]["frac"])
print("decode", d["decode"])
print("e2e", d["e2e"])
PY
