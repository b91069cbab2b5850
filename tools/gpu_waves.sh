mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for w in 1 4; do
  PE_PREFILL_WAVES=$w timeout 300 python bench.py --no-cpu --no-decode --steps 3 --warmup 3 > gpurun_out/waves_$w.txt 2>&1
  python - "$w" <<'PY'
import json,sys
w=sys.argv[1]
line=[l for l in open(f"gpurun_out/waves_{w}.txt") if l.startswith("{")][-1]
d=json.loads(line); print("waves",w,"prefill",d["prefill"]["ms_per_layer_p50"],"ms", d["prefill"]["gbs"],"GB/s frac",d["prefill"]["frac"], "value", d["value"])
PY
done
