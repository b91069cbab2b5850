mkdir -p gpurun_out
for ut in 256 1024 2048 4096; do
  PE_UNIT_TOKENS=$ut timeout 300 python bench.py --no-cpu --no-decode --steps 5 --warmup 3 > gpurun_out/ut_$ut.txt 2>&1
  python - "$ut" <<'PY'
import json,sys
s=sys.argv[1]
line=[l for l in open(f"gpurun_out/ut_{s}.txt") if l.startswith("{")][-1]
d=json.loads(line); print("unit",s,"prefill",d["prefill"]["ms_per_layer_p50"],"ms frac",d["prefill"]["frac"])
PY
done
