mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "prefill or smoke or facade" 2>&1 | tail -2
for cfg in "512 0" "512 2" "512 8" "256 0" "1024 0"; do
  set -- $cfg
  if [ "$2" = "0" ]; then unset PE_FUSED_LAG; else export PE_FUSED_LAG=$2; fi
  PE_UNIT_TOKENS=$1 timeout 300 python bench.py --no-cpu --no-decode --steps 5 --warmup 3 > gpurun_out/lag_$1_$2.txt 2>&1
  python - "$1" "$2" <<'PY'
import json,sys
u,l=sys.argv[1],sys.argv[2]
line=[x for x in open(f"gpurun_out/lag_{u}_{l}.txt") if x.startswith("{")][-1]
d=json.loads(line); print("unit",u,"lag",l,"prefill",d["prefill"]["ms_per_layer_p50"],"ms frac",d["prefill"]["frac"])
PY
done
unset PE_FUSED_LAG
PE_PREFILL_FUSED=0 timeout 300 python bench.py --no-cpu --no-decode --steps 5 --warmup 3 > gpurun_out/lag_unfused.txt 2>&1; python -c "
import json; d=json.loads([x for x in open('gpurun_out/lag_unfused.txt') if x.startswith('{')][-1]); print('unfused', d['prefill']['ms_per_layer_p50'], d['prefill']['frac'])"
