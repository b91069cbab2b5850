mkdir -p gpurun_out
for sel in cta cluster; do for w in 1 4 8; do
  PE_SELECT=$sel PE_PREFILL_WAVES=$w timeout 300 python bench.py --no-cpu --no-decode --steps 3 --warmup 3 > gpurun_out/sv_${sel}_$w.txt 2>&1
  python - "$sel" "$w" <<'PY'
import json,sys
s,w=sys.argv[1],sys.argv[2]
line=[l for l in open(f"gpurun_out/sv_{s}_{w}.txt") if l.startswith("{")][-1]
d=json.loads(line); print(s,"waves",w,"prefill",d["prefill"]["ms_per_layer_p50"],"ms frac",d["prefill"]["frac"])
PY
done; done
PE_SELECT=cluster PE_PREFILL_WAVES=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"prefill" --csv --log-file gpurun_out/prefill_times_cluster.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-decode > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/prefill_times_cluster.csv
