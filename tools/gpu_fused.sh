mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for fz in 1 0 1 0; do
  PE_PREFILL_FUSED=$fz timeout 300 python bench.py --no-cpu --no-decode --steps 5 --warmup 3 > gpurun_out/fz_$fz.txt 2>&1
  python - "$fz" <<'PY'
import json,sys
s=sys.argv[1]
line=[l for l in open(f"gpurun_out/fz_{s}.txt") if l.startswith("{")][-1]
d=json.loads(line); print("fused",s,"prefill",d["prefill"]["ms_per_layer_p50"],"ms frac",d["prefill"]["frac"], "value", d["value"])
PY
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"prefill" --csv --log-file gpurun_out/prefill_fused_times.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-decode > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/prefill_fused_times.csv
