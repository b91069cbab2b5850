# A/B timing of two builds of libpe_b200.so on the same box (PE_LIB override).
mkdir -p gpurun_out
run() {
  PE_LIB=$2 timeout 300 python bench.py --no-cpu --no-decode --steps 30 > gpurun_out/ab_$1.txt 2>&1
  python - "$1" <<'PY'
import json,sys
t=sys.argv[1]
line=[l for l in open(f"gpurun_out/ab_{t}.txt") if l.startswith("{")][-1]
d=json.loads(line); print(t, "value", d["value"], "K2", d["roofline"]["achieved"], "p50", d["p50_evict_step_us"], "layerK2", d["p50_evict_layer_launch_us"], "prefill", d["prefill"]["ms_per_layer_p50"])
PY
}
run orig1 $PWD/ab/libpe_b200_orig.so
run new1 $PWD/paper_2509_04377_b200/lib/libpe_b200.so
run orig2 $PWD/ab/libpe_b200_orig.so
run orig3 $PWD/ab/libpe_b200_orig.so
run new2 $PWD/paper_2509_04377_b200/lib/libpe_b200.so
run new3 $PWD/paper_2509_04377_b200/lib/libpe_b200.so
