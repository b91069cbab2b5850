# Eviction-step A/B over N values of one environment variable (same build,
# alternating, same box): usage gpu_ab_envn.sh VAR V1 V2 ...
mkdir -p gpurun_out
VAR=$1; shift
timeout 900 python -m pytest tests -m gpu -x -q -k "decode or smoke or golden or facade or exhaust or invariants or cfg3 or table" > gpurun_out/ab_tests.txt 2>&1; tail -1 gpurun_out/ab_tests.txt
run() {
  env $VAR=$2 timeout 300 python bench.py --no-cpu --no-decode --steps 20 > gpurun_out/abenv_$1.txt 2>&1
  python - "$1" <<'PY'
import json,sys
t=sys.argv[1]
line=[l for l in open(f"gpurun_out/abenv_{t}.txt") if l.startswith("{")][-1]
d=json.loads(line); print(t, "value", d["value"], "K2", d["roofline"]["achieved"], "p50", d["p50_evict_step_us"], "layerK2", d["p50_evict_layer_launch_us"], "probe", d["roofline"].get("probe",{}).get("read_gbs"))
PY
}
for r in 1 2; do for v in "$@"; do run ${v}_$r $v; done; done
