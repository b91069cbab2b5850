# A/B (eviction step only) of two builds, alternating, same box.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "decode or smoke or golden or facade or exhaust or invariants or cfg3" 2>&1 | tail -1
run() {
  PE_LIB=$2 timeout 300 python bench.py --no-cpu --no-decode --steps 20 > gpurun_out/ab3_$1.txt 2>&1
  python - "$1" <<'PY'
import json,sys
t=sys.argv[1]
line=[l for l in open(f"gpurun_out/ab3_{t}.txt") if l.startswith("{")][-1]
d=json.loads(line); print(t, "value", d["value"], "K2", d["roofline"]["achieved"], "p50", d["p50_evict_step_us"], "layerK2", d["p50_evict_layer_launch_us"])
PY
}
for r in 1 2 3; do run head$r $PWD/ab/libpe_b200_head.so; run new$r $PWD/ab/libpe_b200_new.so; done
