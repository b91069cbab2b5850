# Prefill (K1) A/B over values of one environment variable, alternating, same
# box: usage gpu_ab_prefill.sh VAR V1 V2 ...  ("-" = unset)
mkdir -p gpurun_out
VAR=$1; shift
run() {
  if [ "$2" = "-" ]; then env -u $VAR timeout 300 python bench.py --no-cpu --no-decode --steps 3 > gpurun_out/abpf_$1.txt 2>&1
  else env $VAR=$2 timeout 300 python bench.py --no-cpu --no-decode --steps 3 > gpurun_out/abpf_$1.txt 2>&1; fi
  python - "$1" <<'PY'
import json,sys
t=sys.argv[1]
line=[l for l in open(f"gpurun_out/abpf_{t}.txt") if l.startswith("{")][-1]
d=json.loads(line); p=d["prefill"]; print(t, "prefill ms/layer", p["ms_per_layer_p50"], "GB/s", p["gbs"], "frac", p["frac"], "checks", d["checks"]["invariant_violations"])
PY
}
for r in 1 2; do for v in "$@"; do run ${v}_$r $v; done; done
