# A/B of two library builds on one box: full bench (decode + e2e), alternating.
mkdir -p gpurun_out
run() {
  PE_LIB=$2 timeout 300 python bench.py --no-cpu > gpurun_out/ab2_$1.txt 2>&1
  python - "$1" <<'PY'
import json,sys
t=sys.argv[1]
line=[l for l in open(f"gpurun_out/ab2_{t}.txt") if l.startswith("{")][-1]
d=json.loads(line); print(t, "value", d["value"], "attn_us", d["decode"]["attention_us_per_layer_p50"], "tok/s", d["decode"]["tokens_per_s"], "e2e", d["e2e"]["value"], d["e2e"]["ms_per_step"], "prefill", d["prefill"]["ms_per_layer_p50"])
PY
}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
run head1 $PWD/ab/libpe_b200_head.so
run new1 $PWD/ab/libpe_b200_new.so
run head2 $PWD/ab/libpe_b200_head.so
run new2 $PWD/ab/libpe_b200_new.so
