mkdir -p gpurun_out
run() {
  PE_LIB=$2 timeout 300 python bench.py --no-cpu --no-decode --steps 20 > gpurun_out/k0_$1.txt 2>&1
  python - "$1" <<'PY'
import json,sys
t=sys.argv[1]
d=json.loads([l for l in open(f"gpurun_out/k0_{t}.txt") if l.startswith("{")][-1]); print(t, "value", d["value"], "K2", d["roofline"]["achieved"], "step ms", d["ms_per_step"])
PY
}
PE_LIB=$PWD/ab/libpe_b200_k0_512.so timeout 600 python -m pytest tests -m gpu -q -x -k "decode or exhaust or invariants" 2>&1 | tail -1
for r in 1 2; do run head$r $PWD/ab/libpe_b200_head.so; run t256_$r $PWD/ab/libpe_b200_k0_256.so; run t512_$r $PWD/ab/libpe_b200_k0_512.so; done
