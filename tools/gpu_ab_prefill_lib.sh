# Prefill (K1) A/B of two builds (ab/libpe_b200_{head,new}.so), alternating.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_engine_gpu.py -x -q -k "prefill" > gpurun_out/abp_tests.txt 2>&1; tail -1 gpurun_out/abp_tests.txt
for r in 1 2; do for b in head new; do
  PE_LIB=$PWD/ab/libpe_b200_$b.so timeout 300 python bench.py --no-cpu --no-decode --steps 3 > gpurun_out/abp_${b}_$r.txt 2>&1
  python - "$b" "$r" <<'PY'
import json,sys
b,r=sys.argv[1],sys.argv[2]
d=json.loads([l for l in open(f"gpurun_out/abp_{b}_{r}.txt") if l.startswith("{")][-1]); p=d["prefill"]
print(b, "prefill ms/layer", p["ms_per_layer_p50"], "frac", p["frac"], "checks", d["checks"]["invariant_violations"])
PY
done; done
