# A/B of two builds (ab/libpe_b200_{head,new}.so), burst (10 steps) and
# sustained (100 steps) eviction-step runs, alternating, same box.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "decode or smoke or golden or facade or exhaust or invariants or cfg3 or table or steplog or token" > gpurun_out/ab_tests.txt 2>&1; tail -1 gpurun_out/ab_tests.txt
for r in 1 2; do for b in head new; do for k in 10 100; do
  PE_LIB=$PWD/ab/libpe_b200_$b.so timeout 300 python bench.py --no-cpu --no-decode --steps $k > gpurun_out/abs_${b}_${k}_$r.txt 2>&1
  tail -1 gpurun_out/abs_${b}_${k}_$r.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$b', $k, d['value'], d['roofline']['achieved'], d['p50_evict_step_us'], d['append_us_per_launch_p50'], d['prefill']['ms_per_layer_p50'], d['clocks']['sm_mhz'])"
done; done; done
