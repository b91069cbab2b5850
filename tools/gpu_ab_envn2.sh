# Eviction-step A/B over values of one environment variable (same build,
# alternating, same box), with the append launch time: gpu_ab_envn2.sh VAR V1 V2 ...
mkdir -p gpurun_out
VAR=$1; shift
for r in 1 2; do for v in "$@"; do
  env $VAR=$v timeout 300 python bench.py --no-cpu --no-decode --steps 10 > gpurun_out/abe_${v}_$r.txt 2>&1
  tail -1 gpurun_out/abe_${v}_$r.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$VAR=$v', d['value'], d['ms_per_step'], 'K2', d['roofline']['achieved'], 'append_us', d['append_us_per_launch_p50'], 'e2e', d['e2e']['value'], d['checks']['invariant_violations'], d['checks']['cadence_ok'])"
done; done
