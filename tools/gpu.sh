#!/usr/bin/env bash
# One parameterised driver for the GPU box (run through gpurun from the repo
# root); every output lands in gpurun_out/<tag>_*. Subcommands, chained with ';':
#
#   tools/gpu.sh tests TAG [pytest -k expr]   pytest -m gpu (optionally filtered)
#   tools/gpu.sh smoke TAG                     __graft_entry__.smoke()
#   tools/gpu.sh bench TAG [bench args...]     one bench.py line (+ clocks)
#   tools/gpu.sh ref TAG                       bench.py --impl reference
#   tools/gpu.sh ab-lib TAG ROUNDS ARGS...     bench.py with ab/libpe_b200_{head,new}.so alternating
#   tools/gpu.sh ab-env TAG VAR "V1 V2 .." ARGS...  bench.py over env values ("-" = unset), alternating
#   tools/gpu.sh launches TAG [bench args...]  ncu launch list (time + dram bytes) of a bench run
#   tools/gpu.sh ncu TAG REGEX SKIP [bench args...]  ncu --set full of one launch -> .ncu-rep
#   tools/gpu.sh configs TAG [configs args...] tools/bench_configs.py (cfg1/2/4/5 with checks)
set -u
mkdir -p gpurun_out
cmd=$1; tag=$2; shift 2
summ() {  # print the key numbers of the last JSON line of a bench log
  python - "$1" <<'PY'
import json, sys
lines = [l for l in open(sys.argv[1]) if l.startswith("{")]
if not lines:
    print(sys.argv[1], "no JSON line"); sys.exit()
d = json.loads(lines[-1])
p = d.get("prefill", {}); r = d.get("roofline", {})
print(sys.argv[1].split("/")[-1], "value", d.get("value"), "k2_frac", r.get("frac"),
      "p50_evict_step_us", d.get("p50_evict_step_us"), "launch_us", d.get("p50_evict_launch_us"),
      "append_us", d.get("append_us_per_launch_p50"),
      "prefill_ms", p.get("ms_per_layer_p50"), "prefill_frac", p.get("frac"),
      "checks", (d.get("checks") or {}).get("invariant_violations"), "clocks", d.get("clocks", {}).get("sm_mhz"))
PY
}
case $cmd in
  tests)
    if [ $# -gt 0 ]; then timeout 2400 python -m pytest tests -m gpu -x -q -k "$1" > gpurun_out/${tag}_tests.txt 2>&1
    else timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_tests.txt 2>&1; fi
    tail -3 gpurun_out/${tag}_tests.txt ;;
  smoke)
    timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.txt 2>&1
    tail -3 gpurun_out/${tag}_smoke.txt ;;
  bench)
    timeout 1200 python bench.py "$@" > gpurun_out/${tag}_bench.txt 2>&1
    tail -1 gpurun_out/${tag}_bench.txt; summ gpurun_out/${tag}_bench.txt ;;
  ref)
    timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${tag}_ref.txt 2>&1
    tail -1 gpurun_out/${tag}_ref.txt ;;
  ab-lib)
    rounds=$1; shift
    for r in $(seq 1 $rounds); do for b in head new; do
      PE_LIB=$PWD/ab/libpe_b200_$b.so timeout 900 python bench.py "$@" > gpurun_out/${tag}_${b}_$r.txt 2>&1
      summ gpurun_out/${tag}_${b}_$r.txt
    done; done ;;
  ab-env)
    var=$1; vals=$2; shift 2
    for r in 1 2; do for v in $vals; do
      if [ "$v" = "-" ]; then env -u $var timeout 900 python bench.py "$@" > gpurun_out/${tag}_${v}_$r.txt 2>&1
      else env $var=$v timeout 900 python bench.py "$@" > gpurun_out/${tag}_${v}_$r.txt 2>&1; fi
      summ gpurun_out/${tag}_${v}_$r.txt
    done; done ;;
  launches)
    timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file gpurun_out/${tag}_launches.csv python bench.py --no-cpu "$@" > gpurun_out/${tag}_under_ncu.txt 2>&1
    python tools/launch_summary.py gpurun_out/${tag}_launches.csv ;;
  ncu)
    regex=$1; skip=$2; shift 2
    timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"$regex" -s $skip -c 1 \
      -o gpurun_out/${tag} python bench.py --no-cpu "$@" > gpurun_out/${tag}_ncu_log.txt 2>&1
    ls -la gpurun_out/${tag}.ncu-rep ;;
  configs)
    timeout 2400 python tools/bench_configs.py "$@" > gpurun_out/${tag}_configs.txt 2>&1
    tail -8 gpurun_out/${tag}_configs.txt ;;
  *) echo "unknown subcommand $cmd"; exit 2 ;;
esac
