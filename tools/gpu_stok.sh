mkdir -p gpurun_out
for cfg in "64 2" "64 1" "64 3" "96 2" "128 2" "64 2" "256 4"; do
  set -- $cfg
  PE_SCORE_TOKENS=$1 PE_PREFILL_WAVES=$2 timeout 300 python bench.py --no-cpu --no-decode --steps 3 --warmup 3 > gpurun_out/stok.txt 2>&1
  python -c "
import json; d=json.loads([x for x in open('gpurun_out/stok.txt') if x.startswith('{')][-1]); print('tokens $1 waves $2 prefill', d['prefill']['ms_per_layer_p50'], d['prefill']['frac'])"
done
