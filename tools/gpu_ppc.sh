mkdir -p gpurun_out
for p in 0 32 64 96 129 257 64 0; do
  if [ "$p" = "0" ]; then unset PE_EVICT_PPC; else export PE_EVICT_PPC=$p; fi
  timeout 300 python bench.py --no-cpu --no-decode --steps 20 > gpurun_out/ppc.txt 2>&1
  python -c "
import json; d=json.loads([x for x in open('gpurun_out/ppc.txt') if x.startswith('{')][-1]); print('ppc $p value', d['value'], 'K2', d['roofline']['achieved'], 'p50', d['p50_evict_step_us'], 'layer', d['p50_evict_layer_launch_us'])"
done
