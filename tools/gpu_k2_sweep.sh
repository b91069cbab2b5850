for v in 28 8 14 20 40 56 28; do
  PE_K2_CTAS_PER_SM=$v timeout 300 python bench.py --no-cpu --no-decode --steps 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($v, 'layer_us', d['p50_evict_layer_launch_us'], 'layer_gbs', d['evict_layer_launch_gbs'], 'step_K2', d['roofline']['achieved'])"
done
