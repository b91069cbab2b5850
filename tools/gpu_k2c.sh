mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "decode or invariants or smoke or facade" 2>&1 | tail -2
timeout 300 python bench.py --no-cpu --no-decode --steps 5 > gpurun_out/k2c.txt 2>&1; python -c "
import json; d=json.loads([x for x in open('gpurun_out/k2c.txt') if x.startswith('{')][-1]); print('cached p50', d['p50_evict_step_us_cached'], 'value', d['value'], 'checks', d['checks']['cadence_ok'], d['checks']['invariant_violations'])"
