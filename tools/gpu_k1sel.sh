mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "prefill or smoke or golden or cfg3 or facade or cfg1" 2>&1 | tail -2
for r in 1 2; do
timeout 300 python bench.py --no-cpu --no-decode --steps 3 --warmup 3 > gpurun_out/k1s.txt 2>&1; python -c "
import json; d=json.loads([x for x in open('gpurun_out/k1s.txt') if x.startswith('{')][-1]); print('cfg3 prefill', d['prefill']['ms_per_layer_p50'], d['prefill']['frac'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"prefill" --csv --log-file gpurun_out/pf_times.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-decode > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/pf_times.csv
