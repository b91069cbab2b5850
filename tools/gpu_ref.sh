timeout 600 python bench.py --impl reference > gpurun_out/ref.txt 2>&1; tail -1 gpurun_out/ref.txt
timeout 600 python bench.py --no-decode --steps 3 > gpurun_out/cpu.txt 2>&1; python -c "
import json; d=json.loads([x for x in open('gpurun_out/cpu.txt') if x.startswith('{')][-1]); print(d['cpu_baseline'])"
