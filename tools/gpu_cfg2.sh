for w in 1 2 4; do PE_PREFILL_WAVES=$w timeout 600 python tools/bench_configs.py --configs cfg2 > /tmp/c2.txt 2>/tmp/c2.err; tail -2 /tmp/c2.err; python -c "
import json; d=json.loads(open('/tmp/c2.txt').readline()); print('waves $w', d['prefill'])"; done
