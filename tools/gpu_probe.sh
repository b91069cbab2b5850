timeout 600 python bench.py --no-cpu --no-decode --steps 5 > /tmp/bp.txt 2>&1; python -c "
import json; d=json.loads([x for x in open('/tmp/bp.txt') if x.startswith('{')][-1]); print(d['roofline'])"
