timeout 900 python -m pytest tests -m gpu -q -x -k "prefill or smoke or golden or cfg3 or facade or cfg1" 2>&1 | tail -1
timeout 300 python tools/sel_timing.py
