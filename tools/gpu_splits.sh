mkdir -p gpurun_out
for sp in 2 3 4 5 6 8 12; do
  PE_ATTN_SPLITS=$sp timeout 300 python bench.py --no-cpu --steps 3 --warmup 3 > gpurun_out/sp_$sp.txt 2>&1
  python - "$sp" <<'PY'
import json,sys
s=sys.argv[1]
line=[l for l in open(f"gpurun_out/sp_{s}.txt") if l.startswith("{")][-1]
d=json.loads(line); print("splits",s,"attn",d["decode"]["attention_us_per_layer_p50"],"us", d["decode"]["attention_gbs"], "tok/s", d["decode"]["tokens_per_s"])
PY
done
