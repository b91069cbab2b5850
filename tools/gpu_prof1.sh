set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"evict_score_kernel|prefill_kernel|attention_split_kernel|append_kernel" -c 6 -o gpurun_out/prof1 python tools/prof_kernels.py --layers 2 > gpurun_out/ncu1.log 2>&1
tail -3 gpurun_out/ncu1.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches1.csv python tools/prof_kernels.py --layers 4 > /dev/null 2>&1
wc -l gpurun_out/launches1.csv
