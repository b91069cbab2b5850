mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench2.txt 2>&1; tail -3 gpurun_out/bench2.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"evict_score_kernel|prefill_score|prefill_pack|append_kernel" -c 4 -o gpurun_out/prof3 python tools/prof_kernels.py --layers 1 > gpurun_out/ncu3.log 2>&1
tail -1 gpurun_out/ncu3.log
