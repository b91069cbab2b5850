mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"prefill_select_cta_kernel|prefill_copy_kernel|prefill_score_kernel" -s 3 -c 3 -o gpurun_out/prof_prefill python bench.py --steps 1 --warmup 3 --no-cpu --no-decode > gpurun_out/prof_prefill.log 2>&1
ls -la gpurun_out/prof_prefill.ncu-rep
