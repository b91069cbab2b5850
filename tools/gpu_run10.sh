mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench10.txt 2>&1; tail -1 gpurun_out/bench10.txt | cut -c1-2200
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"prefill_select|append_kernel" -c 3 -o gpurun_out/prof10 python tools/prof_kernels.py --layers 1 > gpurun_out/ncu10.log 2>&1
tail -1 gpurun_out/ncu10.log
