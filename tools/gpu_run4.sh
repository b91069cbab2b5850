mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-decode > gpurun_out/bench4.txt 2>&1; tail -1 gpurun_out/bench4.txt | cut -c1-1500
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches4.csv python tools/prof_kernels.py --layers 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"evict_score_kernel|prefill_score|prefill_pack" -c 3 -o gpurun_out/prof4 python tools/prof_kernels.py --layers 1 > gpurun_out/ncu4.log 2>&1
tail -1 gpurun_out/ncu4.log
