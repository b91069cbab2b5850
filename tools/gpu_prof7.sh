mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"prefill_pack|attention_mma|evict_score_kernel|prefill_score" -c 4 -o gpurun_out/prof7 python tools/prof_kernels.py --layers 1 > gpurun_out/ncu7.log 2>&1
tail -1 gpurun_out/ncu7.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"plan|append|evict|prefill|attention" --csv --log-file gpurun_out/bench_launches_r1.csv python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_under_ncu.txt 2>&1
python tools/launch_summary.py gpurun_out/bench_launches_r1.csv
