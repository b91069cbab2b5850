mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench20.txt 2>&1; tail -1 gpurun_out/bench20.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"append|evict|prefill|attention" --csv --log-file gpurun_out/bench_launches_r1b.csv python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_under_ncu20.txt 2>&1
python tools/launch_summary.py gpurun_out/bench_launches_r1b.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"evict_score_kernel" -s 1 -c 1 -o gpurun_out/prof20_k2 python bench.py --steps 1 --warmup 3 --no-cpu --no-decode > /dev/null 2>&1
ls -la gpurun_out/prof20_k2.ncu-rep
