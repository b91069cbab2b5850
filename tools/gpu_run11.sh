mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench11.txt 2>&1; tail -1 gpurun_out/bench11.txt | cut -c1-2200
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches11.csv python tools/prof_kernels.py --layers 2 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches11.csv | head -12
