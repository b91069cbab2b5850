mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-decode > gpurun_out/bench5.txt 2>&1; tail -1 gpurun_out/bench5.txt | cut -c1-1500
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none --csv --log-file gpurun_out/launches5.csv python tools/prof_kernels.py --layers 2 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches5.csv
