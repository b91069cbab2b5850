mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches14.csv python tools/prof_kernels.py --layers 2 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches14.csv | grep -E "select|copy|score"
PE_SELECT=cluster timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:select --csv --log-file gpurun_out/launches14b.csv python tools/prof_kernels.py --layers 2 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches14b.csv | grep -E "select"
