mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "prefill or golden" 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:select --csv --log-file gpurun_out/launches16.csv python tools/prof_kernels.py --layers 2 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches16.csv | grep -E "select"
PE_SELECT=cluster timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:select --csv --log-file gpurun_out/launches16b.csv python tools/prof_kernels.py --layers 2 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches16b.csv | grep -E "select"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"prefill_select" -c 1 -o gpurun_out/prof16 python tools/prof_kernels.py --layers 1 > /dev/null 2>&1
