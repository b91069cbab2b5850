mkdir -p gpurun_out
export PE_PREFILL_WAVES=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"prefill" --csv --log-file gpurun_out/prefill_times.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-decode > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"prefill_select_cta_kernel" -s 2 -c 1 -o gpurun_out/prof_select python bench.py --steps 1 --warmup 3 --no-cpu --no-decode > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/prefill_times.csv
