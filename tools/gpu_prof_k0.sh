mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"append_kernel" -s 40 -c 1 -o gpurun_out/prof_k0 python bench.py --steps 3 --warmup 3 --no-cpu --no-decode > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"append_kernel" --csv --log-file gpurun_out/k0_times.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-decode > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/k0_times.csv
