timeout 900 ncu --set full --clock-control none --import-source on -k regex:"evict_cached_kernel" -s 0 -c 1 -o gpurun_out/prof_k2c python bench.py --steps 1 --warmup 3 --no-cpu --no-decode > /dev/null 2>&1
ls -la gpurun_out/prof_k2c.ncu-rep
