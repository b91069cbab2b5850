timeout 900 ncu --set full --clock-control none --import-source on -k regex:"prefill_select_cta_kernel" -s 2 -c 1 -o gpurun_out/prof_sel2 python bench.py --steps 1 --warmup 3 --no-cpu --no-decode > /dev/null 2>&1
ls -la gpurun_out/prof_sel2.ncu-rep
