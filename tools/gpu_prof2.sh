mkdir -p gpurun_out
./tools/ubench_fp64 | tee gpurun_out/ubench.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"evict_score_kernel|attention_split_kernel" -c 2 -o gpurun_out/prof2 python tools/prof_kernels.py --layers 1 > gpurun_out/ncu2.log 2>&1
tail -2 gpurun_out/ncu2.log
