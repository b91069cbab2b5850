mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"prefill_select" -c 1 -o gpurun_out/prof13 python tools/prof_kernels.py --layers 1 > gpurun_out/ncu13.log 2>&1
PE_SELECT=cluster timeout 600 ncu --set full --clock-control none --import-source on -k regex:"prefill_select" -c 1 -o gpurun_out/prof13b python tools/prof_kernels.py --layers 1 > gpurun_out/ncu13b.log 2>&1
tail -1 gpurun_out/ncu13.log gpurun_out/ncu13b.log
