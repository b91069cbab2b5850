mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attention_mma_kernel" -s 2 -c 1 -o gpurun_out/prof_attn python bench.py --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
ls -la gpurun_out/prof_attn.ncu-rep
