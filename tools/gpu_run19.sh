mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-decode > gpurun_out/bench19a.txt 2>&1; tail -1 gpurun_out/bench19a.txt | cut -c1-1500
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-decode --evict-launch step > gpurun_out/bench19b.txt 2>&1; tail -1 gpurun_out/bench19b.txt | cut -c1-1500
