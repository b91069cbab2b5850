set -u
mkdir -p gpurun_out
N="timeout 1500 ncu --set full --clock-control none --import-source on"
$N -k regex:evict_score_kernel -s 3 -c 1 -o gpurun_out/r2_k2 python bench.py --no-cpu --no-decode --steps 2 --warmup 3 > gpurun_out/r2_k2_log.txt 2>&1
$N -k regex:append_kernel -s 40 -c 1 -o gpurun_out/r2_k0 python bench.py --no-cpu --no-decode --steps 2 --warmup 3 > gpurun_out/r2_k0_log.txt 2>&1
$N -k regex:"prefill_score_kernel|prefill_copy_score|gsel_" -s 8 -c 7 -o gpurun_out/r2_k1 python tools/prefill_ab.py --rounds 2 --variant base: > gpurun_out/r2_k1_log.txt 2>&1
$N -k regex:attention_tma -s 40 -c 1 -o gpurun_out/r2_k3 python bench.py --no-cpu --steps 2 --warmup 3 > gpurun_out/r2_k3_log.txt 2>&1
ls -la gpurun_out/*.ncu-rep
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2_torchrun1.txt 2>&1; tail -1 gpurun_out/r2_torchrun1.txt | cut -c1-300
timeout 900 python bench.py --gpus 2 > gpurun_out/r2_gpus2.txt 2>&1; echo "gpus2 rc=$?"; tail -2 gpurun_out/r2_gpus2.txt | cut -c1-300
