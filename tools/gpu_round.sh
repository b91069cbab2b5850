# Round measurement: GPU tests, default bench line, reference arm, launch list
# of the bench command and ncu --set full captures of K2 and the prefill kernels.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/round_tests.txt 2>&1; tail -2 gpurun_out/round_tests.txt
timeout 600 python bench.py > gpurun_out/bench_round.txt 2>&1; tail -1 gpurun_out/bench_round.txt
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_round.txt 2>&1; tail -1 gpurun_out/bench_ref_round.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"append|evict|prefill|attention" --csv --log-file gpurun_out/bench_launches_round.csv python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_under_ncu_round.txt 2>&1
python tools/launch_summary.py gpurun_out/bench_launches_round.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"evict_score_kernel" -s 1 -c 1 -o gpurun_out/prof_round_k2 python bench.py --steps 1 --warmup 3 --no-cpu --no-decode > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"prefill_score_kernel|prefill_select_stream512_kernel|prefill_copy_kernel" -s 3 -c 3 -o gpurun_out/prof_round_k1 python bench.py --steps 1 --warmup 3 --no-cpu --no-decode > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attention_tma_kernel" -s 2 -c 1 -o gpurun_out/prof_round_k3 python bench.py --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"append_kernel" -s 40 -c 1 -o gpurun_out/prof_round_k0 python bench.py --steps 3 --warmup 3 --no-cpu --no-decode > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
