set -x
python -c "from paper_1208_4772_b200 import gpu; gpu.lib(); print(gpu.measure_fp64_peak())"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err
tail -3 gpurun_out/bench_r1.err; cat gpurun_out/bench_r1.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_bench.log 2>&1
tail -2 gpurun_out/ncu_launch_bench.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_rhs -s 3 -c 1 -o gpurun_out/prof_rhs_r1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_traces -s 3 -c 1 -o gpurun_out/prof_tr_r1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_tr.log 2>&1
ls -la gpurun_out
