# ncu evidence for the current build; usage: bash scripts/gpu_ncu.sh TAG
TAG=${1:-x}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_$TAG.log 2>&1
tail -1 gpurun_out/ncu_launch_$TAG.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_rhs -s 3 -c 1 -o gpurun_out/prof_rhs_$TAG python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_$TAG.log 2>&1
tail -1 gpurun_out/ncu_full_$TAG.log
timeout 900 ncu --set full --clock-control none -k regex:k_traces -s 3 -c 1 -o gpurun_out/prof_tr_$TAG python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_tr_$TAG.log 2>&1
tail -1 gpurun_out/ncu_full_tr_$TAG.log
