# round evidence for the default build: bench line (with cpu baseline), ncu launch list, ncu full capture
TAG=${1:-final}
mkdir -p gpurun_out/ev
timeout 900 python bench.py > gpurun_out/ev/bench_$TAG.json 2> gpurun_out/ev/bench_$TAG.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_rhs|k_interp|k_timestep|k_residual" -c 40 --csv --log-file gpurun_out/ev/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ev/ncu_launch_$TAG.log 2>&1; echo "launches rc=$?"
bash scripts/gpu_ncu2.sh rhs_$TAG k_rhs_row ""
