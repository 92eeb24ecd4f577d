# round-2 checkpoint: GPU test suite + smoke + 1-GPU bench (default args, the driver's command)
mkdir -p gpurun_out/r2
( lscpu; nproc; free -g; nvidia-smi ) > gpurun_out/r2/box.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS:-} > gpurun_out/r2/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/r2/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2/smoke.log
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/r2/bench.json 2> gpurun_out/r2/bench.err; echo "bench rc=$?"; tail -c 600 gpurun_out/r2/bench.err
timeout 600 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/r2/bench_ref.json 2> gpurun_out/r2/bench_ref.err; echo "ref rc=$?"
