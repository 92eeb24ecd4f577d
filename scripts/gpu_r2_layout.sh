# compact device layout check: full GPU suite + order sweep
mkdir -p gpurun_out/r2
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2/pytest_gpu.log
bash scripts/order_sweep.sh
