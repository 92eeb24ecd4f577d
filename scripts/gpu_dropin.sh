# the reference's own tests linked against the GPU adapter (drop-in evidence)
mkdir -p gpurun_out
timeout 600 ./oracle/_ref/test_solver_gpu > gpurun_out/test_solver_gpu.log 2>&1; echo "test_solver_gpu rc=$?"; tail -4 gpurun_out/test_solver_gpu.log
timeout 2400 ./oracle/_ref/acceptance_gpu ${1:-3 4 6 12 10 11} --fixture-dir /tmp/accfx > gpurun_out/acceptance_gpu.log 2>&1; echo "acceptance_gpu rc=$?"; grep -E "PASS|FAIL|EXCEPTION|cost model|asymmetry" gpurun_out/acceptance_gpu.log
