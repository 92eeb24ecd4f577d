# microbench + full gpu test suite; usage: bash scripts/gpu_tests.sh TAG
TAG=${1:-x}
mkdir -p gpurun_out
[ -x microbench/fp64_mix ] && timeout 120 ./microbench/fp64_mix > gpurun_out/fp64_mix_$TAG.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/pytest_$TAG.log
