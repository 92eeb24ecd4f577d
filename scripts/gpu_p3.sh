# p=3 warp-tile kernel vs CTA kernel + parity; usage: bash scripts/gpu_p3.sh TAG
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition.py tests/test_gpu_curved.py -q -x -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
for p in 1 2 3; do for nw in 0 1; do
  CDG_NOWARP=$nw timeout 600 python bench.py --p $p --n 70 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_${TAG}_p${p}_nw$nw.json 2> gpurun_out/b_${TAG}_p${p}_nw$nw.err
  python -c "
import json; d=json.load(open('gpurun_out/b_${TAG}_p${p}_nw$nw.json')); r=d['roofline']
print('p=$p nowarp=$nw: value %.3e rhs %.2f ms trace %.2f ms frac %.3f' % (d['value'], r['kernel_ms_avg'], r['trace_kernel_ms_avg'], r['frac']))" 2>&1 | tail -1
done; done
