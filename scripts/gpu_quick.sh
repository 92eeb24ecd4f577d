# quick: parity subset + bench + dbg1 ; usage: bash scripts/gpu_quick.sh TAG
TAG=${1:-x}
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for dbg in 0 1; do
  CDG_KDBG=$dbg timeout 600 python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/q_${TAG}_$dbg.json 2> gpurun_out/q_${TAG}_$dbg.err
  python -c "
import json; d=json.load(open('gpurun_out/q_${TAG}_$dbg.json')); r=d['roofline']
print('$TAG dbg $dbg: value %.3e rhs %.2f ms trace %.2f ms frac %.3f' % (d['value'], r['kernel_ms_avg'], r['trace_kernel_ms_avg'], r['frac']))" 2>&1 | tail -1
done
