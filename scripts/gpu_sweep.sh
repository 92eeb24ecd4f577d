# variant sweep for the P=4 kernel; usage: bash scripts/gpu_sweep.sh TAG "0 1 2 3 4"
TAG=${1:-x}; VARS=${2:-"0 1 2 3 4"}
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for v in $VARS; do
  CDG_KCFG=$v timeout 600 python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/sweep_${TAG}_$v.json 2> gpurun_out/sweep_${TAG}_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/sweep_${TAG}_$v.json')); r=d['roofline']
print('variant $v: value %.3e rhs %.2f ms trace %.2f ms frac %.3f' % (d['value'], r['kernel_ms_avg'], r['trace_kernel_ms_avg'], r['frac']))" || tail -3 gpurun_out/sweep_${TAG}_$v.err
done
