# kernel-config sweep (CDG_KCFG) + prefetch masks; usage: bash scripts/gpu_sweep.sh TAG "cfgs" "prefetch masks" "bench args"
TAG=${1:-x}; CFGS=${2:-"0 1 2 3 4"}; PFS=${3:-"15"}; BARGS=${4:-""}
mkdir -p gpurun_out
for k in $CFGS; do
  CDG_KCFG=$k timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "rhs_matches_oracle and 4 or rk_steps_match and 4" > gpurun_out/pytest_${TAG}_$k.log 2>&1; echo "cfg $k pytest rc=$? $(tail -1 gpurun_out/pytest_${TAG}_$k.log)"
  for pf in $PFS; do
  CDG_KCFG=$k CDG_PREFETCH=$pf timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $BARGS > gpurun_out/s_${TAG}_${k}_${pf}.json 2> gpurun_out/s_${TAG}_${k}_${pf}.err
  python -c "
import json; d=json.load(open('gpurun_out/s_${TAG}_${k}_${pf}.json')); r=d['roofline']
print('cfg $k pf $pf: value %.3e rhs %.2f ms trace %.2f ms frac %.3f' % (d['value'], r['kernel_ms_avg'], r['trace_kernel_ms_avg'], r['frac']))" 2>&1 | tail -1
done; done
