for v in 2 3; do CDG_KCFG=$v timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "p4 or rk_steps or determinism or inadmissible or zero_rhs or freestream" 2>&1 | tail -1; done
for v in 2 3 0; do
  CDG_KCFG=$v timeout 600 python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/sp_$v.json 2> gpurun_out/sp_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/sp_$v.json')); r=d['roofline']
print('kcfg $v: value %.3e rhs %.2f ms trace %.2f ms frac %.3f' % (d['value'], r['kernel_ms_avg'], r['trace_kernel_ms_avg'], r['frac']))" 2>&1 | tail -1
done
