mkdir -p gpurun_out/r2
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2/pytest_gpu.log
mkdir -p gpurun_out/sweep
for p in 1 2 3; do
  timeout 900 python bench.py --p $p --n 44 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --curved-n 0 > gpurun_out/sweep/p$p.json 2> gpurun_out/sweep/p$p.err
  python -c "
import json; d=json.load(open('gpurun_out/sweep/p$p.json')); r=d['roofline']
print('p=$p value %.3e DOF-upd/s  rhs %.3f ms trace %.3f ms  fp64 frac %.3f  hbm %.0f GB/s (%.2f) fused %s' % (d['value'], r['kernel_ms_avg'], r['trace_kernel_ms_avg'], r['frac'], r['hbm_achieved_gbs'], r['hbm_frac'], r['fused_traces']))" 2>&1 | tail -1
done
