# warp-autonomous default: full GPU suite + smoke + bench (default) + order sweep p=1..5
mkdir -p gpurun_out/r2wa gpurun_out/sweep
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2wa/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2wa/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/r2wa/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2wa/smoke.log
timeout 900 python bench.py > gpurun_out/r2wa/bench.json 2> gpurun_out/r2wa/bench.err; echo "bench rc=$?"
for p in 1 2 3 4 5; do
  timeout 900 python bench.py --p $p --n 44 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --curved-n 0 > gpurun_out/sweep/p$p.json 2> gpurun_out/sweep/p$p.err
  python -c "
import json; d=json.load(open('gpurun_out/sweep/p$p.json')); r=d['roofline']
print('p=$p value %.3e rhs %.3f ms fp64 frac %.3f hbm frac %.2f fused %s' % (d['value'], r['kernel_ms_avg'], r['frac'], r['hbm_frac'], r['fused_traces']))" 2>&1 | tail -1
done
