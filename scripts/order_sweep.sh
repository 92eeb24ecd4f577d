# BASELINE config 4: order sweep P=1..8 on one fixed synthetic mesh (make_cube_mesh(44) = 511,104 tets)
mkdir -p gpurun_out/sweep
for p in 1 2 3 4 5 6 7 8; do
  CFL=0.5; [ $p -ge 7 ] && CFL=0.2; [ $p -ge 8 ] && CFL=0.05  # the random state is unstable at CFL 0.5 for p >= 7 (oracle agrees)
  timeout 900 python bench.py --p $p --n ${N:-44} --steps 5 --warmup 3 --cfl $CFL --no-cpu-baseline --no-e2e --curved-n 0 > gpurun_out/sweep/p$p.json 2> gpurun_out/sweep/p$p.err
  python -c "
import json; d=json.load(open('gpurun_out/sweep/p$p.json')); r=d['roofline']
print('p=$p value %.3e DOF-upd/s  rhs %.2f ms trace %.2f ms  fp64 frac %.3f  hbm %.0f GB/s (%.2f)' % (d['value'], r['kernel_ms_avg'], r['trace_kernel_ms_avg'], r['frac'], r['hbm_achieved_gbs'], r['hbm_frac']))" 2>&1 | tail -1
done
