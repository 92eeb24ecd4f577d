# kernel-time distribution of viscous (AV forced) RK steps: curved P=4 (all curved) and affine P=4
mkdir -p gpurun_out
for a in "--n 24 --visc" "--n 24 --visc --frac 0" "--n 24 --visc --riemann hllc"; do
  timeout 600 python scripts/bench_curved.py $a --steps 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$a', 'ms/step %.2f dof/s %.3e' % (d['ms_per_step'], d['dof_updates_per_s']))"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/visc_launches.csv python scripts/bench_curved.py --n 24 --visc --steps 1 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/visc_launches_affine.csv python scripts/bench_curved.py --n 24 --visc --frac 0 --steps 1 > /dev/null 2>&1
ls -la gpurun_out/visc_launches*.csv
