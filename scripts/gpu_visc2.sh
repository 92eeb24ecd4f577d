# viscous row kernels: gpu tests + AV throughput + headline bench unchanged
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for a in "--n 24 --visc" "--n 24 --visc --frac 0" "--n 32 --visc --frac 0"; do
  timeout 600 python scripts/bench_curved.py $a --steps 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$a', 'ms/step %.2f dof/s %.3e' % (d['ms_per_step'], d['dof_updates_per_s']))"
done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_chk.json 2>gpurun_out/bench_chk.err
python -c "import json; d=json.load(open('gpurun_out/bench_chk.json')); print('bench value %.4e frac %.3f e2e %.3e' % (d['value'], d['roofline']['frac'], d['e2e']['value']))"
