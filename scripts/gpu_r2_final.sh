# round-2 evidence for the warp-autonomous kernels: GPU suite, smoke, bench (both arms),
# launch list, ncu of k_rhs_wa (4.09M tets) and k_rhs_wac (curved block), sanitizer, order sweep
mkdir -p gpurun_out/r2f gpurun_out/ncu gpurun_out/san gpurun_out/sweep
( lscpu; nproc; free -g; nvidia-smi ) > gpurun_out/r2f/box.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2f/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2f/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/r2f/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2f/smoke.log
timeout 900 python bench.py > gpurun_out/r2f/bench.json 2> gpurun_out/r2f/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/r2f/bench_ref.json 2> gpurun_out/r2f/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2f/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --curved-n 0 > gpurun_out/r2f/launches.log 2>&1; echo "launches rc=$?"
bash scripts/gpu_ncu2.sh r2wa k_rhs_wa "--curved-n 0"
bash scripts/gpu_ncu2.sh r2wac k_rhs_wac "--n 8 --curved-n 32"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 python scripts/sanitize_case.py > gpurun_out/san/$tool.txt 2>&1
  echo "$tool rc=$?"; tail -1 gpurun_out/san/$tool.txt
done
for p in 1 2 3 4 5 6 7 8; do
  CFL=0.5; [ $p -ge 7 ] && CFL=0.2; [ $p -ge 8 ] && CFL=0.05
  timeout 900 python bench.py --p $p --n 44 --steps 5 --warmup 3 --cfl $CFL --no-cpu-baseline --no-e2e --curved-n 0 > gpurun_out/sweep/p$p.json 2> gpurun_out/sweep/p$p.err
  python -c "
import json; d=json.load(open('gpurun_out/sweep/p$p.json')); r=d['roofline']
print('p=$p value %.3e rhs %.3f ms trace %.3f fp64 frac %.3f hbm frac %.2f %s' % (d['value'], r['kernel_ms_avg'], r['trace_kernel_ms_avg'], r['frac'], r['hbm_frac'], r['kernel'][:12]))" 2>&1 | tail -1
done
