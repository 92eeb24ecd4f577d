# curved row kernel: parity tests + throughput (rowc vs the CTA curved kernel)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_curved.py tests/test_gpu_parity.py -q -x 2>&1 | tail -4
for a in "--n 24" "--n 32" "--n 32 --frac 0.4" "--n 32 --riemann hllc"; do
  timeout 600 python scripts/bench_curved.py $a 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('rowc', '$a', 'rhs %.3f ms tr %.3f frac %.3f dof/s %.3e hbm %.0f' % (d['rhs_kernel_ms'], d['trace_kernel_ms'], d['frac'], d['dof_updates_per_s'], d['hbm_gbs']))"
done
CDG_NOROWC=1 timeout 600 python scripts/bench_curved.py --n 32 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cta n32', 'rhs %.3f ms frac %.3f' % (d['rhs_kernel_ms'], d['frac']))"
