# k_rhs_rowc tuning variants (CDG_KCFG) on the curved P=4 bench
for k in ${KS:-0 1 2 3}; do
  CDG_KCFG=$k timeout 600 python scripts/bench_curved.py --n ${N:-24} ${BARGS} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('kcfg $k', 'rhs %.3f ms frac %.3f hbm %.0f' % (d['rhs_kernel_ms'], d['frac'], d['hbm_gbs']))"
done
