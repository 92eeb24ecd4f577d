# k_rhs_rowc prefetch-mask sweep (CDG_PREFETCH_ROWC), curved P=4 at 197k tets
for pf in ${PFS:-0 1 2 3 4 7}; do
  CDG_PREFETCH_ROWC=$pf timeout 600 python scripts/bench_curved.py --n 32 ${BARGS} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pf $pf', 'rhs %.3f ms frac %.3f hbm %.0f' % (d['rhs_kernel_ms'], d['frac'], d['hbm_gbs']))"
done
