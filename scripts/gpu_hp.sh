# high-p kernel variants on make_cube_mesh(44)
for pk in ${1:-"5 0" "6 0" "7 0" "7 1" "7 2" "8 0" "8 1" "8 2"}; do
  set -- $pk; p=$1; k=$2; CFL=0.5; [ $p -ge 7 ] && CFL=0.2
  CDG_KCFG=$k timeout 900 python bench.py --p $p --n 44 --cfl $CFL --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > /tmp/hp_${p}_$k.json 2>/tmp/hp_${p}_$k.err
  python -c "
import json; d=json.load(open('/tmp/hp_${p}_$k.json')); r=d['roofline']
print('p=$p cfg $k: value %.3e rhs %.2f ms trace %.2f ms frac %.3f' % (d['value'], r['kernel_ms_avg'], r['trace_kernel_ms_avg'], r['frac']))" 2>&1 | tail -1
done
for k in 0 1 2; do CDG_KCFG=$k timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "rhs_matches_oracle and (5 or 6 or 7 or 8)" 2>&1 | tail -1; done
