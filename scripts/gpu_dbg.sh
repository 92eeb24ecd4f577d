# phase breakdown of k_rhs (P=4): full / no-SIMT / no-GEMM, with and without carveout
for cfg in "0 0" "1 0" "2 0" "0 1"; do
  set -- $cfg
  if [ "$2" = "1" ]; then export CDG_CARVEOUT=1; else unset CDG_CARVEOUT; fi
  CDG_KDBG=$1 timeout 600 python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/dbg_$1_$2.json 2> gpurun_out/dbg_$1_$2.err
  python -c "
import json; d=json.load(open('gpurun_out/dbg_$1_$2.json')); r=d['roofline']
print('dbg $1 carve $2: rhs %.2f ms trace %.2f ms' % (r['kernel_ms_avg'], r['trace_kernel_ms_avg']))" 2>&1 | tail -1
done
