# curved-path throughput at GPU-filling sizes + one ncu capture of k_rhs_curved
mkdir -p gpurun_out/ncu
for a in "--n 24 --frac 1.0" "--n 32 --frac 1.0" "--n 32 --frac 0.4" "--n 32 --frac 1.0 --riemann hllc"; do
  timeout 600 python scripts/bench_curved.py $a >> gpurun_out/curved.jsonl 2>> gpurun_out/curved.err
done
cat gpurun_out/curved.jsonl; tail -3 gpurun_out/curved.err
REP=/tmp/prof_curved
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rhs_curved -s 3 -c 1 -f -o $REP python scripts/bench_curved.py --n 16 --steps 1 > gpurun_out/ncu/log_curved.txt 2>&1
ncu -i $REP.ncu-rep --page raw --csv > gpurun_out/ncu/raw_curved.csv 2>/dev/null
ncu -i $REP.ncu-rep --page details --csv > gpurun_out/ncu/details_curved.csv 2>/dev/null
ncu -i $REP.ncu-rep --page source --csv --print-source cuda > gpurun_out/ncu/cuda_curved.csv 2>/dev/null
ls -la gpurun_out/ncu | grep curved
