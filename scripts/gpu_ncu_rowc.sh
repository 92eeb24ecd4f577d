# ncu full capture of k_rhs_rowc (curved P=4) + text exports
mkdir -p gpurun_out/ncu
REP=/tmp/prof_rowc
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rhs_rowc -s 3 -c 1 -f -o $REP python scripts/bench_curved.py --n 24 --steps 1 > gpurun_out/ncu/log_rowc.txt 2>&1
tail -2 gpurun_out/ncu/log_rowc.txt
ncu -i $REP.ncu-rep --page raw --csv > gpurun_out/ncu/raw_rowc.csv 2>/dev/null
ncu -i $REP.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu/sass_rowc.csv 2>/dev/null
gzip -f gpurun_out/ncu/sass_rowc.csv
ncu -i $REP.ncu-rep --page details --csv > gpurun_out/ncu/details_rowc.csv 2>/dev/null
ls -la gpurun_out/ncu | grep rowc
