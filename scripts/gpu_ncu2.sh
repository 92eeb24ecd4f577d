# ncu full capture of one kernel + text exports (the .ncu-rep stays on the box unless small)
# usage: bash scripts/gpu_ncu2.sh TAG KREGEX "bench args"
TAG=$1; KRE=$2; BARGS=$3
mkdir -p gpurun_out/ncu
REP=/tmp/prof_$TAG
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$KRE -s 3 -c 1 -f -o $REP python bench.py $BARGS --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu/log_$TAG.txt 2>&1
tail -1 gpurun_out/ncu/log_$TAG.txt
ncu -i $REP.ncu-rep --page raw --csv > gpurun_out/ncu/raw_$TAG.csv 2>/dev/null
ncu -i $REP.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu/sass_$TAG.csv 2>/dev/null
ncu -i $REP.ncu-rep --page source --csv --print-source cuda > gpurun_out/ncu/cuda_$TAG.csv 2>/dev/null
ncu -i $REP.ncu-rep --page details --csv > gpurun_out/ncu/details_$TAG.csv 2>/dev/null
SZ=$(stat -c %s $REP.ncu-rep); if [ "$SZ" -lt 15000000 ]; then cp $REP.ncu-rep gpurun_out/ncu/; fi
gzip -f gpurun_out/ncu/sass_$TAG.csv
ls -la gpurun_out/ncu | tail -8
