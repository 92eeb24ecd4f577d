# ncu full capture of one kernel launch of a given library build (tuning variants)
# usage: bash scripts/gpu_ncu_lib.sh TAG KREGEX LIB "tune_p4 args"
TAG=$1; KRE=$2; LIB=$3; TARGS=$4
mkdir -p gpurun_out/ncu
REP=/tmp/prof_$TAG
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$KRE -s 4 -c 1 -f -o $REP python scripts/tune_p4.py --child $TARGS --steps 1 $LIB > gpurun_out/ncu/log_$TAG.txt 2>&1
tail -1 gpurun_out/ncu/log_$TAG.txt
ncu -i $REP.ncu-rep --page raw --csv > gpurun_out/ncu/raw_$TAG.csv 2>/dev/null
ncu -i $REP.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu/sass_$TAG.csv 2>/dev/null
ncu -i $REP.ncu-rep --page details --csv > gpurun_out/ncu/details_$TAG.csv 2>/dev/null
gzip -f gpurun_out/ncu/sass_$TAG.csv
ls -la gpurun_out/ncu | tail -4
