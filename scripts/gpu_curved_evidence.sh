# curved-path evidence: bench_configs (C1-C3 vs the reference CPU), curved throughput lines, ncu of k_rhs_rowc
mkdir -p gpurun_out/cev gpurun_out/ncu
timeout 1500 python scripts/bench_configs.py > gpurun_out/cev/configs.jsonl 2> gpurun_out/cev/configs.err; echo "configs rc=$?"
for a in "--n 32" "--n 32 --riemann hllc" "--n 32 --frac 0.4" "--n 24 --visc"; do
  timeout 600 python scripts/bench_curved.py $a >> gpurun_out/cev/curved.jsonl 2>> gpurun_out/cev/curved.err
done
bash scripts/gpu_ncu_rowc.sh
