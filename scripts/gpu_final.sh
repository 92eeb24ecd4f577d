# final round evidence: bench line, BASELINE configs, order sweep, curved lines
mkdir -p gpurun_out/fin gpurun_out/sweep
timeout 900 python bench.py > gpurun_out/fin/bench.json 2> gpurun_out/fin/bench.err; echo "bench rc=$?"
timeout 1500 python scripts/bench_configs.py > gpurun_out/fin/configs.jsonl 2> gpurun_out/fin/configs.err; echo "configs rc=$?"
bash scripts/order_sweep.sh
for a in "--n 32" "--n 32 --riemann hllc" "--n 32 --frac 0.4" "--n 24 --visc"; do
  timeout 600 python scripts/bench_curved.py $a >> gpurun_out/fin/curved.jsonl 2>> gpurun_out/fin/curved.err
done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fin/bench_ref.json 2> gpurun_out/fin/bench_ref.err; echo "ref rc=$?"
