# parity + bench (no profiler); usage: bash scripts/gpu_check.sh TAG
TAG=${1:-x}
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -2 gpurun_out/bench_$TAG.err
python -c "
import json; d=json.load(open('gpurun_out/bench_$TAG.json'))
r=d['roofline']; print('value %.3e ms/step %.1f rhs %.2f ms trace %.2f ms achieved %.2f TF frac %.3f hbm %.0f GB/s e2e %.3e' % (d['value'], d['ms_per_step'], r['kernel_ms_avg'], r['trace_kernel_ms_avg'], r['achieved'], r['frac'], r['hbm_achieved_gbs'], d['e2e']['value']))
print('peaks', r['peak'], r['fp64_dfma_peak_tflops'], r['fp64_dmma_k8_tflops'])
"
