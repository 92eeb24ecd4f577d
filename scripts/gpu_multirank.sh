# functional check of bench.py's N>1 path on a 1-GPU box: 2 ranks on cuda:0,
# gloo with host-staged halos (not a measurement)
mkdir -p gpurun_out
CDG_BENCH_DIST=gloo CDG_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline \
  > gpurun_out/mr2.json 2> gpurun_out/mr2.err
echo "exit $?"; cat gpurun_out/mr2.json; tail -5 gpurun_out/mr2.err
