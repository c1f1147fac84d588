# bench.py's N > 1 paths on one GPU: two ranks sharing it over gloo (the
# driver's 8-GPU run uses NCCL, one GPU per rank)
for mode in queries records; do
SAIR_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 3 --warmup 3 \
  --records 2097152 --queries 512 --shard $mode --no-pareto --no-cpu-baseline \
  > gpurun_out/mr_$mode.json 2> gpurun_out/mr_$mode.err
echo "$mode rc=$?"; tail -c 600 gpurun_out/mr_$mode.json; tail -2 gpurun_out/mr_$mode.err
done
