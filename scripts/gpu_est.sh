set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests/test_gpu_wide.py tests/test_gpu_wide_variants.py tests/test_gpu_configs.py -x -q 2>&1 | tail -4
for a in 2.5 0; do
 export SAIR_WIDE_AGGR=$a
 TAG=c5aggr$a timeout 600 python scripts/c5_time.py 2>&1 | tail -1
 TAG=16M$a timeout 600 python scripts/ab_time.py 2>&1 | tail -1
 N=2097152 TAG=2M$a timeout 600 python scripts/ab_time.py 2>&1 | tail -1
done
