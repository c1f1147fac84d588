timeout 1200 python -m pytest tests/test_gpu_wide_variants.py -x -q 2>&1 | tail -3
for a in 2.5 1.5 0; do
 export SAIR_WIDE_AGGR=$a
 TAG=c5aggr$a timeout 600 python scripts/c5_time.py 2>&1 | tail -2
done
