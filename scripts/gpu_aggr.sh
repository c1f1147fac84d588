N=1048576 NQ=256 TAG=sanity timeout 120 python scripts/ab_time.py 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_wide.py -x -q 2>&1 | tail -3
for r in 1 2; do
for b in 0 1; do
for g in 0 2.5; do
  SAIR_WIDE_BF16=$b SAIR_WIDE_AGGR=$g N=16777216 NQ=512 TAG=bf${b}_aggr$g timeout 200 python scripts/ab_time.py 2>&1 | tail -1
done; done; done
for b in 0 1; do SAIR_WIDE_BF16=$b TAG=bf${b}_4096 timeout 300 python scripts/ab_time.py 2>&1 | tail -1; done
SAIR_WIDE_TRACE=1 N=16777216 NQ=512 timeout 300 python scripts/ab_time.py > gpurun_out/trace512_aggr.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_configs.py -x -q 2>&1 | tail -3
