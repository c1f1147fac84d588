# CTA-pair stream pass: hang guard on a small store first, then A/B (SAIR_WIDE_CG=1) and parity
N=1048576 NQ=256 TAG=cg2_1M timeout 120 python scripts/ab_time.py 2>&1 | tail -3
if [ $? -ne 0 ]; then echo "small run failed"; fi
for r in 1 2; do
  SAIR_WIDE_CG=1 N=16777216 NQ=512 TAG=cg1 timeout 200 python scripts/ab_time.py 2>&1 | tail -1
  N=16777216 NQ=512 TAG=cg2 timeout 200 python scripts/ab_time.py 2>&1 | tail -1
done
SAIR_WIDE_CG=1 TAG=cg1_4096 timeout 300 python scripts/ab_time.py 2>&1 | tail -1
TAG=cg2_4096 timeout 300 python scripts/ab_time.py 2>&1 | tail -1
SAIR_WIDE_TRACE=1 N=16777216 NQ=512 timeout 300 python scripts/ab_time.py > gpurun_out/trace512_cg2.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_wide.py tests/test_gpu_configs.py -x -q 2>&1 | tail -3
