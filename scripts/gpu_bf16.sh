# bf16 wide pass: correctness first (hang-guarded), then A/B against SAIR_WIDE_BF16=0
N=1048576 NQ=256 TAG=bf16_1M timeout 120 python scripts/ab_time.py 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_wide.py -x -q 2>&1 | tail -5
for r in 1 2; do
  SAIR_WIDE_BF16=0 N=16777216 NQ=512 TAG=tf32 timeout 200 python scripts/ab_time.py 2>&1 | tail -1
  N=16777216 NQ=512 TAG=bf16 timeout 200 python scripts/ab_time.py 2>&1 | tail -1
done
SAIR_WIDE_BF16=0 TAG=tf32_4096 timeout 300 python scripts/ab_time.py 2>&1 | tail -1
TAG=bf16_4096 timeout 300 python scripts/ab_time.py 2>&1 | tail -1
SAIR_WIDE_TRACE=1 N=16777216 NQ=512 timeout 300 python scripts/ab_time.py > gpurun_out/trace512_bf16.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_configs.py -x -q 2>&1 | tail -3
