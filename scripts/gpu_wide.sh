set -x
timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_gpu_parity.py -x -q 2>&1 | tail -25
timeout 300 python scripts/wide_time.py 2>&1 | tail -12
