set -x
timeout 600 python -m pytest tests/test_gpu_wide.py -x -q 2>&1 | tail -25
timeout 300 python scripts/wide_time.py 2>&1 | tail -12
SAIR_PROBE_WIDE=1 timeout 300 python scripts/wide_time.py 2>&1 | tail -12
