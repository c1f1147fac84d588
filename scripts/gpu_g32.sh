N=100000 NQ=16 TAG=sanity timeout 120 python scripts/lam_time.py 2>&1 | tail -3
timeout 1500 python -m pytest tests/test_gpu_greedy32.py -x -q 2>&1 | tail -8
TAG=g32 timeout 300 python scripts/lam_time.py 2>&1 | tail -1
SAIR_GREEDY64=1 TAG=g64 timeout 600 python scripts/lam_time.py 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_greedy.py tests/test_gpu_configs.py -x -q -k "greedy or lambda or config1 or configs1" 2>&1 | tail -3
