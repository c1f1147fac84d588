timeout 1500 python -m pytest tests/test_gpu_greedy32.py -x -q 2>&1 | tail -2
TAG=g32 timeout 300 python scripts/lam_time.py 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_g32_launches.csv python scripts/lam_time.py > /dev/null 2>&1
