N=100000 NQ=16 TAG=sanity timeout 120 python scripts/lam_time.py 2>&1 | tail -3
timeout 1500 python -m pytest tests/test_gpu_greedy32.py -x -q 2>&1 | tail -4
TAG=g32 timeout 300 python scripts/lam_time.py 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_g32_launches.csv python scripts/lam_time.py > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"g32_step_kernel|g32_pick_kernel" -s 100 -c 2 -o gpurun_out/r02_g32 python scripts/lam_time.py > gpurun_out/r02_ncu_g32.log 2>&1
