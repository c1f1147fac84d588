timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -k "pareto or frontier or dominance or score or config2 or configs2" 2>&1 | tail -3
DISTS=uniform,anti,corr,grid KS=3 NS=262144 timeout 600 python scripts/pareto_time.py 2>&1 | tail -8
T=4194304 DISTS=uniform,anti KS=4 NS=1024 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"score_batch_kernel" -c 2 -o gpurun_out/r02_score2 python scripts/pareto_time.py > gpurun_out/r02_ncu_score2.log 2>&1
