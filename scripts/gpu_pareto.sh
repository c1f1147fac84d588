timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -k "pareto or frontier or dominance or score or config2 or configs2" 2>&1 | tail -3
NS=262144,1048576 timeout 600 python scripts/pareto_time.py 2>&1 | tail -8
KS=3,4 NS=4194304 DISTS=uniform timeout 900 python scripts/pareto_time.py 2>&1 | tail -3
T=4194304 KS=4 NS=262144 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"score_batch_kernel|dominance4_kernel|member_kernel|compact_kernel|batch_keys_kernel" -c 12 -o gpurun_out/r02_pareto_k678 python scripts/pareto_time.py > gpurun_out/r02_ncu_pareto2.log 2>&1
