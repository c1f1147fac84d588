#!/bin/bash
# K6 pre-filter: parity tests + timing (filtered vs SAIR_K6_NOFILTER)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/j_smi.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_golden.py -x -q -m gpu -k "frontier or insert or config2 or golden or pareto" > gpurun_out/j_pytest.txt 2>&1
echo "pytest rc $?" >> gpurun_out/j_pytest.txt
timeout 300 python scripts/k6_time.py > gpurun_out/j_k6.txt 2>&1
SAIR_K6_NOFILTER=1 timeout 300 python scripts/k6_time.py > gpurun_out/j_k6_nofilter.txt 2>&1
DISTS=uniform T=4194304 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/j_k6_launches.csv python scripts/k6_time.py > /dev/null 2>&1
tail -3 gpurun_out/j_pytest.txt; cat gpurun_out/j_k6.txt gpurun_out/j_k6_nofilter.txt
