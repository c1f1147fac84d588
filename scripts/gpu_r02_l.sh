#!/bin/bash
# host-side phase trace of configs[1]'s call, K6 with the staged H2D, parity
mkdir -p gpurun_out
N=1048576 NQ=256 timeout 300 python scripts/ab_time.py > gpurun_out/l_ab_c1.txt 2>&1
N=1048576 NQ=256 SAIR_TRACE_SELECT=1 timeout 300 python scripts/ab_time.py > gpurun_out/l_trace_c1.txt 2>&1
N=16777216 NQ=4096 SAIR_TRACE_SELECT=1 timeout 300 python scripts/ab_time.py > gpurun_out/l_trace_c3.txt 2>&1
timeout 300 python scripts/k6_time.py > gpurun_out/l_k6.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_wide.py tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -m gpu > gpurun_out/l_pytest.txt 2>&1
echo "pytest rc $?" >> gpurun_out/l_pytest.txt
tail -3 gpurun_out/l_pytest.txt; tail -3 gpurun_out/l_ab_c1.txt; tail -4 gpurun_out/l_trace_c1.txt; tail -3 gpurun_out/l_trace_c3.txt; cat gpurun_out/l_k6.txt
