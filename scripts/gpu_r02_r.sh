#!/bin/bash
mkdir -p gpurun_out
STEPS=200 timeout 300 python scripts/dec_time.py > gpurun_out/r_dec.txt 2>&1
SAIR_TRACE_DECISION=1 STEPS=30 timeout 300 python scripts/dec_time.py > gpurun_out/r_dec_trace.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_decision_step.py tests/test_gpu_small.py tests/test_dropin.py -x -q -m gpu > gpurun_out/r_pytest.txt 2>&1
echo "pytest rc $?" >> gpurun_out/r_pytest.txt
tail -3 gpurun_out/r_pytest.txt; cat gpurun_out/r_dec.txt; tail -4 gpurun_out/r_dec_trace.txt
