timeout 900 python -m pytest tests/test_gpu_small.py tests/test_gpu_decision_step.py tests/test_gpu_parity.py tests/test_gpu_greedy.py -x -q 2>&1 | tail -3
SAIR_SMALL_TRACE=1 timeout 300 python scripts/small_trace.py 2>&1 | tail -1
SAIR_SMALL_NOZS=1 SAIR_SMALL_TRACE=1 timeout 300 python scripts/small_trace.py 2>&1 | tail -1
STEPS=60 timeout 300 python scripts/dec_time.py 2>&1 | tail -1
