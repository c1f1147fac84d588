timeout 900 python -m pytest tests/test_gpu_decision_step.py tests/test_gpu_small.py -x -q 2>&1 | tail -2
for i in 1 2; do STEPS=60 timeout 300 python scripts/dec_time.py 2>&1 | tail -1; done
SAIR_TRACE_DECISION=1 STEPS=20 timeout 300 python scripts/dec_time.py 2>&1 | tail -3
ls tests/cpp/; ls oracle/_ref/ 2>/dev/null | head
