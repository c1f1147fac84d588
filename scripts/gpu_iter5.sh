set -x
timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_gpu_parity.py tests/test_gpu_decision_step.py -x -q 2>&1 | tail -5
bash scripts/gpu_ab.sh 2>&1 | grep -v "^+"
