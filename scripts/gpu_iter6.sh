set -x
timeout 1500 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -3
bash scripts/gpu_ab.sh 2>&1 | grep -v "^+"
