# parity + bench (MMA and CUDA-core) + bounded ncu capture; fail fast
set -e
timeout 600 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -4
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1
SAIR_NO_MMA=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-pareto 2>&1 | tail -1
timeout 300 bash scripts/gpu_prof.sh
