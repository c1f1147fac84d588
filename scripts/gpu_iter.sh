# quick iteration: parity tests + bench + bounded ncu capture of the stream kernel
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -15
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -2
bash scripts/gpu_prof.sh
