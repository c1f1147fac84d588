set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; free -g | head -2; lscpu | grep -i "model name"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1500 python -m pytest tests/ -x -q -m gpu --durations=15 2>&1 | tail -30
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench0.json 2> gpurun_out/r2_bench0.err; tail -c 2000 gpurun_out/r2_bench0.json
