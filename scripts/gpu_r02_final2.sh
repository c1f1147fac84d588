set -x
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/g_pytest.txt
timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err
for n in 2097152 4194304 8388608 16777216; do for b in 0 1; do SAIR_WIDE_BF16=$b N=$n TAG=bf$b timeout 300 python scripts/ab_time.py 2>&1 | tail -1; done; done > gpurun_out/g_shards.txt
