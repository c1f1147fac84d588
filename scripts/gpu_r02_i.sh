timeout 2700 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/i_pytest.txt
timeout 1800 python bench.py > gpurun_out/i_bench.json 2> gpurun_out/i_bench.err
