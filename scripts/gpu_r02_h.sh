timeout 2700 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/h_pytest.txt
timeout 1800 python bench.py > gpurun_out/h_bench.json 2> gpurun_out/h_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/h_bench_ref.json 2> gpurun_out/h_bench_ref.err
