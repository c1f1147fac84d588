#!/bin/bash
# full GPU suite, smoke, bench (own arm + reference arm), launch list of the bench's Pareto leg
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/n_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/n_smoke.txt 2>&1
timeout 1800 python bench.py > gpurun_out/n_bench.json 2> gpurun_out/n_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/n_bench_ref.json 2> gpurun_out/n_bench_ref.err
cat gpurun_out/n_pytest.txt gpurun_out/n_smoke.txt; head -c 600 gpurun_out/n_bench.json; echo; head -c 300 gpurun_out/n_bench_ref.json
