#!/bin/bash
# HEAD, final: full GPU suite, smoke, bench (own arm)
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/y_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/y_smoke.txt 2>&1
timeout 1800 python bench.py > gpurun_out/y_bench.json 2> gpurun_out/y_bench.err
cat gpurun_out/y_pytest.txt gpurun_out/y_smoke.txt; head -c 300 gpurun_out/y_bench.json
