#!/bin/bash
# HEAD, final (after the K7b 128-tuple j-tiles): suite, smoke, 4M box == pairwise, bench
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/z_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z_smoke.txt 2>&1
timeout 900 python scripts/dom_check.py > gpurun_out/z_dom.txt 2>&1
timeout 1800 python bench.py > gpurun_out/z_bench.json 2> gpurun_out/z_bench.err
cat gpurun_out/z_pytest.txt gpurun_out/z_smoke.txt; tail -5 gpurun_out/z_dom.txt; head -c 300 gpurun_out/z_bench.json
