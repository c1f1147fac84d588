#!/bin/bash
# round-end state: full GPU suite, smoke, both bench arms, the bench's launch list
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/s_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s_smoke.txt 2>&1
timeout 1800 python bench.py > gpurun_out/s_bench.json 2> gpurun_out/s_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/s_bench_ref.json 2> gpurun_out/s_bench_ref.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/s_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/s_ncu.log 2>&1
cat gpurun_out/s_pytest.txt gpurun_out/s_smoke.txt; head -c 400 gpurun_out/s_bench.json; echo; head -c 200 gpurun_out/s_bench_ref.json
