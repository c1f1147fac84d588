#!/bin/bash
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/o_pytest.txt
timeout 900 python scripts/harness_time.py > gpurun_out/o_harness.json 2> gpurun_out/o_harness.err
cat gpurun_out/o_pytest.txt; cat gpurun_out/o_harness.json
