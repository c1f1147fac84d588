#!/bin/bash
# K7b box-pruned dominance counts: parity + timing vs the pairwise kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_multigpu_capi.py -x -q -m gpu -k "dominance or objective or count" > gpurun_out/m_pytest.txt 2>&1
echo "pytest rc $?" >> gpurun_out/m_pytest.txt
timeout 900 python scripts/dom_check.py > gpurun_out/m_dom.txt 2>&1
T=262144 timeout 300 ncu --set full --clock-control none -k regex:dominance_box --launch-skip 1 -c 1 -o gpurun_out/m_box python scripts/dom_check.py > /dev/null 2>&1 || true
CHECK=0 T=4194304 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m_launches.csv python -c "
import sys; sys.path.insert(0,'.')
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import synth
t = synth.tuples(2031, 4194304, 3, 'uniform'); sair.dominance_counts(t)" > /dev/null 2>&1 || true
tail -3 gpurun_out/m_pytest.txt; cat gpurun_out/m_dom.txt
