#!/bin/bash
# where configs[0]'s decision step and configs[1]'s 256-query call spend their time
mkdir -p gpurun_out
SAIR_TRACE_DECISION=1 STEPS=40 timeout 300 python scripts/dec_time.py > gpurun_out/k_dec.txt 2>&1
N=1048576 NQ=256 timeout 300 python scripts/timeline.py > gpurun_out/k_tl_c1.txt 2>&1
cp gpurun_out/timeline.json gpurun_out/k_tl_c1.json 2>/dev/null
N=1048576 NQ=256 timeout 300 python scripts/ab_time.py > gpurun_out/k_ab_c1.txt 2>&1
tail -5 gpurun_out/k_dec.txt; cat gpurun_out/k_tl_c1.txt | head -40; tail gpurun_out/k_ab_c1.txt
