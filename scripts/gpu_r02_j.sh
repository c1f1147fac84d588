STEPS=60 timeout 300 python scripts/dec_time.py 2>&1 | tail -1 > gpurun_out/j_dec.txt
SAIR_TRACE_DECISION=1 STEPS=20 timeout 300 python scripts/dec_time.py 2>&1 | tail -6 >> gpurun_out/j_dec.txt
SAIR_SMALL_TRACE=1 STEPS=8 timeout 300 python scripts/dec_time.py 2>&1 | tail -4 >> gpurun_out/j_dec.txt
STEPS=20 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/j_dec_launches.csv python scripts/dec_time.py > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/j_dec_launches.csv > gpurun_out/j_dec_table.txt 2>&1
N=1048576 NQ=256 timeout 300 python scripts/timeline.py > gpurun_out/j_tl_c1.txt 2>&1
N=16777216 NQ=4096 timeout 600 python scripts/timeline.py > gpurun_out/j_tl_c3.txt 2>&1
