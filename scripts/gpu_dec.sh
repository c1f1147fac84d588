STEPS=60 timeout 300 python scripts/dec_time.py 2>&1 | tail -1
SAIR_TRACE_DECISION=1 STEPS=20 timeout 300 python scripts/dec_time.py 2>&1 | tail -6
STEPS=20 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dec_launches.csv python scripts/dec_time.py > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/dec_launches.csv 2>&1 | head -30
