SAIR_WIDE_TRACE=1 N=16777216 NQ=256 timeout 300 python scripts/ab_time.py > gpurun_out/trace256.txt 2>&1
SAIR_WIDE_TRACE=1 N=16777216 NQ=512 timeout 300 python scripts/ab_time.py > gpurun_out/trace512.txt 2>&1
