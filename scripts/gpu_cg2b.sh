N=1048576 NQ=256 TAG=cg2_1M timeout 120 python scripts/ab_time.py 2>&1 | tail -1
for r in 1 2; do
  SAIR_WIDE_CG=1 N=16777216 NQ=512 TAG=cg1 timeout 200 python scripts/ab_time.py 2>&1 | tail -1
  N=16777216 NQ=512 TAG=cg2 timeout 200 python scripts/ab_time.py 2>&1 | tail -1
  SAIR_WIDE_NST2=4 N=16777216 NQ=512 TAG=cg2nst4 timeout 200 python scripts/ab_time.py 2>&1 | tail -1
done
SAIR_WIDE_TRACE=1 N=16777216 NQ=512 timeout 300 python scripts/ab_time.py > gpurun_out/trace512_cg2b.txt 2>&1
SAIR_PROBE_WIDE=1 N=16777216 NQ=512 TAG=cg2probe1 timeout 300 python scripts/ab_time.py 2>&1 | tail -1
