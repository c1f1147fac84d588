for r in 1 2; do
for pf in 0 4 8 16 32; do
  SAIR_WIDE_PF=$pf N=16777216 NQ=512 TAG=pf$pf timeout 300 python scripts/ab_time.py 2>&1 | tail -1
done
done
SAIR_WIDE_PF=16 SAIR_WIDE_TRACE=1 N=16777216 NQ=512 timeout 300 python scripts/ab_time.py > gpurun_out/trace512_pf16.txt 2>&1
SAIR_PROBE_WIDE=2 SAIR_WIDE_PF=16 N=16777216 NQ=512 TAG=probe2pf16 timeout 300 python scripts/ab_time.py 2>&1 | tail -1
SAIR_PROBE_WIDE=2 SAIR_WIDE_PF=0 N=16777216 NQ=512 TAG=probe2pf0 timeout 300 python scripts/ab_time.py 2>&1 | tail -1
