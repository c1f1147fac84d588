# Decompose one 256-query wide pass over 16M records: full / no epilogue math / no MMA either
for p in 0 1 2 0; do
  SAIR_PROBE_WIDE=$p N=16777216 NQ=256 TAG=probe$p timeout 300 python scripts/ab_time.py 2>&1 | tail -1
done
N=16777216 NQ=256 timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_wide_kernel -s 3 -c 2 -o gpurun_out/r02_wide_pair python scripts/ab_time.py > gpurun_out/r02_ncu_pair.log 2>&1
