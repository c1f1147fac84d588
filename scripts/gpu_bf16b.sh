for c in 5 20 80; do
  SAIR_SAMPLE_C=$c N=16777216 NQ=512 TAG=bf16_c$c timeout 200 python scripts/ab_time.py 2>&1 | tail -1
  SAIR_WIDE_BF16=0 SAIR_SAMPLE_C=$c N=16777216 NQ=512 TAG=tf32_c$c timeout 200 python scripts/ab_time.py 2>&1 | tail -1
done
SAIR_PROBE_WIDE=1 N=16777216 NQ=512 TAG=bf16_probe1 timeout 300 python scripts/ab_time.py 2>&1 | tail -1
SAIR_PROBE_WIDE=2 N=16777216 NQ=512 TAG=bf16_probe2 timeout 300 python scripts/ab_time.py 2>&1 | tail -1
