./scripts/tmem_bw
for r in 1 2; do
  for c in 2 3 5; do SAIR_SAMPLE_C=$c TAG=c$c timeout 120 python scripts/ab_time.py 2>&1 | tail -1; done
done
