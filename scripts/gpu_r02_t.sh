#!/bin/bash
# bf16 page copy below 8M records? same-box A/B of SAIR_WIDE_BF16 at 1M / 2M / 4M
for N in 1048576 2097152 4194304; do
  for NQ in 256 4096; do
    for B in 0 1; do
      TAG="bf16=$B" SAIR_WIDE_BF16=$B N=$N NQ=$NQ timeout 300 python scripts/ab_time.py 2>&1 | tail -1
    done
  done
done
