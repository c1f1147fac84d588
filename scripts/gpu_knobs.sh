for r in 1 2; do
for n in 4 8; do SAIR_WIDE_NST16=$n N=16777216 NQ=1024 TAG=nst$n timeout 200 python scripts/ab_time.py 2>&1 | tail -1; done
for g in 1.5 2.5 4; do SAIR_WIDE_AGGR=$g N=16777216 NQ=1024 TAG=aggr$g timeout 200 python scripts/ab_time.py 2>&1 | tail -1; done
for b in 0 1; do SAIR_WIDE_BF16=$b N=1048576 NQ=256 TAG=c1_bf$b timeout 200 python scripts/ab_time.py 2>&1 | tail -1; done
for b in 0 1; do SAIR_WIDE_BF16=$b N=4194304 NQ=256 TAG=c4M_bf$b timeout 200 python scripts/ab_time.py 2>&1 | tail -1; done
done
