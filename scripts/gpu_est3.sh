export SAIR_WIDE_AGGR=0
SAIR_WIDE_DEBUG=1 N=8388608 NQ=4096 timeout 600 python scripts/ab_time.py 2>&1 | grep -v "^\[wide\] QW" | grep -v "same CTA 0, across CTAs 0" | head -20
TAG=16M0 timeout 600 python scripts/ab_time.py 2>&1 | tail -1
TAG=c5aggr0 timeout 600 python scripts/c5_time.py 2>&1 | tail -1
