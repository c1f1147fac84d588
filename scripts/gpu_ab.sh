# A/B: ab/libsair_A.so vs the in-tree build, alternating, same box
set -x
for r in 1 2; do
  SAIR_LIB_PATH=ab/libsair_A.so TAG=A timeout 120 python scripts/ab_time.py 2>&1 | tail -1
  TAG=B timeout 120 python scripts/ab_time.py 2>&1 | tail -1
done
for r in 1 2; do
  NQ=128 SAIR_LIB_PATH=ab/libsair_A.so TAG=A timeout 120 python scripts/ab_time.py 2>&1 | tail -1
  NQ=128 TAG=B timeout 120 python scripts/ab_time.py 2>&1 | tail -1
done
