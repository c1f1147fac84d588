for r in 1 2; do
  TAG=base timeout 120 python scripts/ab_time.py 2>&1 | tail -1
  SAIR_LIB_PATH=ab/libsair_us.so TAG=usplit timeout 120 python scripts/ab_time.py 2>&1 | tail -1
  SAIR_LIB_PATH=ab/libsair_sn.so TAG=suspend timeout 120 python scripts/ab_time.py 2>&1 | tail -1
  SAIR_LIB_PATH=ab/libsair_ussn.so TAG=us+sn timeout 120 python scripts/ab_time.py 2>&1 | tail -1
done
for L in ab/libsair_us.so ab/libsair_sn.so ab/libsair_ussn.so; do
  SAIR_LIB_PATH=$L SAIR_WIDE_QW=128 TAG=$L-qw128 timeout 120 python scripts/ab_time.py 2>&1 | tail -1
done
SAIR_WIDE_QW=128 TAG=base-qw128 timeout 120 python scripts/ab_time.py 2>&1 | tail -1
