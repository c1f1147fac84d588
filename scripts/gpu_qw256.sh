timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_gpu_configs.py -x -q -k "wide or config3 or config1" 2>&1 | tail -3
for r in 1 2; do
  TAG=qw256 timeout 120 python scripts/ab_time.py 2>&1 | tail -1
  SAIR_WIDE_QW=128 TAG=qw128 timeout 120 python scripts/ab_time.py 2>&1 | tail -1
done
N=1048576 NQ=256 TAG=c1_qw256 timeout 120 python scripts/ab_time.py 2>&1 | tail -1
N=16777216 NQ=256 timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_wide_kernel -s 3 -c 1 -o gpurun_out/qw256u_stream python scripts/ab_time.py > gpurun_out/ncu_qw256u.log 2>&1
