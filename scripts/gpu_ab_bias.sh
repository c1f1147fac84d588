# A/B (same box): ab/libsair_A.so (previous build) vs the in-tree build; then the wide/config parity tests
for r in 1 2; do
  SAIR_LIB_PATH=ab/libsair_A.so N=16777216 NQ=256 TAG=A256 timeout 300 python scripts/ab_time.py 2>&1 | tail -1
  N=16777216 NQ=256 TAG=B256 timeout 300 python scripts/ab_time.py 2>&1 | tail -1
done
SAIR_LIB_PATH=ab/libsair_A.so TAG=A4096 timeout 300 python scripts/ab_time.py 2>&1 | tail -1
TAG=B4096 timeout 300 python scripts/ab_time.py 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_wide.py tests/test_gpu_configs.py -x -q 2>&1 | tail -3
N=16777216 NQ=256 timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_wide_kernel -s 3 -c 1 -o gpurun_out/r02_bias_stream python scripts/ab_time.py > gpurun_out/r02_ncu_bias.log 2>&1
