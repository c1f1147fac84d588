set -x
export SAIR_WIDE_AGGR=0
SAIR_LIB_PATH=$PWD/gpurun_in_head.so TAG=head16M timeout 600 python scripts/ab_time.py 2>&1 | tail -1
N=8388608 TAG=new8M timeout 600 python scripts/ab_time.py 2>&1 | tail -1
CUDA_LAUNCH_BLOCKING=1 TAG=new16Mblk timeout 600 python scripts/ab_time.py 2>&1 | tail -3
NQ=256 timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python scripts/ab_time.py 2>&1 | grep -v "^=========     " | head -40
