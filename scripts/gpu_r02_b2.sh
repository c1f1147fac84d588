./scripts/mma_rate 2>&1 | tee gpurun_out/mma_rate.txt
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/r02b2_pytest.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02b2_bench.json 2> gpurun_out/r02b2_bench.err
N=16777216 NQ=4096 timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_wide16 -s 3 -c 1 -o gpurun_out/r02b2_wide16 python scripts/ab_time.py > gpurun_out/r02b2_ncu.log 2>&1
