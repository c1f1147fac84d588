# Round-2 baseline on one B200: GPU tests, bench (both arms), launch list, ncu captures
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/r02_pytest.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02_bench_ref.json 2>gpurun_out/r02_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
N=16777216 NQ=4096 timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_wide_kernel -s 4 -c 1 -o gpurun_out/r02_stream_wide python scripts/ab_time.py > gpurun_out/r02_ncu_wide.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"score_batch_kernel|dominance_kernel|compact_kernel|member_kernel" -c 6 -o gpurun_out/r02_pareto python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r02_ncu_pareto.log 2>&1
ls -la gpurun_out
