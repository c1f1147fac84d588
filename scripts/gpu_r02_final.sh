# Round-2 measurement: GPU tests, bench (both arms), launch list, ncu captures
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/f_pytest.txt
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/f_bench_ref.json 2> gpurun_out/f_bench_ref.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-pareto > /dev/null 2>&1
N=16777216 NQ=4096 timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_wide16 -s 3 -c 1 -o gpurun_out/f_wide16 python scripts/ab_time.py > gpurun_out/f_ncu_wide16.log 2>&1
N=16777216 NQ=4096 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stream_wide_kernel" -s 4 -c 1 -o gpurun_out/f_sample python scripts/ab_time.py > gpurun_out/f_ncu_sample.log 2>&1
N=16777216 NQ=8 timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_mma_kernel -s 3 -c 1 -o gpurun_out/f_k3 python scripts/ab_time.py > gpurun_out/f_ncu_k3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"g32_step_kernel|g32_pick_kernel" -s 40 -c 2 -o gpurun_out/f_g32 python scripts/lam_time.py > gpurun_out/f_ncu_g32.log 2>&1
T=4194304 DISTS=uniform,anti KS=4 NS=262144 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"score_batch_kernel|score_window_kernel|dominance4_kernel|member_kernel|compact_kernel|batch_keys_kernel" -c 10 -o gpurun_out/f_pareto python scripts/pareto_time.py > gpurun_out/f_ncu_pareto.log 2>&1
ls -la gpurun_out | tail -30
