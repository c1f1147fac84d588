# iteration: wide/parity tests, select timing, sample-size sweep, launch list
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_gpu_parity.py tests/test_gpu_decision_step.py -x -q 2>&1 | tail -5
timeout 300 python scripts/wide_time.py 2>&1 | tail -6
timeout 300 python scripts/sample_sweep.py 2>&1 | tail -8
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_iter.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-pareto > gpurun_out/ncu_iter.log 2>&1
python scripts/launch_table.py gpurun_out/launches_iter.csv > gpurun_out/lt.txt; head -6 gpurun_out/lt.txt
