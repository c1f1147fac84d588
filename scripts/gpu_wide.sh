set -x
timeout 600 python -m pytest tests/test_gpu_wide.py -x -q 2>&1 | tail -25
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_wide.csv python scripts/wide_prof.py 1048576 256 > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/launches_wide.csv | head -20
timeout 300 python scripts/wide_time.py 2>&1 | tail -12
