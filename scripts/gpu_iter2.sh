# quick parity + short bench + warm per-kernel launch times + refine/merge source profile
set -e
bash scripts/gpu_quick.sh
timeout 180 python bench.py --no-cpu-baseline --no-pareto --steps 10 --warmup 3 > gpurun_out/bq.log 2>&1
tail -c 700 gpurun_out/bq.log
set +e
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"refine|merge_|sample_|stream_mma" -c 40 --csv --log-file gpurun_out/launches_warm.csv python bench.py --no-cpu-baseline --no-pareto --steps 3 --warmup 3 > gpurun_out/bl.log 2>&1
timeout 300 ncu --section WarpStateStats --section SourceCounters --metrics gpu__time_duration.sum --clock-control none --cache-control none --import-source on -k regex:"refine|merge_" -s 6 -c 2 -o gpurun_out/prof_small python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-pareto > gpurun_out/ncu_small.log 2>&1
tail -1 gpurun_out/ncu_small.log
