# profile the small per-step kernels (pre-pass, merge, refine) with source counters
set -x
timeout 300 ncu --section SpeedOfLight --section WarpStateStats --section SourceCounters --section LaunchStats --metrics gpu__time_duration.sum --clock-control none --import-source on -k regex:"refine|merge_kernel|sample_" -s 6 -c 4 -o gpurun_out/prof_small python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-pareto > gpurun_out/ncu_small.log 2>&1
tail -2 gpurun_out/ncu_small.log
