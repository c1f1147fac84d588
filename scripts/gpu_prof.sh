# profile the stream kernel with a bounded section set (full-set replay is slow)
set -x
timeout 300 ncu --section SpeedOfLight --section WarpStateStats --section SourceCounters --section MemoryWorkloadAnalysis --section LaunchStats --section Occupancy --section ComputeWorkloadAnalysis --metrics dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --import-source on -k regex:stream_ -s 4 -c 1 -o gpurun_out/prof_stream python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-pareto > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
