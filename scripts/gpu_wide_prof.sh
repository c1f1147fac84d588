set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stream_wide -s 2 -c 2 -o gpurun_out/prof_wide4 python scripts/wide_prof.py 16777216 128 > gpurun_out/ncu_wide.log 2>&1
tail -3 gpurun_out/ncu_wide.log
