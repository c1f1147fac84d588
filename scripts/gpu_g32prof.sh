timeout 900 ncu --set full --clock-control none --import-source on -k regex:"g32_step_kernel|g32_pick_kernel" -s 200 -c 2 -o gpurun_out/r02_g32 python scripts/lam_time.py > gpurun_out/r02_ncu_g32.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_g32_launches.csv python scripts/lam_time.py > /dev/null 2>&1
