N=1048576 timeout 900 ncu --set full --clock-control none --import-source on -k regex:g32_mma_step -s 5 -c 1 -o gpurun_out/g32mma_step python scripts/lam_time.py > gpurun_out/g32prof.log 2>&1
ls -la gpurun_out/*.ncu-rep
