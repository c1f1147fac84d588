timeout 120 python scripts/sanitize_workload.py 2>&1 | tail -2
for tool in memcheck racecheck synccheck; do
  for part in select pareto decision; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python scripts/sanitize_workload.py $part > gpurun_out/san_${tool}_${part}.txt 2>&1
    echo "$tool $part rc=$? $(grep -c 'ERROR SUMMARY' gpurun_out/san_${tool}_${part}.txt) $(grep 'ERROR SUMMARY\|RACECHECK SUMMARY' gpurun_out/san_${tool}_${part}.txt | tail -1)"
  done
done
