SAIR_NO_MMA=1 SAIR_NO_WIDE=1 timeout 600 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize_workload.py select 2>&1 | grep -A3 "Error\|Warning\|SUMMARY" | head -30
timeout 600 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize_workload.py select 2>&1 | grep -A2 "Error\|Warning\|SUMMARY" | grep -v "stream_wide" | head -30
timeout 1500 python -m pytest tests/test_gpu_sanitizer.py tests/test_gpu_parity.py tests/test_gpu_greedy.py -x -q 2>&1 | tail -3
