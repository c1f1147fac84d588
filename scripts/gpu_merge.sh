timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_gpu_wide_variants.py -x -q 2>&1 | tail -2
for c in 5 3 2; do SAIR_SAMPLE_C=$c TAG=c$c timeout 300 python scripts/ab_time.py 2>&1 | tail -1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m_launches.csv python scripts/ab_time.py > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_configs.py -x -q -k "config3 or config1 or configs1" 2>&1 | tail -2
