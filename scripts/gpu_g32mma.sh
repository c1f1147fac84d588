timeout 900 python -m pytest tests/test_gpu_greedy32.py -x -q 2>&1 | tail -2
TAG=mma timeout 600 python scripts/lam_time.py 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g32mma_launches.csv python scripts/lam_time.py > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open("gpurun_out/g32mma_launches.csv")) if len(r)>10]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
v=[float(r[vi].replace(",",""))/1000 for r in rows[1:] if "mma_step" in r[ki]]
print("step kernel us per launch (first call):", [round(x) for x in v[:32]])
PY
python - <<'PY'
import csv
rows=[r for r in csv.reader(open("gpurun_out/g32mma_launches.csv")) if len(r)>10]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
v=[float(r[vi].replace(",",""))/1000 for r in rows[1:] if "pick" in r[ki]]
print("pick kernel us per launch (first call):", [round(x) for x in v[:32]])
PY
