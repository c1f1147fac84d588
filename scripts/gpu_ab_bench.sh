# A/B of the bench's headline value: ab/libsair_A.so vs the in-tree build, alternating
for r in 1 2; do
  SAIR_LIB_PATH=ab/libsair_A.so timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-pareto 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('A', d['value'], d['e2e']['value'], d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
  timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-pareto 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('B', d['value'], d['e2e']['value'], d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
done
