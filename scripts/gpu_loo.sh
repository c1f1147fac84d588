timeout 900 python -m pytest tests -m gpu -q -k "local or loo or weighted" 2>&1 | tail -3
NS=10000,20000,40000 timeout 600 python scripts/loo_time.py 2>&1 | tail -3
SAIR_LOO_SIMPLE=1 NS=10000 timeout 600 python scripts/loo_time.py 2>&1 | tail -1
