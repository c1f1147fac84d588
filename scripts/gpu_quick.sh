# fail-fast quick check with short timeouts
set -e
timeout 60 python scripts/mma_check.py 300000 64 | tail -1
timeout 60 python scripts/mma_check.py 3000 23 | tail -1
timeout 60 python scripts/mma_check.py 2000000 16 | tail -1
