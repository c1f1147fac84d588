"""bench.py --gpus N starts its own N ranks when no torchrun environment is
set (the driver's plain `python bench.py --gpus N`): the launcher re-execs
through torch.distributed.run on 127.0.0.1, every rank rendezvous, and rank 0
alone prints the JSON line with n_gpus == N.  Run with gloo on CPU through the
launcher self-check (no kernels)."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("n", [1, 2])
def test_bench_launches_n_ranks(n):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", str(n),
                          "--launcher-check"], capture_output=True, text=True, timeout=300,
                         env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    j = json.loads(lines[0])
    assert j["n_gpus"] == n and j["max_over_ranks"] == float(n)
    assert j["shard"] == "records"
