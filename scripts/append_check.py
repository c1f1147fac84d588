"""A store with a freshly appended batch of high-reward records (config 5's
decision step): certification, the retry pass, and time."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
db = sair.ExperienceBuffer(0.0)
db.store_synthetic(2026, n, 64)
rng = np.random.default_rng(1)
P = 30000
db.store_many(synth.queries(5, P, 64), rng.uniform(0.01, 5.0, P), np.arange(P, dtype=np.int32))
xq = synth.queries(9, 4096, 64)
cfg = sair.SelectionConfig(m=32, lambda_div=0.0)
t0 = time.perf_counter()
db.select_batch(xq, cfg, nearest=True)
print(f"n={n}: {time.perf_counter() - t0:.3f} s", db.last_stats(), flush=True)
