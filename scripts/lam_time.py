"""configs[1] (1M x 64, 256-query batches, k = 32) at lambda 0.1: the
filtered greedy vs the fp64 greedy (SAIR_GREEDY64=1)."""
import os, sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import synth
n, nq = int(os.environ.get("N", 1 << 20)), int(os.environ.get("NQ", 256))
db = sair.ExperienceBuffer(0.0)
db.store_synthetic(2026, n, 64)
xq = synth.queries(7, nq * 3, 64).reshape(3, nq, 64)
cfg = sair.SelectionConfig(m=32, lambda_div=0.1)
db.select_batch(xq[0], cfg)
ts = []
for i in (1, 2):
    t0 = time.perf_counter(); db.select_batch(xq[i], cfg); ts.append(time.perf_counter() - t0)
st = db.last_stats()
print(f"{os.environ.get('TAG','')} n={n} nq={nq} lambda 0.1: {np.median(ts)*1e3:.1f} ms/call, "
      f"greedy32={st['greedy32']} candidates/(query*step)={st['greedy32_candidates']/max(1,nq*32):.2f}", flush=True)
