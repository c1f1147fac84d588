"""Quick timing of the select paths at the configs' shapes (public API, CUDA
events from last_stats); not the bench."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import synth

for n, nq in [(1 << 20, 256), (1 << 21, 512), (1 << 24, 128), (1 << 24, 8), (1 << 24, 4096)]:
    db = sair.ExperienceBuffer(0.0)
    db.store_synthetic(2026, n, 64)
    xq = synth.queries(7, nq * 4, 64).reshape(4, nq, 64)
    cfg = sair.SelectionConfig(m=32, lambda_div=0.0)
    db.select_batch(xq[0], cfg)
    for i in range(1, 4):
        t0 = time.perf_counter()
        db.select_batch(xq[i], cfg)
        dt = time.perf_counter() - t0
        st = db.last_stats()
    print(f"n={n} nq={nq}: wall {dt*1e3:.3f} ms -> {nq/dt:,.0f} q/s; {st}", flush=True)
