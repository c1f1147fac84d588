"""configs[4]'s retrieval on one GPU (16M store, 30000 queries, veto scan):
stats per call with and without the veto lists, and after a bulk append of
30000 outcomes (the decision step's pattern), to see what the 190 ms holds."""
import os, sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import synth
n, P = 1 << 24, int(os.environ.get("P", 30000))
db = sair.ExperienceBuffer(0.0)
db.store_synthetic(2026, n, 64)
cfg = sair.SelectionConfig(m=32, lambda_div=0.0)
rng = np.random.default_rng(1)
for it in range(4):
    xq = synth.queries(100 + it, P, 64)
    for nn in (False, True):
        t0 = time.perf_counter(); db.select_batch(xq, cfg, nearest=nn); dt = time.perf_counter() - t0
        st = db.last_stats()
        keys = ("stream_launches", "stream_ms", "prepass_ms", "total_ms", "retried", "certified",
                "exact_fallbacks")
        print(f"it {it} nearest={nn}: {dt*1e3:.1f} ms wall; " +
              ", ".join(f"{k}={st.get(k)}" for k in keys), flush=True)
    if it >= 1:  # the decision step's bulk append of this step's outcomes
        db.store_many(xq, rng.normal(size=P), np.full(P, 1000 + it, np.int32))
