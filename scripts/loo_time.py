"""locally_weighted_mean select: the exact local-LOO pass at a few store sizes."""
import os, sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import synth
for n in [int(x) for x in os.environ.get("NS", "10000,20000,40000").split(",")]:
    db = sair.ExperienceBuffer(0.0)
    db.store_synthetic(5, n, 32)
    cfg = sair.SelectionConfig(m=8, lambda_div=0.1, locally_weighted_mean=True)
    q = synth.queries(6, 4, 32)
    db.select_batch(q[:1], cfg)
    t0 = time.perf_counter(); db.select_batch(q[1:2], cfg); t1 = time.perf_counter()
    print(f"n={n}: {1e3*(t1-t0):.2f} ms per select (1 query)", flush=True)
