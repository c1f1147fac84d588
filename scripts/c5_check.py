import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import synth, decision
P = int(sys.argv[1]) if len(sys.argv) > 1 else 30000
db = sair.ExperienceBuffer(0.0)
db.store_synthetic(2026, 1 << 24, 64)
rng = np.random.default_rng(0)
fs = sair.FrontierSet(P, 2000.0, 10.0)
scfg = sair.SelectionConfig(m=32, lambda_div=0.0)
for s in range(3):
    ctx = synth.queries(100 + s, P, 64)
    inputs = np.stack([rng.uniform(100, 2500, P), rng.uniform(50, 2600, P),
                       rng.uniform(0.5, 10, P), rng.uniform(0.5, 11, P)], 1)
    t0 = time.perf_counter()
    decision.retrieve(db, ctx, scfg)
    t1 = time.perf_counter()
    print(f"step {s}: retrieve {t1 - t0:.3f} s", db.last_stats(), flush=True)
    rw, k = decision.score_and_store(db, fs, ctx, inputs, np.zeros((P, 3, 4), np.int32),
                                     np.ones(P, np.uint8), np.full(P, s, np.int32), sair.RewardConfig())
    print(f"  reward+store {time.perf_counter() - t1:.3f} s, stored {k}, reward range {rw[:,5].min():.2f}..{rw[:,5].max():.2f}", flush=True)
