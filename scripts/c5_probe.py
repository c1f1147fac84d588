"""Where config 5's retrieve time goes: nearest on/off, before/after appends."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import synth, decision
P = 30000
db = sair.ExperienceBuffer(0.0)
db.store_synthetic(2026, 1 << 24, 64)
rng = np.random.default_rng(0)
fs = sair.FrontierSet(P, 2000.0, 10.0)
scfg = sair.SelectionConfig(m=32, lambda_div=0.0)
def run(tag, ctx, nearest):
    t0 = time.perf_counter()
    db.select_batch(ctx, scfg, nearest=nearest)
    print(f"{tag} nearest={nearest}: {time.perf_counter() - t0:.3f} s", db.last_stats(), flush=True)
for s in range(3):
    ctx = synth.queries(100 + s, P, 64)
    run(f"step{s}", ctx, False)
    run(f"step{s}", ctx, True)
    inputs = np.stack([rng.uniform(100, 2500, P), rng.uniform(50, 2600, P),
                       rng.uniform(0.5, 10, P), rng.uniform(0.5, 11, P)], 1)
    rw, k = decision.score_and_store(db, fs, ctx, inputs, rng.integers(-2, 3, size=(P, 3, 4)).astype(np.int32),
                                     np.ones(P, np.uint8), np.full(P, s, np.int32), sair.RewardConfig())
    print(f"  stored {k}, reward range {rw[:,5].min():.2f}..{rw[:,5].max():.2f}", flush=True)
