"""configs[0] per-decision split: select wall vs device span, and each call of the step."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import synth
db = sair.ExperienceBuffer(0.0)
db.store_synthetic(2029, 10000, 32)
fr = sair.ParetoFrontier(2000.0, 10.0)
cfg = sair.SelectionConfig(m=8, lambda_div=0.1)
rc = sair.RewardConfig()
act = sair.ScalingAction.noop(3)
rng = np.random.default_rng(0)
T = {"select": [], "dev": [], "reward": [], "update": [], "store": []}
for s in range(60):
    x = synth.queries(300 + s, 1, 32)
    inp = sair.RewardInputs(rng.uniform(300, 900), rng.uniform(300, 900), rng.uniform(1, 5), rng.uniform(1, 5))
    t0 = time.perf_counter(); db.select_batch(x, cfg, nearest=True); t1 = time.perf_counter()
    r = sair.compute_reward(inp, act, fr, rc); t2 = time.perf_counter()
    fr.update(inp.l_after_ms, inp.c_after); t3 = time.perf_counter()
    db.store(sair.Experience(list(x[0]), act, r.total, 10000 + s)); t4 = time.perf_counter()
    if s >= 10:
        T["select"].append(t1 - t0); T["reward"].append(t2 - t1); T["update"].append(t3 - t2)
        T["store"].append(t4 - t3); T["dev"].append(db.last_stats()["total_ms"] / 1e3)
print({k: round(float(np.median(v)) * 1e6, 1) for k, v in T.items()})
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for s in range(50):
    x = synth.queries(400 + s, 1, 32)
    db.select_batch(x, cfg, nearest=True)
pr.disable(); pstats.Stats(pr).sort_stats("tottime").print_stats(6)
