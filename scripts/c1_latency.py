"""configs[0] decision-step latency: 10k records, d = 32, select m = 8 with
the fused veto scan, compute_reward + update against a small frontier,
store() of the new experience -- through the public API."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import synth
db = sair.ExperienceBuffer(0.0)
db.store_synthetic(1, 10000, 32)
f = sair.ParetoFrontier(2000.0, 10.0)
rng = np.random.default_rng(0)
cfg = sair.SelectionConfig(m=8, lambda_div=0.1)
rc = sair.RewardConfig()
act = sair.ScalingAction.noop(3)
ts = {"select": [], "reward": [], "update": [], "store": []}
for step in range(60):
    x = synth.queries(100 + step, 1, 32)
    t0 = time.perf_counter()
    db.select_batch(x, cfg, nearest=True)
    t1 = time.perf_counter()
    inp = sair.RewardInputs(rng.uniform(300, 900), rng.uniform(300, 900), rng.uniform(1, 5), rng.uniform(1, 5))
    r = sair.compute_reward(inp, act, f, rc)
    t2 = time.perf_counter()
    f.update(inp.l_after_ms, inp.c_after)
    t3 = time.perf_counter()
    db.store(sair.Experience(list(x[0]), act, r.total, 10000 + step))
    t4 = time.perf_counter()
    if step >= 10:
        for k, v in zip(ts, (t1 - t0, t2 - t1, t3 - t2, t4 - t3)):
            ts[k].append(v * 1e6)
print({k: round(float(np.median(v)), 1) for k, v in ts.items()}, "us (median)")
