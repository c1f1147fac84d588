"""configs[0]'s decision step latency (bench.bench_config1's fused path)."""
import os, sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import decision, synth
cfg = sair.SelectionConfig(m=8, lambda_div=0.1)
rc, act = sair.RewardConfig(), sair.ScalingAction.noop(3)
db = sair.ExperienceBuffer(0.0)
db.store_synthetic(2029, 10000, 32)
fr = sair.ParetoFrontier(2000.0, 10.0)
rng = np.random.default_rng(1)
lat = []
for s in range(int(os.environ.get("STEPS", 60))):
    x = synth.queries(2300 + s, 1, 32)
    inp = sair.RewardInputs(rng.uniform(300, 900), rng.uniform(300, 900), rng.uniform(1, 5), rng.uniform(1, 5))
    t0 = time.perf_counter()
    decision.replay_step(db, fr, x[0], cfg, inp, act, rc, update=True, round=10000 + s)
    lat.append(time.perf_counter() - t0)
print(f"median {np.median(lat[5:])*1e6:.1f} us, min {np.min(lat[5:])*1e6:.1f} us", flush=True)
