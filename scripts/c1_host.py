"""configs[0] decision step: wall per replay_step vs the device span, and the
Python-side share (the same call with the device work skipped is not
possible, so: time the marshalling alone)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import decision, synth
db = sair.ExperienceBuffer(0.0)
db.store_synthetic(2031, 10000, 32)
fr = sair.ParetoFrontier(2000.0, 10.0)
cfg = sair.SelectionConfig(m=8, lambda_div=0.1)
rc = sair.RewardConfig()
act = sair.ScalingAction.noop(3)
rng = np.random.default_rng(0)
w, dev = [], []
for s in range(120):
    x = synth.queries(500 + s, 1, 32)[0]
    inp = sair.RewardInputs(rng.uniform(300, 900), rng.uniform(300, 900), rng.uniform(1, 5), rng.uniform(1, 5))
    t0 = time.perf_counter()
    decision.replay_step(db, fr, x, cfg, inp, act, rc, update=True, round=20000 + s)
    w.append(time.perf_counter() - t0)
    dev.append(db.last_stats()["total_ms"] * 1e3)
print(f"replay_step wall median {np.median(w[20:])*1e6:.1f} us, select device span {np.median(dev[20:]):.1f} us")
t0 = time.perf_counter()
for s in range(1000):
    c = cfg._c(); r = rc._c(); d = act.deltas()
    idx = np.full(8, -1, np.int64); sim = np.zeros(8); sc = np.zeros(8)
print(f"marshalling ~{(time.perf_counter()-t0)*1e3:.1f} us per call")
