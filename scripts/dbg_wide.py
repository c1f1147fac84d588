import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import synth
from oracle.oracle import COracle
orc = COracle()
n, d, nq, m = 70000, 64, 128, 32
db = sair.ExperienceBuffer(0.0)
db.store_synthetic(n + d, n, d)
ctx, rew, rnd = synth.contexts(n + d, 0, n, d), synth.rewards(n + d, 0, n), synth.rounds(0, n)
sigma = db.effective_sigma()
xq = synth.queries(n + d + 1, nq, d)
idx, sim, sc, cnt = db.select_batch(xq, sair.SelectionConfig(m=m, lambda_div=0.0))
print(db.last_stats())
oi, osim, osc, ocnt = orc.select_batch(ctx, rew, rnd, xq, m, 0.0, sigma)
bad = [q for q in range(nq) if not np.array_equal(idx[q], oi[q])]
print("bad queries", len(bad), bad[:10])
for q in bad[:3]:
    print(q, idx[q][:8], oi[q][:8])
    print(sc[q][:8], osc[q][:8])
