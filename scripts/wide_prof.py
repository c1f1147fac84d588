import sys
sys.path.insert(0, ".")
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import synth
n, nq = int(sys.argv[1]), int(sys.argv[2])
db = sair.ExperienceBuffer(0.0)
db.store_synthetic(2026, n, 64)
xq = synth.queries(7, nq, 64)
cfg = sair.SelectionConfig(m=32, lambda_div=0.0)
for _ in range(2):
    db.select_batch(xq, cfg)
    print(db.last_stats(), flush=True)
