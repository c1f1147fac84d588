import sys
sys.path.insert(0, ".")
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import synth
n, d, m, lam = 10000, 32, 8, float(sys.argv[1]) if len(sys.argv) > 1 else 0.1
db = sair.ExperienceBuffer(0.0)
db.store_synthetic(5, n, d)
xq = synth.queries(6, 4, d)
cfg = sair.SelectionConfig(m=m, lambda_div=lam)
for i in range(4):
    db.select_batch(xq[i:i + 1], cfg, nearest=True)
print(db.last_stats())
