import sys
sys.path.insert(0, ".")
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import synth
db = sair.ExperienceBuffer(0.0)
db.store_synthetic(2026, 1 << 20, 64)
xq = synth.queries(7, 128, 64)
db.select_batch(xq, sair.SelectionConfig(m=4, lambda_div=0.1))
print(db.last_stats())
