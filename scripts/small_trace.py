"""Phase trace of the small select kernel (SAIR_SMALL_TRACE) at configs[0]'s shape."""
import sys
sys.path.insert(0, ".")
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import synth
db = sair.ExperienceBuffer(0.0)
db.store_synthetic(2029, 10000, 32)
cfg = sair.SelectionConfig(m=8, lambda_div=0.1)
for s in range(4):
    db.select_batch(synth.queries(2300 + s, 1, 32), cfg, nearest=True)
