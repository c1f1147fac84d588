import os, sys
sys.path.insert(0, ".")
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import synth
db = sair.ExperienceBuffer(0.0)
db.store_synthetic(2026, 1 << 24, 64)
xq = synth.queries(7, 128, 64)
cfg = sair.SelectionConfig(m=4, lambda_div=0.0)
for p in ["0", "2", "0", "2"]:
    os.environ["SAIR_PROBE_WIDE"] = p
    db.select_batch(xq, cfg)
    st = db.last_stats()
    print(f"probe {p}: stream {st['stream_ms']:.3f} ms prepass {st['prepass_ms']:.3f}", flush=True)
