import os, sys
sys.path.insert(0, ".")
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import synth
n, nq = int(sys.argv[1]), int(sys.argv[2])
db = sair.ExperienceBuffer(0.0)
db.store_synthetic(2026, n, 64)
xq = synth.queries(7, nq, 64)
cfg = sair.SelectionConfig(m=32, lambda_div=0.0)
for p in ["0", "1", "2", "3", "4", "0"]:
    os.environ["SAIR_PROBE_WIDE"] = p
    db.select_batch(xq, cfg)
    db.select_batch(xq, cfg)
    st = db.last_stats()
    print(f"probe {p}: stream {st['stream_ms']:.3f} ms prepass {st['prepass_ms']:.3f} total {st['total_ms']:.3f}", flush=True)
