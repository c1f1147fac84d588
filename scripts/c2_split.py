"""configs[1] per-call split: host wall vs the device span of the call (ev0..ev3)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import synth
db = sair.ExperienceBuffer(0.0)
db.store_synthetic(2027, 1 << 20, 64)
cfg = sair.SelectionConfig(m=32, lambda_div=0.0)
qs = synth.queries(9, 256 * 40, 64).reshape(40, 256, 64)
for i in range(5):
    db.select_batch(qs[i], cfg)
w, dev, st = [], [], []
for i in range(5, 40):
    t0 = time.perf_counter()
    db.select_batch(qs[i], cfg)
    w.append(time.perf_counter() - t0)
    s = db.last_stats()
    dev.append(s["total_ms"]); st.append((s["stream_ms"], s["prepass_ms"]))
print(f"wall {np.median(w)*1e3:.3f} ms, device span {np.median(dev):.3f} ms, stream {np.median([a for a,b in st]):.3f}, prepass {np.median([b for a,b in st]):.3f}")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for i in range(5, 40):
    db.select_batch(qs[i], cfg)
pr.disable(); pstats.Stats(pr).sort_stats("tottime").print_stats(8)
