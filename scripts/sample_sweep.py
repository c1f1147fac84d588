import os, sys, time
sys.path.insert(0, ".")
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import synth
for n in (1 << 24, 1 << 20):
    db = sair.ExperienceBuffer(0.0)
    db.store_synthetic(2026, n, 64)
    xq = synth.queries(7, 1024, 64)
    cfg = sair.SelectionConfig(m=32, lambda_div=0.0)
    for c in ("5", "2.5", "3.5", "7"):
        os.environ["SAIR_SAMPLE_C"] = c
        db.select_batch(xq, cfg)
        t0 = time.perf_counter()
        db.select_batch(xq, cfg)
        dt = time.perf_counter() - t0
        st = db.last_stats()
        print(f"n={n} c={c}: {dt*1e3:.2f} ms, stream {st['stream_ms']:.2f} prepass {st['prepass_ms']:.2f} total {st['total_ms']:.2f} cert {st['certified']}", flush=True)
