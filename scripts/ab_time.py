"""A/B timing of one select shape (SAIR_LIB_PATH picks the library build)."""
import os, sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import synth
n, nq = int(os.environ.get("N", 1 << 24)), int(os.environ.get("NQ", 4096))
db = sair.ExperienceBuffer(0.0)
db.store_synthetic(2026, n, 64)
xq = synth.queries(7, nq * 6, 64).reshape(6, nq, 64)
cfg = sair.SelectionConfig(m=32, lambda_div=0.0)
db.select_batch(xq[0], cfg)
ts, ss, rq, tt, pp = [], [], [], [], []
for i in range(1, 6):
    t0 = time.perf_counter()
    db.select_batch(xq[i], cfg)
    ts.append(time.perf_counter() - t0)
    st = db.last_stats()
    ss.append(st["stream_ms"] / st["stream_launches"])
    rq.append(st["retried"])
    tt.append(st["total_ms"])
    pp.append(st["prepass_ms"])
print(f"{os.environ.get('TAG', '')} n={n} nq={nq}: median {np.median(ts)*1e3:.2f} ms, stream {np.median(ss):.3f} ms/launch, retried {rq}, device total {np.median(tt):.2f} ms, prepass {np.median(pp):.2f} ms", flush=True)
