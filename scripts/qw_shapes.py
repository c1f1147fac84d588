"""16M x 64 store, query batches that pick the 32- and 64-query wide kernels
(nst 5 shared stages < ntm 8 TMEM stages): completes, certified."""
import sys, time
sys.path.insert(0, ".")
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import synth
db = sair.ExperienceBuffer(0.0)
db.store_synthetic(2026, 1 << 24, 64)
for nq in (40, 100, 300):
    xq = synth.queries(11, nq, 64)
    t0 = time.perf_counter()
    db.select_batch(xq, sair.SelectionConfig(m=32, lambda_div=0.0))
    st = db.last_stats()
    print(nq, f"{(time.perf_counter() - t0) * 1e3:.2f} ms", {k: st[k] for k in ("qb", "certified", "exact_fallbacks", "retried", "stream_ms")}, flush=True)
