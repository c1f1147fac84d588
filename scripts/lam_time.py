"""lambda > 0 behaviour: certification rate and time per call."""
import sys, time
sys.path.insert(0, ".")
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import synth
for n, d, nq, m, lam in [(10000, 32, 1, 8, 0.1), (10000, 32, 1, 8, 0.0), (100000, 64, 8, 32, 0.1),
                         (1 << 20, 64, 8, 32, 0.1), (1 << 20, 64, 128, 32, 0.1), (1 << 20, 64, 8, 32, 0.01)]:
    db = sair.ExperienceBuffer(0.0)
    db.store_synthetic(5, n, d)
    xq = synth.queries(6, nq * 3, d).reshape(3, nq, d)
    cfg = sair.SelectionConfig(m=m, lambda_div=lam)
    db.select_batch(xq[0], cfg)
    t0 = time.perf_counter()
    db.select_batch(xq[1], cfg)
    dt = time.perf_counter() - t0
    print(f"n={n} d={d} nq={nq} m={m} lam={lam}: {dt*1e3:.2f} ms/call; {db.last_stats()}", flush=True)
