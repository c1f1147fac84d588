"""The wide pass on a 16M store before and after appending one batch of
high-reward experiences (config 5's store after a decision step)."""
import sys, time, os
import numpy as np
sys.path.insert(0, ".")
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import synth
db = sair.ExperienceBuffer(0.0)
db.store_synthetic(2026, 1 << 24, 64)
cfg = sair.SelectionConfig(m=32, lambda_div=0.0)
nq = int(os.environ.get("NQ", 4096))
def run(tag):
    xq = synth.queries(11, nq, 64)
    t0 = time.perf_counter()
    db.select_batch(xq, cfg)
    st = db.last_stats()
    print(f"{tag}: {1e3*(time.perf_counter()-t0):.1f} ms, stream {st['stream_ms']/st['stream_launches']:.3f} ms/launch", st, flush=True)
run("before")
run("before")
rng = np.random.default_rng(1)
k = int(os.environ.get("NAPP", 12000))
db.store_many(synth.queries(5, k, 64), rng.uniform(-5, 5, k), np.full(k, 9, np.int32))
run("after")
run("after")
