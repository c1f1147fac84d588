"""Quick A/B of the tensor-core stream kernel vs the CUDA-core one vs exact."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22397_b200 as sair  # noqa: E402
from paper_2601_22397_b200 import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 50000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 64
b = sair.ExperienceBuffer(0.0)
b.store_synthetic(11, n, d)
xq = synth.queries(11, 8, d)
for lam in (0.0,):
    cfg = sair.SelectionConfig(m=32, lambda_div=lam)
    t = time.time()
    fast = b.select_batch(xq, cfg, nearest=True)
    print("mma", b.last_stats(), time.time() - t, flush=True)
    os.environ["SAIR_NO_MMA"] = "1"
    core = b.select_batch(xq, cfg, nearest=True)
    print("core", b.last_stats(), flush=True)
    del os.environ["SAIR_NO_MMA"]
    ex = b.select_batch(xq, sair.SelectionConfig(m=32, lambda_div=lam, mode=sair.SELECT_EXACT),
                        nearest=True)
    print("idx equal mma/exact", np.array_equal(fast[0], ex[0]), "core/exact",
          np.array_equal(core[0], ex[0]), "nn", np.array_equal(fast[4], ex[4]))
