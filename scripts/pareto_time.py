"""configs[2] timing: K8 scoring (cold L2) on uniform / anti-correlated 4M-tuple
frontiers, K6 batch insert, K7 dominance counts for K = 3 / 4 (262k and 4M)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import synth
T = int(os.environ.get("T", 4 * 1024 * 1024))
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
for dist in os.environ.get("DISTS", "uniform,anti").split(","):
    pts = synth.tuples(2026 + (5 if dist != "uniform" else 0), T, 2, dist)
    f = sair.ParetoFrontier(1.0, 1.0)
    t0 = time.perf_counter(); F = f.insert_batch(pts); ins = time.perf_counter() - t0
    dp = torch.from_numpy(pts).cuda(); out = torch.empty(T, dtype=torch.float64, device="cuda")
    dom = torch.empty(T, dtype=torch.uint8, device="cuda")
    f.score_batch_device(dp.data_ptr(), T, out.data_ptr(), dom.data_ptr(), s.cuda_stream)
    ts = []
    for _ in range(5):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); f.score_batch_device(dp.data_ptr(), T, out.data_ptr(), dom.data_ptr(), s.cuda_stream); e1.record(s)
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(f"{dist}: F={F} insert {ins*1e3:.1f} ms e2e, score {np.median(ts):.4f} ms "
          f"({T*25/np.median(ts)/1e6:.0f} GB/s)", flush=True)
for K in [int(k) for k in os.environ.get("KS", "3,4").split(",")]:
    for n in [int(x) for x in os.environ.get("NS", "262144").split(",")]:
        tp = synth.tuples(2028, n, K, "uniform")
        sair.dominance_counts(tp[:4096])
        t0 = time.perf_counter(); c, m = sair.dominance_counts(tp); dt = time.perf_counter() - t0
        print(f"K={K} T={n}: counts {dt*1e3:.1f} ms e2e, frontier {int(m.sum())}, "
              f"mean count {c.mean():.1f}", flush=True)
