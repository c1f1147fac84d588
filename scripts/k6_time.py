"""K6 batch insert timing (configs[2], 4M 2-objective tuples): first call on a
fresh frontier (scratch allocation included) and warm calls (a frontier whose
buffers already hold a batch of that size), e2e from the host array, plus the
device time of the warm call (CUDA events on the frontier's stream are not
reachable from here: wall time around a synchronising call)."""
import os, sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import synth
T = int(os.environ.get("T", 4 * 1024 * 1024))
for dist in os.environ.get("DISTS", "uniform,anti,corr,grid").split(","):
    pts = synth.tuples(2026, T, 2, dist)
    warm = synth.tuples(3026, T, 2, dist)
    f = sair.ParetoFrontier(1.0, 1.0)
    t0 = time.perf_counter(); F = f.insert_batch(pts); cold = time.perf_counter() - t0
    ws = []
    for r in range(5):
        g = sair.ParetoFrontier(1.0, 1.0)
        g.insert_batch(warm)          # sizes the buffers
        g2 = g                        # then the timed batch into the same handle
        t0 = time.perf_counter(); g2.insert_batch(pts); ws.append(time.perf_counter() - t0)
    print(f"{dist}: F={F} first call {cold*1e3:.2f} ms, warm median {np.median(ws)*1e3:.2f} ms "
          f"({T/np.median(ws)/1e6:.0f} M tuples/s)", flush=True)
