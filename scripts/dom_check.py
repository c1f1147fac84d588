"""K7b (Morton tiles, box-pruned) against the rank-sum pairwise kernel
(SAIR_DOM_PAIRWISE=1, run in a child process) on 4M tuples: counts and
membership equal, both timed."""
import os, subprocess, sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import synth
T = int(os.environ.get("T", 4 * 1024 * 1024))
mode = os.environ.get("MODE", "parent")
for K, dist in [(3, "uniform"), (4, "uniform"), (3, "anti"), (4, "corr"), (3, "grid")]:
    t = synth.tuples(2028 + K, T, K, dist)
    sair.dominance_counts(t[:4096])
    t0 = time.perf_counter(); c, m = sair.dominance_counts(t); dt = time.perf_counter() - t0
    tag = f"K{K}_{dist}"
    if mode == "child":
        np.save(f"/tmp/dom_{tag}_c.npy", c); np.save(f"/tmp/dom_{tag}_m.npy", m)
        print(f"pairwise {tag}: {dt*1e3:.1f} ms", flush=True)
    else:
        t0 = time.perf_counter(); sair.dominance_counts(t, counts=False); dm = time.perf_counter() - t0
        print(f"box {tag}: membership only {dm*1e3:.1f} ms", flush=True)
        print(f"box {tag}: {dt*1e3:.1f} ms, frontier {int(m.sum())}, mean count {c.mean():.1f}", flush=True)
        np.save(f"/tmp/dombox_{tag}_c.npy", c); np.save(f"/tmp/dombox_{tag}_m.npy", m)
if mode == "parent" and os.environ.get("CHECK", "1") == "1":
    env = dict(os.environ, MODE="child", SAIR_DOM_PAIRWISE="1")
    subprocess.run([sys.executable, __file__], env=env, check=True)
    for K, dist in [(3, "uniform"), (4, "uniform"), (3, "anti"), (4, "corr"), (3, "grid")]:
        tag = f"K{K}_{dist}"
        ok = (np.array_equal(np.load(f"/tmp/dom_{tag}_c.npy"), np.load(f"/tmp/dombox_{tag}_c.npy")) and
              np.array_equal(np.load(f"/tmp/dom_{tag}_m.npy"), np.load(f"/tmp/dombox_{tag}_m.npy")))
        print(f"{tag}: box == pairwise: {ok}", flush=True)
