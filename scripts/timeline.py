"""Device timeline of one N x NQ select_batch (env N, NQ, LAM; default 16M x 4096) (torch.profiler / CUPTI sees
the library's kernels and copies): per-op totals and the idle gaps between ops."""
import json, os, sys
sys.path.insert(0, ".")
import torch
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import synth
from torch.profiler import profile, ProfilerActivity

n, nq = int(os.environ.get("N", 1 << 24)), int(os.environ.get("NQ", 4096))
db = sair.ExperienceBuffer(0.0)
db.store_synthetic(2026, n, 64)
xq = synth.queries(7, nq * 3, 64).reshape(3, nq, 64)
cfg = sair.SelectionConfig(m=32, lambda_div=float(os.environ.get("LAM", 0.0)))
db.select_batch(xq[0], cfg)
db.select_batch(xq[1], cfg)
import time
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    t_0 = time.perf_counter()
    db.select_batch(xq[2], cfg)
    torch.cuda.synchronize()
    print(f"host wall {(time.perf_counter() - t_0) * 1e3:.3f} ms (under the profiler)")
prof.export_chrome_trace("gpurun_out/timeline.json")
ev = [e for e in json.load(open("gpurun_out/timeline.json"))["traceEvents"]
      if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
t0, t1 = ev[0]["ts"], max(e["ts"] + e["dur"] for e in ev)
tot = {}
for e in ev:
    k = e["cat"] + ":" + e["name"][:60]
    c, d = tot.get(k, (0, 0.0))
    tot[k] = (c + 1, d + e["dur"])
busy, gaps, end = 0.0, [], t0
for e in ev:
    if e["ts"] > end:
        gaps.append((e["ts"] - end, e["name"][:50]))
    busy += max(0.0, e["ts"] + e["dur"] - max(end, e["ts"]))
    end = max(end, e["ts"] + e["dur"])
print(f"span {(t1 - t0) / 1e3:.3f} ms, busy {busy / 1e3:.3f} ms, idle {(t1 - t0 - busy) / 1e3:.3f} ms in {len(gaps)} gaps")
for k, (c, d) in sorted(tot.items(), key=lambda x: -x[1][1])[:14]:
    print(f"  {d / 1e3:8.3f} ms  {c:4d}x  {k}")
gaps.sort(reverse=True)
print("largest gaps (us, before):", [(round(g, 1), nm) for g, nm in gaps[:8]])
