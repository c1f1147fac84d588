import sys, time
import numpy as np
sys.path.insert(0, ".")
import torch
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import synth
T = 4 * 1024 * 1024
for kind in ("uniform", "anti"):
    if kind == "anti":
        l = np.random.default_rng(1).uniform(size=T)
        pts = np.stack([l, 1 - l], 1) + np.random.default_rng(2).uniform(0, 0.01, (T, 2))
    else:
        pts = synth.tuples(2026, T, 2, "uniform")
    f = sair.ParetoFrontier(1.0, 1.0)
    F = f.insert_batch(pts)
    dp = torch.from_numpy(pts).cuda()
    out = torch.empty(T, dtype=torch.float64, device="cuda")
    dom = torch.empty(T, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    for _ in range(3):
        f.score_batch_device(dp.data_ptr(), T, out.data_ptr(), dom.data_ptr(), s.cuda_stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(10):
        f.score_batch_device(dp.data_ptr(), T, out.data_ptr(), dom.data_ptr(), s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{kind}: F={F} score {ms*1e3:.1f} us -> {T/ms/1e6:.2f} G tuples/s", flush=True)
