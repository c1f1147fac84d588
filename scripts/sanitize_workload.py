"""A small workload over every kernel family, for compute-sanitizer (memcheck /
racecheck / synccheck): the one-launch small select (lambda 0.1, veto), the
8-query and wide tcgen05 passes with merge and refine, the filtered and the
fp64 greedy, the batched decision step, and the Pareto kernels (K6 insert, K8
scoring incl. the windowed path, K7 counts)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22397_b200 as sair  # noqa: E402
from paper_2601_22397_b200 import decision, synth  # noqa: E402

part = sys.argv[1] if len(sys.argv) > 1 else "all"
if part in ("all", "select"):
    small = sair.ExperienceBuffer(0.0)
    small.store_synthetic(3, 3000, 16)
    small.select_batch(synth.queries(4, 3, 16), sair.SelectionConfig(m=6, lambda_div=0.1),
                       nearest=True)
    big = sair.ExperienceBuffer(0.0)
    big.store_synthetic(5, 70000, 64)
    for nq in (4, 40):
        big.select_batch(synth.queries(6 + nq, nq, 64), sair.SelectionConfig(m=8, lambda_div=0.0),
                         nearest=True)
    big.select_batch(synth.queries(9, 6, 64), sair.SelectionConfig(m=6, lambda_div=0.1))
    os.environ["SAIR_GREEDY64"] = "1"
    big.select_batch(synth.queries(10, 3, 64), sair.SelectionConfig(m=4, lambda_div=0.1))
    os.environ.pop("SAIR_GREEDY64")
if part in ("all", "pareto"):
    f = sair.ParetoFrontier(1.0, 1.0)
    pts = synth.tuples(7, 20000, 2, "anti")
    f.insert_batch(pts)
    f.score_batch(pts[:3000])
    f.score_batch(synth.tuples(8, 70000, 2, "anti"))
    sair.dominance_counts(synth.tuples(9, 3000, 3, "uniform"))
    sair.dominance_counts(synth.tuples(9, 3000, 2, "grid"))
if part in ("all", "decision"):
    buf = sair.ExperienceBuffer(0.0)
    buf.store_synthetic(11, 2000, 32)
    fr = sair.ParetoFrontier(2000.0, 10.0)
    x = synth.queries(12, 1, 32)[0]
    decision.replay_step(buf, fr, x, sair.SelectionConfig(m=8, lambda_div=0.1),
                         sair.RewardInputs(700.0, 430.0, 2.4, 3.1), sair.ScalingAction.noop(3),
                         sair.RewardConfig(), round=5000)
print("workload done")
