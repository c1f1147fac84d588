"""Generate the golden fixtures in this directory from the REFERENCE itself
(oracle/_ref: /root/reference/proj/src/{experience,pareto,reward}.cpp compiled
unmodified).  Run here, where /root/reference exists:

    python tests/golden/make_golden.py

The fixtures travel with the repo, so tests on a machine without
/root/reference still check against the reference's own outputs.
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.oracle import Ref, RefBuffer, RefFrontier, ref_compute_reward  # noqa: E402

OUT = Path(__file__).resolve().parent


def retrieval_cases(ref):
    cases = []
    specs = [  # (name, n, d, m, lambda, sigma_sim, seed, kind)
        ("tiny_lambda0", 5, 2, 3, 0.0, 2.0, 1, "normal"),
        ("small_default", 60, 23, 15, 0.1, 0.0, 2, "scenario"),
        ("medium_lambda0", 700, 32, 8, 0.0, 0.0, 3, "scenario"),
        ("medium_greedy", 700, 32, 8, 0.1, 0.0, 4, "scenario"),
        ("ties", 40, 3, 10, 0.1, 1.0, 5, "ties"),
        ("wide", 600, 64, 32, 0.0, 0.0, 6, "normal"),
        ("gated", 300, 7, 12, 0.1, 0.0, 7, "gated"),
    ]
    for name, n, d, m, lam, ss, seed, kind in specs:
        rng = np.random.default_rng(seed)
        if kind == "scenario":  # mixed units like context_features (experience.cpp:13-28)
            scale = rng.choice([1.0, 500.0, 256.0, 0.1, 10.0, 0.3, 0.3], size=d)
            ctx = np.abs(rng.normal(size=(n, d))) * scale + rng.integers(0, 4, d) * scale
        elif kind == "ties":
            ctx = np.round(rng.normal(size=(n, d)))
        else:
            ctx = rng.normal(size=(n, d))
        rew = rng.uniform(-0.3 if kind == "gated" else 0.01, 1.5, n)
        if kind == "ties":
            rew = np.round(rew * 4) / 4 + 0.25
        rounds = rng.permutation(n).astype(np.int32)
        b = RefBuffer(ref, 0.0)
        acc = [b.store(ctx[i], rew[i], int(rounds[i])) for i in range(n)]
        sigma = b.effective_sigma(ss)
        queries = rng.normal(size=(4, d)) * ctx.std(0) + ctx.mean(0)
        res = []
        for x in queries:
            r_round, r_sim, r_score = b.select(x, m, lam, ss)
            res.append({"rounds": r_round.tolist(), "sim": r_sim.tolist(),
                        "score": r_score.tolist()})
        cases.append({"name": name, "m": m, "lambda_div": lam, "sigma_sim": ss,
                      "context": ctx.tolist(), "reward": rew.tolist(), "round": rounds.tolist(),
                      "accepted": acc, "rejected": int(b.rejected()), "sigma": sigma,
                      "queries": queries.tolist(), "select": res})
    return cases


def pareto_cases(ref):
    rng = np.random.default_rng(20240817)
    cases = []
    for t in range(40):
        n = int(rng.integers(1, 60))
        grid = [8.0, 16.0, 1e9][t % 3]
        pts = np.round(rng.uniform(size=(n, 2)) * grid) / grid
        f = RefFrontier(ref, 1.0, 1.0)
        ins = f.insert_batch(pts)
        fl, fc = f.points()
        probes = np.round(rng.uniform(size=(12, 2)) * 16) / 16
        cases.append({"points": pts.tolist(), "inserted": ins.tolist(), "frontier_l": fl.tolist(),
                      "frontier_c": fc.tolist(), "hypervolume": f.hypervolume(),
                      "probes": probes.tolist(), "reward": f.reward_batch(probes).tolist(),
                      "dominated": [f.strictly_dominated(*p) for p in probes]})
    return cases


def reward_cases(ref):
    rng = np.random.default_rng(424242)
    cases = []
    for t in range(40):
        f = RefFrontier(ref, 2000.0, 10.0)
        upd = rng.uniform(size=(int(rng.integers(0, 6)), 2)) * [2400.0, 12.0]
        for p in upd:
            f.update(*p)
        inp = rng.uniform(size=4) * [3000.0, 3000.0, 12.0, 12.0]
        deltas = rng.integers(-2, 3, size=(3, 4)) * [1, 500, 256, 1]
        cfg = (500.0, 0.0 if t % 2 else 400.0, 10.0, 0.7, 0.3, 0.3, 5.0)
        out = ref_compute_reward(ref, inp, deltas, f, cfg)
        cases.append({"updates": upd.tolist(), "inputs": inp.tolist(), "deltas": deltas.tolist(),
                      "config": cfg, "breakdown": out.tolist()})
    return cases


def main():
    ref = Ref()
    (OUT / "retrieval.json").write_text(json.dumps(retrieval_cases(ref)))
    (OUT / "pareto.json").write_text(json.dumps(pareto_cases(ref)))
    (OUT / "reward.json").write_text(json.dumps(reward_cases(ref)))
    print("wrote", [p.name for p in OUT.glob("*.json")])


if __name__ == "__main__":
    main()
