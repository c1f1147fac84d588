"""The reference's acceptance checks on the hot path (tests/acceptance/
acceptance_main.cpp), restated against the device implementation: 1 (the
frontier reward separates dominance classes, :95-131), 3 (frontier,
hypervolume and contribution against brute force on coarse grids,
:237-280) and 8 (greedy selection quality against random subsets and the
exhaustive optimum, :466-530).  The reference draws from std::mt19937_64;
these draw the same distributions from numpy with the same seeds (the checks
are properties, not golden values)."""
import itertools

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2601_22397_b200 as sair  # noqa: E402
from paper_2601_22397_b200 import ExperienceBuffer, ParetoFrontier, SelectionConfig  # noqa: E402


def brute_frontier(pts):
    """Non-dominated distinct points sorted by latency (test_pareto.cpp:17-33)."""
    out = []
    for i, (l, c) in enumerate(pts):
        if any((pl <= l and pc <= c and (pl < l or pc < c)) for pl, pc in pts):
            continue
        if (l, c) in out:
            continue
        out.append((l, c))
    return sorted(out)


def brute_hv(pts):
    f = brute_frontier(pts)
    hv = 0.0
    for i, (l, c) in enumerate(f):
        nl = f[i + 1][0] if i + 1 < len(f) else 1.0
        hv += (nl - l) * (1.0 - c)
    return hv


def test_acceptance_1_reward_separates_dominance_classes():
    gen = np.random.default_rng(20260823)
    min_gap, scored = 1e300, 0
    for trial in range(2000):
        f = ParetoFrontier(1.0, 1.0)
        n = 1 + int(gen.integers(0, 6))
        for _ in range(n):
            f.update(gen.uniform(), gen.uniform())
        probe = gen.uniform(size=(12, 2))
        r, dom = f.score_batch(probe)
        if dom.any() and (~dom).any():
            min_gap = min(min_gap, r[~dom].min() - r[dom].max())
            scored += 1
    assert scored > 1000 and min_gap >= 0.2 - 1e-12, (scored, min_gap)


def test_acceptance_3_frontier_hypervolume_contribution_against_brute_force():
    gen = np.random.default_rng(31337)
    worst = 0.0
    for trial in range(500):
        f = ParetoFrontier(1.0, 1.0)
        n = 1 + int(gen.integers(0, 6))
        pts = [(round(gen.uniform() * 8) / 8, round(gen.uniform() * 8) / 8) for _ in range(n)]
        for l, c in pts:
            f.update(l, c)
        l, c = f.points_array()
        assert list(zip(l, c)) == brute_frontier(pts)
        worst = max(worst, abs(f.hypervolume() - brute_hv(pts)))
        p = (round(gen.uniform() * 16) / 16, round(gen.uniform() * 16) / 16)
        if not f.strictly_dominated(p):
            want = brute_hv(pts + [p]) - brute_hv(pts)
            worst = max(worst, abs(f.contribution(p) - want))
    assert worst <= 1e-12


def _objective(ctx, rew, subset, x, lam, sigma):
    """selection_objective (acceptance_main.cpp:448-463): sum of surprisals
    minus lambda x pairwise similarity, in the reference's formulas."""
    n = len(rew)
    mean = ctx.mean(0)
    var = np.maximum(0.0, (ctx ** 2).mean(0) - mean ** 2)
    sd = np.sqrt(var)
    sd[sd < 1e-12] = 1.0
    z = (ctx - mean) / sd
    zx = (x - mean) / sd
    sim = lambda a, b: np.exp(-np.sum((a - b) ** 2) / (2 * sigma * sigma))
    total = rew.sum()
    val = 0.0
    for i in subset:
        loo = (total - rew[i]) / (n - 1)
        val += sim(z[i], zx) * abs(rew[i] - loo)
    for a, b in itertools.combinations(subset, 2):
        val -= lam * sim(z[a], z[b])
    return val


def test_acceptance_8_selection_quality():
    gen = np.random.default_rng(90210)
    cfg = SelectionConfig(m=3, lambda_div=0.1, sigma_sim=0.8)
    x = np.array([1.5, 1.5])

    def buffer(n):
        ctx = gen.uniform(size=(n, 2)) * 3.0
        rew = 0.05 + gen.uniform(size=n)
        db = ExperienceBuffer(0.0)
        db.store_many(ctx, rew, np.arange(n, dtype=np.int32))
        return db, ctx, rew

    wins = 0
    for trial in range(200):
        n = 8 + int(gen.integers(0, 25))
        db, ctx, rew = buffer(n)
        idx, _, _, cnt = db.select_batch(x[None], cfg)
        greedy = _objective(ctx, rew, list(idx[0, :cnt[0]]), x, 0.1, 0.8)
        rand = np.mean([_objective(ctx, rew, list(gen.permutation(n)[:3]), x, 0.1, 0.8)
                        for _ in range(100)])
        wins += greedy >= rand - 1e-9
    ok = 0
    for trial in range(50):
        db, ctx, rew = buffer(8)
        idx, _, _, cnt = db.select_batch(x[None], cfg)
        greedy = _objective(ctx, rew, list(idx[0, :cnt[0]]), x, 0.1, 0.8)
        best = max(_objective(ctx, rew, list(s), x, 0.1, 0.8)
                   for s in itertools.combinations(range(8), 3))
        ok += greedy >= 0.5 * best - 1e-9
    assert wins >= 190 and ok == 50, (wins, ok)
