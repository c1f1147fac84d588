"""Parity of the CUDA path (libsair.so through the C-ABI) with the oracle.

Checkers: `ref` = the reference's own code compiled in place (oracle/_ref,
travels to the GPU box as a prebuilt .so), `orc` = the C restatement pinned to
it (tests/test_oracle.py), and the committed golden fixtures.  Bars
(SURVEY.md 8(d)): indices / memberships / counts bit-exact, scores within
1e-5 * max(1, |ref|) -- asserted much tighter here where the math allows.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2601_22397_b200 as sair  # noqa: E402
from paper_2601_22397_b200 import (ExperienceBuffer, Experience, ParetoFrontier,  # noqa: E402
                                   RewardConfig, RewardInputs, ScalingAction, SelectionConfig,
                                   synth)
from oracle.oracle import RefBuffer, RefFrontier, ref_compute_reward  # noqa: E402

TOL = 1e-5  # the north-star score tolerance (relative, acceptance_main.cpp:51-53 style)


def near(got, want, rel):
    got, want = np.asarray(got, float), np.asarray(want, float)
    return np.all(np.abs(got - want) <= rel * np.maximum(1.0, np.abs(want)))


def mk(ctx, reward, rnd):
    return Experience(list(map(float, ctx)), ScalingAction.noop(1), float(reward), int(rnd))


def dev_buffer(ctx, rew, rounds, r_min=0.0):
    b = ExperienceBuffer(r_min)
    b.store_many(ctx, rew, rounds, keep_mirror=True)
    return b


# ------------------------------------------------ test_experience.cpp KATs ---

def test_gate_and_rejections():
    b = ExperienceBuffer(0.0)
    assert b.store(mk([1.0, 2.0], 0.5, 0))
    assert not b.store(mk([1.0, 2.0], -0.2, 1))
    assert not b.store(mk([1.0, 2.0], 0.0, 2))
    assert b.size() == 1 and b.rejected() == 2
    s = ExperienceBuffer(0.0)
    for i in range(100):
        s.store(mk([float(i), 0.0], -1.0 if i % 10 < 3 else 1.0, i))
    assert s.size() == 70 and s.rejected() == 30


def test_dimension_change_is_invalid_argument():
    b = ExperienceBuffer(0.0)
    b.store(mk([1.0, 2.0], 0.5, 0))
    with pytest.raises(sair.InvalidArgument):
        b.store(mk([1.0], 0.5, 1))
    with pytest.raises(sair.InvalidArgument):
        b.select([1.0, 2.0, 3.0], SelectionConfig(m=2))
    with pytest.raises(sair.OutOfRange):
        b.surprisal(5, [1.0, 2.0])


def test_surprisal_kats():
    cfg = SelectionConfig(sigma_sim=1e9)
    b = ExperienceBuffer(-10.0)
    for i, r in enumerate([0.5, 0.5, 0.5]):
        b.store(mk([0.0], r, i))
    assert abs(b.surprisal(1, [0.0], cfg)) <= 1e-9
    b2 = ExperienceBuffer(-10.0)
    for i, r in enumerate([1.0, 0.4, 0.6]):
        b2.store(mk([0.0], r, i))
    assert abs(b2.surprisal(0, [0.0], cfg) - 0.5) <= 1e-9 * 0.5
    lone = ExperienceBuffer(-10.0)
    lone.store(mk([0.0], 0.7, 0))
    assert abs(lone.surprisal(0, [0.0], cfg) - 0.7) <= 1e-9


def test_top_m_without_diversity_and_curriculum():
    cfg = SelectionConfig(m=3, lambda_div=0.0, sigma_sim=2.0)
    b = ExperienceBuffer(0.0)
    for i, (c, r) in enumerate([([0.0, 0.0], 0.9), ([0.5, 0.1], 0.2), ([1.0, 0.2], 1.4),
                                ([1.5, 0.3], 0.4), ([2.0, 0.4], 0.6)]):
        b.store(mk(c, r, i))
    x = [0.4, 0.1]
    sel = b.select(x, cfg)
    assert len(sel) == 3
    direct = sorted(((b.surprisal(i, x, cfg), i) for i in range(5)), reverse=True)[:3]
    assert {s.experience.round for s in sel} == {i for _, i in direct}
    assert all(sel[i - 1].experience.reward <= sel[i].experience.reward for i in range(1, 3))


def test_small_buffer_edge_cases():
    cfg = SelectionConfig(m=15)
    assert ExperienceBuffer(0.0).select([1.0, 2.0], cfg) == []
    b = ExperienceBuffer(0.0)
    b.store(mk([1.0, 0.0], 0.3, 0))
    b.store(mk([0.0, 1.0], 0.8, 1))
    a1, a2 = b.select([0.5, 0.5], cfg), b.select([0.5, 0.5], cfg)
    assert len(a1) == 2 and [s.experience.round for s in a1] == [s.experience.round for s in a2]
    assert b.select([0.5, 0.5], SelectionConfig(m=0)) == []


# ------------------------------------------------ parity with the reference ---

@pytest.mark.parametrize("lam", [0.0, 0.1])
@pytest.mark.parametrize("n,d,m", [(1, 2, 3), (7, 2, 3), (300, 5, 8), (2000, 23, 15),
                                   (5000, 32, 8)])
def test_select_matches_reference(ref, lam, n, d, m):
    rng = np.random.default_rng(7 * n + d)
    # real-valued, not fp32-representable contexts with mixed units
    ctx = rng.normal(size=(n, d)) * rng.uniform(0.5, 50, d) + rng.uniform(-100, 100, d)
    rew = rng.uniform(0.01, 1.01, n)
    rounds = rng.permutation(n).astype(np.int32)
    rb = RefBuffer(ref, 0.0)
    rb.store_many(ctx, rew, rounds)
    db = dev_buffer(ctx, rew, rounds)
    assert db.effective_sigma() == rb.effective_sigma(0.0)
    xq = rng.normal(size=(5, d)) * ctx.std(0) + ctx.mean(0)
    idx, sim, sc, cnt, nn_i, nn_s = db.select_batch(xq, SelectionConfig(m=m, lambda_div=lam),
                                                    nearest=True)
    for q in range(len(xq)):
        r_round, r_sim, r_score = rb.select(xq[q], m, lam, 0.0)
        k = int(cnt[q])
        assert k == len(r_round)
        assert np.array_equal(rounds[idx[q, :k]], r_round)
        assert near(sc[q, :k], r_score, 1e-12) and near(sim[q, :k], r_sim, 1e-12)
        # veto scan (policy.cpp:140-157) restated with the reference's standardize
        zc = rb.standardize(xq[q])
        sims = [math.exp(-sum((a - b) ** 2 for a, b in zip(rb.standardize(ctx[i]), zc))
                         / (2.0 * rb.effective_sigma(0.0) ** 2)) for i in range(n)]
        best = int(np.argmax(sims))
        assert nn_i[q] == best and abs(nn_s[q] - sims[best]) <= 1e-12


@pytest.mark.parametrize("n,d", [(600, 300), (70000, 300)])
def test_wide_contexts_beyond_the_page_width(ref, orc, n, d):
    """d > 256 (37+ stages): the page rows hold 256 columns, the fp64 rows all
    d -- sigma, get, select (one-launch small path below 64k records, the exact
    passes above) against the reference / its pinned restatement."""
    rng = np.random.default_rng(d + n)
    ctx = rng.normal(size=(n, d)) * rng.uniform(0.5, 5, d)
    rew = rng.uniform(0.01, 1.01, n)
    rounds = np.arange(n, dtype=np.int32)
    db = ExperienceBuffer(0.0)
    db.store_many(ctx, rew, rounds)
    c, r, _ = db.get(n - 1)
    assert np.array_equal(c, ctx[n - 1]) and r == rew[n - 1]
    sigma = db.effective_sigma()
    assert sigma == orc.sigma_median(ctx)
    xq = rng.normal(size=(3, d))
    for lam in (0.0, 0.1):
        idx, sim, sc, cnt = db.select_batch(xq, SelectionConfig(m=8, lambda_div=lam))
        oi, osim, osc, _ = orc.select_batch(ctx, rew, rounds, xq, 8, lam, sigma)
        assert np.array_equal(idx, oi)
        assert near(sc, osc, 1e-12)
    if n <= 1000:
        rb = RefBuffer(ref, 0.0)
        rb.store_many(ctx, rew, rounds)
        r_round, _, r_score = rb.select(xq[0], 8, 0.1, 0.0)
        assert np.array_equal(rounds[idx[0, :len(r_round)]], r_round)


@pytest.mark.parametrize("n", [3000, 100000])
def test_negative_lambda_takes_the_exact_path(orc, n):
    """lambda_div < 0 (accepted by the reference, scenario.cpp:197) rewards
    similarity: the score bound cannot certify it, the answer is the exact one."""
    d = 16
    db = ExperienceBuffer(0.0)
    db.store_synthetic(21, n, d)
    ctx, rew, rnd = synth.contexts(21, 0, n, d), synth.rewards(21, 0, n), synth.rounds(0, n)
    xq = synth.queries(22, 40, d)
    idx, sim, sc, cnt = db.select_batch(xq, SelectionConfig(m=8, lambda_div=-0.3))
    oi, osim, osc, _ = orc.select_batch(ctx, rew, rnd, xq, 8, -0.3, db.effective_sigma())
    assert np.array_equal(idx, oi)
    assert near(sc, osc, 1e-12)


def test_exact_mode_and_fast_path_agree(orc):
    n, d = 50000, 64
    ctx = synth.contexts(11, 0, n, d)
    rew = synth.rewards(11, 0, n)
    rounds = synth.rounds(0, n)
    db = ExperienceBuffer(0.0)
    db.store_synthetic(11, n, d)
    # the device generator is the numpy generator
    c0, r0, rd0 = db.get(12345)
    assert np.array_equal(c0, ctx[12345]) and r0 == rew[12345] and rd0 == 12345
    sigma = db.effective_sigma()
    assert sigma == orc.sigma_median(ctx)
    xq = synth.queries(11, 11, d)
    for lam in (0.0, 0.1):
        cfg = SelectionConfig(m=32, lambda_div=lam)
        fast = db.select_batch(xq, cfg)
        st = db.last_stats()
        exact = db.select_batch(xq, SelectionConfig(m=32, lambda_div=lam, mode=sair.SELECT_EXACT))
        assert np.array_equal(fast[0], exact[0])
        assert np.array_equal(fast[2], exact[2])
        if lam == 0.0:
            assert st["certified"] == len(xq), st
        oi, osim, osc, ocnt = orc.select_batch(ctx, rew, rounds, xq, 32, lam, sigma)
        assert np.array_equal(fast[0], oi)
        assert near(fast[2], osc, 1e-12)


def test_clustered_store_parity(orc):
    n, d = 20000, 32
    db = ExperienceBuffer(0.0)
    db.store_synthetic(3, n, d, clustered=True)
    ctx = synth.contexts(3, 0, n, d, clustered=True)
    rew = synth.rewards(3, 0, n)
    c, r, _ = db.get(777)
    assert np.array_equal(c, ctx[777])
    xq = synth.queries(3, 8, d, clustered=True)
    sigma = db.effective_sigma()
    for lam in (0.0, 0.1):
        idx, sim, sc, cnt = db.select_batch(xq, SelectionConfig(m=16, lambda_div=lam))
        oi, osim, osc, _ = orc.select_batch(ctx, rew, synth.rounds(0, n), xq, 16, lam, sigma)
        assert np.array_equal(idx, oi)
        assert near(sc, osc, 1e-12)


def test_sigma_cache_state_machine(ref):
    rng = np.random.default_rng(5)
    d = 4
    rb, db = RefBuffer(ref, 0.0), ExperienceBuffer(0.0)
    for step in range(700):
        x = rng.normal(size=d) * [1, 10, 100, 0.1]
        r = rng.uniform(0.01, 1)
        rb.store(x, r, step)
        db.store(mk(x, r, step))
        if step % 37 == 0 or step in (1, 2, 511, 512, 513, 699):
            assert db.effective_sigma() == rb.effective_sigma(0.0)
            assert db.effective_sigma(SelectionConfig(sigma_sim=0.3)) == 0.3


def test_surprisal_and_local_mean_match_reference(ref):
    rng = np.random.default_rng(9)
    n, d = 120, 3
    ctx = rng.normal(size=(n, d))
    rew = rng.uniform(0.01, 1.0, n)
    rb = RefBuffer(ref, 0.0)
    rb.store_many(ctx, rew, np.arange(n))
    db = dev_buffer(ctx, rew, np.arange(n))
    x = rng.normal(size=d)
    for lm in (False, True):
        cfg = SelectionConfig(m=6, lambda_div=0.1, sigma_sim=0.9, locally_weighted_mean=lm)
        for i in (0, 7, n - 1):
            assert near(db.surprisal(i, x, cfg), rb.surprisal(i, x, 0.9, lm), 1e-13)
        r_round, _, r_score = rb.select(x, 6, 0.1, 0.9, lm)
        sel = db.select(x, cfg)
        assert [s.experience.round for s in sel] == list(r_round)
        assert near([s.score for s in sel], r_score, 1e-12)


@pytest.mark.slow
def test_full_size_16m_properties():
    """BASELINE config at full size: 16M x 64 on one GPU.  The fast path must be
    certified and equal the device's full fp64 pass (the oracle's algorithm)."""
    n, d = 16 * 1024 * 1024, 64
    db = ExperienceBuffer(0.0)
    db.store_synthetic(2026, n, d)
    assert db.size() == n
    xq = synth.queries(2026, 8, d)
    cfg = SelectionConfig(m=32, lambda_div=0.0)
    fast = db.select_batch(xq, cfg, nearest=True)
    st = db.last_stats()
    assert st["certified"] == 8, st
    exact = db.select_batch(xq[:2], SelectionConfig(m=32, lambda_div=0.0,
                                                    mode=sair.SELECT_EXACT), nearest=True)
    assert np.array_equal(fast[0][:2], exact[0])
    assert np.array_equal(fast[2][:2], exact[2])
    assert np.array_equal(fast[4][:2], exact[4])
    # curriculum order: rewards ascending within every query
    for q in range(8):
        rw = [db.get(int(i))[1] for i in fast[0][q]]
        assert all(a <= b for a, b in zip(rw, rw[1:]))


# ------------------------------------------------------------ pareto (2-D) ---

def test_pareto_kats():
    f = ParetoFrontier(1000.0, 10.0)
    assert f.update(600.0, 4.0)[0] and f.update(200.0, 8.0)[0]
    assert not f.update(700.0, 5.0)[0] and not f.update(600.0, 4.0)[0]
    assert f.size() == 2
    assert f.update(100.0, 1.0)[0]
    assert f.points() == [sair.ObjectivePoint(0.1, 0.1)]
    g = ParetoFrontier(1000.0, 10.0)
    assert g.hypervolume() == 0.0
    g.update(200.0, 8.0)
    g.update(600.0, 4.0)
    assert abs(g.hypervolume() - 0.32) <= 1e-12
    assert abs(g.contribution((0.4, 0.5)) - 0.06) <= 1e-12
    with pytest.raises(sair.LogicError):
        g.contribution((0.7, 0.9))
    d = min(math.hypot(0.7 - 0.2, 0.9 - 0.8), math.hypot(0.7 - 0.6, 0.9 - 0.4))
    assert abs(g.reward((0.7, 0.9)) - 0.8 / (1 + d)) <= 1e-12
    assert abs(g.reward((0.4, 0.5)) - 1.06) <= 1e-12
    assert abs(g.reward((0.2, 0.8)) - 1.0) <= 1e-12
    h = ParetoFrontier(1000.0, 10.0)
    assert abs(h.reward((0.3, 0.4)) - (1.0 + 0.7 * 0.6)) <= 1e-12
    assert h.distance((0.3, 0.4)) is None
    p, cl = h.normalize(2500.0, 3.0)
    assert p.latency == 1.0 and cl
    with pytest.raises(sair.InvalidArgument):
        ParetoFrontier(0.0, 1.0)
    with pytest.raises(sair.InvalidArgument):
        ParetoFrontier(1.0, -2.0)
    assert sair.dominates((0.2, 0.3), (0.3, 0.3)) and not sair.dominates((0.2, 0.3), (0.2, 0.3))
    assert not sair.dominates((0.1, 0.9), (0.9, 0.1))


def test_frontier_sequences_match_reference(ref):
    gen = np.random.default_rng(20240817)
    for trial in range(120):
        n = int(gen.integers(1, 41))
        pts = np.round(gen.uniform(size=(n, 2)) * 8.0) / 8.0
        rf = RefFrontier(ref, 1.0, 1.0)
        df = ParetoFrontier(1.0, 1.0)
        for p in pts:
            assert df.update(*p)[0] == rf.update(*p)[0]
        rl, rc = rf.points()
        dl, dc = df.points_array()
        assert np.array_equal(dl, rl) and np.array_equal(dc, rc)
        assert df.hypervolume() == rf.hypervolume()
        probes = np.round(gen.uniform(size=(16, 2)) * 16.0) / 16.0
        got, dom = df.score_batch(probes)
        want = rf.reward_batch(probes)
        assert np.array_equal(got, want)  # small frontiers replay the reference sequence
        for p, dm in zip(probes, dom):
            assert dm == rf.strictly_dominated(*p)


def test_batch_insert_prefilter_edge_cases(ref):
    """K6's CTA pre-filter (pareto.cu prefilter_kernel: 4096-tuple CTAs, runs
    from 8192 tuples) against the reference's own insert_normalized loop
    (pareto.cpp:43-54): coarse grids (latency ties inside and across CTAs),
    exact duplicates whose first occurrence carries -0.0 vs +0.0 bits, a
    staircase spanning CTA boundaries, a non-empty frontier beforehand, and a
    NaN tuple (the host falls back to the unfiltered sort path)."""
    gen = np.random.default_rng(7)
    cases = []
    T = 3 * 4096 + 777
    cases.append(np.round(gen.uniform(size=(T, 2)) * 4.0) / 4.0)          # heavy ties
    z = np.round(gen.uniform(size=(T, 2)) * 16.0) / 16.0
    z[gen.integers(0, T, 500)] = (0.0, 0.5)
    z[gen.integers(0, T, 500)] = (-0.0, 0.5)                                  # signed zeros
    z[gen.integers(0, T, 300)] = (0.25, -0.0)
    cases.append(z)
    x = np.linspace(0.0, 1.0, T)
    stair = np.stack([x, 1.0 - x], 1)[gen.permutation(T)]                   # every tuple on the frontier
    cases.append(stair)
    for pts in cases:
        rf = RefFrontier(ref, 1.0, 1.0)
        df = ParetoFrontier(1.0, 1.0)
        pre = np.round(gen.uniform(size=(64, 2)) * 8.0) / 8.0
        for p in pre:
            rf.insert_normalized(*p)
        df.insert_batch(pre)
        for p in pts:
            rf.insert_normalized(*p)
        F = df.insert_batch(pts)
        rl, rc = rf.points()
        dl, dc = df.points_array()
        assert F == len(rl)
        assert np.array_equal(np.signbit(dl), np.signbit(rl))
        assert np.array_equal(np.signbit(dc), np.signbit(rc))
        assert np.array_equal(dl, rl) and np.array_equal(dc, rc)
        assert df.hypervolume() == rf.hypervolume()
    # a NaN anywhere sends the batch down the unfiltered sort path (the
    # pre-filter's order argument needs totally ordered coordinates)
    pts = gen.uniform(size=(20000, 2))
    pts[12345] = (np.nan, 0.5)
    dn = ParetoFrontier(1.0, 1.0)
    F = dn.insert_batch(pts)
    assert F == len(dn.points_array()[0])


def test_batch_insert_and_scoring_at_scale(orc):
    for dist in ("uniform", "anti", "grid", "corr"):
        pts = synth.tuples(17, 200000, 2, dist)
        df = ParetoFrontier(1.0, 1.0)
        F = df.insert_batch(pts[:120000])
        F = df.insert_batch(pts[120000:])
        fl, fc, _ = orc.frontier_from_points(pts)
        dl, dc = df.points_array()
        assert F == len(fl)
        assert np.array_equal(dl, fl) and np.array_equal(dc, fc)
        probes = synth.tuples(18, 4000, 2, dist)
        got, dom = df.score_batch(probes)
        want = orc.pareto_reward_batch(fl, fc, probes)
        assert near(got, want, 1e-12), dist


def test_reward_matches_reference(ref):
    gen = np.random.default_rng(424242)
    cfg = RewardConfig()
    cfgv = (cfg.t_sla_ms, cfg.l_baseline_ms, cfg.c_budget, cfg.w_latency, cfg.w_cost,
            cfg.w_proactive, cfg.r_max)
    for trial in range(60):
        rf = RefFrontier(ref, 2000.0, 10.0)
        df = ParetoFrontier(2000.0, 10.0)
        for p in gen.uniform(size=(int(gen.integers(0, 6)), 2)) * [2400.0, 12.0]:
            rf.update(*p)
            df.update(*p)
        inp = gen.uniform(size=4) * [3000.0, 3000.0, 12.0, 12.0]
        deltas = gen.integers(-2, 3, size=(3, 4)) * [1, 500, 256, 1]
        act = ScalingAction([sair.StageDelta(*map(int, r)) for r in deltas])
        want = ref_compute_reward(ref, inp, deltas, rf, cfgv)
        got = sair.compute_reward(RewardInputs(*inp), act, df, cfg)
        assert np.array_equal([got.latency, got.cost, got.sla, got.proactive, got.pareto,
                               got.total, float(got.clipped)], want)
    with pytest.raises(sair.InvalidArgument):
        sair.compute_reward(RewardInputs(1, 1, 1, 1), ScalingAction.noop(1), df,
                            RewardConfig(t_sla_ms=0.0))
    with pytest.raises(sair.InvalidArgument):
        sair.compute_reward(RewardInputs(1, 1, 1, 1), ScalingAction.noop(1), df,
                            RewardConfig(c_budget=0.0))


def test_reward_golden_and_batch():
    # test_reward.cpp:57-76
    f = ParetoFrontier(400.0, 10.0)
    f.update(100.0, 1.2)
    a = ScalingAction.noop(1)
    a.stages[0].replicas = 1
    r = sair.compute_reward(RewardInputs(400.0, 300.0, 1.0, 1.2), a, f,
                            RewardConfig(500.0, 400.0, 10.0))
    assert abs(r.latency - 0.175) <= 1e-9 and abs(r.cost + 0.006) <= 1e-9
    assert r.sla == 0.0 and r.proactive == 0.0 and not r.clipped
    assert abs(r.pareto - 0.8 / 1.5) <= 1e-9
    assert sair.action_magnitude(a) == 1.5
    rows = np.array([[400.0, 300.0, 1.0, 1.2], [40000.0, 100.0, 5.0, 1.0],
                     [100.0, 40000.0, 1.0, 5.0]])
    deltas = np.array([[[1, 0, 0, 0]], [[1, 0, 0, 0]], [[0, 0, 0, 0]]])
    out = sair.compute_reward_batch(rows, deltas, f, RewardConfig(500.0, 400.0, 10.0))
    assert out[0, 5] == r.total
    assert out[1, 5] == 5.0 and out[1, 6] == 1.0 and out[2, 5] == -5.0


# ----------------------------------------------------- k-D dominance counts ---

@pytest.mark.parametrize("K", [1, 2, 3, 4])
def test_dominance_counts_match_oracle(orc, K):
    for dist in ("uniform", "grid", "anti", "corr"):
        t = synth.tuples(23 + K, 3000, K, dist)
        if dist == "grid":
            t = np.floor(t * 8) / 8  # many duplicates and ties
        cnt, mem = sair.dominance_counts(t)
        ocnt, omem = orc.dominance_counts(t)
        assert np.array_equal(cnt, ocnt) and np.array_equal(mem, omem)
        _, mem2 = sair.dominance_counts(t, counts=False)
        assert np.array_equal(mem2, omem)


@pytest.mark.parametrize("K", [1, 2])
@pytest.mark.parametrize("dist", ["uniform", "grid", "anti"])
def test_two_objective_counting_equals_pairwise_tiles(K, dist):
    """K <= 2 counts by the O(T log T) merge counting equal the pairwise tile
    kernel (the K >= 3 path, forced with SAIR_DOM_TILES) at 150k tuples."""
    import os
    T = 150000
    if dist == "anti":
        l = np.random.default_rng(K).uniform(size=T)
        t = np.stack([l, 1.0 - l + np.random.default_rng(K + 1).uniform(-1e-3, 1e-3, T)], 1)[:, :K]
    else:
        t = synth.tuples(31 + K, T, K, "grid" if dist == "grid" else "uniform")
        if dist == "grid":
            t = np.floor(t * 32) / 32
    cnt, mem = sair.dominance_counts(t)
    os.environ["SAIR_DOM_TILES"] = "1"
    try:
        c2, m2 = sair.dominance_counts(t)
    finally:
        os.environ.pop("SAIR_DOM_TILES")
    assert np.array_equal(cnt, c2) and np.array_equal(mem, m2)
    # and the parts combine by a sum (only part 0 does the work for K <= 2)
    p0 = sair.dominance_counts(t, part=0, nparts=2)
    p1 = sair.dominance_counts(t, part=1, nparts=2)
    assert np.array_equal(p0[0] + p1[0], cnt) and np.array_equal(p0[1] | p1[1], mem)


def test_shard_merges_agree():
    """The two cross-shard merges (host arrays: sair_merge_topk; the
    all-gathered device buffer: sair_merge_topk_packed) on random per-shard
    top-m with ties in score and round and ragged counts."""
    import ctypes as C
    from paper_2601_22397_b200 import _lib
    from paper_2601_22397_b200.sharded import merge_parts
    rng = np.random.default_rng(8)
    R, nq, m = 3, 60, 8
    parts = []
    gid = rng.permutation(R * nq * m).reshape(R, nq, m)
    for r in range(R):
        sc = np.sort(rng.integers(0, 6, (nq, m)) / 8.0, axis=1)[:, ::-1]
        cnt = rng.integers(0, m + 1, nq)
        parts.append(np.concatenate([sc, rng.uniform(size=(nq, m)), rng.integers(0, 3, (nq, m)) / 2.0,
                                     gid[r].astype(np.float64), rng.integers(0, 4, (nq, m)).astype(np.float64),
                                     cnt[:, None].astype(np.float64)], axis=1))
    i1, s1, c1, n1 = merge_parts(parts, nq, m, 0)
    dev = torch.from_numpy(np.stack(parts)).cuda()
    out = torch.empty((nq, 3 * m + 1), dtype=torch.float64, device="cuda")
    assert sair.lib().sair_merge_topk_packed(dev.data_ptr(), R, nq, m, 0, None, out.data_ptr()) == 0
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    n2 = o[:, 3 * m].astype(np.int64)
    assert np.array_equal(n1, n2)
    for q in range(nq):
        k = n1[q]
        assert np.array_equal(i1[q, :k], o[q, :k].astype(np.int64))
        assert np.array_equal(s1[q, :k], o[q, m:m + k]) and np.array_equal(c1[q, :k], o[q, 2 * m:2 * m + k])
