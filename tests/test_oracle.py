"""Pin the C restatement (oracle/sair_oracle.c) to the reference itself.

`ref` is the reference's own experience/pareto/reward.cpp compiled unmodified
(oracle/_ref); `orc` is the restatement.  Retrieval and frontier results must be
bit-identical (same operations, same order).  The known-answer vectors are the
reference's unit/acceptance tests, restated (doctest is not in the image):
proj/tests/test_experience.cpp, test_pareto.cpp, test_reward.cpp and
proj/tests/acceptance/acceptance_main.cpp.
"""
import math

import numpy as np
import pytest

from oracle.oracle import RefBuffer, RefFrontier, ref_compute_reward
from paper_2601_22397_b200 import synth


def _buffer(ref, ctx, rew, rounds, r_min=0.0):
    b = RefBuffer(ref, r_min)
    b.store_many(ctx, rew, rounds)
    return b


# ---------------------------------------------------------------- retrieval ---

@pytest.mark.parametrize("n,d", [(1, 3), (2, 2), (37, 5), (600, 7), (1500, 23)])
def test_standardize_and_sigma_bit_identical(orc, ref, n, d):
    rng = np.random.default_rng(n * 7 + d)
    ctx = rng.normal(size=(n, d)) * rng.uniform(0.1, 100, size=d) + rng.uniform(-50, 50, d)
    ctx[:, 0] = 3.0  # a zero-variance dimension (sd := 1, experience.cpp:74)
    rew = rng.uniform(0.01, 1.0, n)
    b = _buffer(ref, ctx, rew, np.arange(n))
    s, ss = orc.stats(ctx)
    x = rng.normal(size=d)
    assert np.array_equal(orc.standardize(n, s, ss, x), b.standardize(x))
    want = b.effective_sigma(0.0)
    got = orc.sigma_median(ctx) if n >= 2 else 1.0
    assert got == want


@pytest.mark.parametrize("lam", [0.0, 0.1, 0.7])
@pytest.mark.parametrize("n,d,m", [(1, 2, 3), (5, 2, 3), (64, 4, 8), (400, 23, 15), (2000, 32, 8)])
def test_select_bit_identical(orc, ref, n, d, m, lam):
    rng = np.random.default_rng(1000 + n + d + m)
    ctx = rng.normal(size=(n, d))
    rew = rng.uniform(0.01, 1.01, n)
    rounds = rng.permutation(n).astype(np.int32)  # rounds != index to exercise tie-breaks
    b = _buffer(ref, ctx, rew, rounds)
    sigma = b.effective_sigma(0.0)
    for q in range(3):
        x = rng.normal(size=d)
        r_round, r_sim, r_score = b.select(x, m, lam, 0.0)
        idx, sim, sc = orc.select(ctx, rew, rounds, x, m, lam, sigma)
        assert np.array_equal(rounds[idx], r_round)
        assert np.array_equal(sim, r_sim)
        assert np.array_equal(sc, r_score)


def test_select_ties_go_to_lower_round(orc, ref):
    # identical records: every score ties, so picks follow the round order
    n, d = 12, 3
    ctx = np.ones((n, d))
    rew = np.full(n, 0.5)
    rew[::3] = 0.9
    rounds = np.array([7, 3, 11, 0, 5, 9, 1, 8, 2, 10, 4, 6], np.int32)
    b = _buffer(ref, ctx, rew, rounds)
    for lam in (0.0, 0.1):
        r_round, _, r_score = b.select(np.ones(d), 5, lam, 1.0)
        idx, _, sc = orc.select(ctx, rew, rounds, np.ones(d), 5, lam, 1.0)
        assert np.array_equal(rounds[idx], r_round)
        assert np.array_equal(sc, r_score)


def test_select_synthetic_fp32_exact_store(orc, ref):
    n, d = 3000, 64
    ctx = synth.contexts(5, 0, n, d)
    assert np.array_equal(ctx, ctx.astype(np.float32).astype(np.float64))
    rew = synth.rewards(5, 0, n)
    rounds = synth.rounds(0, n)
    b = _buffer(ref, ctx, rew, rounds)
    sigma = b.effective_sigma(0.0)
    xq = synth.queries(5, 4, d)
    for lam in (0.0, 0.1):
        rr, rc, _ = b.select_batch(xq, 32, lam, 0.0, nthreads=4)
        idx, sim, sc, cnt = orc.select_batch(ctx, rew, rounds, xq, 32, lam, sigma, nthreads=4)
        assert np.array_equal(rounds[idx], rr)
        assert np.array_equal(sc, rc)


def test_surprisal_and_local_mean(orc, ref):
    rng = np.random.default_rng(9)
    n, d = 50, 3
    ctx = rng.normal(size=(n, d))
    rew = rng.uniform(0.01, 1.0, n)
    b = _buffer(ref, ctx, rew, np.arange(n))
    x = rng.normal(size=d)
    for lm in (False, True):
        for i in (0, 7, 49):
            want = b.surprisal(i, x, 0.9, lm)
            assert orc.surprisal(ctx, rew, i, x, 0.9, lm) == want
        r_round, _, r_score = b.select(x, 6, 0.1, 0.9, lm)
        idx, _, sc = orc.select(ctx, rew, np.arange(n), x, 6, 0.1, 0.9, local_mean=lm)
        assert np.array_equal(idx, r_round)
        assert np.array_equal(sc, r_score)


def test_nearest_matches_veto_scan(orc, ref):
    # policy.cpp:140-153 restated with the reference's own standardize/similarity
    rng = np.random.default_rng(4)
    n, d = 300, 6
    ctx = rng.normal(size=(n, d))
    ctx[17] = ctx[3]  # an exact duplicate: the first index must win
    b = _buffer(ref, ctx, rng.uniform(0.1, 1, n), np.arange(n))
    sigma = b.effective_sigma(0.0)
    x = ctx[3] + 1e-3
    zc = b.standardize(x)
    best, best_sim = -1, -1.0
    for i in range(n):
        s = math.exp(-np.sum((b.standardize(ctx[i]) - zc) ** 2) / (2.0 * sigma * sigma))
        zi = b.standardize(ctx[i])
        d2 = 0.0
        for k in range(d):
            t = zi[k] - zc[k]
            d2 += t * t
        s = math.exp(-d2 / (2.0 * sigma * sigma))
        if s > best_sim:
            best, best_sim = i, s
    i, s = orc.nearest(ctx, x, sigma)
    assert (i, s) == (best, best_sim) and i == 3


# --------------------------------------------- test_experience.cpp restated ---

def test_kat_gate(ref):
    b = RefBuffer(ref, 0.0)
    assert b.store([1.0, 2.0], 0.5, 0)
    assert not b.store([1.0, 2.0], -0.2, 1)
    assert not b.store([1.0, 2.0], 0.0, 2)  # floor is strict
    assert b.size() == 1 and b.rejected() == 2
    s = RefBuffer(ref, 0.0)
    for i in range(100):
        s.store([float(i), 0.0], -1.0 if i % 10 < 3 else 1.0, i)
    assert s.size() == 70 and s.rejected() == 30


def test_kat_kernel(orc):
    a = np.zeros(2)
    assert orc.lib.orc_similarity(a.ctypes.data_as(__import__("ctypes").POINTER(__import__("ctypes").c_double)),
                                  a.ctypes.data_as(__import__("ctypes").POINTER(__import__("ctypes").c_double)), 2, 1.0) == 1.0
    c = np.array([math.sqrt(2.0), 0.0])
    import ctypes as C
    v = orc.lib.orc_similarity(a.ctypes.data_as(C.POINTER(C.c_double)),
                               c.ctypes.data_as(C.POINTER(C.c_double)), 2, 1.0)
    assert abs(v - math.exp(-1.0)) <= 1e-12 * math.exp(-1.0)


def test_kat_surprisal(orc):
    ctx = np.zeros((3, 1))
    assert abs(orc.surprisal(ctx, [0.5, 0.5, 0.5], 1, [0.0], 1e9)) <= 1e-9
    assert abs(orc.surprisal(ctx, [1.0, 0.4, 0.6], 0, [0.0], 1e9) - 0.5) <= 1e-9 * 0.5
    assert abs(orc.surprisal(np.zeros((1, 1)), [0.7], 0, [0.0], 1e9) - 0.7) <= 1e-9


def test_kat_top_m_without_diversity(orc):
    ctx = np.array([[0.0, 0.0], [0.5, 0.1], [1.0, 0.2], [1.5, 0.3], [2.0, 0.4]])
    rew = np.array([0.9, 0.2, 1.4, 0.4, 0.6])
    x = np.array([0.4, 0.1])
    idx, _, _ = orc.select(ctx, rew, np.arange(5), x, 3, 0.0, 2.0)
    direct = sorted(((orc.surprisal(ctx, rew, i, x, 2.0), i) for i in range(5)), reverse=True)
    assert set(idx.tolist()) == {direct[0][1], direct[1][1], direct[2][1]}
    assert all(rew[idx[i - 1]] <= rew[idx[i]] for i in range(1, 3))


# ------------------------------------------------------------------- pareto ---

def test_frontier_sequences_bit_identical(orc, ref):
    gen = np.random.default_rng(20240817)
    for trial in range(300):
        n = int(gen.integers(1, 41))
        pts = np.round(gen.uniform(size=(n, 2)) * 8.0) / 8.0
        f = RefFrontier(ref, 1.0, 1.0)
        ins_ref = f.insert_batch(pts)
        fl, fc, ins = orc.frontier_from_points(pts)
        rl, rc = f.points()
        assert np.array_equal(fl, rl) and np.array_equal(fc, rc)
        assert np.array_equal(ins, ins_ref)
        assert orc.hypervolume(fl, fc) == f.hypervolume()
        probes = np.round(gen.uniform(size=(8, 2)) * 16.0) / 16.0
        assert np.array_equal(orc.pareto_reward_batch(fl, fc, probes), f.reward_batch(probes))


def test_frontier_order_independent(orc):
    # the sequential update result is the non-dominated set (8(a) A13)
    gen = np.random.default_rng(7)
    pts = np.round(gen.uniform(size=(500, 2)) * 32.0) / 32.0
    a = orc.frontier_from_points(pts)[:2]
    b = orc.frontier_from_points(pts[::-1])[:2]
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_kat_pareto(ref):
    # test_pareto.cpp:55-125
    f = RefFrontier(ref, 1000.0, 10.0)
    assert f.update(600.0, 4.0)[0] and f.update(200.0, 8.0)[0]
    assert not f.update(700.0, 5.0)[0] and not f.update(600.0, 4.0)[0]
    assert len(f.points()[0]) == 2
    assert f.update(100.0, 1.0)[0]
    assert list(zip(*f.points())) == [(0.1, 0.1)]
    g = RefFrontier(ref, 1000.0, 10.0)
    g.update(200.0, 8.0)
    g.update(600.0, 4.0)
    assert abs(g.hypervolume() - 0.32) <= 1e-12 * 0.32
    assert abs(g.contribution(0.4, 0.5) - 0.06) <= 1e-12
    with pytest.raises(RuntimeError):
        g.contribution(0.7, 0.9)
    assert abs(g.reward(0.4, 0.5) - 1.06) <= 1e-12
    assert abs(g.reward(0.2, 0.8) - 1.0) <= 1e-12
    with pytest.raises(ValueError):
        RefFrontier(ref, 0.0, 1.0)


def test_dominance_counts_brute(orc):
    gen = np.random.default_rng(3)
    for K in (2, 3, 4):
        t = np.floor(gen.uniform(size=(300, K)) * 6) / 6
        cnt, mem = orc.dominance_counts(t)
        le = (t[:, None, :] <= t[None, :, :]).all(-1)
        lt = (t[:, None, :] < t[None, :, :]).any(-1)
        dom = le & lt  # dom[j, i]: j dominates i
        assert np.array_equal(cnt, dom.sum(0))
        eq = (t[:, None, :] == t[None, :, :]).all(-1)
        first = ~np.tril(eq, -1).any(1)
        assert np.array_equal(mem, (cnt == 0) & first)
        if K == 2:
            fl, fc, _ = orc.frontier_from_points(t)
            fr = sorted(map(tuple, t[mem]))
            assert fr == list(zip(fl, fc))



def test_scalable_pareto_checkers_equal_brute_force(orc):
    """The checkers the full-size (4M-tuple) GPU parity tests use -- the
    threaded k-D counts, the O(T log T) two-objective counts and the sorted
    frontier -- equal the brute-force loop and the sequential insert loop
    (src/pareto.cpp:43-54) on tie-heavy grids and continuous data."""
    gen = np.random.default_rng(17)
    for K in (2, 3, 4):
        for grid in (4, 16, 0):
            t = gen.uniform(size=(2000, K))
            if grid:
                t = np.floor(t * grid) / grid
            cnt, mem = orc.dominance_counts(t)
            c2, m2 = orc.dominance_counts_mt(t, nthreads=5)
            assert np.array_equal(cnt, c2) and np.array_equal(mem, m2)
            if K == 2:
                c3, m3 = orc.dominance_counts2_sorted(t)
                assert np.array_equal(cnt, c3) and np.array_equal(mem, m3)
                fl, fc, _ = orc.frontier_from_points(t)
                sl, sc = orc.frontier_sorted(t)
                assert np.array_equal(fl, sl) and np.array_equal(fc, sc)
    # anti-correlated: a frontier of most of the points
    x = gen.uniform(size=3000)
    t = np.stack([x, 1.0 - x + gen.uniform(-0.01, 0.01, 3000)], 1)
    fl, fc, _ = orc.frontier_from_points(t)
    sl, sc = orc.frontier_sorted(t)
    assert len(fl) > 100 and np.array_equal(fl, sl) and np.array_equal(fc, sc)
    assert np.array_equal(orc.dominance_counts2_sorted(t)[0], orc.dominance_counts(t)[0])

# ------------------------------------------------------------------- reward ---

CFG_DEFAULT = (500.0, 0.0, 10.0, 0.7, 0.3, 0.3, 5.0)


def test_reward_matches_reference(orc, ref):
    gen = np.random.default_rng(424242)
    for trial in range(200):
        l_max, c_max = 2000.0, 10.0
        f = RefFrontier(ref, l_max, c_max)
        pts = gen.uniform(size=(int(gen.integers(0, 6)), 2)) * [2400.0, 12.0]
        for p in pts:
            f.update(*p)
        fl, fc = f.points()
        inp = gen.uniform(size=4) * [3000.0, 3000.0, 12.0, 12.0]
        deltas = gen.integers(-2, 3, size=(3, 4)) * [1, 500, 256, 1]
        want = ref_compute_reward(ref, inp, deltas, f, CFG_DEFAULT)
        got = orc.compute_reward(inp, deltas, fl, fc, l_max, c_max, CFG_DEFAULT)
        assert np.array_equal(got, want)


def test_kat_reward_golden(orc):
    # test_reward.cpp:57-76
    fl, fc = np.array([0.25]), np.array([0.12])
    out = orc.compute_reward([400.0, 300.0, 1.0, 1.2], [[1, 0, 0, 0]], fl, fc, 400.0, 10.0,
                             (500.0, 400.0, 10.0, 0.7, 0.3, 0.3, 5.0))
    lat, cost, sla, pro, par, tot, clip = out
    assert abs(lat - 0.175) <= 1e-9 and abs(cost + 0.006) <= 1e-9
    assert sla == 0.0 and pro == 0.0 and clip == 0.0
    assert abs(par - 0.8 / 1.5) <= 1e-9 and abs(tot - (0.175 - 0.006 + 0.8 / 1.5)) <= 1e-9


def test_kat_reward_acceptance_vectors(orc, ref):
    # acceptance_main.cpp:140-233 (check 2), frontier {(0.3,0.4),(0.7,0.2)}
    f = RefFrontier(ref, 1000.0, 10.0)
    f.update(300.0, 4.0)
    f.update(700.0, 2.0)
    fl, fc = f.points()
    cfg = (500.0, 400.0, 10.0, 0.7, 0.3, 0.3, 5.0)
    cases = [
        ([900.0, 650.0, 2.0, 2.6], [[1, 0, 0, 0], [0, 0, 0, 0]], 1.0 + 0.05 * 0.14),
        ([820.0, 820.0, 3.0, 3.0], [[0, 0, 0, 0]] * 3, 0.8 / (1.0 + math.sqrt(0.12 ** 2 + 0.1 ** 2))),
        ([4000.0, 3500.0, 1.0, 1.5], [[0, 0, 0, 0]] * 2, 1.0),
        ([700.0, 430.0, 2.4, 3.1], [[1, 0, 0, 0], [0, 0, 0, 0], [0, 500, 0, 0]], 1.0 + 0.27 * 0.09),
        ([150.0, 180.0, 4.0, 3.2], [[0, 0, 0, 0], [-1, 0, 0, 0], [0, 0, 0, 0]],
         1.0 + 0.12 * 0.68 + 0.4 * 0.08),
        ([500.0, 500.0, 2.0, 2.0], [[0, 0, 0, 0]], 1.0 + 0.2 * 0.2),
    ]
    for inp, deltas, pareto in cases:
        got = orc.compute_reward(inp, deltas, fl, fc, 1000.0, 10.0, cfg)
        want = ref_compute_reward(ref, inp, deltas, f, cfg)
        assert np.array_equal(got, want)
        assert abs(got[4] - pareto) <= 1e-9 * max(1.0, abs(pareto))
    with pytest.raises(ValueError):
        orc.compute_reward([1, 1, 1, 1], [[0, 0, 0, 0]], fl, fc, 1000.0, 10.0,
                           (0.0, 0.0, 10.0, 0.7, 0.3, 0.3, 5.0))


def test_action_magnitude(orc, ref):
    d = np.array([[2, -500, 0, 0], [0, 0, 0, 1]], np.int32)
    assert abs(orc.action_magnitude(d) - (2.0 + 0.5 + 0.05 + 1.0)) <= 1e-12
    import ctypes as C
    assert orc.action_magnitude(d) == ref.lib.ref_action_magnitude(
        d.ctypes.data_as(C.POINTER(C.c_int32)), 2)


def test_threaded_synth_equals_synth_py(orc):
    from paper_2601_22397_b200 import synth
    for seed, start, count, d in ((2026, 0, 3000, 64), (7, 123457, 999, 23), (11, 0, 5, 1)):
        assert np.array_equal(orc.synth_contexts(seed, start, count, d, nthreads=3),
                              synth.contexts(seed, start, count, d))
