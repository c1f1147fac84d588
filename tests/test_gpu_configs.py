"""Parity at every BASELINE.json config's stated size, each
against the CPU oracle (oracle/sair_oracle.c, pinned == oracle/_ref in
test_oracle.py) or against the reference compiled in place (oracle/_ref):

  configs[0]  10k x 32, m = 8, lambda_div = 0.1 (the reference default,
              experience.hpp:29) with the veto scan: 60 decision steps of
              harness.cpp:197-261 through sair_decision_step, each checked
              against the reference's own ExperienceBuffer / ParetoFrontier /
              compute_reward stepped in the same order;
  configs[1]  1M x 64, one 256-query call (the wide tcgen05 pass), all 256
              queries vs the oracle at lambda 0; 16 queries at lambda 0.1;
  configs[2]  4M tuples: the 2-objective frontier and the dominance counts of
              every tuple for four distributions (O(T log T) oracle), the
              Pareto reward of a sample; 3 and 4 objectives at 262,144 tuples
              (the threaded brute-force oracle);
  configs[3]  16M x 64, one 4096-query call (32 wide passes), 64 queries
              spread over all 32 query groups vs the oracle.

Bars (SURVEY 8(d) parity rule, tightened): indices / counts / membership
bit-exact; scores and similarities within 1e-12 relative (the contract is
1e-5: the device computes the reference's fp64 arithmetic, only exp() may
differ by an ulp).
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2601_22397_b200 as sair  # noqa: E402
from paper_2601_22397_b200 import decision, synth  # noqa: E402

THREADS = os.cpu_count() or 1
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def near(got, want, rel=1e-12):
    got, want = np.asarray(got, float), np.asarray(want, float)
    return np.all(np.abs(got - want) <= rel * np.maximum(1.0, np.abs(want)))


def host_store(orc, seed, n, d):
    """The host copy of a device-generated synthetic store (synth.py)."""
    return (orc.synth_contexts(seed, 0, n, d), synth.rewards(seed, 0, n),
            synth.rounds(0, n))


def check_queries(orc, ctx, rew, rnd, xq, got, m, lam, sigma, stats):
    idx, sim, sc, cnt = got
    oi, osim, osc, ocnt = orc.select_batch(ctx, rew, rnd, xq, m, lam, sigma,
                                           nthreads=THREADS, stats=stats)
    assert np.array_equal(cnt, ocnt)
    bad = [q for q in range(len(xq)) if not np.array_equal(idx[q], oi[q])]
    assert not bad, f"queries {bad[:8]} differ from the oracle"
    assert near(sc, osc) and near(sim, osim)


# ---------------------------------------------------------------- configs[3] --

def test_config3_16m_4096_queries_vs_oracle(orc):
    n, d, nq, m, seed = 16 * 1024 * 1024, 64, 4096, 32, 2026
    db = sair.ExperienceBuffer(0.0)
    db.store_synthetic(seed, n, d)
    xq = synth.queries(seed + 1, nq, d)
    got = db.select_batch(xq, sair.SelectionConfig(m=m, lambda_div=0.0), nearest=True)
    st = db.last_stats()
    assert st["tensor_core"] == 3 and st["stream_launches"] == nq // st["qb"], st
    assert st["certified"] == nq and st["exact_fallbacks"] == 0, st
    ctx, rew, rnd = host_store(orc, seed, n, d)
    stats = orc.stats(ctx)
    sigma = db.effective_sigma()
    assert sigma == orc.sigma_median(ctx)
    # two queries in every one of the 32 groups of 128 (first/last lanes too)
    pick = np.array(sorted({g * 128 + (g * 37) % 128 for g in range(32)}
                           | {g * 128 + 127 - (g * 11) % 128 for g in range(32)}
                           | {0, 127, 4095}))
    assert len(pick) >= 64
    check_queries(orc, ctx, rew, rnd, xq[pick], tuple(a[pick] for a in got[:4]), m, 0.0,
                  sigma, stats)
    # the fused veto scan of the same call (policy.cpp:140-157)
    for q in pick[:6]:
        j, s = orc.nearest(ctx, xq[q], sigma)
        assert got[4][q] == j and abs(got[5][q] - s) <= 1e-12


# ---------------------------------------------------------------- configs[1] --

def test_config1_1m_256_queries_vs_oracle(orc):
    n, d, nq, m, seed = 1 << 20, 64, 256, 32, 2027
    db = sair.ExperienceBuffer(0.0)
    db.store_synthetic(seed, n, d)
    ctx, rew, rnd = host_store(orc, seed, n, d)
    stats = orc.stats(ctx)
    sigma = db.effective_sigma()
    assert sigma == orc.sigma_median(ctx)
    xq = synth.queries(seed + 1, nq, d)
    got = db.select_batch(xq, sair.SelectionConfig(m=m, lambda_div=0.0))
    st = db.last_stats()
    assert st["tensor_core"] == 2 and st["certified"] == nq, st
    check_queries(orc, ctx, rew, rnd, xq, got, m, 0.0, sigma, stats)
    # the reference's default diversity weight on a bounded sample
    xl = synth.queries(seed + 2, 16, d)
    got = db.select_batch(xl, sair.SelectionConfig(m=m, lambda_div=0.1))
    check_queries(orc, ctx, rew, rnd, xl, got, m, 0.1, sigma, stats)


# ---------------------------------------------------------------- configs[0] --

def test_config0_decision_steps_vs_reference(orc, ref):
    """60 decisions at configs[0]'s shape, the device's sair_decision_step
    against the reference's own classes (oracle/_ref) in harness order:
    select (experience.cpp:151-205) + veto scan (policy.cpp:140-157, oracle
    restatement), compute_reward against the pre-insert frontier
    (reward.cpp:21-44), frontier.update (pareto.cpp:36-54), store()
    (experience.cpp:44-62) -- across the 50-insertion sigma refresh
    (experience.cpp:116-121) and r_min rejections."""
    from oracle.oracle import RefBuffer, RefFrontier, ref_compute_reward
    n, d, seed, steps = 10000, 32, 31, 60
    cfg = sair.SelectionConfig(m=8, lambda_div=0.1)
    rc = sair.RewardConfig()
    rcv = (rc.t_sla_ms, rc.l_baseline_ms, rc.c_budget, rc.w_latency, rc.w_cost, rc.w_proactive,
           rc.r_max)
    db = sair.ExperienceBuffer(0.0)
    db.store_synthetic(seed, n, d)
    fr = sair.ParetoFrontier(2000.0, 10.0)
    ctx, rew, rnd = host_store(orc, seed, n, d)
    rb = RefBuffer(ref, 0.0)
    rb.store_many(ctx, rew, rnd)
    rf = RefFrontier(ref, 2000.0, 10.0)
    rows, rounds = [ctx], list(rnd)
    rng = np.random.default_rng(seed)
    for s in range(steps):
        x = synth.queries(seed + 100 + s, 1, d)[0]
        inp = sair.RewardInputs(rng.uniform(200, 1500), rng.uniform(200, 2600),
                                rng.uniform(0.5, 9), rng.uniform(0.5, 11))
        deltas = rng.integers(-2, 3, size=(3, 4)).astype(np.int32)
        act = sair.ScalingAction([sair.StageDelta(*map(int, r)) for r in deltas])
        upd = bool(rng.uniform() < 0.8)
        got = decision.replay_step(db, fr, x, cfg, inp, act, rc, update=upd, round=n + s)
        # the reference, same order
        want_r, want_sim, want_sc = rb.select(x, m=8, lambda_div=0.1)
        assert np.array_equal(np.asarray(rounds)[got.idx], want_r), f"step {s}: picks differ"
        assert near(got.sim, want_sim) and near(got.score, want_sc)
        allc = np.concatenate(rows) if len(rows) > 1 else rows[0]
        j, sj = orc.nearest(allc, x, rb.effective_sigma())
        assert got.nn_idx == j and abs(got.nn_sim - sj) <= 1e-12, f"step {s}: veto scan"
        out = ref_compute_reward(ref, [inp.l_before_ms, inp.l_after_ms, inp.c_before,
                                       inp.c_after], deltas, rf, rcv)
        r = got.reward
        assert (r.latency, r.cost, r.sla, r.proactive, r.pareto, r.total, float(r.clipped)) == \
            tuple(out), f"step {s}: reward"
        ins = rf.update(inp.l_after_ms, inp.c_after)[0] if upd else False
        assert got.inserted == ins
        sto = rb.store(x, r.total, n + s)
        assert got.stored == sto
        if sto:
            rows.append(x[None, :])
            rounds.append(n + s)
        assert db.size() == rb.size() and db.rejected() == rb.rejected()
        assert db.effective_sigma() == rb.effective_sigma()
    gl, gc = fr.points_array()
    fl, fc = rf.points()
    assert np.array_equal(gl, fl) and np.array_equal(gc, fc)
    assert fr.hypervolume() == rf.hypervolume()


# ---------------------------------------------------------------- configs[2] --

@pytest.mark.parametrize("dist", ["uniform", "anti", "corr", "grid"])
def test_config2_4m_two_objectives_vs_oracle(orc, dist):
    T = 4 * 1024 * 1024
    pts = synth.tuples(2028, T, 2, dist)
    f = sair.ParetoFrontier(1.0, 1.0)
    F = f.insert_batch(pts)
    fl, fc = orc.frontier_sorted(pts)
    gl, gc = f.points_array()
    assert F == len(fl) and np.array_equal(gl, fl) and np.array_equal(gc, fc)
    cnt, mem = sair.dominance_counts(pts)
    ocnt, omem = orc.dominance_counts2_sorted(pts)
    assert np.array_equal(cnt, ocnt) and np.array_equal(mem, omem)
    assert int(mem.sum()) == F
    # the reward of a sample of the tuples against the final frontier
    probe = pts[:: max(1, T // (4096 if F > 1000 else 65536))]
    got, dom = f.score_batch(probe)
    assert near(got, orc.pareto_reward_batch(fl, fc, probe))


@pytest.mark.parametrize("K,dist", [(3, "uniform"), (4, "uniform"), (4, "grid")])
def test_config2_k_objective_counts_vs_oracle(orc, K, dist):
    T = 262144
    t = synth.tuples(2029 + K, T, K, dist)
    cnt, mem = sair.dominance_counts(t)
    ocnt, omem = orc.dominance_counts_mt(t, nthreads=THREADS)
    assert np.array_equal(cnt, ocnt) and np.array_equal(mem, omem)


def test_config2_k7b_box_pruned_equals_pairwise(tmp_path):
    """K7b (Morton tiles, FULL / NONE / PARTIAL boxes; pareto.cu
    dominance_box_kernel) against the rank-sum pairwise kernel
    (SAIR_DOM_PAIRWISE=1, a child process: the switch is read once) at 1M
    tuples: uniform and anti-correlated K = 3, correlated and grid K = 4
    (grid: long runs of equal vectors -- the duplicate rule)."""
    import subprocess
    import sys
    T = 1 << 20
    cases = [(3, "uniform"), (3, "anti"), (4, "corr"), (4, "grid")]
    code = ("import sys, numpy as np; sys.path.insert(0, %r)\n"
            "import paper_2601_22397_b200 as sair\nfrom paper_2601_22397_b200 import synth\n"
            "for K, dist in %r:\n"
            "    c, m = sair.dominance_counts(synth.tuples(3100 + K, %d, K, dist))\n"
            "    np.save(%r + f'/c{K}{dist}.npy', c); np.save(%r + f'/m{K}{dist}.npy', m)\n"
            % (str(ROOT), cases, T, str(tmp_path), str(tmp_path)))
    env = dict(os.environ, SAIR_DOM_PAIRWISE="1")
    subprocess.run([sys.executable, "-c", code], env=env, check=True, timeout=600)
    for K, dist in cases:
        c, m = sair.dominance_counts(synth.tuples(3100 + K, T, K, dist))
        assert np.array_equal(c, np.load(tmp_path / f"c{K}{dist}.npy")), (K, dist)
        assert np.array_equal(m, np.load(tmp_path / f"m{K}{dist}.npy")), (K, dist)
        _, mo = sair.dominance_counts(synth.tuples(3100 + K, T, K, dist), counts=False)
        assert np.array_equal(mo, m), (K, dist)


@pytest.mark.parametrize("K,dist", [(3, "uniform"), (4, "grid")])
def test_k7b_parts_combine_by_a_sum(orc, K, dist):
    """K7b split into parts (sair_dominance_counts_part: an equal share of the
    j-tiles each, the multi-GPU split): the parts' counts sum to the whole and
    their memberships OR to it; the whole equals the oracle."""
    t = synth.tuples(4100 + K, 50000, K, dist)
    cnt, mem = sair.dominance_counts(t)
    ocnt, omem = orc.dominance_counts_mt(t, nthreads=THREADS)
    assert np.array_equal(cnt, ocnt) and np.array_equal(mem, omem)
    parts = [sair.dominance_counts(t, part=p, nparts=3) for p in range(3)]
    assert np.array_equal(sum(p[0].astype(np.int64) for p in parts), cnt.astype(np.int64))
    assert np.array_equal(parts[0][1] | parts[1][1] | parts[2][1], mem)


def test_config2_windowed_scoring_of_every_tuple(orc):
    """K8 on a frontier beyond shared memory (anti-correlated 4M tuples, F ~
    17.6k): the bucketed windowed path (T >= 64k) scores every tuple exactly
    as the direct kernel does (chunks below 64k) and as the oracle (sample)."""
    T = 4 * 1024 * 1024
    pts = synth.tuples(2031, T, 2, "anti")
    f = sair.ParetoFrontier(1.0, 1.0)
    F = f.insert_batch(pts)
    assert F > 6144
    got, dom = f.score_batch(pts)
    ref_r = np.empty(T)
    ref_d = np.empty(T, bool)
    for s in range(0, T, 60000):
        r, d = f.score_batch(pts[s:s + 60000])
        ref_r[s:s + 60000], ref_d[s:s + 60000] = r, d
    assert np.array_equal(got, ref_r) and np.array_equal(dom, ref_d)
    fl, fc = orc.frontier_sorted(pts)
    probe = np.arange(0, T, 997)
    assert near(got[probe], orc.pareto_reward_batch(fl, fc, pts[probe]))
