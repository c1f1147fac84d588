"""Parity of the wide tensor-core pass (select_wide.cu, K4: 32-128 queries per
store pass) with the oracle, and with the
8-query pass it replaces for large batches.  Same bars as test_gpu_parity.py:
indices bit-exact, scores within 1e-12 relative (the contract is 1e-5)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2601_22397_b200 as sair  # noqa: E402
from paper_2601_22397_b200 import ExperienceBuffer, SelectionConfig, synth  # noqa: E402


def near(got, want, rel):
    got, want = np.asarray(got, float), np.asarray(want, float)
    return np.all(np.abs(got - want) <= rel * np.maximum(1.0, np.abs(want)))


def synth_store(seed, n, d, clustered=False):
    db = ExperienceBuffer(0.0)
    db.store_synthetic(seed, n, d, clustered=clustered)
    ctx = synth.contexts(seed, 0, n, d, clustered=clustered)
    return db, ctx, synth.rewards(seed, 0, n), synth.rounds(0, n)


class no_wide:
    def __enter__(self):
        os.environ["SAIR_NO_WIDE"] = "1"

    def __exit__(self, *a):
        os.environ.pop("SAIR_NO_WIDE", None)


@pytest.mark.parametrize("n,d,nq,m,lam", [(70000, 64, 128, 32, 0.0), (66000, 64, 72, 16, 0.1),
                                          (70001, 23, 40, 8, 0.0), (100000, 32, 200, 32, 0.0),
                                          (66000, 8, 33, 8, 0.1)])
def test_wide_matches_oracle(orc, n, d, nq, m, lam):
    db, ctx, rew, rnd = synth_store(n + d, n, d)
    sigma = db.effective_sigma()
    xq = synth.queries(n + d + 1, nq, d)
    idx, sim, sc, cnt = db.select_batch(xq, SelectionConfig(m=m, lambda_div=lam))
    st = db.last_stats()
    assert st["tensor_core"] == 2, st
    if lam == 0.0:
        assert st["certified"] == nq and st["exact_fallbacks"] == 0, st
    oi, osim, osc, ocnt = orc.select_batch(ctx, rew, rnd, xq, m, lam, sigma)
    assert np.array_equal(cnt, ocnt)
    assert np.array_equal(idx, oi)
    assert near(sc, osc, 1e-12) and near(sim, osim, 1e-12)


def test_wide_equals_eight_query_pass_with_veto():
    n, d, nq = 80000, 64, 96
    db, ctx, rew, rnd = synth_store(5, n, d, clustered=True)
    xq = synth.queries(6, nq, d, clustered=True)
    cfg = SelectionConfig(m=32, lambda_div=0.0)
    wide = db.select_batch(xq, cfg, nearest=True)
    assert db.last_stats()["tensor_core"] == 2
    with no_wide():
        narrow = db.select_batch(xq, cfg, nearest=True)
        assert db.last_stats()["tensor_core"] == 1
    for a, b in zip(wide, narrow):
        assert np.array_equal(a, b)


def test_wide_ties_and_duplicates(orc):
    # a store of 64 distinct rows repeated: every score ties 500 ways, the
    # reference's (round asc, index asc) tie-break decides
    n, d, nq = 96000, 16, 64
    base = synth.contexts(9, 0, 64, d)
    ctx = np.tile(base, (n // 64, 1))
    rew = np.tile(synth.rewards(9, 0, 64), n // 64)
    rnd = (np.arange(n, dtype=np.int32) * 7919) % n
    db = ExperienceBuffer(0.0)
    db.store_many(ctx, rew, rnd)
    sigma = db.effective_sigma()
    xq = synth.queries(10, nq, d)
    idx, sim, sc, cnt = db.select_batch(xq, SelectionConfig(m=16, lambda_div=0.0))
    assert db.last_stats()["tensor_core"] == 2
    oi, osim, osc, _ = orc.select_batch(ctx, rew, rnd, xq, 16, 0.0, sigma)
    assert np.array_equal(idx, oi)
    assert near(sc, osc, 1e-12)


def test_wide_small_and_ragged_stores(orc):
    # below 64k records the batch goes through the 8-query pass; ragged page
    # counts above it through the wide one
    for n in (1, 31, 129, 4097, 65537, 65536 + 127):
        d = 12
        db, ctx, rew, rnd = synth_store(n, n, d)
        sigma = db.effective_sigma()
        xq = synth.queries(n + 3, 48, d)
        idx, sim, sc, cnt = db.select_batch(xq, SelectionConfig(m=8, lambda_div=0.0))
        oi, osim, osc, ocnt = orc.select_batch(ctx, rew, rnd, xq, 8, 0.0, sigma)
        assert np.array_equal(cnt, ocnt)
        for q in range(len(xq)):
            k = int(cnt[q])
            assert np.array_equal(idx[q, :k], oi[q, :k])
            assert near(sc[q, :k], osc[q, :k], 1e-12)


def test_config2_1m_256_queries_against_exact():
    """configs[1]: 1M x 64, 256 queries, k = 32 -- certified, and equal to the
    full fp64 pass for a sample of the queries."""
    n, d = 1 << 20, 64
    db = ExperienceBuffer(0.0)
    db.store_synthetic(2026, n, d)
    xq = synth.queries(2027, 256, d)
    cfg = SelectionConfig(m=32, lambda_div=0.0)
    fast = db.select_batch(xq, cfg, nearest=True)
    st = db.last_stats()
    assert st["tensor_core"] == 2 and st["certified"] == 256, st
    pick = [0, 77, 128, 255]
    exact = db.select_batch(xq[pick], SelectionConfig(m=32, lambda_div=0.0,
                                                      mode=sair.SELECT_EXACT), nearest=True)
    for a, b in zip(fast, exact):
        assert np.array_equal(np.asarray(a)[pick], b)


def test_wide_after_high_residual_append(orc):
    """Config 5's store after a decision step: a batch of outcomes far from the
    store's mean appended at the end.  The sample's highest-residual pages
    put the start threshold next to the K'-th key, so every query certifies in
    the first pass (no retry); results equal the oracle's, before and after a
    second append (the hot-page list is rebuilt when the store grows)."""
    n, d, nq, m = 90000, 32, 128, 16
    db, ctx, rew, rnd = synth_store(31, n, d)
    rng = np.random.default_rng(3)
    cfg = SelectionConfig(m=m, lambda_div=0.0)
    for step in range(2):
        k = 1500
        c = synth.queries(40 + step, k, d)
        r = rng.uniform(3, 6, k)  # above the r_min gate, far above the mean
        db.store_many(c, r, np.full(k, 7 + step, np.int32))
        ctx = np.concatenate([ctx, c])
        rew = np.concatenate([rew, r])
        rnd = np.concatenate([rnd, np.full(k, 7 + step, np.int32)])
        xq = synth.queries(50 + step, nq, d)
        for _ in range(2):  # the second call reuses the hot-page list
            idx, sim, sc, cnt, _, _ = db.select_batch(xq, cfg, nearest=True)
            st = db.last_stats()
            assert st["tensor_core"] == 2 and st["certified"] == nq, st
            assert st["retried"] == 0 and st["exact_fallbacks"] == 0, st
        oi, osim, osc, ocnt = orc.select_batch(ctx, rew, rnd, xq, m, 0.0, db.effective_sigma())
        assert np.array_equal(cnt, ocnt) and np.array_equal(idx, oi)
        assert near(sc, osc, 1e-12) and near(sim, osim, 1e-12)


@pytest.mark.parametrize("cap", [1, 4])
def test_wide_full_lists_retry_and_fallback(orc, cap):
    """Per-CTA lists far too small (SAIR_WIDE_CAP): lists overflow, the
    dropped-key bound leaves queries uncertified, the threshold retry pass
    (start thresholds uploaded with the group constants) and the exact
    fallback finish them -- the answer is still the oracle's."""
    n, d, nq, m = 70000, 32, 160, 16
    db, ctx, rew, rnd = synth_store(n + 7, n, d)
    sigma = db.effective_sigma()
    xq = synth.queries(n + 8, nq, d)
    os.environ["SAIR_WIDE_CAP"] = str(cap)
    try:
        idx, sim, sc, cnt = db.select_batch(xq, SelectionConfig(m=m, lambda_div=0.0))
        st = db.last_stats()
    finally:
        os.environ.pop("SAIR_WIDE_CAP", None)
    assert st["tensor_core"] == 2 and st["retried"] > 0, st
    oi, osim, osc, ocnt = orc.select_batch(ctx, rew, rnd, xq, m, 0.0, sigma)
    assert np.array_equal(cnt, ocnt)
    assert np.array_equal(idx, oi)
    assert near(sc, osc, 1e-12) and near(sim, osim, 1e-12)
    # and the next call (default capacity) is unaffected
    idx2, _, sc2, _ = db.select_batch(xq, SelectionConfig(m=m, lambda_div=0.0))
    assert db.last_stats()["retried"] == 0
    assert np.array_equal(idx2, oi) and near(sc2, osc, 1e-12)


def test_wide_32_and_64_query_kernels_many_pages_per_cta():
    """The 32- and 64-query wide kernels (5 shared page stages, 8 TMEM stages)
    over 4M records (~220 pages per CTA: the rings wrap many times) certify
    every query and give the 8-query pass's answer."""
    db = ExperienceBuffer(0.0)
    db.store_synthetic(4242, 1 << 22, 64)
    cfg = SelectionConfig(m=32, lambda_div=0.0)
    for nq, qb in ((40, 32), (100, 64)):
        xq = synth.queries(4243 + nq, nq, 64)
        idx, sim, sc, cnt = db.select_batch(xq, cfg)
        st = db.last_stats()
        assert st["qb"] == qb and st["tensor_core"] == 2, st
        assert st["certified"] == nq and st["exact_fallbacks"] == 0, st
        with no_wide():
            idx8, sim8, sc8, cnt8 = db.select_batch(xq, cfg)
        assert db.last_stats()["tensor_core"] == 1
        assert np.array_equal(cnt, cnt8) and np.array_equal(idx, idx8)
        assert near(sc, sc8, 1e-12) and near(sim, sim8, 1e-12)
