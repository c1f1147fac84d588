"""sair_decision_step: one decision of harness.cpp:197-261
replayed on the device with one host synchronisation must equal the four
calls it replaces -- select + veto scan, compute_reward, frontier.update,
store() -- bit for bit, on twin stores and frontiers, through rejected rewards,
updates that do not insert, the small-store path (deferred copy-out) and the
filter path, and an empty store (store() fixes the dimension)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2601_22397_b200 as sair  # noqa: E402
from paper_2601_22397_b200 import decision, synth  # noqa: E402


def twins(n, d, seed):
    a, b = sair.ExperienceBuffer(0.0), sair.ExperienceBuffer(0.0)
    if n:
        a.store_synthetic(seed, n, d)
        b.store_synthetic(seed, n, d)
    return a, b, sair.ParetoFrontier(2000.0, 10.0), sair.ParetoFrontier(2000.0, 10.0)


def run(n, d, cfg, steps, seed):
    ba, bb, fa, fb = twins(n, d, seed)
    rng = np.random.default_rng(seed)
    rc = sair.RewardConfig()
    for s in range(steps):
        x = synth.queries(seed + 100 + s, 1, d)[0]
        # outcomes on both sides of the r_min gate and of the frontier
        inp = sair.RewardInputs(rng.uniform(200, 1500), rng.uniform(200, 2600),
                                rng.uniform(0.5, 9), rng.uniform(0.5, 11))
        act = sair.ScalingAction([sair.StageDelta(*map(int, r))
                                  for r in rng.integers(-2, 3, size=(3, 4))])
        upd = bool(rng.uniform() < 0.8)
        got = decision.replay_step(ba, fa, x, cfg, inp, act, rc, update=upd, round=500 + s)
        want = bb.select_batch(x[None, :], cfg, nearest=True) if bb.size() else None
        r = sair.compute_reward(inp, act, fb, rc)
        ins = fb.update(inp.l_after_ms, inp.c_after)[0] if upd else False
        sto = bb.store(sair.Experience(list(x), act, r.total, 500 + s))
        if want is not None:
            k = int(want[3][0])
            assert np.array_equal(got.idx, want[0][0, :k])
            assert np.array_equal(got.sim, want[1][0, :k])
            assert np.array_equal(got.score, want[2][0, :k])
            assert got.nn_idx == want[4][0] and got.nn_sim == want[5][0]
        else:
            assert len(got.idx) == 0
        assert got.reward == r
        assert got.inserted == ins and got.stored == sto
        assert ba.size() == bb.size() and ba.rejected() == bb.rejected()
        assert fa.size() == fb.size() and fa.hypervolume() == fb.hypervolume()
        for u, v in zip(fa.points_array(), fb.points_array()):
            assert np.array_equal(u, v)
    for u, v in zip(ba.export(), bb.export()):
        assert np.array_equal(u, v)
    assert ba.effective_sigma() == bb.effective_sigma()
    return ba


def test_decision_step_small_store_path():
    # config 1's shape: 10k x 32, m = 8, lambda 0.1 (the one-launch small select)
    run(10000, 32, sair.SelectionConfig(m=8, lambda_div=0.1), 70, 1)


def test_decision_step_filter_path_and_empty_store():
    run(20000, 64, sair.SelectionConfig(m=16, lambda_div=0.0), 12, 2)
    run(0, 8, sair.SelectionConfig(m=4, lambda_div=0.1), 20, 3)
