"""Prefix-sequential replay: sair_compute_reward_replay
against the reference's own sequential loop (scalelab_cli.cpp:118-147:
compute_reward against the current frontier, then update() unless guarded),
run with the reference compiled in place."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2601_22397_b200 as sair  # noqa: E402
from oracle.oracle import RefFrontier, ref_compute_reward  # noqa: E402

CFG = sair.RewardConfig()
CFGV = (CFG.t_sla_ms, CFG.l_baseline_ms, CFG.c_budget, CFG.w_latency, CFG.w_cost,
        CFG.w_proactive, CFG.r_max)
L_MAX, C_MAX = 2000.0, 10.0


def _rounds(rng, T, kind):
    lb = rng.uniform(100, 2500, T)
    if kind == "anti":   # every point on the frontier: F grows with T
        la = rng.uniform(50, 1900, T)
        ca = (1.0 - la / L_MAX) * C_MAX + rng.uniform(-1e-3, 1e-3, T)
    elif kind == "grid":  # ties and exact duplicates
        la = np.round(rng.uniform(0, 2400, T) / 250) * 250
        ca = np.round(rng.uniform(0, 12, T) * 2) / 2
    else:
        la = rng.uniform(50, 2600, T)   # some clamp at l_max
        ca = rng.uniform(0.5, 11, T)
    cb = rng.uniform(0.5, 10, T)
    inputs = np.stack([lb, la, cb, ca], 1)
    deltas = rng.integers(-3, 4, size=(T, 3, 4)).astype(np.int32) * [1, 100, 64, 1]
    update = (rng.uniform(size=T) < 0.85).astype(np.uint8)
    return inputs, deltas.astype(np.int32), update


def _reference(ref, inputs, deltas, update, seed_pts=()):
    rf = RefFrontier(ref, L_MAX, C_MAX)
    for l, c in seed_pts:
        rf.update(l, c)
    out = []
    for t in range(len(inputs)):
        out.append(ref_compute_reward(ref, inputs[t], deltas[t], rf, CFGV))
        if update[t]:
            rf.update(inputs[t, 1], inputs[t, 3])
    return np.array(out), rf.points()


@pytest.mark.parametrize("kind,T", [("uniform", 5000), ("grid", 4000), ("anti", 3000),
                                    ("uniform", 40)])
def test_replay_matches_sequential_reference(ref, kind, T):
    rng = np.random.default_rng(T + len(kind))
    inputs, deltas, update = _rounds(rng, T, kind)
    seed = [(300.0, 6.0), (900.0, 2.0)]
    want, (wl, wc) = _reference(ref, inputs, deltas, update, seed)
    f = sair.ParetoFrontier(L_MAX, C_MAX)
    for l, c in seed:
        f.update(l, c)
    got = sair.compute_reward_replay(inputs, deltas, update, f, CFG)
    gl, gc = f.points_array()
    assert np.array_equal(gl, wl) and np.array_equal(gc, wc)
    # every term except pareto is per-row arithmetic: bit-exact
    assert np.array_equal(got[:, [0, 1, 2, 3, 6]], want[:, [0, 1, 2, 3, 6]])
    if kind != "anti":
        assert np.array_equal(got, want)   # frontiers <= 64 points: the reference's sequence
    else:
        # > 64 points: the local exclusive area instead of HV(F u p) - HV(F)
        assert np.all(np.abs(got[:, 4] - want[:, 4]) <= 1e-12)
        assert np.all(np.abs(got[:, 5] - want[:, 5]) <= 1e-12)


def test_frontier_set_matches_independent_reference_frontiers(ref):
    """config 5's per-pipeline frontiers: P frontiers stepped together for
    several decision rounds against P reference frontiers stepped one by one."""
    rng = np.random.default_rng(11)
    P, rounds = 300, 12
    fs = sair.FrontierSet(P, L_MAX, C_MAX)
    rfs = [RefFrontier(ref, L_MAX, C_MAX) for _ in range(P)]
    for r in range(rounds):
        inputs, deltas, update = _rounds(rng, P, "grid" if r % 3 == 0 else "uniform")
        got = fs.step(inputs, deltas, update, CFG)
        for p in range(P):
            want = ref_compute_reward(ref, inputs[p], deltas[p], rfs[p], CFGV)
            assert np.array_equal(got[p], want), (r, p)
            if update[p]:
                rfs[p].update(inputs[p, 1], inputs[p, 3])
    for p in range(0, P, 7):
        gl, gc = fs.points_array(p)
        wl, wc = rfs[p].points()
        assert np.array_equal(gl, wl) and np.array_equal(gc, wc)
        assert fs.hypervolume(p) == rfs[p].hypervolume()
