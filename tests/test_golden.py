"""Committed golden fixtures from the reference itself (tests/golden/make_golden.py
runs oracle/_ref).  The oracle restatement must reproduce them bit for bit;
the device path (gpu) must reproduce indices exactly and values within 1e-12
relative (1e-5 is the contract; exp() may differ by an ulp)."""
import json
from pathlib import Path

import numpy as np
import pytest

G = Path(__file__).resolve().parent / "golden"
RET = json.loads((G / "retrieval.json").read_text())
PAR = json.loads((G / "pareto.json").read_text())
REW = json.loads((G / "reward.json").read_text())


def _accepted(case):
    ctx = np.array(case["context"])
    rew = np.array(case["reward"])
    rnd = np.array(case["round"], np.int32)
    acc = np.array(case["accepted"], bool)
    return ctx[acc], rew[acc], rnd[acc]


@pytest.mark.parametrize("case", RET, ids=[c["name"] for c in RET])
def test_oracle_reproduces_reference_retrieval(orc, case):
    ctx, rew, rnd = _accepted(case)
    assert len(ctx) + case["rejected"] == len(case["context"])
    sigma = case["sigma_sim"] if case["sigma_sim"] > 0 else (orc.sigma_median(ctx) if len(ctx) >= 2 else 1.0)
    assert sigma == case["sigma"]
    for x, want in zip(case["queries"], case["select"]):
        idx, sim, sc = orc.select(ctx, rew, rnd, x, case["m"], case["lambda_div"], sigma)
        assert rnd[idx].tolist() == want["rounds"]
        assert sim.tolist() == want["sim"] and sc.tolist() == want["score"]


def test_oracle_reproduces_reference_pareto(orc):
    for case in PAR:
        fl, fc, ins = orc.frontier_from_points(case["points"])
        assert fl.tolist() == case["frontier_l"] and fc.tolist() == case["frontier_c"]
        assert ins.tolist() == case["inserted"]
        assert orc.hypervolume(fl, fc) == case["hypervolume"]
        assert orc.pareto_reward_batch(fl, fc, case["probes"]).tolist() == case["reward"]


def test_oracle_reproduces_reference_reward(orc):
    for case in REW:
        fl, fc = np.zeros(8), np.zeros(8)
        F = 0
        pts = []
        for l_ms, c in case["updates"]:
            l, cc = min(l_ms / 2000.0, 1.0), min(c / 10.0, 1.0)
            pts.append((max(l, 0.0), max(cc, 0.0)))
        fl, fc, _ = orc.frontier_from_points(np.array(pts).reshape(-1, 2))
        cfg = list(case["config"])
        got = orc.compute_reward(case["inputs"], case["deltas"], fl, fc, 2000.0, 10.0, cfg)
        assert got.tolist() == case["breakdown"]


def _near(a, b, rel=1e-12):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return np.all(np.abs(a - b) <= rel * np.maximum(1.0, np.abs(b)))


@pytest.mark.gpu
@pytest.mark.parametrize("case", RET, ids=[c["name"] for c in RET])
def test_device_reproduces_reference_retrieval(case):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2601_22397_b200 as sair
    buf = sair.ExperienceBuffer(0.0)
    ctx = np.array(case["context"])
    acc = [buf.store(sair.Experience(list(ctx[i]), sair.ScalingAction(), case["reward"][i],
                                     case["round"][i])) for i in range(len(ctx))]
    assert acc == case["accepted"] and buf.rejected() == case["rejected"]
    cfg = sair.SelectionConfig(m=case["m"], lambda_div=case["lambda_div"],
                               sigma_sim=case["sigma_sim"])
    assert buf.effective_sigma(cfg) == case["sigma"]
    for x, want in zip(case["queries"], case["select"]):
        sel = buf.select(x, cfg)
        assert [s.experience.round for s in sel] == want["rounds"]
        assert _near([s.score for s in sel], want["score"])
        assert _near([s.similarity_to_current for s in sel], want["sim"])


@pytest.mark.gpu
def test_device_reproduces_reference_pareto_and_reward():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2601_22397_b200 as sair
    for case in PAR:
        f = sair.ParetoFrontier(1.0, 1.0)
        ins = [f.insert_normalized(p) for p in case["points"]]
        assert ins == case["inserted"]
        l, c = f.points_array()
        assert l.tolist() == case["frontier_l"] and c.tolist() == case["frontier_c"]
        assert f.hypervolume() == case["hypervolume"]
        r, dom = f.score_batch(case["probes"])
        assert r.tolist() == case["reward"] and dom.tolist() == case["dominated"]
        g = sair.ParetoFrontier(1.0, 1.0)
        g.insert_batch(case["points"])
        gl, gc = g.points_array()
        assert gl.tolist() == case["frontier_l"] and gc.tolist() == case["frontier_c"]
    for case in REW:
        f = sair.ParetoFrontier(2000.0, 10.0)
        for u in case["updates"]:
            f.update(*u)
        act = sair.ScalingAction([sair.StageDelta(*map(int, d)) for d in case["deltas"]])
        r = sair.compute_reward(sair.RewardInputs(*case["inputs"]), act, f,
                                sair.RewardConfig(*case["config"]))
        got = [r.latency, r.cost, r.sla, r.proactive, r.pareto, r.total, float(r.clipped)]
        assert got == case["breakdown"]
