"""Persistence of the device store in the reference's JSONL format (SURVEY.md
8(f) row 3; experience.cpp:232-271): sair_store_load_jsonl / persist_jsonl
against the reference's own load() / persist() compiled in place."""
import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2601_22397_b200 as sair  # noqa: E402
from paper_2601_22397_b200 import ExperienceBuffer, SelectionConfig, synth  # noqa: E402
from oracle.oracle import RefBuffer  # noqa: E402


def _lines(rng, n, d):
    out = []
    for i in range(n):
        ctx = list(rng.normal(size=d) * rng.uniform(0.1, 1e3))
        act = [{"cpu_millicores": int(rng.integers(-500, 500)), "memory_mb": 0,
                "rate_ratio_tenths": 0, "replicas": int(rng.integers(-2, 3))}]
        out.append(json.dumps({"action": act, "context": ctx, "reward": float(rng.normal()),
                               "round": i, "source": "llm"}))
    return out


def test_load_matches_reference_load(ref, tmp_path):
    rng = np.random.default_rng(3)
    d = 9
    lines = _lines(rng, 4000, d)
    lines[17] = "{not json"                                  # corrupt
    lines[99] = json.dumps({"context": [1.0] * d, "reward": 0.5})  # missing keys: corrupt
    lines[500] = ""                                          # skipped
    bad_action = json.loads(lines[700])
    bad_action["action"] = [{"replicas": "x"}]
    lines[700] = json.dumps(bad_action)                      # wrong type: corrupt
    p = tmp_path / "buf.jsonl"
    p.write_text("\n".join(lines))                           # no trailing newline
    rb, rbad = RefBuffer.load(ref, p, 0.1)
    db, dbad = ExperienceBuffer.load(p, 0.1)
    assert dbad == rbad == 3
    assert db.size() == rb.size() and db.rejected() == rb.rejected()
    ctx, rw, rd = db.export()
    for i in range(0, db.size(), 97):
        c, r, k = rb.get(i, d)
        assert np.array_equal(ctx[i], c) and rw[i] == r and rd[i] == k
    assert db.effective_sigma() == rb.effective_sigma(0.0)
    x = rng.normal(size=d)
    r_round, _, r_score = rb.select(x, 8, 0.1, 0.0)
    idx, sim, sc, cnt = db.select_batch(x[None], SelectionConfig(m=8, lambda_div=0.1))
    assert list(rd[idx[0, :cnt[0]]]) == list(r_round)


def test_dimension_change_and_missing_file(tmp_path):
    p = tmp_path / "bad.jsonl"
    p.write_text(json.dumps({"action": [], "context": [1.0, 2.0], "reward": 1.0, "round": 0,
                             "source": "s"}) + "\n" +
                 json.dumps({"action": [], "context": [1.0, 2.0, 3.0], "reward": -1.0,
                             "round": 1, "source": "s"}) + "\n" +   # rejected: dim ignored
                 json.dumps({"action": [], "context": [1.0], "reward": 1.0, "round": 2,
                             "source": "s"}) + "\n")
    with pytest.raises(sair.InvalidArgument):
        ExperienceBuffer.load(p, 0.0)
    with pytest.raises(sair.SairError):
        ExperienceBuffer.load(tmp_path / "missing.jsonl", 0.0)


def test_persist_round_trip_through_the_reference(ref, tmp_path):
    n, d = 20000, 16
    db = ExperienceBuffer(0.0)
    db.store_synthetic(5, n, d)
    p = tmp_path / "out.jsonl"
    with pytest.raises(sair.LogicError):   # bulk rows: no source/action to write
        db.persist(p)
    db.persist(p, lossy=True)
    rb, bad = RefBuffer.load(ref, p, 0.0)
    assert bad == 0 and rb.size() == n
    q = tmp_path / "ref.jsonl"
    rb.persist(q)
    assert p.read_bytes() == q.read_bytes()   # the reference re-writes it byte for byte
    back, bad = ExperienceBuffer.load(q, 0.0)
    a, b = db.export(), back.export()
    assert bad == 0 and all(np.array_equal(u, v) for u, v in zip(a, b))
    assert np.array_equal(a[0][123], synth.contexts(5, 123, 1, d)[0])


def test_persist_from_the_mirror_keeps_source_and_action(ref, tmp_path):
    """Rows stored one by one keep the host mirror: persist() writes their
    source and action, byte-identical to the reference's own persist()."""
    rng = np.random.default_rng(9)
    db = ExperienceBuffer(0.0)
    for i in range(40):
        act = sair.ScalingAction([sair.StageDelta(int(rng.integers(-2, 3)), int(rng.integers(-500, 500)),
                                                  int(rng.integers(-64, 64)), int(rng.integers(-3, 4)))
                                  for _ in range(3)])
        db.store(sair.Experience(list(rng.normal(size=23) * rng.uniform(0.1, 1e3)), act,
                                 float(rng.normal()), i, ["llm", "mock", "explore"][i % 3]))
    p = tmp_path / "mirror.jsonl"
    db.persist(p)
    lines = p.read_text().splitlines()
    assert len(lines) == db.size() and all(json.loads(x)["action"] for x in lines)
    rb, bad = RefBuffer.load(ref, p, 0.0)
    assert bad == 0 and rb.size() == db.size()
    q = tmp_path / "ref.jsonl"
    rb.persist(q)
    assert p.read_bytes() == q.read_bytes()
