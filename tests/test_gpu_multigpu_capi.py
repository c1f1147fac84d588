"""The C ABI's one-process multi-GPU buffer and frontier (sharded.cpp, SURVEY.md
8(e)): select() over shards equals select() over one buffer holding the same
records (lambda 0: the all-gathered per-shard candidates merged; lambda 0.1:
the distributed greedy), bit for bit.  One B200 per box: the shards share
device 0 (device-to-device copies), and a one-device communicator drives
the NCCL transport (SAIR_COMM_NCCL=1)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2601_22397_b200 import ExperienceBuffer, ParetoFrontier, SelectionConfig, synth  # noqa: E402
from paper_2601_22397_b200.sharded import (DeviceComm, MultiGPUExperienceBuffer,  # noqa: E402
                                           frontier_insert_batch_multi)


def same(a, b):
    for x, y in zip(a, b):
        assert np.array_equal(np.asarray(x), np.asarray(y))


@pytest.mark.parametrize("shards,n,d,nq,lam", [(3, 300000, 64, 256, 0.0), (2, 150000, 32, 40, 0.0),
                                               (3, 90000, 23, 12, 0.1), (4, 5000, 16, 9, 0.1)])
def test_sharded_select_equals_one_buffer(shards, n, d, nq, lam):
    comm = DeviceComm([0] * shards)
    assert comm.info() == (shards, False)
    mg = MultiGPUExperienceBuffer(comm, 0.0, capacity=n)
    mg.store_synthetic(n + d, n, d)
    one = ExperienceBuffer(0.0)
    one.store_synthetic(n + d, n, d)
    tot, rej, per = mg.size()
    assert tot == n and rej == 0 and per.sum() == n and (per > 0).all()
    assert mg.effective_sigma() == one.effective_sigma()
    xq = synth.queries(n + d + 1, nq, d)
    cfg = SelectionConfig(m=16, lambda_div=lam)
    same(mg.select_batch(xq, cfg), one.select_batch(xq, cfg))


def test_nccl_transport_one_device():
    os.environ["SAIR_COMM_NCCL"] = "1"
    try:
        comm = DeviceComm([0])
    finally:
        os.environ.pop("SAIR_COMM_NCCL", None)
    assert comm.info() == (1, True)
    n, d = 200000, 64
    mg = MultiGPUExperienceBuffer(comm, 0.0, capacity=n)
    mg.store_synthetic(5, n, d)
    one = ExperienceBuffer(0.0)
    one.store_synthetic(5, n, d)
    xq = synth.queries(6, 64, d)
    cfg = SelectionConfig(m=32, lambda_div=0.0)
    same(mg.select_batch(xq, cfg), one.select_batch(xq, cfg))


def test_appends_gate_quota_overflow_and_sigma_refresh():
    """store() semantics through the shards: rejected rows only count, shards
    fill in order (the last takes the overflow), the sigma cache refreshes
    every 50 stored records like one buffer's."""
    d = 12
    rng = np.random.default_rng(3)
    comm = DeviceComm([0, 0, 0])
    mg = MultiGPUExperienceBuffer(comm, r_min=0.2, capacity=900)
    one = ExperienceBuffer(0.2)
    cfg = SelectionConfig(m=8, lambda_div=0.1)
    rnd0 = 0
    for batch in (400, 7, 333, 40, 600):
        x = rng.normal(size=(batch, d)) * 3.0
        r = rng.uniform(-0.5, 1.5, size=batch)
        rd = np.arange(rnd0, rnd0 + batch, dtype=np.int32)
        rnd0 += batch
        assert mg.store_many(x, r, rd) == one.store_many(x, r, rd)
        assert mg.effective_sigma() == one.effective_sigma()
        xq = rng.normal(size=(5, d)) * 3.0
        same(mg.select_batch(xq, cfg), one.select_batch(xq, cfg)[:4])
    tot, rej, per = mg.size()
    assert tot == one.size() and rej == one.rejected()
    assert per[0] == 300 and per[1] == 300 and per[2] == tot - 600


def test_sharded_frontier_insert():
    for dist in ("uniform", "anti", "grid"):
        pts = synth.tuples(31, 300000, 2, dist)
        f1 = ParetoFrontier(1.0, 1.0)
        F1 = f1.insert_batch(pts)
        f2 = ParetoFrontier(1.0, 1.0)
        F2 = frontier_insert_batch_multi(DeviceComm([0, 0, 0, 0]), f2, pts)
        assert F1 == F2
        same(f1.points_array(), f2.points_array())
