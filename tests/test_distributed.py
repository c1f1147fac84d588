"""The multi-GPU (record-sharded) path, world_size 2.

CPU (gloo): the exchange protocol of paper_2601_22397_b200/sharded.py --
shard ranges, rank-ordered statistics combination, the sigma subsample
gather, and the candidate merge rule -- with the oracle's shard restatement
(orc_select_shard) standing in for each rank's device select; the merged
answer must equal the oracle's single-buffer select bit for bit.

GPU: two ranks sharing cuda:0 run the real ShardedExperienceBuffer (device
select per shard + device merge) against the single-store device answer.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2601_22397_b200 import synth
from paper_2601_22397_b200.sharded import combine_stats, moments, shard_range

N, D, M, SEED = 3000, 16, 12, 41


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _gather(arr):
    t = torch.from_numpy(np.ascontiguousarray(arr))
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [o.numpy() for o in out]


def merge_checker(parts, m):
    """The merge rule, restated in numpy (test-side checker): top-m by
    (score desc, round asc, global index asc), then (reward asc, round asc,
    pick order)."""
    rows = [r for p in parts for r in p]
    rows.sort(key=lambda r: (-r[0], r[2], r[3]))
    picks = rows[:m]
    order = sorted(range(len(picks)), key=lambda i: (picks[i][1], picks[i][2], i))
    return [picks[i] for i in order]


def _cpu_worker(rank, world, port, q):
    from oracle.oracle import COracle
    _init(rank, world, port)
    orc = COracle()
    lo, hi = shard_range(N, rank, world)
    ctx = synth.contexts(SEED, lo, hi - lo, D)
    rew = synth.rewards(SEED, lo, hi - lo)
    rnd = synth.rounds(lo, hi - lo)
    s, ss = orc.stats(ctx)
    mine = np.concatenate([s, ss, np.abs(ctx).max(0), [hi - lo, orc.lib.orc_reward_total(
        rew.ctypes.data_as(__import__("ctypes").POINTER(__import__("ctypes").c_double)), hi - lo),
        np.abs(rew).max()]])
    n, gs, gss, gxa, total, rabs = combine_stats(_gather(mine), D)
    # sigma over the buffer's subsample, rows from their owners
    stride = n / 512.0
    idx = np.array([int(k * stride) for k in range(512)]) if n > 512 else np.arange(n)
    owned = (idx >= lo) & (idx < hi)
    rows = np.zeros((len(idx), D + 1))
    rows[owned, 0] = 1
    rows[owned, 1:] = ctx[idx[owned] - lo]
    full = np.zeros((len(idx), D))
    for g in _gather(rows):
        full[g[:, 0] > 0] = g[g[:, 0] > 0, 1:]
    sigma = orc.sigma_rows(full, n, gs, gss)
    xq = synth.queries(SEED, 3, D)
    results = []
    for x in xq:
        li, lsim, lsc = orc.select_shard(ctx, rew, rnd, x, M, sigma, n, gs, gss, total)
        part = np.array([[lsc[j], rew[li[j]], rnd[li[j]], lo + li[j]] for j in range(len(li))])
        pad = np.full((M - len(part), 4), np.nan)
        parts = _gather(np.concatenate([part, pad]) if len(part) < M else part)
        merged = merge_checker([[tuple(r) for r in p if not np.isnan(r[0])] for p in parts], M)
        results.append([(r[3], r[0]) for r in merged])
    if rank == 0:
        q.put((n, gs, gss, total, sigma, results))
    dist.destroy_process_group()


def test_sharded_protocol_matches_single_buffer_cpu(orc):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cpu_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    n, gs, gss, total, sigma, results = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ctx_all = synth.contexts(SEED, 0, N, D)
    rew = synth.rewards(SEED, 0, N)
    rnd = synth.rounds(0, N)
    s, ss = orc.stats(ctx_all)
    assert n == N and np.array_equal(gs, s) and np.array_equal(gss, ss)
    assert total == orc.lib.orc_reward_total(
        rew.ctypes.data_as(__import__("ctypes").POINTER(__import__("ctypes").c_double)), N)
    assert sigma == orc.sigma_median(ctx_all)
    mean, sd = moments(n, gs, gss)
    assert np.array_equal(orc.standardize(n, s, ss, ctx_all[5]), (ctx_all[5] - mean) / sd)
    for x, got in zip(synth.queries(SEED, 3, D), results):
        idx, sim, sc = orc.select(ctx_all, rew, rnd, x, M, 0.0, sigma)
        assert [int(i) for i, _ in got] == list(idx)
        assert np.array_equal([v for _, v in got], sc)


def test_sharded_greedy_rules_cpu():
    """The host side of the sharded lambda > 0 select: the global winner rule
    (gain desc, round asc, global index asc; -inf = shard exhausted) and the
    curriculum order (reward asc, round asc, pick order), against a direct
    restatement on random parts with many ties."""
    from paper_2601_22397_b200.sharded import curriculum_order, global_winner
    rng = np.random.default_rng(4)
    R, nq = 5, 200
    parts = np.zeros((R, nq, 3))
    parts[:, :, 0] = rng.integers(0, 3, (R, nq)) / 4.0
    parts[rng.uniform(size=(R, nq)) < 0.1, 0] = -np.inf
    parts[:, :, 1] = rng.integers(0, 3, (R, nq))
    parts[:, :, 2] = rng.permutation(R * nq).reshape(R, nq)
    win = global_winner(parts)
    for q in range(nq):
        want = min(range(R), key=lambda r: (-parts[r, q, 0], parts[r, q, 1], parts[r, q, 2]))
        assert win[q] == want
    rew = rng.integers(0, 3, (12, nq)) / 2.0
    rnd = rng.integers(0, 3, (12, nq))
    order = curriculum_order(rew, rnd)
    for q in range(nq):
        assert list(order[q]) == sorted(range(12), key=lambda i: (rew[i, q], rnd[i, q], i))


def _gpu_worker(rank, world, port, q, nq=10, lam=0.0):
    from paper_2601_22397_b200 import SelectionConfig
    from paper_2601_22397_b200.sharded import ShardedExperienceBuffer
    _init(rank, world, port)
    buf = ShardedExperienceBuffer(dist, device=0)
    buf.store_synthetic(SEED, 200000, 32)
    xq = synth.queries(SEED, nq, 32)
    out = buf.select_batch(xq, SelectionConfig(m=32 if lam == 0.0 else 12, lambda_div=lam))
    if rank == 0:
        q.put((buf.sigma,) + tuple(out))
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("nq,lam", [(10, 0.0), (160, 0.0), (6, 0.1)])  # 8-query / wide / greedy
def test_sharded_select_on_device_matches_single_store(nq, lam):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2601_22397_b200 as sair
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, q, nq, lam))
             for r in range(world)]
    for p in procs:
        p.start()
    sigma, idx, sim, sc, cnt = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    one = sair.ExperienceBuffer(0.0)
    one.store_synthetic(SEED, 200000, 32)
    assert sigma == one.effective_sigma()
    i1, s1, c1, n1 = one.select_batch(synth.queries(SEED, nq, 32),
                                      sair.SelectionConfig(m=32 if lam == 0.0 else 12,
                                                           lambda_div=lam))
    assert np.array_equal(cnt, n1)
    assert np.array_equal(idx, i1)
    assert np.array_equal(sc, c1) and np.array_equal(sim, s1)


# ------------------------------------------------------------------ pareto --

T_P, K_P = 6000, 3


def _pareto_cpu_worker(rank, world, port, q):
    from oracle.oracle import COracle
    from paper_2601_22397_b200.sharded import all_gather_rows, combine_parts
    _init(rank, world, port)
    orc = COracle()
    lo, hi = shard_range(T_P, rank, world)
    pts = synth.tuples(SEED, T_P, 2, "grid")[lo:hi]
    # each rank's device frontier (K6) is restated by the oracle
    fl, fc, _ = orc.frontier_from_points(pts)
    parts = all_gather_rows(dist, np.stack([fl, fc], axis=1), "cpu")
    gl, gc, _ = orc.frontier_from_points(np.concatenate(parts))
    # dominance counts: all-gather, this rank's part (a stripe here), sum
    tk = synth.tuples(SEED + 1, T_P, K_P, "grid")[lo:hi]
    allt = np.concatenate(all_gather_rows(dist, tk, "cpu"))
    cnt, mem = orc.dominance_counts(allt)
    mine = np.arange(len(allt)) % world == rank
    cnt, mem = combine_parts(dist, np.where(mine, cnt, 0), np.where(mine, mem, False), "cpu")
    if rank == 0:
        q.put((gl, gc, cnt, mem))
    dist.destroy_process_group()


def test_sharded_pareto_protocol_cpu(orc):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pareto_cpu_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    gl, gc, cnt, mem = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    fl, fc, _ = orc.frontier_from_points(synth.tuples(SEED, T_P, 2, "grid"))
    assert np.array_equal(gl, fl) and np.array_equal(gc, fc)
    c1, m1 = orc.dominance_counts(synth.tuples(SEED + 1, T_P, K_P, "grid"))
    assert np.array_equal(cnt, c1) and np.array_equal(mem, m1)


def _pareto_gpu_worker(rank, world, port, q):
    from paper_2601_22397_b200.sharded import ShardedParetoFrontier, sharded_dominance_counts
    _init(rank, world, port)
    T = 200000
    lo, hi = shard_range(T, rank, world)
    pts = synth.tuples(SEED, T, 2, "grid")[lo:hi]
    f = ShardedParetoFrontier(dist, 0, 1.0, 1.0)
    f.insert_batch(pts)
    probe = synth.tuples(SEED + 2, 5000, 2, "uniform")
    rw, dom = f.score_batch(probe)
    tk = synth.tuples(SEED + 1, 100000, 4, "grid")
    klo, khi = shard_range(len(tk), rank, world)
    cnt, mem, nf = sharded_dominance_counts(dist, tk[klo:khi], 0)
    parts = [None] * world
    dist.all_gather_object(parts, (cnt, mem))
    if rank == 0:
        l, c = f.points_array()
        q.put((l, c, rw, dom, np.concatenate([p[0] for p in parts]),
               np.concatenate([p[1] for p in parts]), nf))
    dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_pareto_on_device_matches_single():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2601_22397_b200 as sair
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pareto_gpu_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    l, c, rw, dom, cnt, mem, nf = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    one = sair.ParetoFrontier(1.0, 1.0)
    one.insert_batch(synth.tuples(SEED, 200000, 2, "grid"))
    l1, c1 = one.points_array()
    assert np.array_equal(l, l1) and np.array_equal(c, c1)
    r1, d1 = one.score_batch(synth.tuples(SEED + 2, 5000, 2, "uniform"))
    assert np.array_equal(rw, r1) and np.array_equal(dom, d1)
    cf, mf = sair.dominance_counts(synth.tuples(SEED + 1, 100000, 4, "grid"))
    assert np.array_equal(cnt, cf) and np.array_equal(mem, mf) and nf == int(mf.sum())
