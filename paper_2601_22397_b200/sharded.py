"""One logical ExperienceBuffer sharded over the GPUs of a node.

One process per GPU (torch.distributed, NCCL over NVLink; gloo for CPU tests).
Rank r owns the contiguous global slice [lo_r, hi_r) of the buffer.  Exactness
with the single-buffer reference (experience.cpp:151-205) rests on three
exchanges, each deterministic (rank order):

1. statistics -- every rank all-gathers the shards' running sums and combines
   them in rank order (sum_, sum_sq_, the reward total; experience.cpp:55-58,
   :229-230).  For the synthetic generator every partial sum is exact, so the
   combined sums are bit-identical to the sequential reference's;
2. sigma -- the buffer's 512-row subsample (experience.cpp:82-91) is gathered
   from the owning ranks and every rank computes the same median on its device;
3. candidates -- each shard's certified top-m (exact fp64 scores over the
   global statistics, each pick's reward and round) is all-gathered and merged
   by the device merge kernel (score desc, round asc, global index asc, then
   curriculum order).  With lambda_div == 0 the buffer's top-m is a subset of
   the union of the shards' top-m, so the merge is exact.

lambda_div > 0 (the greedy with diversity penalties): every step's arg-max is
taken across shards -- each rank scores its shard exactly (device, fp64, the
reference's rounding order) and reports its best untaken record per query
with everything the others need (gain, round, global index, similarity,
score, reward, standardized row); one all-gather per step, the global winner
by (gain desc, round asc, index asc), and every rank adds the winner's
similarity to its penalties (sair_store_greedy_begin / _next).

Pareto: outcome tuples are sharded the same way.  The
frontier of a union is the frontier of the union of the shards' frontiers, so
each rank reduces its tuples to a local frontier on its device (K6), the
local frontiers are all-gathered (a few hundred points) and every rank inserts
them, in rank order, into its copy of the global frontier; scoring is then
rank-local.  Dominance counts need every pair: the tuples are all-gathered and
each rank computes an equal-work part of the pairwise counts; the parts sum.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Tuple

import numpy as np

from . import SelectionConfig, _check, _dp, _f64, lib
from . import ExperienceBuffer, ParetoFrontier, dominance_counts


def shard_range(n_total: int, rank: int, world: int) -> Tuple[int, int]:
    return n_total * rank // world, n_total * (rank + 1) // world


def combine_stats(parts: List[np.ndarray], d: int):
    """Rank-ordered combination of per-shard (sum[d], sum_sq[d], xabs[d], n,
    total, rabs) vectors -> global (n, sum, sum_sq, xabs, total, rabs)."""
    n = 0
    s = np.zeros(d)
    ss = np.zeros(d)
    xa = np.zeros(d)
    total = 0.0
    rabs = 0.0
    for p in parts:  # rank order: deterministic on every rank
        s = s + p[:d]
        ss = ss + p[d:2 * d]
        xa = np.maximum(xa, p[2 * d:3 * d])
        n += int(p[3 * d])
        total = total + float(p[3 * d + 1])
        rabs = max(rabs, float(p[3 * d + 2]))
    return n, s, ss, xa, total, rabs


def moments(n: int, s: np.ndarray, ss: np.ndarray):
    """standardize()'s mean / sd, experience.cpp:68-74 (numpy fp64, same
    operation order -- used only to feed the device sigma kernel)."""
    mean = s / float(n)
    var = np.maximum(0.0, ss / float(n) - mean * mean)
    sd = np.sqrt(var)
    sd[sd < 1e-12] = 1.0
    return mean, sd


def sigma_sample_indices(n: int) -> np.ndarray:
    idx = np.zeros(512, np.int64)
    m = C.c_size_t()
    _check(lib().sair_sigma_sample_indices(n, idx.ctypes.data_as(C.POINTER(C.c_int64)),
                                           C.byref(m)))
    return idx[:m.value]


def _all_gather(dist, arr: np.ndarray, device) -> List[np.ndarray]:
    import torch
    t = torch.from_numpy(np.ascontiguousarray(arr))
    if dist.get_backend() == "nccl":
        t = t.to(device)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [o.cpu().numpy() for o in out]


class ShardedExperienceBuffer:
    """The rank-local shard of one logical ExperienceBuffer."""

    def __init__(self, dist, device: int, r_min: float = 0.0):
        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.device = device
        self.local = ExperienceBuffer(r_min, device=device)
        self.lo = self.hi = 0
        self.n_global = 0

    def store_synthetic(self, seed: int, n_total: int, dim: int, clustered: bool = False):
        """Every rank generates its slice of the same synthetic buffer."""
        self.lo, self.hi = shard_range(n_total, self.rank, self.world)
        _check(lib().sair_store_set_shard(self.local._h, self.lo))
        self.local.store_synthetic(seed, self.hi - self.lo, dim, clustered)
        self.finalize()

    def finalize(self):
        """Exchange statistics and sigma; switch the shard to global mode."""
        d = self.local.dim()
        s, ss, xa, sc = np.zeros(d), np.zeros(d), np.zeros(d), np.zeros(3)
        _check(lib().sair_store_local_stats(self.local._h, _dp(s), _dp(ss), _dp(xa), _dp(sc)))
        mine = np.concatenate([s, ss, xa, sc])
        dev = f"cuda:{self.device}"
        parts = _all_gather(self.dist, mine, dev)
        n, gs, gss, gxa, total, rabs = combine_stats(parts, d)
        self.n_global = n
        mean, sd = moments(n, gs, gss)
        # sigma over the buffer's subsample: rows come from their owners
        idx = sigma_sample_indices(n)
        rows = np.zeros((len(idx), d))
        owned = (idx >= self.lo) & (idx < self.hi)
        for j in np.nonzero(owned)[0]:
            rows[j] = self.local.get(int(idx[j] - self.lo))[0]
        gathered = _all_gather(self.dist, np.concatenate([owned.astype(np.float64)[:, None], rows],
                                                         axis=1), dev)
        full = np.zeros((len(idx), d))
        for g in gathered:
            own = g[:, 0] > 0
            full[own] = g[own, 1:]
        sigma = C.c_double(1.0)
        if len(idx) >= 2:
            _check(lib().sair_sigma_rows(_dp(np.ascontiguousarray(full)), len(idx), d, _dp(mean),
                                         _dp(sd), self.device, C.byref(sigma)))
        _check(lib().sair_store_set_global(self.local._h, n, _dp(gs), _dp(gss), _dp(gxa), total,
                                           rabs, sigma.value))
        self.sigma = sigma.value

    def select_local(self, queries, cfg: SelectionConfig):
        q = _f64(queries)
        if q.ndim == 1:
            q = q[None, :]
        nq, d = q.shape
        m = max(cfg.m, 1)
        idx = np.full((nq, m), -1, np.int64)
        sim, sc, rw = np.zeros((nq, m)), np.zeros((nq, m)), np.zeros((nq, m))
        rd = np.zeros((nq, m), np.int32)
        cnt = np.zeros(nq, np.uintp)
        c = cfg._c()
        _check(lib().sair_store_select_shard(
            self.local._h, _dp(q), nq, d, C.byref(c), idx.ctypes.data_as(C.POINTER(C.c_int64)),
            _dp(sim), _dp(sc), _dp(rw), rd.ctypes.data_as(C.POINTER(C.c_int32)),
            cnt.ctypes.data_as(C.POINTER(C.c_size_t))))
        return idx, sim, sc, rw, rd, cnt.astype(np.int64)

    def select_batch(self, queries, cfg: SelectionConfig):
        """The buffer's select() for every query: (idx, sim, score, count)."""
        if cfg.lambda_div != 0.0:
            return self._select_greedy(queries, cfg)
        idx, sim, sc, rw, rd, cnt = self.select_local(queries, cfg)
        nq, m = idx.shape
        pack = np.concatenate([sc, sim, rw, idx.astype(np.float64), rd.astype(np.float64),
                               cnt.astype(np.float64)[:, None]], axis=1)
        return merge_gathered(self.dist, pack, nq, m, self.device)


    def _select_greedy(self, queries, cfg: SelectionConfig):
        q = _f64(queries)
        if q.ndim == 1:
            q = q[None, :]
        nq, d = q.shape
        m = max(cfg.m, 1)
        want = min(cfg.m, self.n_global)
        idx = np.full((nq, m), -1, np.int64)
        sim, sc = np.zeros((nq, m)), np.zeros((nq, m))
        cnt = np.full(nq, want, np.int64)
        if want == 0:
            return idx, sim, sc, np.zeros(nq, np.int64)
        best = np.zeros((nq, 6 + d))
        c = cfg._c()
        _check(lib().sair_store_greedy_begin(self.local._h, _dp(q), nq, d, C.byref(c), _dp(best)))
        picks = np.zeros((want, nq, 6), np.float64)
        dev = f"cuda:{self.device}"
        for step in range(want):
            parts = np.stack(_all_gather(self.dist, best, dev))      # [ranks][nq][6 + d]
            win = global_winner(parts)                                # [nq] rank of the winner
            w = parts[win, np.arange(nq)]
            picks[step] = w[:, :6]
            if step + 1 < want:
                g = np.ascontiguousarray(w[:, 2].astype(np.int64))
                rows = np.ascontiguousarray(w[:, 6:])
                _check(lib().sair_store_greedy_next(
                    self.local._h, g.ctypes.data_as(C.POINTER(C.c_int64)), _dp(rows), _dp(best)))
        order = curriculum_order(picks[:, :, 5], picks[:, :, 1])      # [nq][want]
        for qq in range(nq):
            p = picks[order[qq], qq]
            idx[qq, :want] = p[:, 2].astype(np.int64)
            sim[qq, :want] = p[:, 3]
            sc[qq, :want] = p[:, 4]
        return idx, sim, sc, cnt


def global_winner(parts: np.ndarray) -> np.ndarray:
    """Per query the rank whose best wins: gain desc, round asc, global index
    asc (experience.cpp:177-187); parts = [ranks][nq][>= 3] (gain, round, gidx)."""
    gain, rnd, gi = parts[:, :, 0], parts[:, :, 1], parts[:, :, 2]
    # lexsort: last key primary; -inf gains (no candidate) sort last
    keys = np.lexsort((gi, rnd, -gain), axis=0)
    return keys[0]


def curriculum_order(reward: np.ndarray, rnd: np.ndarray) -> np.ndarray:
    """Stable order by (reward asc, round asc) over pick order (:290-294);
    reward / rnd are [want][nq]; returns [nq][want] pick positions."""
    want, nq = reward.shape
    pos = np.arange(want)
    return np.stack([np.lexsort((pos, rnd[:, q], reward[:, q])) for q in range(nq)])


def merge_gathered(dist, pack: np.ndarray, nq: int, m: int, device: int):
    """All-gather every rank's packed top-m ([nq][5m + 1]) into one device
    tensor and merge it there (sair_merge_topk_packed): one host->device copy
    of this rank's part, the collective, the merge kernel, and one
    device->host copy of the [nq][3m + 1] result."""
    import torch
    R = dist.get_world_size()
    dev = torch.device("cuda", device)
    t = torch.from_numpy(np.ascontiguousarray(pack))
    if dist.get_backend() == "nccl":
        t = t.to(dev)
        gathered = torch.empty((R,) + tuple(t.shape), dtype=t.dtype, device=dev)
        dist.all_gather_into_tensor(gathered, t)
    else:  # gloo: gather on the host, merge on the device
        parts = [torch.empty_like(t) for _ in range(R)]
        dist.all_gather(parts, t)
        gathered = torch.stack(parts).to(dev)
    out = torch.empty((nq, 3 * m + 1), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    _check(lib().sair_merge_topk_packed(gathered.data_ptr(), R, nq, m, device, stream,
                                        out.data_ptr()))
    o = out.cpu().numpy()
    cnt = o[:, 3 * m].astype(np.int64)
    idx = o[:, :m].astype(np.int64)
    for q in range(nq):
        idx[q, cnt[q]:] = -1
    return idx, o[:, m:2 * m].copy(), o[:, 2 * m:3 * m].copy(), cnt


def merge_parts(parts: List[np.ndarray], nq: int, m: int, device: int):
    """Device merge (sair_merge_topk) of all-gathered per-shard results."""
    S = len(parts)
    sc = np.stack([p[:, 0:m] for p in parts])
    sim = np.stack([p[:, m:2 * m] for p in parts])
    rw = np.stack([p[:, 2 * m:3 * m] for p in parts])
    gi = np.ascontiguousarray(np.stack([p[:, 3 * m:4 * m] for p in parts]).astype(np.int64))
    rd = np.ascontiguousarray(np.stack([p[:, 4 * m:5 * m] for p in parts]).astype(np.int32))
    ct = np.ascontiguousarray(np.stack([p[:, 5 * m] for p in parts]).astype(np.uintp))
    oi = np.full((nq, m), -1, np.int64)
    osim, osc = np.zeros((nq, m)), np.zeros((nq, m))
    ocnt = np.zeros(nq, np.uintp)
    _check(lib().sair_merge_topk(
        _dp(np.ascontiguousarray(sc)), _dp(np.ascontiguousarray(sim)),
        _dp(np.ascontiguousarray(rw)), rd.ctypes.data_as(C.POINTER(C.c_int32)),
        gi.ctypes.data_as(C.POINTER(C.c_int64)), ct.ctypes.data_as(C.POINTER(C.c_size_t)), S, nq,
        m, device, oi.ctypes.data_as(C.POINTER(C.c_int64)), _dp(osim), _dp(osc),
        ocnt.ctypes.data_as(C.POINTER(C.c_size_t))))
    return oi, osim, osc, ocnt.astype(np.int64)


# ------------------------------------------------------------------ pareto --

def all_gather_rows(dist, arr: np.ndarray, device) -> List[np.ndarray]:
    """All-gather of row blocks whose row count differs per rank (rank order)."""
    import torch
    arr = np.ascontiguousarray(arr, dtype=np.float64)
    width = arr.shape[1]
    sizes = _all_gather(dist, np.array([arr.shape[0]], np.int64), device)
    mx = max(int(x[0]) for x in sizes)
    pad = np.zeros((max(mx, 1), width))
    pad[:arr.shape[0]] = arr
    parts = _all_gather(dist, pad, device)
    return [p[:int(n[0])] for p, n in zip(parts, sizes)]


def combine_parts(dist, counts: np.ndarray, member: np.ndarray, device):
    """Sum of the ranks' partial dominance counts / memberships."""
    parts = _all_gather(dist, np.concatenate([counts.astype(np.float64),
                                              member.astype(np.float64)]), device)
    tot = np.sum(parts, axis=0)
    T = len(counts)
    return tot[:T].astype(np.uint32), tot[T:] > 0


class ShardedParetoFrontier:
    """ParetoFrontier (pareto.hpp:24-70) over outcome tuples sharded by rank."""

    def __init__(self, dist, device: int, latency_max_ms: float = 1.0, cost_max: float = 1.0):
        self.dist = dist
        self.device = device
        self.bounds = (latency_max_ms, cost_max)
        self.front = ParetoFrontier(latency_max_ms, cost_max, device=device)

    def insert_batch(self, local_pts) -> int:
        """Sequential insert_normalized() of every rank's tuples (in any order:
        the result is the non-dominated set of the distinct points)."""
        local = ParetoFrontier(*self.bounds, device=self.device)
        local.insert_batch(_f64(local_pts).reshape(-1, 2))
        fl, fc = local.points_array()
        parts = all_gather_rows(self.dist, np.stack([fl, fc], axis=1).reshape(-1, 2),
                                f"cuda:{self.device}")
        return self.front.insert_batch(np.concatenate(parts) if parts else np.zeros((0, 2)))

    def score_batch(self, local_pts):
        """reward() of this rank's tuples against the global frontier."""
        return self.front.score_batch(local_pts)

    def points_array(self):
        return self.front.points_array()

    def hypervolume(self) -> float:
        return self.front.hypervolume()


def sharded_dominance_counts(dist, local_tuples, device: int):
    """Dominance counts of this rank's tuples against the whole sharded set:
    (counts, member) for the local rows, and the global frontier size."""
    t = _f64(local_tuples)
    parts = all_gather_rows(dist, t, f"cuda:{device}")
    allt = np.concatenate(parts)
    cnt, mem = dominance_counts(allt, device=device, part=dist.get_rank(),
                                nparts=dist.get_world_size())
    cnt, mem = combine_parts(dist, cnt, mem, f"cuda:{device}")
    lo = sum(len(p) for p in parts[:dist.get_rank()])
    return cnt[lo:lo + len(t)], mem[lo:lo + len(t)], int(mem.sum())


# ------------------------------------------------- one process, many GPUs --

class DeviceComm:
    """sair_comm_t: the GPUs of this process (NCCL when the devices are distinct)."""

    def __init__(self, devices):
        devs = (C.c_int * len(devices))(*devices)
        self._h = C.c_void_p()
        _check(lib().sair_comm_create(devs, len(devices), C.byref(self._h)))
        self.devices = list(devices)

    def info(self):
        n, nc = C.c_int(), C.c_int()
        _check(lib().sair_comm_info(self._h, C.byref(n), C.byref(nc)))
        return n.value, bool(nc.value)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().sair_comm_destroy(self._h)
            self._h = None


class MultiGPUExperienceBuffer:
    """One ExperienceBuffer over the GPUs of a DeviceComm, entirely in the C
    ABI (sharded.cpp): the path the C++ drop-in takes without Python."""

    def __init__(self, comm: DeviceComm, r_min: float = 0.0, capacity: int = 1 << 20):
        self.comm = comm
        self._h = C.c_void_p()
        _check(lib().sair_sharded_create(comm._h, r_min, capacity, C.byref(self._h)))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().sair_sharded_destroy(self._h)
            self._h = None

    def store_many(self, contexts, rewards, rounds) -> int:
        x = _f64(contexts)
        r = _f64(rewards)
        rd = np.ascontiguousarray(rounds, dtype=np.int32)
        n, d = x.shape
        acc = np.zeros(n, np.uint8)
        na = C.c_size_t()
        _check(lib().sair_sharded_append(self._h, _dp(x), n, d, _dp(r),
                                         rd.ctypes.data_as(C.POINTER(C.c_int32)),
                                         acc.ctypes.data_as(C.POINTER(C.c_uint8)), C.byref(na)))
        return na.value

    def store_synthetic(self, seed: int, n: int, dim: int, clustered: bool = False):
        _check(lib().sair_sharded_append_synthetic(self._h, seed, n, dim, int(clustered)))

    def size(self):
        n, rej = C.c_size_t(), C.c_uint64()
        sh = np.zeros(len(self.comm.devices), np.uintp)
        _check(lib().sair_sharded_size(self._h, C.byref(n), C.byref(rej),
                                       sh.ctypes.data_as(C.POINTER(C.c_size_t))))
        return n.value, rej.value, sh.astype(np.int64)

    def effective_sigma(self, sigma_sim: float = 0.0) -> float:
        out = C.c_double()
        _check(lib().sair_sharded_effective_sigma(self._h, sigma_sim, C.byref(out)))
        return out.value

    def select_batch(self, queries, cfg: SelectionConfig):
        q = _f64(queries)
        if q.ndim == 1:
            q = q[None, :]
        nq, d = q.shape
        m = max(cfg.m, 1)
        idx = np.full((nq, m), -1, np.int64)
        sim, sc = np.zeros((nq, m)), np.zeros((nq, m))
        cnt = np.zeros(nq, np.uintp)
        c = cfg._c()
        _check(lib().sair_store_select_sharded(
            self._h, _dp(q), nq, d, C.byref(c), idx.ctypes.data_as(C.POINTER(C.c_int64)),
            _dp(sim), _dp(sc), cnt.ctypes.data_as(C.POINTER(C.c_size_t))))
        return idx, sim, sc, cnt.astype(np.int64)


def frontier_insert_batch_multi(comm: DeviceComm, frontier: ParetoFrontier, pts) -> int:
    """insert_batch on one frontier with the batch reduced on every GPU of comm."""
    a = _f64(pts).reshape(-1, 2)
    F = C.c_size_t()
    _check(lib().sair_frontier_insert_batch_sharded(comm._h, frontier._h, _dp(a), len(a),
                                                    C.byref(F)))
    return F.value
