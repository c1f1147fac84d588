"""B200-native SAIR retrieval + Pareto hot path -- Python host mirror.

Mirrors the reference's C++ interface for the path (namespace ``scalelab``,
/root/reference/proj/include/scalelab/{experience,pareto,reward}.hpp): same
class and method names, argument meaning and error behaviour, implemented on
the C-ABI of libsair.so (include/sair.h).  Exceptions map the reference's:

    std::invalid_argument -> InvalidArgument (a ValueError)
    std::logic_error      -> LogicError
    std::out_of_range     -> OutOfRange (an IndexError)

Nothing here computes on the CPU: every score, frontier and reward comes from
the device.  Host-side Python only holds what the reference's callers hold
(the AoS mirror of stored experiences for ``all()``; the action/source payload
never reaches the device).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import SairError, lib

__all__ = [
    "ExperienceBuffer", "Experience", "SelectionConfig", "SelectedExperience", "ScalingAction",
    "StageDelta", "ParetoFrontier", "ObjectivePoint", "dominates", "RewardConfig",
    "RewardInputs", "RewardBreakdown", "compute_reward", "compute_reward_batch",
    "action_magnitude", "context_features", "dominance_counts", "SairError", "InvalidArgument",
    "compute_reward_replay", "FrontierSet",
    "LogicError", "OutOfRange", "SELECT_AUTO", "SELECT_EXACT",
]

SELECT_AUTO, SELECT_EXACT = 0, 1


class InvalidArgument(SairError, ValueError):
    pass


class LogicError(SairError):
    pass


class OutOfRange(LogicError, IndexError):
    pass


_EXC = {_lib.SAIR_EINVAL: InvalidArgument, _lib.SAIR_ELOGIC: LogicError,
        _lib.SAIR_ERANGE: OutOfRange}


def _check(rc: int):
    if rc != _lib.SAIR_OK:
        msg = lib().sair_last_error().decode(errors="replace")
        raise _EXC.get(rc, SairError)(rc, msg)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _f64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


# --------------------------------------------------------------- actions ---

@dataclass
class StageDelta:  # action.hpp:22-33
    replicas: int = 0
    cpu_millicores: int = 0
    memory_mb: int = 0
    rate_ratio_tenths: int = 0

    def is_noop(self) -> bool:
        return not (self.replicas or self.cpu_millicores or self.memory_mb or
                    self.rate_ratio_tenths)


@dataclass
class ScalingAction:  # action.hpp:35-56
    stages: List[StageDelta] = field(default_factory=list)

    @staticmethod
    def noop(n_stages: int) -> "ScalingAction":
        return ScalingAction([StageDelta() for _ in range(n_stages)])

    def is_noop(self) -> bool:
        return all(s.is_noop() for s in self.stages)

    def stages_scaled(self) -> int:
        return sum(0 if s.is_noop() else 1 for s in self.stages)

    def deltas(self) -> np.ndarray:
        return np.array([[s.replicas, s.cpu_millicores, s.memory_mb, s.rate_ratio_tenths]
                         for s in self.stages], dtype=np.int32).reshape(-1, 4)


# ------------------------------------------------------------- retrieval ---

@dataclass
class Experience:  # experience.hpp:19-25
    context: Sequence[float] = ()
    action: ScalingAction = field(default_factory=ScalingAction)
    reward: float = 0.0
    round: int = 0
    source: str = "llm"


@dataclass
class SelectionConfig:  # experience.hpp:27-32
    m: int = 15
    lambda_div: float = 0.1
    sigma_sim: float = 0.0
    locally_weighted_mean: bool = False
    mode: int = SELECT_AUTO  # this library: SELECT_EXACT forces the full fp64 pass

    def _c(self):
        return _lib.SelectConfigC(self.m, self.lambda_div, self.sigma_sim,
                                  int(self.locally_weighted_mean), self.mode)


@dataclass
class SelectedExperience:  # experience.hpp:35-39
    experience: Experience
    similarity_to_current: float
    score: float
    index: int = -1


def context_features(state) -> List[float]:
    """experience.cpp:13-28: per stage [replicas, cpu_mc, mem_mb, rate_ratio,
    queue_depth, u_cpu, u_gpu_quota], then [latency_p99_ms, throughput_rps].
    ``state`` is any object/dict with those fields (PipelineState, types.hpp)."""
    g = (lambda o, k: o[k]) if isinstance(state, dict) else getattr
    x: List[float] = []
    for s in g(state, "stages"):
        cfg = g(s, "config")
        x += [float(g(cfg, "replicas")), float(g(cfg, "cpu_millicores")),
              float(g(cfg, "memory_mb")), float(g(cfg, "rate_ratio")),
              float(g(s, "queue_depth")), float(g(s, "u_cpu")), float(g(s, "u_gpu_quota"))]
    x += [float(g(state, "latency_p99_ms")), float(g(state, "throughput_rps"))]
    return x


class ExperienceBuffer:
    """ExperienceBuffer (experience.hpp:45-89) over a device-resident store."""

    def __init__(self, r_min: float = 0.0, device: int = 0, capacity_hint: int = 0):
        h = C.c_void_p()
        _check(lib().sair_store_create(r_min, device, capacity_hint, C.byref(h)))
        self._h = h
        self._items: List[Experience] = []  # AoS mirror for all() (experience.hpp:54)
        self._mirror = True

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().sair_store_destroy(h)
            except TypeError:  # interpreter shutdown: module globals already cleared
                pass
            self._h = None

    # value semantics (experience.hpp:45)
    def copy(self) -> "ExperienceBuffer":
        o = ExperienceBuffer.__new__(ExperienceBuffer)
        h = C.c_void_p()
        _check(lib().sair_store_clone(self._h, C.byref(h)))
        o._h, o._items, o._mirror = h, list(self._items), self._mirror
        return o

    __copy__ = copy

    @classmethod
    def load(cls, path: str, r_min: float = 0.0, device: int = 0, nthreads: int = 0):
        """ExperienceBuffer::load (experience.cpp:243-271) into the device store:
        returns (buffer, corrupt_lines).  Parsed on all host threads, one bulk
        append; no host mirror (use get(i) / export())."""
        h = C.c_void_p()
        bad = C.c_size_t()
        _check(lib().sair_store_load_jsonl(str(path).encode(), r_min, device, nthreads,
                                           C.byref(bad), C.byref(h)))
        o = cls.__new__(cls)
        o._h = h
        o._items = []
        o._mirror = False
        return o, bad.value

    def persist(self, path: str, lossy: bool = False):
        """ExperienceBuffer::persist (experience.cpp:232-241).  With the AoS mirror
        (rows stored one by one) every record is written from it, source and
        action included, in nlohmann's compact dump format (sorted keys) -- what
        the reference itself writes.  Without it (bulk / synthetic / loaded rows)
        the device store holds no source or action: that export writes them
        empty and must be asked for with ``lossy=True``."""
        if self._mirror:
            import json
            with open(path, "w", encoding="utf-8") as out:
                for e in self._items:
                    act = [{"cpu_millicores": int(st.cpu_millicores), "memory_mb": int(st.memory_mb),
                            "rate_ratio_tenths": int(st.rate_ratio_tenths),
                            "replicas": int(st.replicas)} for st in e.action.stages]
                    j = {"action": act, "context": [float(v) for v in e.context],
                         "reward": float(e.reward), "round": int(e.round), "source": e.source}
                    out.write(json.dumps(j, separators=(",", ":"), ensure_ascii=False) + "\n")
            return
        if not lossy:
            raise LogicError(_lib.SAIR_ELOGIC,
                             "persist(): no host mirror of source/action for bulk rows; "
                             "pass lossy=True to write them empty")
        _check(lib().sair_store_persist_jsonl(self._h, str(path).encode()))

    def export(self, offset: int = 0, count: Optional[int] = None):
        """Bulk copy of records [offset, offset + count): (contexts, rewards, rounds)."""
        n = self.size()
        count = n - offset if count is None else count
        d = max(self.dim(), 1)
        ctx = np.zeros((count, d))
        rw = np.zeros(count)
        rd = np.zeros(count, np.int32)
        _check(lib().sair_store_export(self._h, offset, count, _dp(ctx), _dp(rw),
                                       rd.ctypes.data_as(C.POINTER(C.c_int32))))
        return ctx, rw, rd

    def store(self, e: Experience) -> bool:
        """experience.cpp:44-62: False (and counted) when reward <= r_min."""
        x = _f64(e.context)
        acc = np.zeros(1, np.uint8)
        n_acc = C.c_size_t()
        _check(lib().sair_store_append(self._h, _dp(x), 1, len(x), _dp(_f64([e.reward])),
                                       np.array([e.round], np.int32).ctypes.data_as(
                                           C.POINTER(C.c_int32)),
                                       acc.ctypes.data_as(C.POINTER(C.c_uint8)),
                                       C.byref(n_acc)))
        if acc[0]:
            self._items.append(e)
        return bool(acc[0])

    def store_many(self, contexts, rewards, rounds, keep_mirror: bool = False) -> int:
        """Bulk store() of n rows (each gated).  The AoS mirror is dropped unless
        requested: at millions of rows all() would be a host-memory copy of the
        device store (use get(i))."""
        x = _f64(contexts)
        r = _f64(rewards)
        rd = np.ascontiguousarray(rounds, dtype=np.int32)
        n, d = x.shape
        acc = np.zeros(n, np.uint8)
        n_acc = C.c_size_t()
        rc = lib().sair_store_append(self._h, _dp(x), n, d, _dp(r),
                                     rd.ctypes.data_as(C.POINTER(C.c_int32)),
                                     acc.ctypes.data_as(C.POINTER(C.c_uint8)), C.byref(n_acc))
        if keep_mirror and self._mirror:
            for i in np.nonzero(acc)[0]:
                self._items.append(Experience(list(x[i]), ScalingAction(), float(r[i]),
                                              int(rd[i])))
        else:
            self._mirror = False
        _check(rc)
        return int(n_acc.value)

    def store_synthetic(self, seed: int, count: int, dim: int, clustered: bool = False):
        """Append device-generated synthetic rows (synth.py documents them)."""
        _check(lib().sair_store_append_synthetic(self._h, seed, count, dim, int(clustered)))
        self._mirror = False

    def size(self) -> int:
        n = C.c_size_t()
        _check(lib().sair_store_size(self._h, C.byref(n)))
        return n.value

    __len__ = size

    def empty(self) -> bool:
        return self.size() == 0

    def dim(self) -> int:
        d = C.c_int()
        _check(lib().sair_store_dim(self._h, C.byref(d)))
        return d.value

    def rejected(self) -> int:
        v = C.c_uint64()
        _check(lib().sair_store_rejected(self._h, C.byref(v)))
        return v.value

    def r_min(self) -> float:
        v = C.c_double()
        _check(lib().sair_store_r_min(self._h, C.byref(v)))
        return v.value

    def all(self) -> List[Experience]:
        if not self._mirror:
            raise LogicError(_lib.SAIR_ELOGIC, "all(): the AoS mirror was not kept for bulk rows")
        return self._items

    def get(self, index: int):
        """(context, reward, round) of record `index`, read back from the device."""
        d = self.dim()
        ctx = np.zeros(max(d, 1))
        r = C.c_double()
        rd = C.c_int32()
        _check(lib().sair_store_get(self._h, index, _dp(ctx), C.byref(r), C.byref(rd)))
        return ctx[:d], r.value, rd.value

    def standardize(self, x) -> np.ndarray:
        x = _f64(x)
        z = np.zeros_like(x)
        _check(lib().sair_store_standardize(self._h, _dp(x), len(x), _dp(z)))
        return z

    def effective_sigma(self, cfg: Optional[SelectionConfig] = None) -> float:
        cfg = cfg or SelectionConfig()
        v = C.c_double()
        _check(lib().sair_store_effective_sigma(self._h, cfg.sigma_sim, C.byref(v)))
        return v.value

    def surprisal(self, index: int, x_curr, cfg: Optional[SelectionConfig] = None) -> float:
        cfg = cfg or SelectionConfig()
        x = _f64(x_curr)
        v = C.c_double()
        c = cfg._c()
        _check(lib().sair_store_surprisal(self._h, index, _dp(x), len(x), C.byref(c), C.byref(v)))
        return v.value

    def select_batch(self, queries, cfg: Optional[SelectionConfig] = None, nearest=False):
        """select() for every row of `queries`: one device pass per 128 queries
        (tensor-core wide pass, Q >= 32) or per 8 (Q < 32).
        Returns (idx[nq, m], sim[nq, m], score[nq, m], count[nq]) and, with
        nearest=True, also (nn_idx[nq], nn_sim[nq]) of the veto scan."""
        cfg = cfg or SelectionConfig()
        q = _f64(queries)
        if q.ndim == 1:
            q = q[None, :]
        nq, d = q.shape
        m = max(cfg.m, 1)
        idx = np.full((nq, m), -1, np.int64)
        sim = np.zeros((nq, m))
        sc = np.zeros((nq, m))
        cnt = np.zeros(nq, np.uintp)
        c = cfg._c()
        nn_i = np.full(nq, -1, np.int64) if nearest else None
        nn_s = np.zeros(nq) if nearest else None
        _check(lib().sair_store_select(
            self._h, _dp(q), nq, d, C.byref(c), idx.ctypes.data_as(C.POINTER(C.c_int64)),
            _dp(sim), _dp(sc), cnt.ctypes.data_as(C.POINTER(C.c_size_t)),
            nn_i.ctypes.data_as(C.POINTER(C.c_int64)) if nearest else None,
            _dp(nn_s) if nearest else None))
        out = (idx, sim, sc, cnt.astype(np.int64))
        return out + (nn_i, nn_s) if nearest else out

    def select(self, x_curr, cfg: Optional[SelectionConfig] = None) -> List[SelectedExperience]:
        """experience.cpp:151-205: greedy diversity-regularised pick of up to m
        experiences in curriculum (reward-ascending) order."""
        idx, sim, sc, cnt = self.select_batch(_f64(x_curr)[None, :], cfg)
        out = []
        for j in range(int(cnt[0])):
            i = int(idx[0, j])
            if self._mirror:
                e = self._items[i]
            else:
                ctx, r, rd = self.get(i)
                e = Experience(list(ctx), ScalingAction(), r, rd)
            out.append(SelectedExperience(e, float(sim[0, j]), float(sc[0, j]), i))
        return out

    def nearest(self, queries, sigma_sim: float = 0.0):
        """The MockBackend veto scan (policy.cpp:140-157): (index, similarity)."""
        q = _f64(queries)
        if q.ndim == 1:
            q = q[None, :]
        nq, d = q.shape
        ii = np.zeros(nq, np.int64)
        ss = np.zeros(nq)
        _check(lib().sair_store_nearest(self._h, _dp(q), nq, d, sigma_sim,
                                        ii.ctypes.data_as(C.POINTER(C.c_int64)), _dp(ss)))
        return ii, ss

    def last_stats(self) -> dict:
        s = _lib.SelectStatsC()
        _check(lib().sair_store_last_stats(self._h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in s._fields_}

    def stream_ptr(self) -> int:
        p = C.c_void_p()
        _check(lib().sair_store_stream(self._h, C.byref(p)))
        return p.value or 0


# ---------------------------------------------------------------- pareto ---

@dataclass(frozen=True)
class ObjectivePoint:  # pareto.hpp:10-15
    latency: float = 0.0
    cost: float = 0.0


class ParetoFrontier:
    """ParetoFrontier (pareto.hpp:24-70): 2-objective frontier on the device."""

    def __init__(self, latency_max_ms: float, cost_max: float, device: int = 0):
        h = C.c_void_p()
        _check(lib().sair_frontier_create(latency_max_ms, cost_max, device, C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().sair_frontier_destroy(h)
            except TypeError:  # interpreter shutdown: module globals already cleared
                pass
            self._h = None

    def copy(self) -> "ParetoFrontier":
        o = ParetoFrontier.__new__(ParetoFrontier)
        h = C.c_void_p()
        _check(lib().sair_frontier_clone(self._h, C.byref(h)))
        o._h = h
        return o

    __copy__ = copy

    @staticmethod
    def _pt(p):
        if isinstance(p, ObjectivePoint):
            return p.latency, p.cost
        return float(p[0]), float(p[1])

    def update(self, latency_ms: float, cost: float):
        """Returns (inserted, clamped) -- UpdateResult, pareto.hpp:28-31."""
        ins, cl = C.c_int(), C.c_int()
        _check(lib().sair_frontier_update(self._h, latency_ms, cost, C.byref(ins), C.byref(cl)))
        return bool(ins.value), bool(cl.value)

    def normalize(self, latency_ms: float, cost: float):
        """Returns (ObjectivePoint, clamped)."""
        l, c, cl = C.c_double(), C.c_double(), C.c_int()
        _check(lib().sair_frontier_normalize(self._h, latency_ms, cost, C.byref(l), C.byref(c),
                                             C.byref(cl)))
        return ObjectivePoint(l.value, c.value), bool(cl.value)

    def insert_normalized(self, p) -> bool:
        l, c = self._pt(p)
        ins = C.c_int()
        _check(lib().sair_frontier_insert_normalized(self._h, l, c, C.byref(ins)))
        return bool(ins.value)

    def insert_batch(self, pts) -> int:
        """T sequential insert_normalized() calls; returns the new size."""
        a = _f64(pts).reshape(-1, 2)
        F = C.c_size_t()
        _check(lib().sair_frontier_insert_batch(self._h, _dp(a), len(a), C.byref(F)))
        return F.value

    def size(self) -> int:
        F = C.c_size_t()
        _check(lib().sair_frontier_size(self._h, C.byref(F)))
        return F.value

    __len__ = size

    def empty(self) -> bool:
        return self.size() == 0

    def points_array(self):
        F = self.size()
        l, c = np.zeros(max(F, 1)), np.zeros(max(F, 1))
        out = C.c_size_t()
        _check(lib().sair_frontier_points(self._h, _dp(l), _dp(c), max(F, 1), C.byref(out)))
        return l[:F], c[:F]

    def points(self) -> List[ObjectivePoint]:
        l, c = self.points_array()
        return [ObjectivePoint(float(a), float(b)) for a, b in zip(l, c)]

    def latency_max_ms(self) -> float:
        a, b = C.c_double(), C.c_double()
        _check(lib().sair_frontier_bounds(self._h, C.byref(a), C.byref(b)))
        return a.value

    def cost_max(self) -> float:
        a, b = C.c_double(), C.c_double()
        _check(lib().sair_frontier_bounds(self._h, C.byref(a), C.byref(b)))
        return b.value

    def strictly_dominated(self, p) -> bool:
        l, c = self._pt(p)
        v = C.c_int()
        _check(lib().sair_frontier_strictly_dominated(self._h, l, c, C.byref(v)))
        return bool(v.value)

    def hypervolume(self) -> float:
        v = C.c_double()
        _check(lib().sair_frontier_hypervolume(self._h, C.byref(v)))
        return v.value

    def contribution(self, p) -> float:
        l, c = self._pt(p)
        v = C.c_double()
        _check(lib().sair_frontier_contribution(self._h, l, c, C.byref(v)))
        return v.value

    def distance(self, p) -> Optional[float]:
        l, c = self._pt(p)
        v, has = C.c_double(), C.c_int()
        _check(lib().sair_frontier_distance(self._h, l, c, C.byref(v), C.byref(has)))
        return v.value if has.value else None

    def reward(self, p) -> float:
        l, c = self._pt(p)
        v = C.c_double()
        _check(lib().sair_frontier_reward(self._h, l, c, C.byref(v)))
        return v.value

    def score_batch(self, pts):
        """reward() of every normalized point (T x 2); returns (reward, dominated)."""
        a = _f64(pts).reshape(-1, 2)
        out = np.zeros(len(a))
        dom = np.zeros(len(a), np.uint8)
        _check(lib().sair_frontier_score_batch(self._h, _dp(a), len(a), _dp(out),
                                               dom.ctypes.data_as(C.POINTER(C.c_uint8))))
        return out, dom.astype(bool)

    def score_batch_device(self, pts_ptr: int, T: int, out_ptr: int, dom_ptr: int = 0,
                           stream: int = 0):
        """score_batch on device pointers (e.g. torch tensors' data_ptr()),
        enqueued on `stream` without synchronizing."""
        _check(lib().sair_frontier_score_batch_device(self._h, pts_ptr, T, out_ptr,
                                                      dom_ptr or None, stream or None))


def dominance_counts(tuples, device: int = 0, counts: bool = True, part: int = 0,
                     nparts: int = 1):
    """K-objective dominance counts and frontier membership (see sair.h).
    With nparts > 1 only part `part` of the pairwise work is done (entries
    outside it are 0; the parts of all ranks combine by a sum)."""
    t = _f64(tuples)
    if t.ndim != 2:
        raise InvalidArgument(_lib.SAIR_EINVAL, "tuples must be T x K")
    T, K = t.shape
    cnt = np.zeros(T, np.uint32) if counts else None
    mem = np.zeros(T, np.uint8)
    cp = cnt.ctypes.data_as(C.POINTER(C.c_uint32)) if counts else None
    mp = mem.ctypes.data_as(C.POINTER(C.c_uint8))
    if nparts == 1:
        _check(lib().sair_dominance_counts(_dp(t), T, K, device, cp, mp))
    else:
        _check(lib().sair_dominance_counts_part(_dp(t), T, K, device, part, nparts, cp, mp))
    return cnt, mem.astype(bool)


def dominates(p, q) -> bool:
    """dominates(p, q), pareto.cpp:9-12 (evaluated by the device kernel)."""
    pl, pc = ParetoFrontier._pt(p)
    ql, qc = ParetoFrontier._pt(q)
    cnt, _ = dominance_counts([[pl, pc], [ql, qc]])
    return bool(cnt[1] > 0)


# ---------------------------------------------------------------- reward ---

@dataclass
class RewardConfig:  # reward.hpp:8-20
    t_sla_ms: float = 500.0
    l_baseline_ms: float = 0.0
    c_budget: float = 10.0
    w_latency: float = 0.7
    w_cost: float = 0.3
    w_proactive: float = 0.3
    r_max: float = 5.0

    def resolved_l_baseline(self) -> float:
        return self.l_baseline_ms if self.l_baseline_ms > 0.0 else 4.0 * self.t_sla_ms

    def _c(self):
        return _lib.RewardConfigC(self.t_sla_ms, self.l_baseline_ms, self.c_budget,
                                  self.w_latency, self.w_cost, self.w_proactive, self.r_max)


@dataclass
class RewardInputs:  # reward.hpp:23-28
    l_before_ms: float = 0.0
    l_after_ms: float = 0.0
    c_before: float = 0.0
    c_after: float = 0.0


@dataclass
class RewardBreakdown:  # reward.hpp:30-38
    latency: float = 0.0
    cost: float = 0.0
    sla: float = 0.0
    proactive: float = 0.0
    pareto: float = 0.0
    total: float = 0.0
    clipped: bool = False


def action_magnitude(action: ScalingAction) -> float:
    d = action.deltas()
    v = C.c_double()
    _check(lib().sair_action_magnitude(d.ctypes.data_as(C.POINTER(C.c_int32)), len(d),
                                       C.byref(v)))
    return v.value


def compute_reward(inp: RewardInputs, action: ScalingAction, frontier: ParetoFrontier,
                   cfg: RewardConfig) -> RewardBreakdown:
    """reward.cpp:21-44; the frontier is read-only (score-then-insert)."""
    ri = _lib.RewardInputsC(inp.l_before_ms, inp.l_after_ms, inp.c_before, inp.c_after)
    d = action.deltas()
    out = _lib.RewardBreakdownC()
    c = cfg._c()
    _check(lib().sair_compute_reward(C.byref(ri), d.ctypes.data_as(C.POINTER(C.c_int32)),
                                     len(d), frontier._h, C.byref(c), C.byref(out)))
    return RewardBreakdown(out.latency, out.cost, out.sla, out.proactive, out.pareto, out.total,
                           bool(out.clipped))


def _breakdowns(out, T: int) -> np.ndarray:
    """T sair_reward_breakdown structs -> T x 7 float64 (latency, cost, sla,
    proactive, pareto, total, clipped), without a Python loop."""
    if T == 0:
        return np.zeros((0, 7))
    rec = np.ctypeslib.as_array(out, shape=(len(out),))[:T]
    res = np.empty((T, 7))
    for j, name in enumerate(("latency", "cost", "sla", "proactive", "pareto", "total")):
        res[:, j] = rec[name]
    res[:, 6] = rec["clipped"]
    return res


def compute_reward_batch(inputs, deltas, frontier: ParetoFrontier, cfg: RewardConfig):
    """compute_reward for T rows: inputs T x 4 (l_before, l_after, c_before,
    c_after), deltas T x S x 4.  Returns a T x 7 array (latency, cost, sla,
    proactive, pareto, total, clipped)."""
    x = _f64(inputs).reshape(-1, 4)
    T = len(x)
    d = np.ascontiguousarray(deltas, dtype=np.int32).reshape(T, -1, 4)
    S = d.shape[1]
    out = (_lib.RewardBreakdownC * max(T, 1))()
    c = cfg._c()
    _check(lib().sair_compute_reward_batch(
        x.ctypes.data_as(C.POINTER(_lib.RewardInputsC)), d.ctypes.data_as(C.POINTER(C.c_int32)),
        S, T, frontier._h, C.byref(c), out))
    return _breakdowns(out, T)


def compute_reward_replay(inputs, deltas, update, frontier: ParetoFrontier, cfg: RewardConfig):
    """The replay loop (scalelab_cli.cpp:118-147, harness.cpp:250-251) in one
    call: row t's compute_reward against the frontier as updated by the earlier
    rows with update[s], then frontier.update(l_after_t, c_after_t) if
    update[t].  Returns T x 7 (latency, cost, sla, proactive, pareto, total,
    clipped); `frontier` ends in the final state."""
    x = _f64(inputs).reshape(-1, 4)
    T = len(x)
    d = np.ascontiguousarray(deltas, dtype=np.int32).reshape(T, -1, 4)
    S = d.shape[1]
    u = np.ascontiguousarray(update, dtype=np.uint8).reshape(T)
    out = (_lib.RewardBreakdownC * max(T, 1))()
    c = cfg._c()
    _check(lib().sair_compute_reward_replay(
        x.ctypes.data_as(C.POINTER(_lib.RewardInputsC)), d.ctypes.data_as(C.POINTER(C.c_int32)),
        S, T, u.ctypes.data_as(C.POINTER(C.c_uint8)), frontier._h, C.byref(c), out))
    return _breakdowns(out, T)


class FrontierSet:
    """P independent ParetoFrontiers stepped together (config 5: one frontier
    per simulated pipeline, harness.cpp:150, :250-251)."""

    def __init__(self, P: int, latency_max_ms: float, cost_max: float, device: int = 0):
        h = C.c_void_p()
        _check(lib().sair_frontier_set_create(P, latency_max_ms, cost_max, device, C.byref(h)))
        self._h = h
        self.P = P

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().sair_frontier_set_destroy(h)
            except TypeError:  # interpreter shutdown: module globals already cleared
                pass
            self._h = None

    def step(self, inputs, deltas, update, cfg: RewardConfig):
        """compute_reward of every pipeline's row against its own frontier, then
        its update() where update[p]; returns P x 7 (as compute_reward_batch)."""
        x = _f64(inputs).reshape(self.P, 4)
        d = np.ascontiguousarray(deltas, dtype=np.int32).reshape(self.P, -1, 4)
        u = np.ascontiguousarray(update, dtype=np.uint8).reshape(self.P)
        out = (_lib.RewardBreakdownC * max(self.P, 1))()
        c = cfg._c()
        _check(lib().sair_frontier_set_step(
            self._h, x.ctypes.data_as(C.POINTER(_lib.RewardInputsC)),
            d.ctypes.data_as(C.POINTER(C.c_int32)), d.shape[1],
            u.ctypes.data_as(C.POINTER(C.c_uint8)), C.byref(c), out))
        return _breakdowns(out, self.P)

    def points_array(self, p: int):
        F = C.c_size_t()
        hv = C.c_double()
        _check(lib().sair_frontier_set_points(self._h, p, None, None, 0, C.byref(F), C.byref(hv)))
        n = max(F.value, 1)
        l, c = np.zeros(n), np.zeros(n)
        _check(lib().sair_frontier_set_points(self._h, p, _dp(l), _dp(c), n, C.byref(F),
                                              C.byref(hv)))
        return l[:F.value], c[:F.value]

    def hypervolume(self, p: int) -> float:
        F = C.c_size_t()
        hv = C.c_double()
        _check(lib().sair_frontier_set_points(self._h, p, None, None, 0, C.byref(F), C.byref(hv)))
        return hv.value
