"""The device side of one batched decision step (SURVEY.md 8(f) row 1, config
5: many simulated pipelines sharing one experience store).

Per pipeline p the reference's decision loop (harness.cpp:197-261) does:
retrieve with select() (:205), veto-scan the store for the nearest record
(policy.cpp:140-157), [LLM policy + simulator -- out of scope], score the
outcome with compute_reward against the pipeline's frontier and update it
(:250-251), and store() the new experience (:253-261).  Here the P pipelines'
device work is three calls: one select_batch with the fused veto scan (the
wide tensor-core pass), one FrontierSet.step (every pipeline's reward and
update in one kernel), one bulk store append.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

import ctypes as C

from . import (Experience, ExperienceBuffer, FrontierSet, ParetoFrontier, RewardBreakdown,
               RewardConfig, RewardInputs, ScalingAction, SelectionConfig, _check, _f64, _lib, lib)


@dataclass
class DecisionOutputs:
    idx: np.ndarray        # [P][m] retrieved record indices (curriculum order)
    sim: np.ndarray
    score: np.ndarray
    count: np.ndarray      # [P]
    nn_idx: np.ndarray     # [P] veto scan: nearest record
    nn_sim: np.ndarray
    reward: np.ndarray     # [P][7] compute_reward breakdown of the step's outcome
    stored: int            # experiences appended (after the reward gate)


def retrieve(buf: ExperienceBuffer, contexts, cfg: SelectionConfig):
    """select() + veto scan of every pipeline's current context (one pass)."""
    return buf.select_batch(contexts, cfg, nearest=True)


def score_and_store(buf: ExperienceBuffer, frontiers: FrontierSet, contexts, inputs, deltas,
                    update, rounds, rcfg: RewardConfig):
    """Every pipeline's outcome against its own frontier (then its update),
    and the new experiences (context, reward total, round) into the store."""
    rw = frontiers.step(inputs, deltas, update, rcfg)
    before = buf.size()
    buf.store_many(contexts, rw[:, 5], rounds)
    return rw, buf.size() - before


def decision_step(buf: ExperienceBuffer, frontiers: FrontierSet, contexts, scfg: SelectionConfig,
                  inputs, deltas, update, rounds, rcfg: RewardConfig) -> DecisionOutputs:
    idx, sim, sc, cnt, nn_i, nn_s = retrieve(buf, contexts, scfg)
    rw, stored = score_and_store(buf, frontiers, contexts, inputs, deltas, update, rounds, rcfg)
    return DecisionOutputs(idx, sim, sc, cnt, nn_i, nn_s, rw, stored)


@dataclass
class ReplayOutputs:
    idx: np.ndarray        # [count] retrieved record indices (curriculum order)
    sim: np.ndarray
    score: np.ndarray
    nn_idx: int            # veto scan: nearest record and its similarity
    nn_sim: float
    reward: RewardBreakdown
    inserted: bool         # frontier.update's result
    stored: bool           # store()'s result (the r_min gate)


class _ReplayScratch:
    """replay_step's output arrays, their ctypes pointers and the last
    converted configs, kept per buffer: building them per call (numpy arrays,
    seven pointer casts, two config structs, a package import) was ~30 us of
    a ~130 us decision step."""

    def __init__(self, m: int, d: int):
        self.m, self.d = m, d
        self.x = np.zeros(d)
        self.idx = np.full(m, -1, np.int64)
        self.sim = np.zeros(m)
        self.sc = np.zeros(m)
        self.nn_i = np.full(1, -1, np.int64)
        self.nn_s = np.zeros(1)
        self.cnt = C.c_size_t()
        self.rw = _lib.RewardBreakdownC()
        self.ins, self.sto = C.c_int(), C.c_int()
        self.ri = _lib.RewardInputsC()
        i64, f64 = C.POINTER(C.c_int64), C.POINTER(C.c_double)
        self.p = (self.x.ctypes.data_as(f64), self.idx.ctypes.data_as(i64),
                  self.sim.ctypes.data_as(f64), self.sc.ctypes.data_as(f64), C.byref(self.cnt),
                  self.nn_i.ctypes.data_as(i64), self.nn_s.ctypes.data_as(f64),
                  C.byref(self.rw), C.byref(self.ins), C.byref(self.sto), C.byref(self.ri))
        self.skey = self.rkey = self.akey = None
        self.sc_c = self.rc_c = None
        self.deltas = None
        self.p_deltas = None


def replay_step(buf: ExperienceBuffer, frontier: ParetoFrontier, x, scfg: SelectionConfig,
                inp: RewardInputs, action: ScalingAction, rcfg: RewardConfig,
                update: bool = True, round: int = 0) -> ReplayOutputs:
    """One decision of harness.cpp:197-261 with its outcome known (config 1's
    trace replay): select(x) + veto scan, compute_reward(inp, action) against
    the frontier, frontier.update(inp.l_after_ms, inp.c_after), store() of
    (x, reward total, round) -- one device call, one host synchronisation
    (sair_decision_step); the same results as the four calls in that order."""
    x = np.asarray(x, dtype=np.float64).reshape(-1)
    m = max(scfg.m, 1)
    sc = getattr(buf, "_replay_scratch", None)
    if sc is None or sc.m != m or sc.d != len(x):
        sc = _ReplayScratch(m, len(x))
        buf._replay_scratch = sc
    sc.x[:] = x
    sc.nn_i[0] = -1
    sc.nn_s[0] = 0.0
    skey = (scfg.m, scfg.lambda_div, scfg.sigma_sim, scfg.locally_weighted_mean, scfg.mode)
    if skey != sc.skey:
        sc.skey, sc.sc_c = skey, scfg._c()
    rkey = (rcfg.t_sla_ms, rcfg.l_baseline_ms, rcfg.c_budget, rcfg.w_latency, rcfg.w_cost,
            rcfg.w_proactive, rcfg.r_max)
    if rkey != sc.rkey:
        sc.rkey, sc.rc_c = rkey, rcfg._c()
    akey = tuple((s.replicas, s.cpu_millicores, s.memory_mb, s.rate_ratio_tenths)
                 for s in action.stages)
    if akey != sc.akey:
        sc.akey, sc.deltas = akey, action.deltas()
        sc.p_deltas = sc.deltas.ctypes.data_as(C.POINTER(C.c_int32))
    ri = sc.ri
    ri.l_before_ms, ri.l_after_ms = inp.l_before_ms, inp.l_after_ms
    ri.c_before, ri.c_after = inp.c_before, inp.c_after
    px, pidx, psim, psc, pcnt, pnn_i, pnn_s, prw, pins, psto, pri = sc.p
    _check(lib().sair_decision_step(
        buf._h, frontier._h, px, sc.d, C.byref(sc.sc_c), pri, sc.p_deltas, len(sc.deltas),
        C.byref(sc.rc_c), int(update), int(round), pidx, psim, psc, pcnt, pnn_i, pnn_s, prw, pins,
        psto))
    k = int(sc.cnt.value)
    rw = sc.rw
    r = RewardBreakdown(rw.latency, rw.cost, rw.sla, rw.proactive, rw.pareto, rw.total,
                        bool(rw.clipped))
    stored = bool(sc.sto.value)
    if stored and buf._mirror:
        buf._items.append(Experience(list(x), action, r.total, int(round)))
    return ReplayOutputs(sc.idx[:k].copy(), sc.sim[:k].copy(), sc.sc[:k].copy(),
                         int(sc.nn_i[0]), float(sc.nn_s[0]), r, bool(sc.ins.value), stored)
