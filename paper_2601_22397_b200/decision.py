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
               RewardConfig, RewardInputs, ScalingAction, SelectionConfig, _lib)


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


def replay_step(buf: ExperienceBuffer, frontier: ParetoFrontier, x, scfg: SelectionConfig,
                inp: RewardInputs, action: ScalingAction, rcfg: RewardConfig,
                update: bool = True, round: int = 0) -> ReplayOutputs:
    """One decision of harness.cpp:197-261 with its outcome known (config 1's
    trace replay): select(x) + veto scan, compute_reward(inp, action) against
    the frontier, frontier.update(inp.l_after_ms, inp.c_after), store() of
    (x, reward total, round) -- one device call, one host synchronisation
    (sair_decision_step); the same results as the four calls in that order."""
    from . import _check, _dp, _f64, lib
    x = _f64(x).ravel()
    m = max(scfg.m, 1)
    idx = np.full(m, -1, np.int64)
    sim = np.zeros(m)
    sc = np.zeros(m)
    cnt = C.c_size_t()
    nn_i = np.full(1, -1, np.int64)
    nn_s = np.zeros(1)
    ri = _lib.RewardInputsC(inp.l_before_ms, inp.l_after_ms, inp.c_before, inp.c_after)
    d = action.deltas()
    rw = _lib.RewardBreakdownC()
    ins, sto = C.c_int(), C.c_int()
    c = scfg._c()
    rc = rcfg._c()
    _check(lib().sair_decision_step(
        buf._h, frontier._h, _dp(x), len(x), C.byref(c), C.byref(ri),
        d.ctypes.data_as(C.POINTER(C.c_int32)), len(d), C.byref(rc), int(update), int(round),
        idx.ctypes.data_as(C.POINTER(C.c_int64)), _dp(sim), _dp(sc), C.byref(cnt),
        nn_i.ctypes.data_as(C.POINTER(C.c_int64)), _dp(nn_s), C.byref(rw), C.byref(ins),
        C.byref(sto)))
    k = int(cnt.value)
    r = RewardBreakdown(rw.latency, rw.cost, rw.sla, rw.proactive, rw.pareto, rw.total,
                        bool(rw.clipped))
    if sto.value and buf._mirror:
        buf._items.append(Experience(list(x), action, r.total, int(round)))
    return ReplayOutputs(idx[:k], sim[:k], sc[:k], int(nn_i[0]), float(nn_s[0]), r,
                         bool(ins.value), bool(sto.value))
