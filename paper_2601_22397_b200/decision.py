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

from . import ExperienceBuffer, FrontierSet, RewardConfig, SelectionConfig


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
