"""ctypes binding of libsair.so (include/sair.h).

The library is built in-tree (``make -C paper_2601_22397_b200/csrc``, or
``__graft_entry__.build()``).  There is no fallback: importing the package
without the library raises, and every compute call on a machine without a
CUDA device fails with ``SairError(SAIR_ECUDA)``.
"""
from __future__ import annotations

import ctypes as C
import os
import re
from pathlib import Path

PKG = Path(__file__).resolve().parent
# SAIR_LIB_PATH: a side build for A/B timing (scripts/); unset, the in-tree library
LIB_PATH = Path(os.environ.get("SAIR_LIB_PATH") or PKG / "libsair.so")
HEADER = PKG.parent / "include" / "sair.h"

SAIR_OK, SAIR_EINVAL, SAIR_ELOGIC, SAIR_ERANGE, SAIR_EIO, SAIR_ECUDA, SAIR_ENOMEM, SAIR_ENCCL = range(8)


class SairError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[sair {code}] {msg}")
        self.code = code


class SelectConfigC(C.Structure):
    _fields_ = [("m", C.c_size_t), ("lambda_div", C.c_double), ("sigma_sim", C.c_double),
                ("locally_weighted_mean", C.c_int), ("mode", C.c_int)]


class SelectStatsC(C.Structure):
    _fields_ = [("queries", C.c_size_t), ("certified", C.c_size_t),
                ("exact_fallbacks", C.c_size_t), ("candidates", C.c_size_t), ("qb", C.c_int),
                ("stream_launches", C.c_int), ("stream_ms", C.c_float), ("total_ms", C.c_float),
                ("prepass_ms", C.c_float), ("tensor_core", C.c_int), ("small", C.c_int),
                ("retried", C.c_size_t), ("greedy32", C.c_size_t),
                ("greedy32_candidates", C.c_size_t), ("greedy32_step_ms", C.c_float),
                ("greedy32_steps", C.c_int)]


class RewardConfigC(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("t_sla_ms", "l_baseline_ms", "c_budget", "w_latency",
                                          "w_cost", "w_proactive", "r_max")]


class RewardInputsC(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("l_before_ms", "l_after_ms", "c_before", "c_after")]


class RewardBreakdownC(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("latency", "cost", "sla", "proactive", "pareto",
                                          "total")] + [("clipped", C.c_int)]


_dp = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_u8p = C.POINTER(C.c_uint8)
_u32p = C.POINTER(C.c_uint32)
_szp = C.POINTER(C.c_size_t)
_vp = C.c_void_p

SIGNATURES = {
    "sair_last_error": (C.c_char_p, []),
    "sair_version": (C.c_int, []),
    "sair_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "sair_store_create": (C.c_int, [C.c_double, C.c_int, C.c_size_t, C.POINTER(_vp)]),
    "sair_store_destroy": (C.c_int, [_vp]),
    "sair_store_clone": (C.c_int, [_vp, C.POINTER(_vp)]),
    "sair_store_append": (C.c_int, [_vp, _dp, C.c_size_t, C.c_int, _dp, _i32p, _u8p, _szp]),
    "sair_store_append_synthetic": (C.c_int, [_vp, C.c_uint64, C.c_size_t, C.c_int, C.c_int]),
    "sair_store_size": (C.c_int, [_vp, _szp]),
    "sair_store_dim": (C.c_int, [_vp, C.POINTER(C.c_int)]),
    "sair_store_rejected": (C.c_int, [_vp, C.POINTER(C.c_uint64)]),
    "sair_store_r_min": (C.c_int, [_vp, _dp]),
    "sair_store_get": (C.c_int, [_vp, C.c_size_t, _dp, _dp, _i32p]),
    "sair_store_standardize": (C.c_int, [_vp, _dp, C.c_int, _dp]),
    "sair_store_effective_sigma": (C.c_int, [_vp, C.c_double, _dp]),
    "sair_similarity": (C.c_int, [_dp, C.c_size_t, _dp, C.c_size_t, C.c_double, _dp]),
    "sair_store_surprisal": (C.c_int, [_vp, C.c_size_t, _dp, C.c_int,
                                       C.POINTER(SelectConfigC), _dp]),
    "sair_store_select": (C.c_int, [_vp, _dp, C.c_size_t, C.c_int, C.POINTER(SelectConfigC),
                                    _i64p, _dp, _dp, _szp, _i64p, _dp]),
    "sair_store_nearest": (C.c_int, [_vp, _dp, C.c_size_t, C.c_int, C.c_double, _i64p, _dp]),
    "sair_store_export": (C.c_int, [_vp, C.c_size_t, C.c_size_t, _dp, _dp, C.POINTER(C.c_int32)]),
    "sair_store_load_jsonl": (C.c_int, [C.c_char_p, C.c_double, C.c_int, C.c_int,
                                        C.POINTER(C.c_size_t), C.POINTER(_vp)]),
    "sair_store_persist_jsonl": (C.c_int, [_vp, C.c_char_p]),
    "sair_store_greedy_begin": (C.c_int, [_vp, _dp, C.c_size_t, C.c_int,
                                          C.POINTER(SelectConfigC), _dp]),
    "sair_store_greedy_next": (C.c_int, [_vp, C.POINTER(C.c_int64), _dp, _dp]),
    "sair_merge_topk_packed": (C.c_int, [_vp, C.c_size_t, C.c_size_t, C.c_size_t, C.c_int, _vp,
                                         _vp]),
    "sair_store_last_stats": (C.c_int, [_vp, C.POINTER(SelectStatsC)]),
    "sair_store_stream": (C.c_int, [_vp, C.POINTER(_vp)]),
    "sair_store_set_shard": (C.c_int, [_vp, C.c_int64]),
    "sair_store_local_stats": (C.c_int, [_vp, _dp, _dp, _dp, _dp]),
    "sair_store_set_global": (C.c_int, [_vp, C.c_uint64, _dp, _dp, _dp, C.c_double, C.c_double,
                                        C.c_double]),
    "sair_store_moments": (C.c_int, [_vp, _dp, _dp]),
    "sair_sigma_sample_indices": (C.c_int, [C.c_uint64, _i64p, _szp]),
    "sair_sigma_rows": (C.c_int, [_dp, C.c_size_t, C.c_int, _dp, _dp, C.c_int, _dp]),
    "sair_store_select_shard": (C.c_int, [_vp, _dp, C.c_size_t, C.c_int, C.POINTER(SelectConfigC),
                                          _i64p, _dp, _dp, _dp, _i32p, _szp]),
    "sair_merge_topk": (C.c_int, [_dp, _dp, _dp, _i32p, _i64p, _szp, C.c_size_t, C.c_size_t,
                                  C.c_size_t, C.c_int, _i64p, _dp, _dp, _szp]),
    "sair_comm_create": (C.c_int, [C.POINTER(C.c_int), C.c_int, C.POINTER(_vp)]),
    "sair_comm_destroy": (C.c_int, [_vp]),
    "sair_comm_info": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "sair_sharded_create": (C.c_int, [_vp, C.c_double, C.c_size_t, C.POINTER(_vp)]),
    "sair_sharded_destroy": (C.c_int, [_vp]),
    "sair_sharded_append": (C.c_int, [_vp, _dp, C.c_size_t, C.c_int, _dp, _i32p, _u8p, _szp]),
    "sair_sharded_append_synthetic": (C.c_int, [_vp, C.c_uint64, C.c_size_t, C.c_int, C.c_int]),
    "sair_sharded_size": (C.c_int, [_vp, _szp, C.POINTER(C.c_uint64), _szp]),
    "sair_sharded_effective_sigma": (C.c_int, [_vp, C.c_double, _dp]),
    "sair_store_select_sharded": (C.c_int, [_vp, _dp, C.c_size_t, C.c_int,
                                            C.POINTER(SelectConfigC), _i64p, _dp, _dp, _szp]),
    "sair_frontier_insert_batch_sharded": (C.c_int, [_vp, _vp, _dp, C.c_size_t, _szp]),
    "sair_frontier_create": (C.c_int, [C.c_double, C.c_double, C.c_int, C.POINTER(_vp)]),
    "sair_frontier_destroy": (C.c_int, [_vp]),
    "sair_frontier_clone": (C.c_int, [_vp, C.POINTER(_vp)]),
    "sair_frontier_normalize": (C.c_int, [_vp, C.c_double, C.c_double, _dp, _dp,
                                          C.POINTER(C.c_int)]),
    "sair_frontier_update": (C.c_int, [_vp, C.c_double, C.c_double, C.POINTER(C.c_int),
                                       C.POINTER(C.c_int)]),
    "sair_frontier_insert_normalized": (C.c_int, [_vp, C.c_double, C.c_double,
                                                  C.POINTER(C.c_int)]),
    "sair_frontier_insert_batch": (C.c_int, [_vp, _dp, C.c_size_t, _szp]),
    "sair_frontier_size": (C.c_int, [_vp, _szp]),
    "sair_frontier_points": (C.c_int, [_vp, _dp, _dp, C.c_size_t, _szp]),
    "sair_frontier_bounds": (C.c_int, [_vp, _dp, _dp]),
    "sair_frontier_hypervolume": (C.c_int, [_vp, _dp]),
    "sair_frontier_strictly_dominated": (C.c_int, [_vp, C.c_double, C.c_double,
                                                   C.POINTER(C.c_int)]),
    "sair_frontier_contribution": (C.c_int, [_vp, C.c_double, C.c_double, _dp]),
    "sair_frontier_distance": (C.c_int, [_vp, C.c_double, C.c_double, _dp, C.POINTER(C.c_int)]),
    "sair_frontier_reward": (C.c_int, [_vp, C.c_double, C.c_double, _dp]),
    "sair_frontier_score_batch": (C.c_int, [_vp, _dp, C.c_size_t, _dp, _u8p]),
    "sair_frontier_score_batch_device": (C.c_int, [_vp, C.c_void_p, C.c_size_t, C.c_void_p,
                                                   C.c_void_p, C.c_void_p]),
    "sair_dominance_counts": (C.c_int, [_dp, C.c_size_t, C.c_int, C.c_int, _u32p, _u8p]),
    "sair_dominance_counts_part": (C.c_int, [_dp, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_int,
                                             _u32p, _u8p]),
    "sair_action_magnitude": (C.c_int, [_i32p, C.c_size_t, _dp]),
    "sair_compute_reward": (C.c_int, [C.POINTER(RewardInputsC), _i32p, C.c_size_t, _vp,
                                      C.POINTER(RewardConfigC), C.POINTER(RewardBreakdownC)]),
    "sair_decision_step": (C.c_int, [_vp, _vp, _dp, C.c_int, C.POINTER(SelectConfigC),
                                     C.POINTER(RewardInputsC), _i32p, C.c_size_t,
                                     C.POINTER(RewardConfigC), C.c_int, C.c_int32, _i64p, _dp,
                                     _dp, _szp, _i64p, _dp, C.POINTER(RewardBreakdownC),
                                     C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "sair_compute_reward_batch": (C.c_int, [C.POINTER(RewardInputsC), _i32p, C.c_size_t,
                                            C.c_size_t, _vp, C.POINTER(RewardConfigC),
                                            C.POINTER(RewardBreakdownC)]),
    "sair_frontier_set_create": (C.c_int, [C.c_size_t, C.c_double, C.c_double, C.c_int,
                                           C.POINTER(_vp)]),
    "sair_frontier_set_destroy": (C.c_int, [_vp]),
    "sair_frontier_set_step": (C.c_int, [_vp, C.POINTER(RewardInputsC), _i32p, C.c_size_t,
                                         C.POINTER(C.c_uint8), C.POINTER(RewardConfigC),
                                         C.POINTER(RewardBreakdownC)]),
    "sair_frontier_set_points": (C.c_int, [_vp, C.c_size_t, _dp, _dp, C.c_size_t,
                                           C.POINTER(C.c_size_t), _dp]),
    "sair_compute_reward_replay": (C.c_int, [C.POINTER(RewardInputsC), _i32p, C.c_size_t,
                                             C.c_size_t, C.POINTER(C.c_uint8), _vp,
                                             C.POINTER(RewardConfigC),
                                             C.POINTER(RewardBreakdownC)]),
}


def header_symbols() -> list[str]:
    """Every function include/sair.h declares (SAIR_API ... name(...))."""
    text = HEADER.read_text()
    return sorted(set(re.findall(r"SAIR_API\s+[\w\s\*]+?\b(sair_\w+)\s*\(", text)))


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: build it with `make -C "
                              f"{PKG / 'csrc'}` (there is no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


def check(rc: int):
    if rc != SAIR_OK:
        raise SairError(rc, lib().sair_last_error().decode(errors="replace"))
