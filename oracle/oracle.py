"""ctypes bindings for the CPU checkers (TEST INFRASTRUCTURE ONLY).

* ``C``   -- oracle/liboracle.so, the plain-C restatement (sair_oracle.c).
* ``Ref`` -- oracle/_ref/libsair_ref.so, the reference's own
  experience/pareto/reward.cpp compiled unmodified (oracle/Makefile).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this module.
The product package (paper_2601_22397_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libsair_ref.so"

_dp = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_u32p = C.POINTER(C.c_uint32)
_u8p = C.POINTER(C.c_uint8)
_szp = C.POINTER(C.c_size_t)
_sz = C.c_size_t


def _p(a, t):
    return a.ctypes.data_as(t) if a is not None else None


def build():
    """Compile the checkers (reference part only when /root/reference exists)."""
    import subprocess
    targets = ["oracle"]
    if Path("/root/reference/proj/src/experience.cpp").exists():
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", str(HERE)] + targets, check=True)


# ----------------------------------------------------------------------------
# C restatement
# ----------------------------------------------------------------------------
class COracle:
    def __init__(self, path: Path = ORACLE_SO):
        if not path.exists():
            build()
        L = self.lib = C.CDLL(str(path))
        L.orc_stats.argtypes = [_dp, _sz, C.c_int, _dp, _dp]
        L.orc_reward_total.argtypes = [_dp, _sz]
        L.orc_reward_total.restype = C.c_double
        L.orc_standardize.argtypes = [_sz, C.c_int, _dp, _dp, _dp, _dp]
        L.orc_similarity.argtypes = [_dp, _dp, C.c_int, C.c_double]
        L.orc_similarity.restype = C.c_double
        L.orc_sigma_median.argtypes = [_dp, _sz, C.c_int, _dp, _dp]
        L.orc_sigma_median.restype = C.c_double
        L.orc_select.argtypes = [_dp, _dp, _i32p, _sz, C.c_int, _dp, _dp, _dp, _sz, C.c_double,
                                 C.c_double, C.c_int, _i64p, _dp, _dp]
        L.orc_select.restype = _sz
        L.orc_select_batch.argtypes = [_dp, _dp, _i32p, _sz, C.c_int, _dp, _dp, _dp, _sz, _sz,
                                       C.c_double, C.c_double, C.c_int, _i64p, _dp, _dp, _szp]
        L.orc_select_shard.argtypes = [_dp, _dp, _i32p, _sz, C.c_int, _dp, _dp, _sz, C.c_double,
                                       _dp, _sz, C.c_double, _i64p, _dp, _dp]
        L.orc_select_shard.restype = _sz
        L.orc_sigma_rows.argtypes = [_dp, _sz, C.c_int, _sz, _dp, _dp]
        L.orc_sigma_rows.restype = C.c_double
        L.orc_surprisal.argtypes = [_dp, _dp, _sz, C.c_int, _dp, _dp, _sz, _dp, C.c_double,
                                    C.c_int]
        L.orc_surprisal.restype = C.c_double
        L.orc_nearest.argtypes = [_dp, _sz, C.c_int, _dp, _dp, _dp, C.c_double, _dp]
        L.orc_nearest.restype = C.c_int64
        L.orc_normalize.argtypes = [C.c_double] * 4 + [_dp, _dp, C.POINTER(C.c_int)]
        L.orc_strictly_dominated.argtypes = [_dp, _dp, _sz, C.c_double, C.c_double]
        L.orc_frontier_insert.argtypes = [_dp, _dp, _szp, C.c_double, C.c_double]
        L.orc_hypervolume.argtypes = [_dp, _dp, _sz]
        L.orc_hypervolume.restype = C.c_double
        for f in ("orc_contribution", "orc_distance", "orc_pareto_reward"):
            getattr(L, f).argtypes = [_dp, _dp, _sz, C.c_double, C.c_double]
            getattr(L, f).restype = C.c_double
        L.orc_pareto_reward_batch.argtypes = [_dp, _dp, _sz, _dp, _sz, _dp]
        L.orc_frontier_insert_seq.argtypes = [_dp, _dp, _sz, _dp, _sz, _u8p]
        L.orc_frontier_insert_seq.restype = _sz
        L.orc_dominance_counts.argtypes = [_dp, _sz, C.c_int, _u32p, _u8p]
        L.orc_dominance_counts_mt.argtypes = [_dp, _sz, C.c_int, C.c_int, _u32p, _u8p]
        L.orc_dominance_counts2_sorted.argtypes = [_dp, _sz, _u32p, _u8p]
        L.orc_frontier_sorted.argtypes = [_dp, _sz, _dp, _dp]
        L.orc_frontier_sorted.restype = _sz
        L.orc_synth_contexts.argtypes = [C.c_int64, _sz, _sz, C.c_int, C.c_int, _dp]
        L.orc_action_magnitude.argtypes = [_i32p, _sz]
        L.orc_action_magnitude.restype = C.c_double
        L.orc_compute_reward.argtypes = [_dp, C.c_double, _dp, _dp, _sz, C.c_double, C.c_double,
                                         _dp, _dp]

    # -- retrieval --
    def synth_contexts(self, seed, start, count, d, nthreads=None):
        """synth.contexts (non-clustered) on host threads: [count, d] float64."""
        out = np.empty((count, d), np.float64)
        self.lib.orc_synth_contexts(seed, start, count, d, nthreads or os.cpu_count() or 1,
                                    _p(out, _dp))
        return out

    def stats(self, ctx):
        ctx = np.ascontiguousarray(ctx, np.float64)
        n, d = ctx.shape
        s = np.zeros(d)
        ss = np.zeros(d)
        self.lib.orc_stats(_p(ctx, _dp), n, d, _p(s, _dp), _p(ss, _dp))
        return s, ss

    def standardize(self, n, s, ss, x):
        x = np.ascontiguousarray(x, np.float64)
        z = np.empty_like(x)
        self.lib.orc_standardize(n, len(x), _p(s, _dp), _p(ss, _dp), _p(x, _dp), _p(z, _dp))
        return z

    def sigma_median(self, ctx):
        ctx = np.ascontiguousarray(ctx, np.float64)
        s, ss = self.stats(ctx)
        return self.lib.orc_sigma_median(_p(ctx, _dp), ctx.shape[0], ctx.shape[1], _p(s, _dp),
                                         _p(ss, _dp))

    def select(self, ctx, reward, rounds, x, m, lam, sigma, local_mean=False, stats=None):
        ctx = np.ascontiguousarray(ctx, np.float64)
        reward = np.ascontiguousarray(reward, np.float64)
        rounds = np.ascontiguousarray(rounds, np.int32)
        x = np.ascontiguousarray(x, np.float64)
        n, d = ctx.shape
        s, ss = stats if stats is not None else self.stats(ctx)
        idx = np.full(max(m, 1), -1, np.int64)
        sim = np.zeros(max(m, 1))
        sc = np.zeros(max(m, 1))
        k = self.lib.orc_select(_p(ctx, _dp), _p(reward, _dp), _p(rounds, _i32p), n, d,
                                _p(s, _dp), _p(ss, _dp), _p(x, _dp), m, lam, sigma,
                                int(local_mean), _p(idx, _i64p), _p(sim, _dp), _p(sc, _dp))
        return idx[:k], sim[:k], sc[:k]

    def select_batch(self, ctx, reward, rounds, xq, m, lam, sigma, nthreads=None, stats=None):
        ctx = np.ascontiguousarray(ctx, np.float64)
        reward = np.ascontiguousarray(reward, np.float64)
        rounds = np.ascontiguousarray(rounds, np.int32)
        xq = np.ascontiguousarray(xq, np.float64)
        n, d = ctx.shape
        nq = xq.shape[0]
        s, ss = stats if stats is not None else self.stats(ctx)
        idx = np.full((nq, m), -1, np.int64)
        sim = np.zeros((nq, m))
        sc = np.zeros((nq, m))
        cnt = np.zeros(nq, np.uintp)
        self.lib.orc_select_batch(_p(ctx, _dp), _p(reward, _dp), _p(rounds, _i32p), n, d,
                                  _p(s, _dp), _p(ss, _dp), _p(xq, _dp), nq, m, lam, sigma,
                                  nthreads or os.cpu_count(), _p(idx, _i64p), _p(sim, _dp),
                                  _p(sc, _dp), cnt.ctypes.data_as(_szp))
        return idx, sim, sc, cnt.astype(np.int64)

    def select_shard(self, ctx, reward, rounds, x, m, sigma, n_global, s, ss, total):
        ctx = np.ascontiguousarray(ctx, np.float64)
        reward = np.ascontiguousarray(reward, np.float64)
        rounds = np.ascontiguousarray(rounds, np.int32)
        x = np.ascontiguousarray(x, np.float64)
        s = np.ascontiguousarray(s, np.float64)
        ss = np.ascontiguousarray(ss, np.float64)
        n, d = ctx.shape
        idx = np.full(max(m, 1), -1, np.int64)
        sim = np.zeros(max(m, 1))
        sc = np.zeros(max(m, 1))
        k = self.lib.orc_select_shard(_p(ctx, _dp), _p(reward, _dp), _p(rounds, _i32p), n, d,
                                      _p(s, _dp), _p(ss, _dp), n_global, total, _p(x, _dp), m,
                                      sigma, _p(idx, _i64p), _p(sim, _dp), _p(sc, _dp))
        return idx[:k], sim[:k], sc[:k]

    def sigma_rows(self, rows, n, s, ss):
        rows = np.ascontiguousarray(rows, np.float64)
        return self.lib.orc_sigma_rows(_p(rows, _dp), rows.shape[0], rows.shape[1], n,
                                       _p(np.ascontiguousarray(s), _dp),
                                       _p(np.ascontiguousarray(ss), _dp))

    def surprisal(self, ctx, reward, index, x, sigma, local_mean=False):
        ctx = np.ascontiguousarray(ctx, np.float64)
        reward = np.ascontiguousarray(reward, np.float64)
        x = np.ascontiguousarray(x, np.float64)
        s, ss = self.stats(ctx)
        return self.lib.orc_surprisal(_p(ctx, _dp), _p(reward, _dp), ctx.shape[0], ctx.shape[1],
                                      _p(s, _dp), _p(ss, _dp), index, _p(x, _dp), sigma,
                                      int(local_mean))

    def nearest(self, ctx, x, sigma):
        ctx = np.ascontiguousarray(ctx, np.float64)
        x = np.ascontiguousarray(x, np.float64)
        s, ss = self.stats(ctx)
        out = C.c_double()
        i = self.lib.orc_nearest(_p(ctx, _dp), ctx.shape[0], ctx.shape[1], _p(s, _dp),
                                 _p(ss, _dp), _p(x, _dp), sigma, C.byref(out))
        return i, out.value

    # -- pareto --
    def frontier_from_points(self, pts):
        """Sequential insert of normalized points into an empty frontier."""
        pts = np.ascontiguousarray(pts, np.float64).reshape(-1, 2)
        fl = np.zeros(len(pts) + 1)
        fc = np.zeros(len(pts) + 1)
        ins = np.zeros(len(pts), np.uint8)
        F = self.lib.orc_frontier_insert_seq(_p(fl, _dp), _p(fc, _dp), 0, _p(pts, _dp),
                                             len(pts), _p(ins, _u8p))
        return fl[:F].copy(), fc[:F].copy(), ins.astype(bool)

    def pareto_reward_batch(self, fl, fc, pts):
        fl = np.ascontiguousarray(fl, np.float64)
        fc = np.ascontiguousarray(fc, np.float64)
        pts = np.ascontiguousarray(pts, np.float64).reshape(-1, 2)
        out = np.zeros(len(pts))
        self.lib.orc_pareto_reward_batch(_p(fl, _dp), _p(fc, _dp), len(fl), _p(pts, _dp),
                                         len(pts), _p(out, _dp))
        return out

    def hypervolume(self, fl, fc):
        fl = np.ascontiguousarray(fl, np.float64)
        fc = np.ascontiguousarray(fc, np.float64)
        return self.lib.orc_hypervolume(_p(fl, _dp), _p(fc, _dp), len(fl))

    def contribution(self, fl, fc, l, c):
        fl = np.ascontiguousarray(fl, np.float64)
        fc = np.ascontiguousarray(fc, np.float64)
        return self.lib.orc_contribution(_p(fl, _dp), _p(fc, _dp), len(fl), l, c)

    def distance(self, fl, fc, l, c):
        fl = np.ascontiguousarray(fl, np.float64)
        fc = np.ascontiguousarray(fc, np.float64)
        return self.lib.orc_distance(_p(fl, _dp), _p(fc, _dp), len(fl), l, c)

    def dominance_counts(self, tuples):
        t = np.ascontiguousarray(tuples, np.float64)
        T, K = t.shape
        cnt = np.zeros(T, np.uint32)
        mem = np.zeros(T, np.uint8)
        self.lib.orc_dominance_counts(_p(t, _dp), T, K, _p(cnt, _u32p), _p(mem, _u8p))
        return cnt, mem.astype(bool)

    def dominance_counts_mt(self, tuples, nthreads=None):
        """dominance_counts on all host threads (same per-tuple loop)."""
        t = np.ascontiguousarray(tuples, np.float64)
        T, K = t.shape
        cnt = np.zeros(T, np.uint32)
        mem = np.zeros(T, np.uint8)
        self.lib.orc_dominance_counts_mt(_p(t, _dp), T, K, nthreads or os.cpu_count() or 1,
                                         _p(cnt, _u32p), _p(mem, _u8p))
        return cnt, mem.astype(bool)

    def dominance_counts2_sorted(self, tuples):
        """Two-objective counts in O(T log T) (sweep + Fenwick tree)."""
        t = np.ascontiguousarray(tuples, np.float64).reshape(-1, 2)
        cnt = np.zeros(len(t), np.uint32)
        mem = np.zeros(len(t), np.uint8)
        self.lib.orc_dominance_counts2_sorted(_p(t, _dp), len(t), _p(cnt, _u32p), _p(mem, _u8p))
        return cnt, mem.astype(bool)

    def frontier_sorted(self, pts):
        """The frontier the sequential insert loop leaves, for millions of points."""
        t = np.ascontiguousarray(pts, np.float64).reshape(-1, 2)
        fl = np.zeros(max(len(t), 1))
        fc = np.zeros(max(len(t), 1))
        F = self.lib.orc_frontier_sorted(_p(t, _dp), len(t), _p(fl, _dp), _p(fc, _dp))
        return fl[:F].copy(), fc[:F].copy()

    def action_magnitude(self, deltas):
        d = np.ascontiguousarray(deltas, np.int32).reshape(-1, 4)
        return self.lib.orc_action_magnitude(_p(d, _i32p), len(d))

    def compute_reward(self, inputs, deltas, fl, fc, l_max, c_max, cfg):
        """cfg = (t_sla, l_baseline(0 => 4*t_sla), c_budget, w_l, w_c, w_p, r_max)."""
        cfg = np.array(cfg, np.float64)
        if cfg[1] <= 0:
            cfg[1] = 4.0 * cfg[0]
        fl = np.ascontiguousarray(fl, np.float64)
        fc = np.ascontiguousarray(fc, np.float64)
        inp = np.array(inputs, np.float64)
        out = np.zeros(7)
        rc = self.lib.orc_compute_reward(_p(inp, _dp), self.action_magnitude(deltas), _p(fl, _dp),
                                         _p(fc, _dp), len(fl), l_max, c_max, _p(cfg, _dp),
                                         _p(out, _dp))
        if rc != 0:
            raise ValueError("reward: invalid configuration")
        return out


# ----------------------------------------------------------------------------
# The reference itself
# ----------------------------------------------------------------------------
class RefError(Exception):
    pass


class Ref:
    def __init__(self, path: Path = REF_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (make -C oracle ref)")
        L = self.lib = C.CDLL(str(path))
        L.ref_last_error.restype = C.c_char_p
        L.ref_buffer_new.argtypes = [C.c_double]
        L.ref_buffer_new.restype = C.c_void_p
        L.ref_buffer_free.argtypes = [C.c_void_p]
        L.ref_buffer_store.argtypes = [C.c_void_p, _dp, C.c_int, C.c_double, C.c_int,
                                       C.POINTER(C.c_int)]
        L.ref_buffer_store_many.argtypes = [C.c_void_p, _dp, _sz, C.c_int, _dp, _i32p]
        L.ref_buffer_size.argtypes = [C.c_void_p]
        L.ref_buffer_size.restype = _sz
        L.ref_buffer_rejected.argtypes = [C.c_void_p]
        L.ref_buffer_rejected.restype = C.c_uint64
        L.ref_buffer_standardize.argtypes = [C.c_void_p, _dp, C.c_int, _dp]
        L.ref_buffer_effective_sigma.argtypes = [C.c_void_p, C.c_double, _dp]
        L.ref_buffer_surprisal.argtypes = [C.c_void_p, _sz, _dp, C.c_int, C.c_double, C.c_int,
                                           _dp]
        L.ref_buffer_select.argtypes = [C.c_void_p, _dp, C.c_int, _sz, C.c_double, C.c_double,
                                        C.c_int, _i32p, _dp, _dp, _szp]
        L.ref_buffer_select_batch.argtypes = [C.c_void_p, _dp, _sz, C.c_int, _sz, C.c_double,
                                              C.c_double, C.c_int, _i32p, _dp, _szp]
        L.ref_similarity.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_double, _dp]
        L.ref_frontier_new.argtypes = [C.c_double, C.c_double, C.POINTER(C.c_void_p)]
        L.ref_frontier_free.argtypes = [C.c_void_p]
        L.ref_frontier_update.argtypes = [C.c_void_p, C.c_double, C.c_double,
                                          C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.ref_frontier_insert_normalized.argtypes = [C.c_void_p, C.c_double, C.c_double]
        L.ref_frontier_points.argtypes = [C.c_void_p, _dp, _dp]
        L.ref_frontier_points.restype = _sz
        L.ref_frontier_hypervolume.argtypes = [C.c_void_p]
        L.ref_frontier_hypervolume.restype = C.c_double
        L.ref_frontier_contribution.argtypes = [C.c_void_p, C.c_double, C.c_double, _dp]
        L.ref_frontier_strictly_dominated.argtypes = [C.c_void_p, C.c_double, C.c_double]
        for f in ("ref_frontier_distance", "ref_frontier_reward"):
            getattr(L, f).argtypes = [C.c_void_p, C.c_double, C.c_double]
            getattr(L, f).restype = C.c_double
        L.ref_frontier_normalize.argtypes = [C.c_void_p, C.c_double, C.c_double, _dp, _dp,
                                             C.POINTER(C.c_int)]
        L.ref_frontier_reward_batch.argtypes = [C.c_void_p, _dp, _sz, _dp]
        L.ref_frontier_insert_batch.argtypes = [C.c_void_p, _dp, _sz, _u8p]
        L.ref_compute_reward.argtypes = [_dp, _i32p, _sz, C.c_void_p, _dp, _dp]
        L.ref_action_magnitude.argtypes = [_i32p, _sz]
        L.ref_action_magnitude.restype = C.c_double
        L.ref_buffer_load.argtypes = [C.c_char_p, C.c_double, _szp]
        L.ref_buffer_load.restype = C.c_void_p
        L.ref_buffer_persist.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_buffer_get.argtypes = [C.c_void_p, _sz, _dp, _dp, C.POINTER(C.c_int)]

    def _chk(self, rc):
        if rc:
            msg = self.lib.ref_last_error().decode()
            raise {1: ValueError, 2: RuntimeError}.get(rc, RefError)(msg)


class RefBuffer:
    """The reference ExperienceBuffer (experience.hpp:45-89) behind ctypes."""

    def __init__(self, ref: Ref, r_min=0.0):
        self.ref, self.L = ref, ref.lib
        self.h = self.L.ref_buffer_new(r_min)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_buffer_free(self.h)
            self.h = None

    def store(self, ctx, reward, round_):
        x = np.ascontiguousarray(ctx, np.float64)
        acc = C.c_int()
        self.ref._chk(self.L.ref_buffer_store(self.h, _p(x, _dp), len(x), reward, round_,
                                              C.byref(acc)))
        return bool(acc.value)

    def store_many(self, ctx, reward, rounds):
        ctx = np.ascontiguousarray(ctx, np.float64)
        reward = np.ascontiguousarray(reward, np.float64)
        rounds = np.ascontiguousarray(rounds, np.int32)
        self.ref._chk(self.L.ref_buffer_store_many(self.h, _p(ctx, _dp), ctx.shape[0],
                                                   ctx.shape[1], _p(reward, _dp),
                                                   _p(rounds, _i32p)))

    def size(self):
        return self.L.ref_buffer_size(self.h)

    @classmethod
    def load(cls, ref: "Ref", path, r_min=0.0):
        """ExperienceBuffer::load (experience.cpp:243-271): (buffer, corrupt)."""
        bad = C.c_size_t()
        h = ref.lib.ref_buffer_load(str(path).encode(), r_min, C.byref(bad))
        if not h:
            raise ValueError(ref.lib.ref_last_error().decode())
        o = cls.__new__(cls)
        o.ref, o.L, o.h = ref, ref.lib, h
        return o, bad.value

    def persist(self, path):
        self.ref._chk(self.L.ref_buffer_persist(self.h, str(path).encode()))

    def get(self, i, d):
        ctx = np.zeros(d)
        r = C.c_double()
        rd = C.c_int()
        self.ref._chk(self.L.ref_buffer_get(self.h, i, _p(ctx, _dp), C.byref(r), C.byref(rd)))
        return ctx, r.value, rd.value

    def rejected(self):
        return self.L.ref_buffer_rejected(self.h)

    def standardize(self, x):
        x = np.ascontiguousarray(x, np.float64)
        z = np.empty_like(x)
        self.ref._chk(self.L.ref_buffer_standardize(self.h, _p(x, _dp), len(x), _p(z, _dp)))
        return z

    def effective_sigma(self, sigma_sim=0.0):
        out = C.c_double()
        self.ref._chk(self.L.ref_buffer_effective_sigma(self.h, sigma_sim, C.byref(out)))
        return out.value

    def surprisal(self, index, x, sigma_sim=0.0, local_mean=False):
        x = np.ascontiguousarray(x, np.float64)
        out = C.c_double()
        self.ref._chk(self.L.ref_buffer_surprisal(self.h, index, _p(x, _dp), len(x), sigma_sim,
                                                  int(local_mean), C.byref(out)))
        return out.value

    def select(self, x, m=15, lambda_div=0.1, sigma_sim=0.0, local_mean=False):
        x = np.ascontiguousarray(x, np.float64)
        r = np.zeros(max(m, 1), np.int32)
        sim = np.zeros(max(m, 1))
        sc = np.zeros(max(m, 1))
        cnt = C.c_size_t()
        self.ref._chk(self.L.ref_buffer_select(self.h, _p(x, _dp), len(x), m, lambda_div,
                                               sigma_sim, int(local_mean), _p(r, _i32p),
                                               _p(sim, _dp), _p(sc, _dp), C.byref(cnt)))
        k = cnt.value
        return r[:k], sim[:k], sc[:k]

    def select_batch(self, xq, m, lambda_div, sigma_sim=0.0, nthreads=None):
        xq = np.ascontiguousarray(xq, np.float64)
        nq, d = xq.shape
        r = np.full((nq, m), -1, np.int32)
        sc = np.zeros((nq, m))
        cnt = np.zeros(nq, np.uintp)
        self.ref._chk(self.L.ref_buffer_select_batch(self.h, _p(xq, _dp), nq, d, m, lambda_div,
                                                     sigma_sim, nthreads or os.cpu_count(),
                                                     _p(r, _i32p), _p(sc, _dp),
                                                     cnt.ctypes.data_as(_szp)))
        return r, sc, cnt.astype(np.int64)


class RefFrontier:
    """The reference ParetoFrontier (pareto.hpp:24-70) behind ctypes."""

    def __init__(self, ref: Ref, l_max=1.0, c_max=1.0):
        self.ref, self.L = ref, ref.lib
        h = C.c_void_p()
        ref._chk(self.L.ref_frontier_new(l_max, c_max, C.byref(h)))
        self.h = h.value

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_frontier_free(self.h)
            self.h = None

    def update(self, l_ms, cost):
        ins, cl = C.c_int(), C.c_int()
        self.ref._chk(self.L.ref_frontier_update(self.h, l_ms, cost, C.byref(ins), C.byref(cl)))
        return bool(ins.value), bool(cl.value)

    def insert_normalized(self, l, c):
        return bool(self.L.ref_frontier_insert_normalized(self.h, l, c))

    def points(self):
        F = self.L.ref_frontier_points(self.h, None, None)
        fl, fc = np.zeros(F), np.zeros(F)
        self.L.ref_frontier_points(self.h, _p(fl, _dp), _p(fc, _dp))
        return fl, fc

    def hypervolume(self):
        return self.L.ref_frontier_hypervolume(self.h)

    def contribution(self, l, c):
        out = C.c_double()
        self.ref._chk(self.L.ref_frontier_contribution(self.h, l, c, C.byref(out)))
        return out.value

    def strictly_dominated(self, l, c):
        return bool(self.L.ref_frontier_strictly_dominated(self.h, l, c))

    def distance(self, l, c):
        d = self.L.ref_frontier_distance(self.h, l, c)
        return None if d < 0 else d

    def reward(self, l, c):
        return self.L.ref_frontier_reward(self.h, l, c)

    def normalize(self, l_ms, cost):
        l, c, cl = C.c_double(), C.c_double(), C.c_int()
        self.L.ref_frontier_normalize(self.h, l_ms, cost, C.byref(l), C.byref(c), C.byref(cl))
        return l.value, c.value, bool(cl.value)

    def reward_batch(self, pts):
        pts = np.ascontiguousarray(pts, np.float64).reshape(-1, 2)
        out = np.zeros(len(pts))
        self.L.ref_frontier_reward_batch(self.h, _p(pts, _dp), len(pts), _p(out, _dp))
        return out

    def insert_batch(self, pts):
        pts = np.ascontiguousarray(pts, np.float64).reshape(-1, 2)
        ins = np.zeros(len(pts), np.uint8)
        self.L.ref_frontier_insert_batch(self.h, _p(pts, _dp), len(pts), _p(ins, _u8p))
        return ins.astype(bool)


def ref_compute_reward(ref: Ref, inputs, deltas, frontier: RefFrontier, cfg):
    inp = np.array(inputs, np.float64)
    d = np.ascontiguousarray(deltas, np.int32).reshape(-1, 4)
    cfgv = np.array(cfg, np.float64)
    out = np.zeros(7)
    ref._chk(ref.lib.ref_compute_reward(_p(inp, _dp), _p(d, _i32p), len(d), frontier.h,
                                        _p(cfgv, _dp), _p(out, _dp)))
    return out
