#!/usr/bin/env python
"""Benchmark: surprisal-guided retrieval over a 16M x 64 experience store
(BASELINE.json metric "retrieval queries/s @16M exps k=32; Pareto-scored
tuples/s; % HBM roofline"; configs[3]: 16M experiences, 4096 queries/batch,
k=32).

A step = one select() of a Q=4096 query batch (k = m = 32, lambda_div = 0, the
fused veto scan off) over the whole device-resident store: 16 wide tensor-core
passes of 256 queries over the store's bf16 page copy (select_wide.cu), each
after a TF32 sample pass for its start thresholds.  Also measured in the same run:
"hbm_target" -- Q=8 queries per step, the single HBM-bound pass of the north
star's >= 70% HBM target (select_mma.cu); "config2" -- configs[1], 1M x 64
with 256-query batches; "pareto" -- configs[2], 4M 2-objective tuples
(frontier maintenance + per-tuple reward) and k-D dominance counts.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun, one rank per GPU): the 16M records are sharded contiguously
(strong scaling); each rank selects its shard's top-k and the per-shard
candidates are merged after an NCCL all-gather.  Timing is CUDA events on the
store's stream, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_RECORDS = 16 * 1024 * 1024
DIM = 64
Q = 4096
Q_HBM = 8
K_SEL = 32
SEED = 2026
PARETO_T = 4 * 1024 * 1024


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--records", type=int, default=N_RECORDS)
    ap.add_argument("--queries", type=int, default=Q)
    ap.add_argument("--lambda-div", type=float, default=0.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-pareto", action="store_true")
    # N > 1: "records" (configs[3]: "16M experiences sharded over 8 B200 ...
    # per-shard top-k merged via NCCL allgather") -- the store is sharded by
    # records (sharded.py) and every query's per-shard top-m are merged after
    # an NCCL all-gather; "queries" -- every rank holds the whole store and
    # serves a slice of each step's queries, no collective (reported as an
    # extra key, "query_shards", when the headline runs record shards)
    ap.add_argument("--shard", default=os.environ.get("SAIR_BENCH_SHARD", "records"),
                    choices=["queries", "records"])
    # launcher self-test (CPU, gloo): start the ranks, rendezvous, print the line
    ap.add_argument("--launcher-check", action="store_true", help=argparse.SUPPRESS)
    return ap.parse_args()


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        j = json.loads(p.read_text())
        return float(j["hbm_gbs"]), float(j.get("bf16_tflops", 1622.7)), "measured"
    return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.rows, self._stop = gpu, [], threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.FIELDS,
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ------------------------------------------------------------------ ours ---

def _launches(stats):
    """Our kernels per select() call, from its stats: per query group the
    threshold pre-pass (2), the stream pass and the list merge (wide: per-list
    top-K') and refine; 3 + 3m per exact fallback query."""
    per = {3: 5, 2: 5, 1: 5, 0: 3}
    return sum(per[s["tensor_core"]] * s["stream_launches"] + s["exact_fallbacks"] * (3 + 3 * K_SEL)
               for s in stats)


def _stream_roofline(stats, n_local, hbm_peak, peak_kind, bf16_peak, qw):
    """Roofline of the dominant kernel (the stream pass): algorithmic bytes =
    records x (4 d_pad + 4) per launch (the fp32 page row + the fp32 reward)
    / its CUDA-event time; the wide pass (qw > 0) reads the call's cached
    (P, log residual) pair instead of the reward: 4 d_pad + 8; on the bf16
    page copy (tensor_core 3) 2 d_pad + 8, and its GEMM runs at the bf16 rate."""
    launches = sum(s["stream_launches"] for s in stats)
    stream_ms = sum(s["stream_ms"] for s in stats)
    dp = 64 if DIM > 32 else 32
    b16 = bool(stats) and stats[0]["tensor_core"] == 3
    alg_bytes = n_local * ((2 if b16 else 4) * dp + (8 if qw else 4))
    per_launch_s = max(stream_ms / 1e3 / max(launches, 1), 1e-12)
    achieved = alg_bytes / per_launch_s / 1e9 if launches else 0.0
    out = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
           "frac": round(achieved / hbm_peak, 4), "peak_kind": peak_kind,
           "algorithmic_bytes_per_launch": alg_bytes, "avg_launch_ms": round(per_launch_s * 1e3, 4),
           "prepass_ms_per_launch": round(sum(s["prepass_ms"] for s in stats) / max(launches, 1), 4)}
    if qw:
        # the same launch as a GEMM: 2 x records x d_pad x QW flops, TF32 or bf16
        tf = 2.0 * n_local * dp * qw / per_launch_s / 1e12
        tpeak = bf16_peak if b16 else bf16_peak / 2
        out["tensor"] = {"achieved_tflops": round(tf, 1), "dtype": "bf16" if b16 else "tf32",
                         "peak_tflops": round(tpeak, 1), "frac": round(tf / tpeak, 4),
                         "peak_note": ("bf16 dense, measured (MEASURED_PEAKS.json)" if b16 else
                                       "TF32 dense = measured bf16 / 2 (nominal ratio)")}
        if out["tensor"]["frac"] > out["frac"]:
            # 256 queries per page visit: the launch does twice the tensor work
            # per HBM byte of a 128-query pass -- report it against the tensor
            # roofline (the HBM figures stay under "hbm")
            out["hbm"] = {k: out[k] for k in ("achieved", "peak", "unit", "frac", "peak_kind")}
            out.update({"bound": "tensor", "achieved": round(tf, 1), "peak": round(tpeak, 1),
                        "unit": "TFLOP/s", "frac": out["tensor"]["frac"],
                        "peak_kind": peak_kind + ("" if b16 else " (bf16 / 2)")})
    return out


def run_ours(a, rank, world, local_rank):
    import torch
    import paper_2601_22397_b200 as sair
    from paper_2601_22397_b200 import synth

    # one GPU per rank; SAIR_BENCH_BACKEND=gloo (with ranks sharing the
    # visible GPUs) only exercises the multi-rank code path on a smaller box
    backend = os.environ.get("SAIR_BENCH_BACKEND", "nccl")
    dev = local_rank % max(1, torch.cuda.device_count()) if backend != "nccl" else local_rank
    torch.cuda.set_device(dev)
    dist = None
    n_total = a.records
    cfg = sair.SelectionConfig(m=K_SEL, lambda_div=a.lambda_div)
    t0 = time.time()
    qlo, qhi = 0, a.queries
    if world > 1:
        import torch.distributed as dist
        from paper_2601_22397_b200.sharded import ShardedExperienceBuffer, shard_range
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)

    def make(mode):
        """(buffer, select, select_whole, lo, hi) for one way of spreading the
        step over the ranks."""
        if world > 1 and mode == "queries":
            # the whole store on every rank (device-generated from the same
            # seed: identical replicas); this rank's slice of every step's queries
            b = sair.ExperienceBuffer(0.0, device=dev)
            b.store_synthetic(SEED, n_total, DIM)

            def sel(q):
                a_, b_ = shard_range(len(q), rank, world)
                return b.select_batch(q[a_:b_], cfg)

            return b, sel, (lambda q: b.select_batch(q, cfg)), 0, n_total
        if world > 1:
            lo_, hi_ = shard_range(n_total, rank, world)
            sh = ShardedExperienceBuffer(dist, dev)
            sh.store_synthetic(SEED, n_total, DIM)

            def sel(q):
                return sh.select_batch(q, cfg)

            return sh.local, sel, sel, lo_, hi_
        b = sair.ExperienceBuffer(0.0, device=dev)
        b.store_synthetic(SEED, n_total, DIM)

        def sel(q):
            return b.select_batch(q, cfg)

        return b, sel, sel, 0, n_total

    buf, select, select_whole, lo, hi = make(a.shard)
    gen_s = time.time() - t0
    qpool = synth.queries(SEED, (a.warmup + a.steps) * a.queries, DIM).reshape(
        a.warmup + a.steps, a.queries, DIM)
    hbm_peak, bf16_peak, peak_kind = measured_peaks()

    def timed(qs, steps, select=select, b=None):
        """device time (CUDA events on the store's stream, max over ranks)"""
        b = b or buf
        stream = torch.cuda.ExternalStream(b.stream_ptr(), device=dev)
        stats = []
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(steps):
            select(qs[i])
            stats.append(b.last_stats())
        e1.record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        ms = e0.elapsed_time(e1)
        if dist:
            t = torch.tensor([ms], device=f"cuda:{dev}" if backend == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, stats

    for i in range(a.warmup):
        select(qpool[i])
    with ClockSampler(dev) as clk:
        ms, stats = timed(qpool[a.warmup:], a.steps)
    value = a.steps * a.queries / (ms / 1e3)

    # e2e: the public API with host queries and host results, wall clock
    # (host->device query copy and device->host result copy inside every step)
    t0 = time.perf_counter()
    for i in range(a.warmup, a.warmup + a.steps):
        select(qpool[i])
    if dist:
        dist.barrier()
    e2e_s = time.perf_counter() - t0
    if dist:
        t = torch.tensor([e2e_s], device=f"cuda:{dev}" if backend == "nccl" else "cpu",
                         dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = a.steps * a.queries / e2e_s

    qw = stats[0]["qb"] if stats[0]["tensor_core"] in (2, 3) else 0
    roof = _stream_roofline(stats, hi - lo, hbm_peak, peak_kind, bf16_peak, qw)
    tc = stats[0]["tensor_core"]
    dp = 64 if DIM > 32 else 32
    roof["kernel"] = (f"sair::stream_wide16_kernel<{qw}> (tcgen05 kind::f16, bf16 page copy, "
                      f"{qw} queries/pass)" if tc == 3
                      else f"sair::stream_wide_kernel<{dp},{qw},1> (tcgen05, {qw} queries/pass)" if tc == 2
                      else f"sair::stream_mma_kernel<{dp},8> (tcgen05)" if tc == 1
                      else f"sair::stream_kernel<{dp},8>")
    tp = ROOT / "profiles" / "stream_kernel_traffic.json"
    roof["traffic"] = None
    if tp.exists():
        tj = json.loads(tp.read_text()).get(roof["kernel"].split(" ")[0], {})
        if tj.get("dram_bytes_per_launch"):
            # ncu capture of a 16M-record launch; a shard's launch reads its share
            scale = (hi - lo) / float(tj.get("records", N_RECORDS))
            roof["traffic"] = round(tj["dram_bytes_per_launch"] * scale)
            roof["traffic_source"] = tj.get("source") + (
                f", scaled x{scale:.3f} to this rank's records" if scale != 1.0 else "")
    gpu_launches = _launches(stats) + (a.steps if dist and a.shard == "records" else 0)

    # the north star's HBM target: Q = 8 queries per step, one memory-bound pass
    qh = synth.queries(SEED + 7, (3 + a.steps) * Q_HBM, DIM).reshape(3 + a.steps, Q_HBM, DIM)
    for i in range(3):
        select_whole(qh[i])
    ms_h, st_h = timed(qh[3:], a.steps, select_whole)
    roof_h = _stream_roofline(st_h, hi - lo, hbm_peak, peak_kind, bf16_peak, 0)
    roof_h["kernel"] = f"sair::stream_mma_kernel<{dp},8> (tcgen05)"
    hbm_target = {"queries_per_step": Q_HBM, "value": round(a.steps * Q_HBM / (ms_h / 1e3), 2),
                  "unit": "queries/s", "ms_per_step": round(ms_h / a.steps, 4), "roofline": roof_h,
                  "certified_queries": sum(s["certified"] for s in st_h)}
    # the rest of the north star's Q in {1, 2, 4, 8}: the same pass, fewer queries
    hbm_target["sweep"] = {}
    for qn in (1, 2, 4):
        for i in range(3):
            select_whole(qh[i][:qn])
        ms_q, st_q = timed([q[:qn] for q in qh[3:]], a.steps, select_whole)
        rq = _stream_roofline(st_q, hi - lo, hbm_peak, peak_kind, bf16_peak, 0)
        hbm_target["sweep"][str(qn)] = {
            "value": round(a.steps * qn / (ms_q / 1e3), 2), "unit": "queries/s",
            "ms_per_step": round(ms_q / a.steps, 4), "frac": rq["frac"]}

    other = None
    if world > 1:
        # the other way to spread the step: query shards over replicated stores
        # (records mode headline) or record shards (queries mode headline)
        mode = "queries" if a.shard == "records" else "records"
        b2, sel2, _, _, _ = make(mode)
        for i in range(a.warmup):
            sel2(qpool[i])
        ms2, _ = timed(qpool[a.warmup:], a.steps, sel2, b2)
        other = {"split": mode, "value": round(a.steps * a.queries / (ms2 / 1e3), 2),
                 "unit": "queries/s", "ms_per_step": round(ms2 / a.steps, 4)}
        del b2, sel2

    out = {
        "metric": "retrieval queries/s @16M exps k=32",
        "value": round(value, 2),
        "unit": "queries/s",
        "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": round(ms / a.steps, 4),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": ("bf16 filter (tcgen05 kind::f16) + f64 refine" if tc == 3
                  else "f32/tf32 filter + f64 refine"),
        "data": "synthetic (device-generated, synth.py; store 16M x 64, i.i.d. Irwin-Hall contexts)",
        "config": {"workload": f"configs[3]: {n_total} records x d={DIM}, Q={a.queries} "
                               f"queries/step, k={K_SEL}, lambda_div={a.lambda_div}",
                   "records": n_total, "dim": DIM, "queries_per_step": a.queries, "k": K_SEL,
                   "lambda_div": a.lambda_div,
                   "parallelism": (f"query shards x{world} (store replicated per GPU, no collective)"
                                   if world > 1 and a.shard == "queries"
                                   else f"record shards x{world}"),
                   "l2": "inputs larger than L2 (4.4 GB store streamed per pass vs 126 MB L2)"},
        "e2e": {"value": round(e2e, 2), "unit": "queries/s",
                "h2d_bytes_per_step": a.queries * DIM * 8,
                "d2h_bytes_per_step": a.queries * K_SEL * 24 + a.queries * 8},
        "gpu_launches": gpu_launches,
        "roofline": roof,
        # the whole step against the Q x N x d contraction it must do (2 Q N d
        # flops at d = 64), at the TF32 and the bf16 measured peaks
        "step_tensor": {"flops_per_step": 2.0 * a.queries * n_total * DIM,
                        "tflops": round(2.0 * a.queries * n_total * DIM / (ms / a.steps / 1e3) / 1e12 / world, 1),
                        "frac_tf32_peak": round(2.0 * a.queries * n_total * DIM / (ms / a.steps / 1e3)
                                                / 1e12 / world / (bf16_peak / 2), 4),
                        "frac_bf16_peak": round(2.0 * a.queries * n_total * DIM / (ms / a.steps / 1e3)
                                                / 1e12 / world / bf16_peak, 4),
                        "note": "per GPU"},
        "certified_queries": sum(s["certified"] for s in stats),
        "exact_fallbacks": sum(s["exact_fallbacks"] for s in stats),
        "retried_queries": sum(s["retried"] for s in stats),
        "store_build_s": round(gen_s, 3),
        "hbm_target": hbm_target,
    }
    if other:
        out["query_shards" if other["split"] == "queries" else "record_shards"] = other
    if rank == 0 and world == 1 and not a.no_pareto:
        out["config1"] = bench_config1(dev)
        out["config1_traces"] = bench_config1_traces()
        out["config2"] = bench_config2(dev, a.steps)
        out["config2_lambda"] = bench_config2(dev, 3, lam=0.1)
        out["config5_step"] = bench_decision_step(buf, dev)
    if rank == 0 and not a.no_pareto:
        out["pareto"] = bench_pareto(dev)
        if not a.no_cpu_baseline:
            out["pareto"]["cpu_baseline"] = cpu_baseline_pareto()
    if rank == 0:
        out["clocks"] = clk.summary()
        if not a.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline_port()
    if dist:
        dist.destroy_process_group()
    return out


def bench_config1_traces():
    """configs[0] on the bundled traces (scripts/harness_time.py): the
    reference's unmodified decision loop over a 10k-record store harvested
    from proj/scenarios, with the reference's own classes vs the drop-in;
    byte-identical episode logs and stores required."""
    if not (ROOT / "oracle" / "_ref" / "harness_ref").exists():
        return {"unavailable": "oracle/_ref harness binaries not built"}
    r = subprocess.run([sys.executable, str(ROOT / "scripts" / "harness_time.py")],
                       capture_output=True, text=True, timeout=1800,
                       env=dict(os.environ, ROUNDS1="40", ROUNDS2="160"))
    if r.returncode != 0:
        return {"unavailable": r.stderr.strip().splitlines()[-1][:200] if r.stderr else "failed"}
    return json.loads(r.stdout.strip().splitlines()[-1])


def bench_config1(dev, steps=50):
    """configs[0]: one decision step at a time over a 10k-record buffer
    (d = 32; the bundled scenarios' contexts are zero-padded 23 -> 32, so a
    synthetic stand-in of that shape): select m = 8 with lambda_div = 0.1 (the
    reference's default) and the fused veto scan, compute_reward + update
    against the frontier, store() of the new experience -- latency per
    decision through the public API (wall clock): `decision.replay_step` (one
    device call, one host synchronisation), and the same four calls made
    separately (each synchronises) for comparison."""
    import paper_2601_22397_b200 as sair
    from paper_2601_22397_b200 import decision, synth
    cfg = sair.SelectionConfig(m=8, lambda_div=0.1)
    rc = sair.RewardConfig()
    act = sair.ScalingAction.noop(3)

    def run(fused):
        db = sair.ExperienceBuffer(0.0, device=dev)
        db.store_synthetic(SEED + 3, 10000, 32)
        fr = sair.ParetoFrontier(2000.0, 10.0, device=dev)
        rng = np.random.default_rng(SEED)
        lat = []
        for s in range(steps + 5):
            x = synth.queries(SEED + 200 + s, 1, 32)
            inp = sair.RewardInputs(rng.uniform(300, 900), rng.uniform(300, 900),
                                    rng.uniform(1, 5), rng.uniform(1, 5))
            t0 = time.perf_counter()
            if fused:
                decision.replay_step(db, fr, x[0], cfg, inp, act, rc, update=True,
                                     round=10000 + s)
            else:
                db.select_batch(x, cfg, nearest=True)
                r = sair.compute_reward(inp, act, fr, rc)
                fr.update(inp.l_after_ms, inp.c_after)
                db.store(sair.Experience(list(x[0]), act, r.total, 10000 + s))
            if s >= 5:
                lat.append(time.perf_counter() - t0)
        return float(np.median(lat))

    fused, four = run(True), run(False)
    return {"workload": "configs[0]: 10k records x d=32, k=8, lambda_div=0.1, veto scan, "
                        "compute_reward + update + store per decision (synthetic stand-in)",
            "us_per_decision_median": round(fused * 1e6, 1),
            "decisions_per_s": round(1.0 / fused, 1),
            "api": "decision.replay_step (sair_decision_step: one host synchronisation)",
            "four_calls_us_per_decision_median": round(four * 1e6, 1)}


def bench_decision_step(buf, dev, P=30000, steps=3):
    """configs[4] on one GPU's shard: the device side of one batched decision
    step for P = 10k pipelines x 3 workload patterns over the 16M-record store
    (128M / 8 GPUs): select + veto scan (wide pass), per-pipeline frontier
    reward + update, bulk append of the P new experiences."""
    import paper_2601_22397_b200 as sair
    from paper_2601_22397_b200 import decision, synth
    rng = np.random.default_rng(SEED)
    fs = sair.FrontierSet(P, 2000.0, 10.0, device=dev)
    scfg = sair.SelectionConfig(m=K_SEL, lambda_div=0.0)
    rcfg = sair.RewardConfig()
    times = {"retrieve": 0.0, "reward_store": 0.0}
    for s in range(steps + 1):
        ctx = synth.queries(SEED + 100 + s, P, DIM)
        inputs = np.stack([rng.uniform(100, 2500, P), rng.uniform(50, 2600, P),
                           rng.uniform(0.5, 10, P), rng.uniform(0.5, 11, P)], 1)
        deltas = rng.integers(-2, 3, size=(P, 3, 4)).astype(np.int32)
        upd = np.ones(P, np.uint8)
        rounds = np.full(P, 1000 + s, np.int32)
        t0 = time.perf_counter()
        decision.retrieve(buf, ctx, scfg)
        t1 = time.perf_counter()
        decision.score_and_store(buf, fs, ctx, inputs, deltas, upd, rounds, rcfg)
        t2 = time.perf_counter()
        if s:  # the first step warms up
            times["retrieve"] += t1 - t0
            times["reward_store"] += t2 - t1
    tot = sum(times.values())
    return {"workload": f"configs[4] per GPU: {P} pipelines, store {buf.size()} records x d={DIM}, "
                        f"k={K_SEL}, lambda_div=0",
            "decisions_per_s": round(P * steps / tot, 1), "ms_per_step": round(tot / steps * 1e3, 3),
            "retrieve_ms": round(times["retrieve"] / steps * 1e3, 3),
            "reward_and_store_ms": round(times["reward_store"] / steps * 1e3, 3)}


def bench_config2(dev, steps, lam=0.0):
    """configs[1]: 1M x 64 store, 256-query batches, k = 32, one GPU; lam =
    0.1 (the reference's default lambda_div, experience.hpp:29): the greedy's
    steps over the whole store, fp32-filtered and fp64-decided
    (select_greedy32.cu)."""
    import torch
    import paper_2601_22397_b200 as sair
    from paper_2601_22397_b200 import synth
    n, nq = 1 << 20, 256
    buf = sair.ExperienceBuffer(0.0, device=dev)
    buf.store_synthetic(SEED + 1, n, DIM)
    cfg = sair.SelectionConfig(m=K_SEL, lambda_div=lam)
    qs = synth.queries(SEED + 2, (3 + steps) * nq, DIM).reshape(3 + steps, nq, DIM)
    for i in range(1 if lam else 3):
        buf.select_batch(qs[i], cfg)
    stream = torch.cuda.ExternalStream(buf.stream_ptr(), device=dev)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stats = []
    e0.record(stream)
    for i in range(3, 3 + steps):
        buf.select_batch(qs[i], cfg)
        stats.append(buf.last_stats())
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    hbm_peak, bf16_peak, peak_kind = measured_peaks()
    qw = stats[0]["qb"] if stats[0]["tensor_core"] in (2, 3) else 0
    roof = _stream_roofline(stats, n, hbm_peak, peak_kind, bf16_peak, qw)
    del buf
    out = {"workload": f"configs[1]: {n} records x d={DIM}, {nq}-query batch, k={K_SEL}, "
                       f"lambda_div={lam}",
           "value": round(steps * nq / (ms / 1e3), 1), "unit": "queries/s",
           "ms_per_step": round(ms / steps, 4),
           "certified_queries": sum(s["certified"] for s in stats)}
    if lam:
        out["greedy32_queries"] = sum(s["greedy32"] for s in stats)
        out["candidates_per_query_step"] = round(
            sum(s["greedy32_candidates"] for s in stats) / max(1, steps * nq * K_SEL), 3)
        nsteps = sum(s["greedy32_steps"] for s in stats)
        if nsteps:
            # the tensor-core greedy step (select_greedy32.cu): per step the
            # fp32 gain of every (query, record) read and written (8 B) and
            # the records' 3xTF32 operand image (hi + lo, 8 B per dimension)
            step_ms = sum(s["greedy32_step_ms"] for s in stats) / nsteps
            alg = nq * n * 8 + n * DIM * 8
            achieved = alg / (step_ms / 1e3) / 1e9
            out["roofline"] = {
                "bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(achieved / hbm_peak, 4), "peak_kind": peak_kind,
                "algorithmic_bytes_per_launch": alg, "avg_launch_ms": round(step_ms, 4),
                "kernel": "sair::g32_mma_step_kernel (tcgen05 kind::tf32 3xTF32, 128 records x "
                          "256 rows per tile, gain update + top-2 epilogue)",
                "traffic": int(1.618604e9 + 1.119989e9),
                "traffic_source": "ncu --set full, profiles/r02/h_g32mma_step_full_summary.txt "
                                  "(dram__bytes_read.sum 1.6186 GB + dram__bytes_write.sum 1.1200 GB)"}
    else:
        out["roofline"] = roof
    return out


def bench_pareto(dev):
    """Config 3: 4M 2-objective tuples -> frontier maintenance (batch insert) and
    Pareto reward of every tuple against the frontier; k-D counts at 256k."""
    import torch
    import paper_2601_22397_b200 as sair
    from paper_2601_22397_b200 import synth
    res = {"metric": "Pareto-scored tuples/s", "tuples": PARETO_T}
    pts = synth.tuples(SEED, PARETO_T, 2, "uniform")
    f = sair.ParetoFrontier(1.0, 1.0, device=dev)
    # warm: the process's one-time costs (the pinned staging ring of large host
    # copies, first launches of the K6 kernels) -- timed and reported apart
    t0 = time.perf_counter()
    f.insert_batch(pts[:1 << 20])
    ins_process_first_s = time.perf_counter() - t0
    f2 = sair.ParetoFrontier(1.0, 1.0, device=dev)
    t0 = time.perf_counter()
    F = f2.insert_batch(pts)
    ins_first_s = time.perf_counter() - t0
    # steady state: a frontier whose scratch already holds a batch of this size
    # (another 4M batch of the distribution), then the timed batch
    ins_ws = []
    for r in range(3):
        fw = sair.ParetoFrontier(1.0, 1.0, device=dev)
        fw.insert_batch(synth.tuples(SEED + 100 + r, PARETO_T, 2, "uniform"))
        t0 = time.perf_counter()
        fw.insert_batch(pts)
        ins_ws.append(time.perf_counter() - t0)
    ins_s = sorted(ins_ws)[1]
    dpts = torch.from_numpy(pts).to(f"cuda:{dev}")
    dout = torch.empty(PARETO_T, dtype=torch.float64, device=f"cuda:{dev}")
    ddom = torch.empty(PARETO_T, dtype=torch.uint8, device=f"cuda:{dev}")
    s = torch.cuda.current_stream(dev)
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=f"cuda:{dev}")

    def score_ms(fr, dp, reps=10):
        """reward() of every tuple (score_batch_kernel), cold L2: a 512 MB
        write (4x the L2) before every launch, CUDA events around the launch
        alone on its stream; mean over reps."""
        fr.score_batch_device(dp.data_ptr(), PARETO_T, dout.data_ptr(), ddom.data_ptr(),
                              s.cuda_stream)
        tot = 0.0
        for _ in range(reps):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            fr.score_batch_device(dp.data_ptr(), PARETO_T, dout.data_ptr(), ddom.data_ptr(),
                                  s.cuda_stream)
            e1.record(s)
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        return tot / reps

    sc_ms = score_ms(f2, dpts)
    hbm_peak, _, peak_kind = measured_peaks()
    # algorithmic bytes per tuple: 16 B in (l, c), 8 B reward + 1 B dominated out
    sbytes = PARETO_T * (16 + 8 + 1)
    res.update({"value": round(PARETO_T / (sc_ms / 1e3), 1), "unit": "tuples/s",
                "score_ms": round(sc_ms, 4), "frontier_size": F,
                "frontier_insert_tuples_per_s": round(PARETO_T / ins_s, 1),
                "frontier_insert_s_e2e": round(ins_s, 4),
                "frontier_insert_s_e2e_first_call": round(ins_first_s, 4),
                "frontier_insert_s_process_first_call": round(ins_process_first_s, 4),
                "frontier_insert_note": "e2e from the host array (67 MB pageable H2D inside); "
                                        "median of 3 on warmed scratch; K6 pre-filter + exact "
                                        "sort path on the survivors; first_call = a fresh "
                                        "frontier (its scratch allocated), process_first_call = "
                                        "the process's first large insert (1M tuples: the pinned "
                                        "staging ring, first kernel launches)",
                "l2": "flushed before every timed launch (512 MB write)",
                "roofline": {"bound": "hbm", "achieved": round(sbytes / (sc_ms / 1e3) / 1e9, 1),
                             "peak": hbm_peak, "unit": "GB/s", "peak_kind": peak_kind,
                             "frac": round(sbytes / (sc_ms / 1e3) / 1e9 / hbm_peak, 4),
                             "algorithmic_bytes_per_launch": sbytes,
                             "kernel": "sair::score_batch_kernel"}})
    # prefix-sequential replay: 4M rounds, 85 % updating
    rng = np.random.default_rng(SEED)
    T = PARETO_T
    inputs = np.stack([rng.uniform(100, 2500, T), rng.uniform(50, 2600, T),
                       rng.uniform(0.5, 10, T), rng.uniform(0.5, 11, T)], 1)
    deltas = np.zeros((T, 3, 4), np.int32)
    upd = (rng.uniform(size=T) < 0.85).astype(np.uint8)
    fr = sair.ParetoFrontier(2000.0, 10.0, device=dev)
    sair.compute_reward_replay(inputs[:4096], deltas[:4096], upd[:4096], fr, sair.RewardConfig())
    fr = sair.ParetoFrontier(2000.0, 10.0, device=dev)
    t0 = time.perf_counter()
    sair.compute_reward_replay(inputs, deltas, upd, fr, sair.RewardConfig())
    dt = time.perf_counter() - t0
    res["replay"] = {"rounds": T, "s_e2e": round(dt, 4), "rounds_per_s": round(T / dt, 1),
                     "final_frontier": fr.size()}
    # configs[2] at full size for two objectives: O(T log T) counting
    t2 = synth.tuples(SEED + 2, PARETO_T, 2, "uniform")
    sair.dominance_counts(t2[:4096])
    t0 = time.perf_counter()
    _, mem2 = sair.dominance_counts(t2)
    dt2 = time.perf_counter() - t0
    res["dominance_counts_K2_4M"] = {"tuples": PARETO_T, "s_e2e": round(dt2, 4),
                                     "tuples_per_s": round(PARETO_T / dt2, 1),
                                     "frontier": int(mem2.sum())}
    # the other configs[2] distributions at full size, two objectives: batch
    # insert (e2e), device scoring against the resulting frontier, counts
    res["distributions"] = {}
    for dist in ("anti", "corr", "grid"):
        pd = synth.tuples(SEED + 5, PARETO_T, 2, dist)
        fd = sair.ParetoFrontier(1.0, 1.0, device=dev)
        t0 = time.perf_counter()
        Fd = fd.insert_batch(pd)
        ins = time.perf_counter() - t0
        dp_ = torch.from_numpy(pd).to(f"cuda:{dev}")
        sms = score_ms(fd, dp_, reps=3)
        t0 = time.perf_counter()
        _, md = sair.dominance_counts(pd)
        dc = time.perf_counter() - t0
        res["distributions"][dist] = {
            "frontier": Fd, "insert_s_e2e": round(ins, 4), "score_ms": round(sms, 4),
            "scored_tuples_per_s": round(PARETO_T / (sms / 1e3), 1),
            "dominance_counts_K2_s_e2e": round(dc, 4), "count_frontier": int(md.sum())}
    for K in (2, 3, 4):
        T = 262144
        t = synth.tuples(SEED + K, T, K, "uniform")
        sair.dominance_counts(t[:4096])
        t0 = time.perf_counter()
        cnt, mem = sair.dominance_counts(t)
        dt = time.perf_counter() - t0
        res[f"dominance_counts_K{K}"] = {"tuples": T, "s_e2e": round(dt, 4),
                                         "tuples_per_s": round(T / dt, 1),
                                         "frontier": int(mem.sum())}
    # configs[2] at its stated size for 3 and 4 objectives: the pairwise K7
    # kernel (dominance4_kernel), T^2/2 rank-vector comparisons
    for K in (3, 4):
        t = synth.tuples(SEED + 10 + K, PARETO_T, K, "uniform")
        t0 = time.perf_counter()
        cnt, mem = sair.dominance_counts(t)
        dt = time.perf_counter() - t0
        res[f"dominance_counts_K{K}_4M"] = {
            "tuples": PARETO_T, "s_e2e": round(dt, 4), "tuples_per_s": round(PARETO_T / dt, 1),
            "pairs_per_s": round(PARETO_T * (PARETO_T - 1) / 2 / dt, 1), "frontier": int(mem.sum())}
    return res


def _host_store(orc, n, threads):
    """The host copy of the bench's device-generated store (synth.py; the
    oracle's threaded restatement of the generator) and its statistics."""
    from paper_2601_22397_b200 import synth
    ctx = orc.synth_contexts(SEED, 0, n, DIM, nthreads=threads)
    return ctx, synth.rewards(SEED, 0, n), synth.rounds(0, n), orc.stats(ctx)


def cpu_baseline_port():
    """The oracle's bit-identical restatement of select (hoisted Sigma r,
    SURVEY F3) on all host threads, at the bench's own size (16M x 64, k = 32,
    lambda 0): a bounded sample of 2 queries per thread, no scaling.  The
    literal reference select is O(N^2) (loo_mean re-sums every reward per
    record, experience.cpp:138-140 inside :163-167): ~2.3 days per query at
    16M, so the restatement is the only CPU path that can run this workload."""
    from oracle.oracle import COracle
    from paper_2601_22397_b200 import synth
    orc = COracle()
    threads = os.cpu_count() or 1
    ctx, rew, rnd, st = _host_store(orc, N_RECORDS, threads)
    sigma = orc.sigma_median(ctx)
    nq = 2 * threads
    xq = synth.queries(SEED + 1, nq, DIM)
    t0 = time.perf_counter()
    orc.select_batch(ctx, rew, rnd, xq, K_SEL, 0.0, sigma, nthreads=threads, stats=st)
    dt = time.perf_counter() - t0
    return {"value": round(nq / dt, 4), "unit": "queries/s", "cores": threads, "kind": "port",
            "sample": f"oracle restatement (oracle/sair_oracle.c), {nq} queries x {N_RECORDS} "
                      f"records x d={DIM}, k={K_SEL}, lambda 0: {dt:.2f}s on {threads} threads",
            "cpu_model": _cpu_model()}


def cpu_baseline_pareto(T=PARETO_T):
    """The reference's own Pareto path (oracle/_ref: pareto.cpp compiled
    unmodified, -O3 -DNDEBUG), single thread like one reference run: the
    literal update loop over the 4M uniform tuples (pareto.cpp:36-54, the
    harness's per-round frontier.update), then reward() of every tuple against
    the resulting frontier (pareto.cpp:86-89, the scoring half of
    compute_reward) -- "Pareto-scored tuples/s"."""
    from oracle.oracle import REF_SO, Ref, RefFrontier
    from paper_2601_22397_b200 import synth
    if not REF_SO.exists():
        return None
    pts = synth.tuples(SEED, T, 2, "uniform")
    f = RefFrontier(Ref(), 1.0, 1.0)
    t0 = time.perf_counter()
    f.insert_batch(pts)
    ins = time.perf_counter() - t0
    t0 = time.perf_counter()
    f.reward_batch(pts)
    sc = time.perf_counter() - t0
    return {"value": round(T / sc, 1), "unit": "tuples/s", "cores": 1, "kind": "reference",
            "sample": f"oracle/_ref ParetoFrontier: {T} uniform 2-objective tuples, literal "
                      f"update loop {ins:.3f}s ({T / ins:.4g} tuples/s), reward() of every "
                      f"tuple vs the {len(f.points()[0])}-point frontier {sc:.3f}s",
            "update_tuples_per_s": round(T / ins, 1), "cpu_model": _cpu_model()}


def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ------------------------------------------------------------- reference ---

def run_reference(a):
    """The reference arm: the reference's CPU implementation of the path on
    the host cores, on this arm's config (16M x 64, Q = 4096 per step, k = 32).

    oracle/_ref is the reference compiled unmodified, but its literal select
    is O(N^2) -- loo_mean re-sums every reward for every record
    (experience.cpp:138-140 inside :163-167): ~2.3 days per query at 16M --
    so the timed path is the oracle's restatement (kind "port"), which is
    bit-identical to _ref (hoisting that loop-invariant sum is the one
    change; pinned == _ref in tests/test_oracle.py): the reference's
    arithmetic at its best possible complexity, on all host threads (queries
    partitioned like the reference's sweep pool, scalelab_cli.cpp:67-76).
    Each step is a bounded sample of the step's 4096 queries: one query per
    thread over the full 16M-record store.  The literal _ref select is timed
    once at n = 8192 for the record (not extrapolated)."""
    from oracle.oracle import REF_SO, COracle, Ref, RefBuffer
    from paper_2601_22397_b200 import synth
    orc = COracle()
    threads = os.cpu_count() or 1
    q_s = min(a.queries, threads)
    ctx, rew, rnd, st = _host_store(orc, a.records, threads)
    sigma = orc.sigma_median(ctx)
    xq = synth.queries(SEED, q_s * (a.warmup + a.steps), DIM)
    for i in range(a.warmup):
        orc.select_batch(ctx, rew, rnd, xq[i * q_s:(i + 1) * q_s], K_SEL, a.lambda_div, sigma,
                         nthreads=threads, stats=st)
    t0 = time.perf_counter()
    for i in range(a.warmup, a.warmup + a.steps):
        orc.select_batch(ctx, rew, rnd, xq[i * q_s:(i + 1) * q_s], K_SEL, a.lambda_div, sigma,
                         nthreads=threads, stats=st)
    dt = time.perf_counter() - t0
    value = a.steps * q_s / dt
    literal = None
    if REF_SO.exists():
        n_l = 8192
        b = RefBuffer(Ref(), 0.0)
        b.store_many(ctx[:n_l], rew[:n_l], rnd[:n_l])
        b.effective_sigma(0.0)
        t1 = time.perf_counter()
        b.select_batch(xq[:threads], K_SEL, a.lambda_div, 0.0, nthreads=threads)
        literal = {"records": n_l, "queries": threads, "threads": threads,
                   "ms_per_query_per_thread": round((time.perf_counter() - t1) * 1e3, 2)}
    sample = (f"oracle restatement of select (hoisted Sigma r, == oracle/_ref), {a.steps} steps x "
              f"{q_s} of the {a.queries} queries (one per thread) over {a.records} records x "
              f"d={DIM}, k={K_SEL}, lambda {a.lambda_div}: {dt:.2f}s on {threads} threads")
    return {
        "metric": "retrieval queries/s @16M exps k=32", "value": round(value, 4),
        "unit": "queries/s", "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": round(a.queries / value * 1e3, 1),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (synth.py, same store and queries as the ours arm)",
        "impl": "reference",
        "config": {"workload": f"configs[3]: {a.records} records x d={DIM}, Q={a.queries} "
                               f"queries/step, k={K_SEL}, lambda_div={a.lambda_div}"},
        "cpu_baseline": {"value": round(value, 4), "unit": "queries/s", "cores": threads,
                         "kind": "port", "sample": sample, "cpu_model": _cpu_model()},
        "e2e": {"value": round(value, 4), "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "reference_literal_select": literal,
    }


def _free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def relaunch(a) -> int:
    """`python bench.py --gpus N` without a torchrun environment: start N
    ranks (one per GPU) through torch.distributed.run on 127.0.0.1 and return
    its exit code; rank 0 prints the JSON line.  NCCL_DEBUG=INFO (unless set)
    puts NCCL's communicator / transport lines on stderr."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT,NVLS")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={a.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.run(cmd, env=env).returncode


def launcher_check(a, rank, world):
    """The multi-rank plumbing without kernels (CPU tests): rendezvous, one
    max-over-ranks all-reduce like the timed region's, rank 0's JSON line."""
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo")
        t = torch.tensor([float(rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        mx = float(t.item())
        dist.destroy_process_group()
    else:
        mx = 1.0
    if rank == 0:
        print(json.dumps({"launcher_check": True, "n_gpus": world, "max_over_ranks": mx,
                          "shard": a.shard}), flush=True)


def main():
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(a))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if a.launcher_check:
        launcher_check(a, rank, world)
        return
    if a.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(a)), flush=True)
        return
    out = run_ours(a, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
