/*
 * sair.h -- C-ABI of the B200-native SAIR retrieval + Pareto hot path.
 *
 * This is the drop-in boundary.  The reference exposes the path as a C++
 * class API (namespace scalelab); it has no FFI of its own.  Each entry point
 * below replaces one reference member, cited as file:line relative to
 * /root/reference/proj.  The host-side mirrors (paper_2601_22397_b200/cpp/: the scalelab
 * classes for C++; paper_2601_22397_b200/__init__.py for Python)
 * call only these functions.  See INTEGRATION.md for the bindings.
 *
 * Conventions
 *   - plain pointers and sizes; no torch / CUDA types in signatures;
 *   - every function returns a sair_status; on failure a thread-local message
 *     is available from sair_last_error();
 *   - status codes map 1:1 onto the exceptions the reference throws
 *     (SAIR_EINVAL -> std::invalid_argument, SAIR_ELOGIC -> std::logic_error,
 *     SAIR_ERANGE -> std::out_of_range, SAIR_EIO -> std::runtime_error);
 *   - host pointers are borrowed for the duration of the call; results are in
 *     caller-provided arrays; the library owns device memory and staging;
 *   - calls are synchronous on return.  Different handles may be used from
 *     different threads; one handle is not thread-safe (the reference mutates
 *     its sigma cache from const methods, experience.hpp:87-88);
 *   - all arithmetic the reference does in fp64 is fp64 here; the fp32 device
 *     copy of the store is only a bandwidth-optimal *filter* whose survivors
 *     are re-scored in fp64 and certified.
 *   - there is no CPU fallback: without a usable CUDA device every compute
 *     entry point fails with SAIR_ECUDA.
 */
#ifndef SAIR_H_
#define SAIR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define SAIR_API __attribute__((visibility("default")))
#else
#define SAIR_API
#endif

typedef enum {
    SAIR_OK = 0,
    SAIR_EINVAL = 1, /* std::invalid_argument */
    SAIR_ELOGIC = 2, /* std::logic_error */
    SAIR_ERANGE = 3, /* std::out_of_range (items_.at) */
    SAIR_EIO = 4,    /* std::runtime_error (persistence) */
    SAIR_ECUDA = 5,  /* CUDA runtime / no device */
    SAIR_ENOMEM = 6,
    SAIR_ENCCL = 7
} sair_status;

typedef struct sair_store_s* sair_store_t;       /* ExperienceBuffer state */
typedef struct sair_frontier_s* sair_frontier_t; /* ParetoFrontier state */
typedef struct sair_frontier_set_s* sair_frontier_set_t; /* P independent ParetoFrontiers */

/* SelectionConfig, experience.hpp:27-32 (+ this library's knobs). */
typedef struct {
    size_t m;                  /* SelectionConfig::m (default 15) */
    double lambda_div;         /* SelectionConfig::lambda_div (default 0.1) */
    double sigma_sim;          /* SelectionConfig::sigma_sim; <= 0 -> buffer median */
    int locally_weighted_mean; /* SelectionConfig::locally_weighted_mean */
    int mode;                  /* SAIR_SELECT_AUTO / SAIR_SELECT_EXACT */
} sair_select_config;

enum { SAIR_SELECT_AUTO = 0, SAIR_SELECT_EXACT = 1 };

/* Counters of the last select call (diagnostics; bench.py reads them). */
typedef struct {
    size_t queries;         /* queries in the call */
    size_t certified;       /* answered by the fp32 filter + fp64 refine */
    size_t exact_fallbacks; /* answered by the full fp64 pass */
    size_t candidates;      /* K' per query used by the filter */
    int qb;                 /* queries per streaming pass */
    int stream_launches;    /* streaming-kernel launches */
    float stream_ms;        /* device time of the streaming kernels (CUDA events) */
    float total_ms;         /* device time of the whole call */
    float prepass_ms;       /* device time of the threshold sample pre-pass (tensor-core path) */
    int tensor_core;        /* 1: tcgen05 8-query stream pass; 2: tcgen05 wide (32-256 query)
                               TF32 pass; 3: the 256-query wide pass on the bf16 page copy */
    int small;              /* 1: the whole call ran as the one-launch exact small-store select */
    size_t retried;         /* queries given a second wide pass with raised thresholds */
    size_t greedy32;        /* queries whose greedy ran fp32-filtered, fp64-decided (lambda != 0) */
    size_t greedy32_candidates; /* (query, step) candidates verified in fp64 by that path */
    float greedy32_step_ms;     /* device time of that path's step kernels (summed) */
    int greedy32_steps;         /* and their launches (tensor-core step: 1 per greedy step) */
} sair_select_stats;

SAIR_API const char* sair_last_error(void);
SAIR_API int sair_version(void);
/* Number of CUDA devices; SAIR_ECUDA if none. */
SAIR_API sair_status sair_device_count(int* out);

/* ------------------------------------------------------------------------
 * Experience store -- ExperienceBuffer (experience.hpp:45-89)
 * ------------------------------------------------------------------------ */

/* ExperienceBuffer(double r_min), experience.cpp:42. Device-resident SoA. */
SAIR_API sair_status sair_store_create(double r_min, int device, size_t capacity_hint,
                                       sair_store_t* out);
SAIR_API sair_status sair_store_destroy(sair_store_t h);
/* Deep copy (the reference's value semantics, experience.hpp:45). */
SAIR_API sair_status sair_store_clone(sair_store_t h, sair_store_t* out);

/* ExperienceBuffer::store for `count` rows, experience.cpp:44-62: each row is
 * gated (reward > r_min, else counted as rejected); the dimension is fixed by
 * the first accepted row and a change is SAIR_EINVAL (rows before the bad one
 * stay stored, as with sequential store() calls).  ctx is count x dim fp64
 * row-major.  accepted (nullable) gets one 0/1 per row. */
SAIR_API sair_status sair_store_append(sair_store_t h, const double* ctx, size_t count, int dim,
                                       const double* reward, const int32_t* round,
                                       uint8_t* accepted, size_t* n_accepted);

/* Benchmark/test helper: append `count` synthetic rows generated on the device
 * (paper_2601_22397_b200/synth.py documents the generator; values are
 * fp32-exact and their running sums exact in fp64).  Record i of the store
 * gets global index base+i, round = global index. */
SAIR_API sair_status sair_store_append_synthetic(sair_store_t h, uint64_t seed, size_t count,
                                                 int dim, int clustered);

SAIR_API sair_status sair_store_size(sair_store_t h, size_t* n);         /* size() */
SAIR_API sair_status sair_store_dim(sair_store_t h, int* dim);           /* 0 if empty */
SAIR_API sair_status sair_store_rejected(sair_store_t h, uint64_t* out); /* rejected() */
SAIR_API sair_status sair_store_r_min(sair_store_t h, double* out);      /* r_min() */

/* Read back record `index` (fp64 context, reward, round): all()[index]. */
SAIR_API sair_status sair_store_get(sair_store_t h, size_t index, double* ctx, double* reward,
                                    int32_t* round);

/* ExperienceBuffer::standardize, experience.cpp:64-78 (fp64, host-kept sums). */
/* Bulk device->host copy of records [offset, offset + count) (each pointer
 * nullable): ctx [count][dim], reward [count], round [count]. */
SAIR_API sair_status sair_store_export(sair_store_t h, size_t offset, size_t count, double* ctx,
                                       double* reward, int32_t* round);

/* ExperienceBuffer::load(path, r_min, corrupt_lines) (experience.hpp:76-77,
 * experience.cpp:243-271) into a new device store: the JSONL lines are parsed
 * on `nthreads` host threads (0 = all) with the reference's parser and
 * store()'s semantics are applied in line order (gate, dimension fixed by the
 * first accepted row -- a change is SAIR_EINVAL), then one bulk append.
 * SAIR_EIO when the file cannot be read. */
SAIR_API sair_status sair_store_load_jsonl(const char* path, double r_min, int device, int nthreads,
                                           size_t* corrupt_lines, sair_store_t* out);
/* ExperienceBuffer::persist(path) (experience.cpp:232-241) from the device
 * store (one bulk export); the device store holds no source / action, so
 * those are written empty ("" and []) -- a host mirror with them persists
 * itself (the C++ drop-in, the Python wrapper with keep_mirror). */
SAIR_API sair_status sair_store_persist_jsonl(sair_store_t h, const char* path);

SAIR_API sair_status sair_store_standardize(sair_store_t h, const double* x, int dim, double* z);

/* ExperienceBuffer::effective_sigma, experience.cpp:116-121, including the
 * stale-after-50-insertions cache; a refresh (experience.cpp:80-114) runs the
 * 512-subsample pairwise median on the device. */
SAIR_API sair_status sair_store_effective_sigma(sair_store_t h, double sigma_sim, double* out);

/* similarity(a, b, sigma), experience.cpp:30-40: SAIR_EINVAL when the
 * lengths differ or sigma <= 0.  Host arithmetic (two host vectors, O(d),
 * bit-identical to the reference), like sair_store_standardize; the
 * data-parallel veto scan is sair_store_nearest. */
SAIR_API sair_status sair_similarity(const double* a, size_t len_a, const double* b, size_t len_b,
                                     double sigma, double* out);

/* ExperienceBuffer::surprisal, experience.cpp:143-149 (SAIR_ERANGE on a bad index). */
SAIR_API sair_status sair_store_surprisal(sair_store_t h, size_t index, const double* x, int dim,
                                          const sair_select_config* cfg, double* out);

/* ExperienceBuffer::select for nq queries, experience.cpp:151-205.
 * queries: nq x dim fp64.  For query q, out_count[q] = min(m, n) picks are
 * written at out_idx/out_sim/out_score[q*m ...] in the reference's curriculum
 * order (stable by reward asc, round asc).  out_idx are store indices
 * (global indices for a shard, see sair_store_set_shard).  out_sim is
 * SelectedExperience::similarity_to_current, out_score ::score.
 * out_nn_idx / out_nn_sim (nullable) additionally return the MockBackend veto
 * scan's nearest record (policy.cpp:140-157) from the same pass. */
SAIR_API sair_status sair_store_select(sair_store_t h, const double* queries, size_t nq, int dim,
                                       const sair_select_config* cfg, int64_t* out_idx,
                                       double* out_sim, double* out_score, size_t* out_count,
                                       int64_t* out_nn_idx, double* out_nn_sim);

/* The veto scan alone, policy.cpp:140-157: argmax similarity, first index on ties. */
SAIR_API sair_status sair_store_nearest(sair_store_t h, const double* queries, size_t nq, int dim,
                                        double sigma_sim, int64_t* out_idx, double* out_sim);

SAIR_API sair_status sair_store_last_stats(sair_store_t h, sair_select_stats* out);

/* ------------------------------------------------------------------------
 * Sharding (one store per GPU, contiguous slices of one logical buffer;
 * SURVEY.md 8(e)).  The reference has one buffer per run (harness.cpp:151);
 * a shard reproduces that buffer's arithmetic exactly by using the buffer's
 * global statistics for standardize / loo_mean / sigma.
 * ------------------------------------------------------------------------ */

/* Global index of this store's first record (call before the first append). */
SAIR_API sair_status sair_store_set_shard(sair_store_t h, int64_t global_offset);
/* This store's own sums (experience.cpp:55-58): sum[d], sum_sq[d], max|x|[d],
 * scalars[3] = {n, reward total (index order), max |reward|}. */
SAIR_API sair_status sair_store_local_stats(sair_store_t h, double* sum, double* sum_sq,
                                            double* xabs, double* scalars);
/* Switch to shard mode with the buffer's statistics and sigma (sigma <= 0:
 * unset -- select then needs SelectionConfig::sigma_sim > 0). */
SAIR_API sair_status sair_store_set_global(sair_store_t h, uint64_t n_global, const double* sum,
                                           const double* sum_sq, const double* xabs,
                                           double reward_total, double reward_absmax,
                                           double sigma);
/* mean[d] and sd[d] of standardize() (experience.cpp:68-74) for this store's
 * statistics (global ones in shard mode). */
SAIR_API sair_status sair_store_moments(sair_store_t h, double* mean, double* sd);
/* The global indices refresh_sigma_cache samples from an n-record buffer
 * (experience.cpp:82-91); m <= 512 returned. */
SAIR_API sair_status sair_sigma_sample_indices(uint64_t n, int64_t* idx, size_t* m);
/* The median pairwise z-distance of m raw rows (m x dim) standardized with
 * mean/sd (experience.cpp:92-112), computed on `device`. */
SAIR_API sair_status sair_sigma_rows(const double* rows, size_t m, int dim, const double* mean,
                                     const double* sd, int device, double* out);
/* select() on a shard: as sair_store_select plus each pick's reward and round
 * (what the cross-shard merge orders by).  out_reward / out_round nullable. */
SAIR_API sair_status sair_store_select_shard(sair_store_t h, const double* queries, size_t nq,
                                             int dim, const sair_select_config* cfg,
                                             int64_t* out_idx, double* out_sim,
                                             double* out_score, double* out_reward,
                                             int32_t* out_round, size_t* out_count);
/* sair_merge_topk on an all-gathered DEVICE buffer (NCCL): d_parts is
 * [nshards][nq][5m + 1] doubles (per rank: score[m], sim[m], reward[m],
 * global index[m], round[m], count), d_out [nq][3m + 1] (index[m], sim[m],
 * score[m], count), ordered on `stream` (a cudaStream_t, 0 = default). */
SAIR_API sair_status sair_merge_topk_packed(const double* d_parts, size_t nshards, size_t nq,
                                            size_t m, int device, void* stream, double* d_out);
/* The shard's side of select() for lambda_div > 0 on a buffer spread over
 * ranks (experience.cpp:170-194 with the arg-max taken across shards by the
 * caller between steps; sharded.py).  greedy_begin scores this shard for nq
 * queries (global statistics, exact fp64) and writes per query the shard's
 * best untaken record as nq x (6 + dim) doubles: gain, round, global index
 * (-1 and gain -inf when none), similarity, score, reward, standardized row.
 * greedy_next takes the step's global picks (global indices, nq) and their
 * rows (nq x dim): local picks become taken, every penalty adds its pick's
 * similarity, and the new bests are written the same way. */
SAIR_API sair_status sair_store_greedy_begin(sair_store_t h, const double* queries, size_t nq,
                                             int dim, const sair_select_config* cfg,
                                             double* out_best);
SAIR_API sair_status sair_store_greedy_next(sair_store_t h, const int64_t* picks,
                                            const double* rows, double* out_best);
/* Merge per-shard top-m lists (shard-major arrays [nshards][nq][m], counts
 * [nshards][nq]) into the buffer's select() result for lambda_div == 0:
 * (score desc, round asc, index asc), then curriculum order. */
SAIR_API sair_status sair_merge_topk(const double* score, const double* sim,
                                     const double* reward, const int32_t* round,
                                     const int64_t* gidx, const size_t* count, size_t nshards,
                                     size_t nq, size_t m, int device, int64_t* out_idx,
                                     double* out_sim, double* out_score, size_t* out_count);

/* The CUDA stream the store's work is ordered on (for event timing). */
SAIR_API sair_status sair_store_stream(sair_store_t h, void** stream);

/* ------------------------------------------------------------------------
 * Pareto frontier -- ParetoFrontier (pareto.hpp:24-70), 2 objectives
 * ------------------------------------------------------------------------ */

/* ParetoFrontier(l_max, c_max), pareto.cpp:14-18: SAIR_EINVAL if either <= 0. */
SAIR_API sair_status sair_frontier_create(double l_max_ms, double c_max, int device,
                                          sair_frontier_t* out);
SAIR_API sair_status sair_frontier_destroy(sair_frontier_t f);
SAIR_API sair_status sair_frontier_clone(sair_frontier_t f, sair_frontier_t* out);

/* normalize, pareto.cpp:20-29 */
SAIR_API sair_status sair_frontier_normalize(sair_frontier_t f, double l_ms, double cost,
                                             double* l, double* c, int* clamped);
/* update, pareto.cpp:36-41 */
SAIR_API sair_status sair_frontier_update(sair_frontier_t f, double l_ms, double cost,
                                          int* inserted, int* clamped);
/* insert_normalized, pareto.cpp:43-54 */
SAIR_API sair_status sair_frontier_insert_normalized(sair_frontier_t f, double l, double c,
                                                     int* inserted);
/* T sequential insert_normalized calls on normalized points (pts: T x 2); the
 * result equals the reference's loop (non-dominated set of F u pts, first
 * occurrence of duplicates). */
SAIR_API sair_status sair_frontier_insert_batch(sair_frontier_t f, const double* pts, size_t T,
                                                size_t* new_size);
SAIR_API sair_status sair_frontier_size(sair_frontier_t f, size_t* F);
/* points(): sorted by latency asc.  l/c may be NULL to query the size. */
SAIR_API sair_status sair_frontier_points(sair_frontier_t f, double* l, double* c, size_t cap,
                                          size_t* F);
SAIR_API sair_status sair_frontier_bounds(sair_frontier_t f, double* l_max, double* c_max);
/* hypervolume, pareto.cpp:56-65 */
SAIR_API sair_status sair_frontier_hypervolume(sair_frontier_t f, double* out);
/* strictly_dominated, pareto.cpp:31-34 */
SAIR_API sair_status sair_frontier_strictly_dominated(sair_frontier_t f, double l, double c,
                                                      int* out);
/* contribution, pareto.cpp:67-73: SAIR_ELOGIC for a dominated point. */
SAIR_API sair_status sair_frontier_contribution(sair_frontier_t f, double l, double c,
                                                double* out);
/* distance, pareto.cpp:75-84: *has = 0 for an empty frontier (nullopt). */
SAIR_API sair_status sair_frontier_distance(sair_frontier_t f, double l, double c, double* out,
                                            int* has);
/* reward, pareto.cpp:86-89 */
SAIR_API sair_status sair_frontier_reward(sair_frontier_t f, double l, double c, double* out);

/* Batch scoring of T normalized points against the (fixed) frontier: the
 * Pareto half of compute_reward for every tuple.  out_dominated nullable. */
SAIR_API sair_status sair_frontier_score_batch(sair_frontier_t f, const double* pts, size_t T,
                                               double* out_reward, uint8_t* out_dominated);

/* Same on device-resident data: pts / out_reward / out_dominated are device
 * pointers, ordered on `stream` (a cudaStream_t, NULL = legacy default);
 * returns without synchronizing. */
SAIR_API sair_status sair_frontier_score_batch_device(sair_frontier_t f, const double* pts,
                                                      size_t T, double* out_reward,
                                                      uint8_t* out_dominated, void* stream);

/* K-objective dominance counts over T tuples (T x K fp64, K in 1..8):
 * counts[i] = #{j : j dominates i} (component-wise dominates(), pareto.cpp:9-12),
 * member[i] = counts[i] == 0 and no equal tuple at a lower index.
 * counts / member nullable (member-only mode exits early). */
SAIR_API sair_status sair_dominance_counts(const double* tuples, size_t T, int K, int device,
                                           uint32_t* counts, uint8_t* member);
/* The same counts split into `nparts` parts of equal pairwise work (a rank of
 * a multi-GPU job computes part = its rank over the all-gathered tuples):
 * entries outside the part are 0, so the parts combine by a sum (SURVEY.md
 * 8(e): dominance counts need every pair across shards). */
SAIR_API sair_status sair_dominance_counts_part(const double* tuples, size_t T, int K, int device,
                                                int part, int nparts, uint32_t* counts,
                                                uint8_t* member);

/* ------------------------------------------------------------------------
 * Reward -- compute_reward / action_magnitude (reward.hpp:42-48)
 * ------------------------------------------------------------------------ */

typedef struct { /* RewardConfig, reward.hpp:8-20 */
    double t_sla_ms, l_baseline_ms, c_budget, w_latency, w_cost, w_proactive, r_max;
} sair_reward_config;

typedef struct { /* RewardInputs, reward.hpp:23-28 */
    double l_before_ms, l_after_ms, c_before, c_after;
} sair_reward_inputs;

typedef struct { /* RewardBreakdown, reward.hpp:30-38 */
    double latency, cost, sla, proactive, pareto, total;
    int clipped;
} sair_reward_breakdown;

/* ------------------------------------------------------------------------
 * Decision step: one iteration of the reference's loop,
 * harness.cpp:197-261, replayed with the step's outcome known (config 1's
 * trace replay): select(x) with the veto scan (:205; policy.cpp:140-157),
 * compute_reward of `in` / `deltas` against the frontier before the update
 * (:250; reward.hpp:44-46), frontier.update(in->l_after_ms, in->c_after) when
 * `update` (:251), store() of (x, reward total, round) through the r_min
 * gate (:253-261).  Same results as sair_store_select + sair_compute_reward +
 * sair_frontier_update + sair_store_append in that order, enqueued on the
 * store's stream with one host synchronisation.  out_count is the select's
 * count (<= cfg->m entries in out_idx / out_sim / out_score); out_nn_* the
 * veto scan; out_inserted / out_stored the update's and store()'s results.
 * ------------------------------------------------------------------------ */
SAIR_API sair_status sair_decision_step(sair_store_t h, sair_frontier_t f, const double* x,
                                        int dim, const sair_select_config* cfg,
                                        const sair_reward_inputs* in, const int32_t* deltas,
                                        size_t stages, const sair_reward_config* rcfg,
                                        int update, int32_t round, int64_t* out_idx,
                                        double* out_sim, double* out_score, size_t* out_count,
                                        int64_t* out_nn_idx, double* out_nn_sim,
                                        sair_reward_breakdown* out_reward, int* out_inserted,
                                        int* out_stored);

/* action_magnitude, reward.cpp:9-19; deltas = stages x {replicas,
 * cpu_millicores, memory_mb, rate_ratio_tenths}. */
SAIR_API sair_status sair_action_magnitude(const int32_t* deltas, size_t stages, double* out);

/* compute_reward, reward.cpp:21-44: the pareto term reads the frontier as the
 * action saw it (read-only).  SAIR_EINVAL on the reference's config errors. */
SAIR_API sair_status sair_compute_reward(const sair_reward_inputs* in, const int32_t* deltas,
                                         size_t stages, sair_frontier_t f,
                                         const sair_reward_config* cfg,
                                         sair_reward_breakdown* out);

/* compute_reward for T independent (inputs, action) rows against one
 * frontier (oracle rollouts, harness.cpp:112-119; config 5).  deltas is
 * T x stages x 4. */
SAIR_API sair_status sair_compute_reward_batch(const sair_reward_inputs* in,
                                               const int32_t* deltas, size_t stages, size_t T,
                                               sair_frontier_t f, const sair_reward_config* cfg,
                                               sair_reward_breakdown* out);

/* Prefix-sequential replay (scalelab_cli.cpp:118-147
 * cmd_replay, harness.cpp:250-251): row t's compute_reward is scored against
 * the frontier `f` as updated by the rows s < t with update[s] != 0, and then
 * f.update(l_after_t, c_after_t) when update[t] != 0 -- the sequential loop's
 * results, computed by parallel replayers from prefix frontiers.  On return f
 * holds the final frontier. */
SAIR_API sair_status sair_compute_reward_replay(const sair_reward_inputs* in,
                                                const int32_t* deltas, size_t stages, size_t T,
                                                const uint8_t* update, sair_frontier_t f,
                                                const sair_reward_config* cfg,
                                                sair_reward_breakdown* out);

/* ------------------------------------------------------------------------
 * A set of P independent frontiers (one
 * ParetoFrontier per simulated pipeline, harness.cpp:150) stepped together.
 * ------------------------------------------------------------------------ */
SAIR_API sair_status sair_frontier_set_create(size_t P, double l_max_ms, double c_max, int device,
                                              sair_frontier_set_t* out);
SAIR_API sair_status sair_frontier_set_destroy(sair_frontier_set_t s);
/* One decision step of every pipeline p (harness.cpp:250-251): out[p] =
 * compute_reward(in[p], deltas[p], frontier_p, cfg), then frontier_p.update(
 * l_after, c_after) when update[p] != 0.  deltas is P x stages x 4. */
SAIR_API sair_status sair_frontier_set_step(sair_frontier_set_t s, const sair_reward_inputs* in,
                                            const int32_t* deltas, size_t stages,
                                            const uint8_t* update, const sair_reward_config* cfg,
                                            sair_reward_breakdown* out);
/* points() / hypervolume() of pipeline p (up to cap points copied). */
SAIR_API sair_status sair_frontier_set_points(sair_frontier_set_t s, size_t p, double* l,
                                              double* c, size_t cap, size_t* F,
                                              double* hypervolume);

/* ---------------------------------------------- multi-GPU (one process) --
 * One logical ExperienceBuffer / ParetoFrontier over several GPUs of this
 * process (the one-process-per-GPU mirror is sharded.py).
 * A communicator spans a device list: NCCL (ncclCommInitAll, loaded at run
 * time) when the devices are distinct, else device-to-device copies.  A
 * sharded store keeps the global insertion order: shard r holds a contiguous
 * slice, appends fill the shards in order (capacity / shards records each),
 * and select() equals the single-buffer select() (experience.cpp:151-205):
 * the buffer's statistics and sigma on every shard, each shard's top-m, an
 * all-gather of the per-shard candidates and the exact merge (lambda 0), or
 * the distributed greedy (lambda != 0). */
typedef struct sair_comm_s* sair_comm_t;
typedef struct sair_sharded_s* sair_sharded_t;
SAIR_API sair_status sair_comm_create(const int* devices, int ndev, sair_comm_t* out);
SAIR_API sair_status sair_comm_destroy(sair_comm_t c);
/* devices in the communicator; *nccl = 1 when NCCL carries its collectives */
SAIR_API sair_status sair_comm_info(sair_comm_t c, int* ndev, int* nccl);
/* capacity: the records the buffer is sized for (shard quota = capacity / ndev) */
SAIR_API sair_status sair_sharded_create(sair_comm_t c, double r_min, size_t capacity,
                                         sair_sharded_t* out);
SAIR_API sair_status sair_sharded_destroy(sair_sharded_t h);
/* store() of count rows in order (experience.cpp:44-62) */
SAIR_API sair_status sair_sharded_append(sair_sharded_t h, const double* ctx, size_t count,
                                         int dim, const double* reward, const int32_t* round,
                                         uint8_t* accepted, size_t* n_accepted);
SAIR_API sair_status sair_sharded_append_synthetic(sair_sharded_t h, uint64_t seed, size_t count,
                                                   int dim, int clustered);
/* records stored / rejected; per-shard sizes into shard_n (ndev entries, or null) */
SAIR_API sair_status sair_sharded_size(sair_sharded_t h, size_t* n, uint64_t* rejected,
                                       size_t* shard_n);
SAIR_API sair_status sair_sharded_effective_sigma(sair_sharded_t h, double sigma_sim, double* out);
/* ExperienceBuffer::select for nq queries over the sharded buffer (global indices) */
SAIR_API sair_status sair_store_select_sharded(sair_sharded_t h, const double* queries, size_t nq,
                                               int dim, const sair_select_config* cfg,
                                               int64_t* out_idx, double* out_sim,
                                               double* out_score, size_t* out_count);
/* T sequential insert_normalized() calls into f (pareto.cpp:36-54), the batch
 * reduced on every device of c first (K6 per slice; frontier of the union) */
SAIR_API sair_status sair_frontier_insert_batch_sharded(sair_comm_t c, sair_frontier_t f,
                                                        const double* pts, size_t T,
                                                        size_t* new_size);

#ifdef __cplusplus
}
#endif
#endif /* SAIR_H_ */
