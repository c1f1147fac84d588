// capi.cpp -- the extern "C" boundary (include/sair.h).  Every entry point
// translates C++ exceptions into sair_status codes + a thread-local message.
#include <cmath>
#include <cstring>
#include <new>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "internal.hpp"

namespace {
thread_local std::string g_err;

// one NVTX range per entry point (the C ABI's name): what a profiler's
// timeline shows around the kernels of a call; free without a tool attached
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

template <class F>
sair_status guard(const char* name, F&& f) {
    NvtxRange r(name);
    try {
        f();
        return SAIR_OK;
    } catch (const sair::Error& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::bad_alloc& e) {
        g_err = "out of memory";
        return SAIR_ENOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SAIR_ECUDA;
    }
}

sair_status bad(const char* msg) {
    g_err = msg;
    return SAIR_EINVAL;
}

sair_select_config defaults(const sair_select_config* c) {
    if (c) return *c;
    sair_select_config d{};
    d.m = 15;
    d.lambda_div = 0.1;
    return d;
}
}  // namespace

extern "C" {

const char* sair_last_error(void) { return g_err.c_str(); }
sair_status sair_internal_fail(sair_status code, const char* msg) {  // hidden: persist.cpp
    g_err = msg;
    return code;
}
int sair_version(void) { return 1; }

sair_status sair_device_count(int* out) {
    return guard(__func__, [&] {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess) n = 0;
        *out = n;
        if (n == 0) throw sair::Error(SAIR_ECUDA, "no CUDA device");
    });
}

// ---------------------------------------------------------------- store --

sair_status sair_store_create(double r_min, int device, size_t capacity_hint, sair_store_t* out) {
    if (!out) return bad("null out");
    return guard(__func__, [&] {
        auto* s = new sair_store_s();
        try {
            sair::store_init(s, r_min, device, capacity_hint);
        } catch (...) {
            delete s;
            throw;
        }
        *out = s;
    });
}

sair_status sair_store_destroy(sair_store_t h) {
    if (!h) return SAIR_OK;
    return guard(__func__, [&] {
        sair::store_free(h);
        delete h;
    });
}

sair_status sair_store_clone(sair_store_t h, sair_store_t* out) {
    if (!h || !out) return bad("null handle");
    return guard(__func__, [&] {
        auto* o = new sair_store_s();
        try {
            sair::store_clone(h, o);
        } catch (...) {
            delete o;
            throw;
        }
        *out = o;
    });
}

sair_status sair_store_append(sair_store_t h, const double* ctx, size_t count, int dim,
                              const double* reward, const int32_t* round, uint8_t* accepted,
                              size_t* n_accepted) {
    if (!h) return bad("null handle");
    if (count && (!ctx || !reward || !round)) return bad("null input");
    return guard(__func__, [&] {
        size_t k = sair::store_append(h, ctx, count, dim, reward, round, accepted);
        if (n_accepted) *n_accepted = k;
    });
}

sair_status sair_store_append_synthetic(sair_store_t h, uint64_t seed, size_t count, int dim,
                                        int clustered) {
    if (!h) return bad("null handle");
    return guard(__func__, [&] { sair::store_append_synthetic(h, seed, count, dim, clustered); });
}

sair_status sair_store_size(sair_store_t h, size_t* n) {
    if (!h || !n) return bad("null handle");
    *n = h->n;
    return SAIR_OK;
}
sair_status sair_store_dim(sair_store_t h, int* dim) {
    if (!h || !dim) return bad("null handle");
    *dim = h->n ? h->d : 0;
    return SAIR_OK;
}
sair_status sair_store_rejected(sair_store_t h, uint64_t* out) {
    if (!h || !out) return bad("null handle");
    *out = h->rejected;
    return SAIR_OK;
}
sair_status sair_store_r_min(sair_store_t h, double* out) {
    if (!h || !out) return bad("null handle");
    *out = h->r_min;
    return SAIR_OK;
}

sair_status sair_store_get(sair_store_t h, size_t index, double* ctx, double* reward,
                           int32_t* round) {
    if (!h) return bad("null handle");
    return guard(__func__, [&] {
        if (index >= h->n) throw sair::Error(SAIR_ERANGE, "vector::_M_range_check");
        sair::DeviceGuard g(h->device);
        if (ctx)
            SAIR_CUDA(cudaMemcpyAsync(ctx, h->x64 + index * h->d, h->d * 8,
                                      cudaMemcpyDeviceToHost, h->st));
        if (reward)
            SAIR_CUDA(cudaMemcpyAsync(reward, h->r64 + index, 8, cudaMemcpyDeviceToHost, h->st));
        if (round)
            SAIR_CUDA(cudaMemcpyAsync(round, h->rnd + index, 4, cudaMemcpyDeviceToHost, h->st));
        SAIR_CUDA(cudaStreamSynchronize(h->st));
    });
}

sair_status sair_store_export(sair_store_t h, size_t offset, size_t count, double* ctx,
                              double* reward, int32_t* round) {
    if (!h) return bad("null handle");
    return guard(__func__, [&] {
        if (offset > h->n || count > h->n - offset)
            throw sair::Error(SAIR_ERANGE, "export range outside the store");
        if (count == 0) return;
        sair::DeviceGuard g(h->device);
        if (ctx)
            SAIR_CUDA(cudaMemcpyAsync(ctx, h->x64 + offset * h->d, count * h->d * 8,
                                      cudaMemcpyDeviceToHost, h->st));
        if (reward)
            SAIR_CUDA(cudaMemcpyAsync(reward, h->r64 + offset, count * 8, cudaMemcpyDeviceToHost,
                                      h->st));
        if (round)
            SAIR_CUDA(cudaMemcpyAsync(round, h->rnd + offset, count * 4, cudaMemcpyDeviceToHost,
                                      h->st));
        SAIR_CUDA(cudaStreamSynchronize(h->st));
    });
}

sair_status sair_store_standardize(sair_store_t h, const double* x, int dim, double* z) {
    if (!h) return bad("null handle");
    return guard(__func__, [&] {
        if (h->n == 0) {  // experience.cpp:65
            std::memcpy(z, x, (size_t)dim * sizeof(double));
            return;
        }
        if (dim != h->d)
            throw sair::Error(SAIR_EINVAL, "experience store: feature dimension mismatch");
        sair::store_standardize(h, x, z);
    });
}

sair_status sair_store_effective_sigma(sair_store_t h, double sigma_sim, double* out) {
    if (!h || !out) return bad("null handle");
    return guard(__func__, [&] { *out = sair::store_effective_sigma(h, sigma_sim); });
}

sair_status sair_similarity(const double* a, size_t len_a, const double* b, size_t len_b,
                            double sigma, double* out) {
    if (!out) return bad("null output");
    // experience.cpp:31-33: the dimension check, then the sigma check
    if (len_a != len_b) return bad("similarity: dimension mismatch");
    if (sigma <= 0.0) return bad("similarity: sigma must be positive");
    // Host arithmetic, like sair_store_standardize: an O(d) function of two
    // host vectors (the reference's own scalar helper, called per stored
    // record by the unmodified policy's veto loop, policy.cpp:146-153).  A
    // device round trip per call would cost ~10 us against ~30 ns; the
    // data-parallel veto scan is sair_store_nearest / the fused select.
    // Same additions in the same order and glibc's exp: bit-identical.
    return guard(__func__, [&] {
        double d2 = 0.0;
        for (size_t i = 0; i < len_a; ++i) {
            const double d = a[i] - b[i];
            d2 += d * d;
        }
        *out = std::exp(-d2 / (2.0 * sigma * sigma));
    });
}

sair_status sair_store_surprisal(sair_store_t h, size_t index, const double* x, int dim,
                                 const sair_select_config* cfg, double* out) {
    if (!h || !out) return bad("null handle");
    return guard(__func__, [&] {
        // items_.at(index) first (experience.cpp:145), then standardize(x)
        if (index >= h->n) throw sair::Error(SAIR_ERANGE, "vector::_M_range_check");
        if (dim != h->d)
            throw sair::Error(SAIR_EINVAL, "experience store: feature dimension mismatch");
        *out = sair::store_surprisal(h, index, x, defaults(cfg));
    });
}

sair_status sair_store_select(sair_store_t h, const double* queries, size_t nq, int dim,
                              const sair_select_config* cfg, int64_t* out_idx, double* out_sim,
                              double* out_score, size_t* out_count, int64_t* out_nn_idx,
                              double* out_nn_sim) {
    if (!h) return bad("null handle");
    if (nq && (!queries || !out_count)) return bad("null input");
    if ((out_nn_idx == nullptr) != (out_nn_sim == nullptr)) return bad("nn outputs come in pairs");
    return guard(__func__, [&] {
        sair::store_select(h, queries, nq, dim, defaults(cfg), out_idx, out_sim, out_score,
                           out_count, out_nn_idx, out_nn_sim);
    });
}

sair_status sair_store_nearest(sair_store_t h, const double* queries, size_t nq, int dim,
                               double sigma_sim, int64_t* out_idx, double* out_sim) {
    if (!h) return bad("null handle");
    return guard(__func__, [&] {
        // a select with m = 1 computes the same pass; only the nearest is kept
        sair_select_config c{};
        c.m = 1;
        c.lambda_div = 0.0;
        c.sigma_sim = sigma_sim;
        std::vector<int64_t> idx(nq);
        std::vector<double> sim(nq), score(nq);
        std::vector<size_t> cnt(nq);
        sair::store_select(h, queries, nq, dim, c, idx.data(), sim.data(), score.data(),
                           cnt.data(), out_idx, out_sim);
    });
}

sair_status sair_store_last_stats(sair_store_t h, sair_select_stats* out) {
    if (!h || !out) return bad("null handle");
    *out = h->last;
    return SAIR_OK;
}

sair_status sair_store_set_shard(sair_store_t h, int64_t global_offset) {
    if (!h) return bad("null handle");
    if (h->n) return bad("set_shard: the store already holds records");
    h->gbase = global_offset;
    return SAIR_OK;
}

sair_status sair_store_local_stats(sair_store_t h, double* sum, double* sum_sq, double* xabs,
                                   double* scalars) {
    if (!h) return bad("null handle");
    for (int k = 0; k < h->d && h->n; ++k) {
        if (sum) sum[k] = h->stats.sum[k];
        if (sum_sq) sum_sq[k] = h->stats.sum_sq[k];
        if (xabs) xabs[k] = h->stats.xabs[k];
    }
    if (scalars) {
        scalars[0] = (double)h->n;
        scalars[1] = h->stats.total;
        scalars[2] = h->stats.rabs;
    }
    return SAIR_OK;
}

sair_status sair_store_set_global(sair_store_t h, uint64_t n_global, const double* sum,
                                  const double* sum_sq, const double* xabs, double reward_total,
                                  double reward_absmax, double sigma) {
    if (!h || !sum || !sum_sq || !xabs) return bad("null input");
    if (!h->n) return bad("set_global: append the shard's records first");
    if (n_global < h->n) return bad("set_global: n_global is smaller than the shard");
    const int d = h->d;
    h->sharded = true;
    h->n_global = n_global;
    h->gst.sum.assign(sum, sum + d);
    h->gst.sum_sq.assign(sum_sq, sum_sq + d);
    h->gst.xabs.assign(xabs, xabs + d);
    h->gst.total = reward_total;
    h->gst.rabs = reward_absmax;
    h->gsigma = sigma;
    return SAIR_OK;
}

sair_status sair_store_moments(sair_store_t h, double* mean, double* sd) {
    if (!h || !mean || !sd) return bad("null input");
    if (!h->n) return bad("moments: empty store");
    sair::store_mean_sd(h, mean, sd);
    return SAIR_OK;
}

sair_status sair_sigma_sample_indices(uint64_t n, int64_t* idx, size_t* m) {
    if (!idx || !m) return bad("null input");
    auto v = sair::sigma_sample(n);
    std::memcpy(idx, v.data(), v.size() * 8);
    *m = v.size();
    return SAIR_OK;
}

sair_status sair_sigma_rows(const double* rows, size_t m, int dim, const double* mean,
                            const double* sd, int device, double* out) {
    if (!out || (m && (!rows || !mean || !sd))) return bad("null input");
    return guard(__func__, [&] { *out = sair::sigma_rows(rows, m, dim, mean, sd, device); });
}

sair_status sair_store_select_shard(sair_store_t h, const double* queries, size_t nq, int dim,
                                    const sair_select_config* cfg, int64_t* out_idx,
                                    double* out_sim, double* out_score, double* out_reward,
                                    int32_t* out_round, size_t* out_count) {
    if (!h) return bad("null handle");
    if (nq && (!queries || !out_count)) return bad("null input");
    return guard(__func__, [&] {
        sair::store_select(h, queries, nq, dim, defaults(cfg), out_idx, out_sim, out_score,
                           out_count, nullptr, nullptr, out_reward, out_round);
    });
}

sair_status sair_store_greedy_begin(sair_store_t h, const double* queries, size_t nq, int dim,
                                    const sair_select_config* cfg, double* out_best) {
    if (!h || !queries || !out_best) return bad("null input");
    return guard(__func__, [&] { sair::greedy_begin(h, queries, nq, dim, defaults(cfg), out_best); });
}

sair_status sair_store_greedy_next(sair_store_t h, const int64_t* picks, const double* rows,
                                   double* out_best) {
    if (!h || !picks || !rows || !out_best) return bad("null input");
    return guard(__func__, [&] { sair::greedy_next(h, picks, rows, out_best); });
}

sair_status sair_merge_topk(const double* score, const double* sim, const double* reward,
                            const int32_t* round, const int64_t* gidx, const size_t* count,
                            size_t nshards, size_t nq, size_t m, int device, int64_t* out_idx,
                            double* out_sim, double* out_score, size_t* out_count) {
    if (nq && (!out_count || !count)) return bad("null input");
    if (m > 4096) return bad("merge: m too large");
    return guard(__func__, [&] {
        sair::merge_topk(score, sim, reward, round, gidx, count, nshards, nq, m, device, out_idx,
                         out_sim, out_score, out_count);
    });
}

sair_status sair_merge_topk_packed(const double* d_parts, size_t nshards, size_t nq, size_t m,
                                   int device, void* stream, double* d_out) {
    if (nq && (!d_parts || !d_out)) return bad("null input");
    if (m > 4096) return bad("merge: m too large");
    return guard(__func__, [&] {
        sair::merge_packed(d_parts, nshards, nq, m, device, static_cast<cudaStream_t>(stream), d_out);
    });
}

sair_status sair_store_stream(sair_store_t h, void** stream) {
    if (!h || !stream) return bad("null handle");
    *stream = h->st;
    return SAIR_OK;
}

// ------------------------------------------------------------- frontier --

sair_status sair_frontier_create(double l_max_ms, double c_max, int device, sair_frontier_t* out) {
    if (!out) return bad("null out");
    return guard(__func__, [&] {
        auto* f = new sair_frontier_s();
        try {
            sair::frontier_init(f, l_max_ms, c_max, device);
        } catch (...) {
            delete f;
            throw;
        }
        *out = f;
    });
}

sair_status sair_frontier_destroy(sair_frontier_t f) {
    if (!f) return SAIR_OK;
    return guard(__func__, [&] {
        sair::frontier_free(f);
        delete f;
    });
}

sair_status sair_frontier_clone(sair_frontier_t f, sair_frontier_t* out) {
    if (!f || !out) return bad("null handle");
    return guard(__func__, [&] {
        auto* o = new sair_frontier_s();
        try {
            sair::frontier_clone(f, o);
        } catch (...) {
            delete o;
            throw;
        }
        *out = o;
    });
}

// normalize, pareto.cpp:20-29 (two divisions and clamps: host arithmetic is
// the reference's own; the device path does the same inside the kernels)
static void normalize_host(const sair_frontier_s* f, double l_ms, double cost, double* l,
                           double* c, int* clamped) {
    double pl = l_ms / f->l_max, pc = cost / f->c_max;
    int hit = 0;
    if (pl > 1.0) { pl = 1.0; hit = 1; }
    if (pc > 1.0) { pc = 1.0; hit = 1; }
    if (pl < 0.0) pl = 0.0;
    if (pc < 0.0) pc = 0.0;
    *l = pl;
    *c = pc;
    if (clamped) *clamped = hit;
}

sair_status sair_frontier_normalize(sair_frontier_t f, double l_ms, double cost, double* l,
                                    double* c, int* clamped) {
    if (!f || !l || !c) return bad("null handle");
    normalize_host(f, l_ms, cost, l, c, clamped);
    return SAIR_OK;
}

sair_status sair_frontier_update(sair_frontier_t f, double l_ms, double cost, int* inserted,
                                 int* clamped) {
    if (!f) return bad("null handle");
    return guard(__func__, [&] {
        double pl, pc;
        int cl = 0;
        normalize_host(f, l_ms, cost, &pl, &pc, &cl);
        bool ins = sair::frontier_insert_one(f, pl, pc);
        if (inserted) *inserted = ins;
        if (clamped) *clamped = cl;
    });
}

sair_status sair_frontier_insert_normalized(sair_frontier_t f, double l, double c, int* inserted) {
    if (!f) return bad("null handle");
    return guard(__func__, [&] {
        bool ins = sair::frontier_insert_one(f, l, c);
        if (inserted) *inserted = ins;
    });
}

sair_status sair_frontier_insert_batch(sair_frontier_t f, const double* pts, size_t T,
                                       size_t* new_size) {
    if (!f) return bad("null handle");
    if (T && !pts) return bad("null input");
    return guard(__func__, [&] {
        size_t F = sair::frontier_insert_batch(f, pts, T);
        if (new_size) *new_size = F;
    });
}

sair_status sair_frontier_size(sair_frontier_t f, size_t* F) {
    if (!f || !F) return bad("null handle");
    *F = f->F;
    return SAIR_OK;
}

sair_status sair_frontier_points(sair_frontier_t f, double* l, double* c, size_t cap, size_t* F) {
    if (!f) return bad("null handle");
    if (F) *F = f->F;
    if (l && c) {
        if (cap < f->F) return bad("points: capacity too small");
        std::memcpy(l, f->hl.data(), f->F * 8);
        std::memcpy(c, f->hc.data(), f->F * 8);
    }
    return SAIR_OK;
}

sair_status sair_frontier_bounds(sair_frontier_t f, double* l_max, double* c_max) {
    if (!f) return bad("null handle");
    if (l_max) *l_max = f->l_max;
    if (c_max) *c_max = f->c_max;
    return SAIR_OK;
}

sair_status sair_frontier_hypervolume(sair_frontier_t f, double* out) {
    if (!f || !out) return bad("null handle");
    return guard(__func__, [&] { *out = sair::frontier_point_query(f, 0.0, 0.0, sair::Q_HV, nullptr); });
}

sair_status sair_frontier_strictly_dominated(sair_frontier_t f, double l, double c, int* out) {
    if (!f || !out) return bad("null handle");
    return guard(__func__, [&] { *out = sair::frontier_point_query(f, l, c, sair::Q_DOMINATED, nullptr) != 0.0; });
}

sair_status sair_frontier_contribution(sair_frontier_t f, double l, double c, double* out) {
    if (!f || !out) return bad("null handle");
    return guard(__func__, [&] {
        double dom = 0.0;
        double v = sair::frontier_point_query(f, l, c, sair::Q_CONTRIB, &dom);
        if (dom != 0.0)  // pareto.cpp:68-69
            throw sair::Error(SAIR_ELOGIC,
                              "contribution: point is dominated, caller must branch first");
        *out = v;
    });
}

sair_status sair_frontier_distance(sair_frontier_t f, double l, double c, double* out, int* has) {
    if (!f || !out) return bad("null handle");
    return guard(__func__, [&] {
        double v = sair::frontier_point_query(f, l, c, sair::Q_DISTANCE, nullptr);
        if (has) *has = f->F > 0;
        *out = f->F > 0 ? v : 0.0;
    });
}

sair_status sair_frontier_reward(sair_frontier_t f, double l, double c, double* out) {
    if (!f || !out) return bad("null handle");
    return guard(__func__, [&] { *out = sair::frontier_point_query(f, l, c, sair::Q_REWARD, nullptr); });
}

sair_status sair_frontier_score_batch(sair_frontier_t f, const double* pts, size_t T,
                                      double* out_reward, uint8_t* out_dominated) {
    if (!f) return bad("null handle");
    if (T && (!pts || !out_reward)) return bad("null input");
    return guard(__func__, [&] { sair::frontier_score_batch(f, pts, T, out_reward, out_dominated); });
}

sair_status sair_frontier_score_batch_device(sair_frontier_t f, const double* pts, size_t T,
                                             double* out_reward, uint8_t* out_dominated,
                                             void* stream) {
    if (!f) return bad("null handle");
    if (T && (!pts || !out_reward)) return bad("null input");
    return guard(__func__, [&] {
        sair::DeviceGuard g(f->device);
        sair::frontier_score_batch_device(f, pts, T, out_reward, out_dominated,
                                          static_cast<cudaStream_t>(stream));
    });
}

sair_status sair_dominance_counts(const double* tuples, size_t T, int K, int device,
                                  uint32_t* counts, uint8_t* member) {
    if (T && !tuples) return bad("null input");
    return guard(__func__, [&] { sair::dominance_counts(tuples, T, K, device, counts, member); });
}

sair_status sair_dominance_counts_part(const double* tuples, size_t T, int K, int device, int part,
                                       int nparts, uint32_t* counts, uint8_t* member) {
    if (T && !tuples) return bad("null input");
    return guard(__func__, [&] { sair::dominance_counts(tuples, T, K, device, counts, member, part, nparts); });
}

// ---------------------------------------------------------------- reward --

sair_status sair_action_magnitude(const int32_t* deltas, size_t stages, double* out) {
    if (!out || (stages && !deltas)) return bad("null input");
    return guard(__func__, [&] { *out = sair::action_magnitude(deltas, stages, 0); });
}

sair_status sair_compute_reward(const sair_reward_inputs* in, const int32_t* deltas, size_t stages,
                                sair_frontier_t f, const sair_reward_config* cfg,
                                sair_reward_breakdown* out) {
    if (!in || !f || !cfg || !out || (stages && !deltas)) return bad("null input");
    return guard(__func__, [&] { sair::compute_reward_batch(in, deltas, stages, 1, f, cfg, out); });
}

sair_status sair_decision_step(sair_store_t h, sair_frontier_t f, const double* x, int dim,
                               const sair_select_config* cfg, const sair_reward_inputs* in,
                               const int32_t* deltas, size_t stages,
                               const sair_reward_config* rcfg, int update, int32_t round,
                               int64_t* out_idx, double* out_sim, double* out_score,
                               size_t* out_count, int64_t* out_nn_idx, double* out_nn_sim,
                               sair_reward_breakdown* out_reward, int* out_inserted,
                               int* out_stored) {
    if (!h || !f) return bad("null handle");
    if (!x || !in || !rcfg || !out_count || !out_reward || !out_inserted || !out_stored ||
        (stages && !deltas))
        return bad("null input");
    if ((out_nn_idx == nullptr) != (out_nn_sim == nullptr)) return bad("nn outputs come in pairs");
    return guard(__func__, [&] {
        double pl = 0.0, pc = 0.0;
        normalize_host(f, in->l_after_ms, in->c_after, &pl, &pc, nullptr);
        sair::decision_step(h, f, x, dim, defaults(cfg), in, deltas, stages, rcfg, update != 0,
                            pl, pc, round, out_idx, out_sim, out_score, out_count, out_nn_idx,
                            out_nn_sim, out_reward, out_inserted, out_stored);
    });
}

sair_status sair_compute_reward_batch(const sair_reward_inputs* in, const int32_t* deltas,
                                      size_t stages, size_t T, sair_frontier_t f,
                                      const sair_reward_config* cfg, sair_reward_breakdown* out) {
    if (!f || !cfg || (T && (!in || !out)) || (T && stages && !deltas)) return bad("null input");
    return guard(__func__, [&] { sair::compute_reward_batch(in, deltas, stages, T, f, cfg, out); });
}

sair_status sair_compute_reward_replay(const sair_reward_inputs* in, const int32_t* deltas,
                                       size_t stages, size_t T, const uint8_t* update,
                                       sair_frontier_t f, const sair_reward_config* cfg,
                                       sair_reward_breakdown* out) {
    if (!f || !cfg || (T && (!in || !out || !update)) || (T && stages && !deltas))
        return bad("null input");
    return guard(__func__, [&] { sair::compute_reward_replay(in, deltas, stages, T, update, f, cfg, out); });
}

// ---------------------------------------------------------- frontier set --

sair_status sair_frontier_set_create(size_t P, double l_max_ms, double c_max, int device,
                                     sair_frontier_set_t* out) {
    if (!out) return bad("null out");
    auto* s = new (std::nothrow) sair_frontier_set_s();
    if (!s) return SAIR_ENOMEM;
    sair_status st = guard(__func__, [&] { sair::frontier_set_init(s, P, l_max_ms, c_max, device); });
    if (st != SAIR_OK) {
        delete s;
        return st;
    }
    *out = s;
    return SAIR_OK;
}

sair_status sair_frontier_set_destroy(sair_frontier_set_t s) {
    if (!s) return SAIR_OK;
    sair_status st = guard(__func__, [&] { sair::frontier_set_free(s); });
    delete s;
    return st;
}

sair_status sair_frontier_set_step(sair_frontier_set_t s, const sair_reward_inputs* in,
                                   const int32_t* deltas, size_t stages, const uint8_t* update,
                                   const sair_reward_config* cfg, sair_reward_breakdown* out) {
    if (!s || !cfg || (s->P && (!in || !out || !update)) || (s->P && stages && !deltas))
        return bad("null input");
    return guard(__func__, [&] { sair::frontier_set_step(s, in, deltas, stages, update, cfg, out); });
}

sair_status sair_frontier_set_points(sair_frontier_set_t s, size_t p, double* l, double* c,
                                     size_t cap, size_t* F, double* hypervolume) {
    if (!s || !F) return bad("null input");
    return guard(__func__, [&] { *F = sair::frontier_set_points(s, p, l, c, cap, hypervolume); });
}

}  // extern "C"

// --------------------------------------------------------- multi-GPU ----

sair_status sair_comm_create(const int* devices, int ndev, sair_comm_t* out) {
    if (!out || !devices) return bad("null input");
    return guard(__func__, [&] {
        auto* c = new sair_comm_s();
        try {
            sair::comm_create(devices, ndev, c);
        } catch (...) {
            sair::comm_free(c);
            delete c;
            throw;
        }
        *out = c;
    });
}

sair_status sair_comm_destroy(sair_comm_t c) {
    if (!c) return SAIR_OK;
    return guard(__func__, [&] {
        sair::comm_free(c);
        delete c;
    });
}

sair_status sair_comm_info(sair_comm_t c, int* ndev, int* nccl) {
    if (!c) return bad("null handle");
    if (ndev) *ndev = (int)c->dev.size();
    if (nccl) *nccl = c->nc.empty() ? 0 : 1;
    return SAIR_OK;
}

sair_status sair_sharded_create(sair_comm_t c, double r_min, size_t capacity, sair_sharded_t* out) {
    if (!c || !out) return bad("null input");
    return guard(__func__, [&] {
        auto* h = new sair_sharded_s();
        try {
            sair::sharded_init(h, c, r_min, capacity);
        } catch (...) {
            sair::sharded_free(h);
            delete h;
            throw;
        }
        *out = h;
    });
}

sair_status sair_sharded_destroy(sair_sharded_t h) {
    if (!h) return SAIR_OK;
    return guard(__func__, [&] {
        sair::sharded_free(h);
        delete h;
    });
}

sair_status sair_sharded_append(sair_sharded_t h, const double* ctx, size_t count, int dim,
                                const double* reward, const int32_t* round, uint8_t* accepted,
                                size_t* n_accepted) {
    if (!h) return bad("null handle");
    if (count && (!ctx || !reward)) return bad("null input");
    if (dim <= 0) return bad("experience store: dimension must be positive");
    return guard(__func__, [&] {
        const size_t a = sair::sharded_append(h, ctx, count, dim, reward, round, accepted);
        if (n_accepted) *n_accepted = a;
    });
}

sair_status sair_sharded_append_synthetic(sair_sharded_t h, uint64_t seed, size_t count, int dim,
                                          int clustered) {
    if (!h) return bad("null handle");
    if (dim <= 0) return bad("experience store: dimension must be positive");
    return guard(__func__, [&] { sair::sharded_append_synthetic(h, seed, count, dim, clustered); });
}

sair_status sair_sharded_size(sair_sharded_t h, size_t* n, uint64_t* rejected, size_t* shard_n) {
    if (!h) return bad("null handle");
    if (n) *n = h->n;
    if (rejected) *rejected = h->rejected;
    if (shard_n)
        for (size_t r = 0; r < h->sh.size(); ++r) shard_n[r] = h->sh[r]->n;
    return SAIR_OK;
}

sair_status sair_sharded_effective_sigma(sair_sharded_t h, double sigma_sim, double* out) {
    if (!h || !out) return bad("null input");
    return guard(__func__, [&] { *out = sair::sharded_effective_sigma(h, sigma_sim); });
}

sair_status sair_store_select_sharded(sair_sharded_t h, const double* queries, size_t nq, int dim,
                                      const sair_select_config* cfg, int64_t* out_idx,
                                      double* out_sim, double* out_score, size_t* out_count) {
    if (!h) return bad("null handle");
    if (nq && (!queries || !out_idx || !out_sim || !out_score || !out_count))
        return bad("null input");
    return guard(__func__, [&] {
        sair::sharded_select(h, queries, nq, dim, defaults(cfg), out_idx, out_sim, out_score,
                             out_count);
    });
}

sair_status sair_frontier_insert_batch_sharded(sair_comm_t c, sair_frontier_t f, const double* pts,
                                               size_t T, size_t* new_size) {
    if (!c || !f) return bad("null handle");
    if (T && !pts) return bad("null input");
    return guard(__func__, [&] {
        const size_t F = sair::frontier_insert_batch_sharded(c, f, pts, T);
        if (new_size) *new_size = F;
    });
}

