// ref_capi.cpp -- a C-ABI veneer over the REFERENCE's own classes.
//
// TEST INFRASTRUCTURE ONLY.  Linked with the unmodified reference sources
// (/root/reference/proj/src/{experience,pareto,reward}.cpp) into
// oracle/_ref/libsair_ref.so by oracle/Makefile; never copied, never shipped.
// It lets the Python tests and bench.py's reference arm drive the reference's
// ExperienceBuffer / ParetoFrontier / compute_reward exactly as its callers do
// (harness.cpp:150-261, policy.cpp:140-157).
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "scalelab/experience.hpp"
#include "scalelab/pareto.hpp"
#include "scalelab/reward.hpp"

using namespace scalelab;

#define REF_API extern "C" __attribute__((visibility("default")))

namespace {
thread_local std::string g_err;

// 0 ok, 1 invalid_argument, 2 logic_error, 3 runtime_error, 9 other
template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

SelectionConfig make_cfg(std::size_t m, double lambda, double sigma_sim, int local_mean) {
    SelectionConfig c;
    c.m = m;
    c.lambda_div = lambda;
    c.sigma_sim = sigma_sim;
    c.locally_weighted_mean = local_mean != 0;
    return c;
}
}  // namespace

REF_API const char* ref_last_error() { return g_err.c_str(); }

// ---- ExperienceBuffer ------------------------------------------------------

REF_API void* ref_buffer_new(double r_min) { return new ExperienceBuffer(r_min); }
REF_API void ref_buffer_free(void* h) { delete static_cast<ExperienceBuffer*>(h); }

REF_API int ref_buffer_store(void* h, const double* ctx, int d, double reward, int round,
                             int* accepted) {
    return guard([&] {
        Experience e;
        e.context.assign(ctx, ctx + d);
        e.reward = reward;
        e.round = round;
        *accepted = static_cast<ExperienceBuffer*>(h)->store(std::move(e)) ? 1 : 0;
    });
}

// bulk store of n rows (each gated like store())
REF_API int ref_buffer_store_many(void* h, const double* ctx, std::size_t n, int d,
                                  const double* reward, const int32_t* round) {
    return guard([&] {
        auto* b = static_cast<ExperienceBuffer*>(h);
        for (std::size_t i = 0; i < n; ++i) {
            Experience e;
            e.context.assign(ctx + i * d, ctx + (i + 1) * d);
            e.reward = reward[i];
            e.round = round[i];
            b->store(std::move(e));
        }
    });
}

// persistence (experience.cpp:232-271), for the persistence parity tests
REF_API void* ref_buffer_load(const char* path, double r_min, std::size_t* corrupt) {
    try {
        return new ExperienceBuffer(ExperienceBuffer::load(path, r_min, corrupt));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
REF_API int ref_buffer_persist(void* h, const char* path) {
    return guard([&] { static_cast<ExperienceBuffer*>(h)->persist(path); });
}
REF_API int ref_buffer_get(void* h, std::size_t i, double* ctx, double* reward, int* round) {
    return guard([&] {
        const Experience& e = static_cast<ExperienceBuffer*>(h)->all().at(i);
        std::copy(e.context.begin(), e.context.end(), ctx);
        *reward = e.reward;
        *round = e.round;
    });
}

REF_API std::size_t ref_buffer_size(void* h) { return static_cast<ExperienceBuffer*>(h)->size(); }
REF_API uint64_t ref_buffer_rejected(void* h) {
    return static_cast<ExperienceBuffer*>(h)->rejected();
}

REF_API int ref_buffer_standardize(void* h, const double* x, int d, double* z) {
    return guard([&] {
        std::vector<double> v(x, x + d);
        auto r = static_cast<ExperienceBuffer*>(h)->standardize(v);
        std::memcpy(z, r.data(), r.size() * sizeof(double));
    });
}

REF_API int ref_buffer_effective_sigma(void* h, double sigma_sim, double* out) {
    return guard([&] {
        *out = static_cast<ExperienceBuffer*>(h)->effective_sigma(make_cfg(15, 0.1, sigma_sim, 0));
    });
}

REF_API int ref_buffer_surprisal(void* h, std::size_t index, const double* x, int d,
                                 double sigma_sim, int local_mean, double* out) {
    return guard([&] {
        std::vector<double> v(x, x + d);
        *out = static_cast<ExperienceBuffer*>(h)->surprisal(index, v,
                                                            make_cfg(15, 0.1, sigma_sim, local_mean));
    });
}

// select(): out_round/out_sim/out_score/out_reward get up to m rows, in the
// reference's curriculum order.  Rounds identify rows (tests use round = index).
REF_API int ref_buffer_select(void* h, const double* x, int d, std::size_t m, double lambda,
                              double sigma_sim, int local_mean, int32_t* out_round,
                              double* out_sim, double* out_score, std::size_t* out_count) {
    return guard([&] {
        std::vector<double> v(x, x + d);
        auto sel = static_cast<ExperienceBuffer*>(h)->select(v, make_cfg(m, lambda, sigma_sim,
                                                                         local_mean));
        for (std::size_t i = 0; i < sel.size(); ++i) {
            out_round[i] = sel[i].experience.round;
            out_sim[i] = sel[i].similarity_to_current;
            out_score[i] = sel[i].score;
        }
        *out_count = sel.size();
    });
}

// select() for nq queries on nthreads threads.  sigma must already be warm
// (effective_sigma called once) because select() mutates the sigma cache.
REF_API int ref_buffer_select_batch(void* h, const double* xq, std::size_t nq, int d,
                                    std::size_t m, double lambda, double sigma_sim,
                                    int nthreads, int32_t* out_round, double* out_score,
                                    std::size_t* out_count) {
    return guard([&] {
        auto* b = static_cast<ExperienceBuffer*>(h);
        SelectionConfig cfg = make_cfg(m, lambda, sigma_sim, 0);
        (void)b->effective_sigma(cfg);
        if (nthreads < 1) nthreads = 1;
        std::vector<std::thread> pool;
        for (int t = 0; t < nthreads; ++t)
            pool.emplace_back([&, t] {
                for (std::size_t q = nq * t / nthreads; q < nq * (t + 1) / nthreads; ++q) {
                    std::vector<double> v(xq + q * d, xq + (q + 1) * d);
                    auto sel = b->select(v, cfg);
                    for (std::size_t i = 0; i < sel.size(); ++i) {
                        out_round[q * m + i] = sel[i].experience.round;
                        out_score[q * m + i] = sel[i].score;
                    }
                    out_count[q] = sel.size();
                }
            });
        for (auto& th : pool) th.join();
    });
}

REF_API int ref_similarity(const double* a, const double* b, int da, int db, double sigma,
                           double* out) {
    return guard([&] {
        *out = similarity(std::vector<double>(a, a + da), std::vector<double>(b, b + db), sigma);
    });
}

// ---- ParetoFrontier ----------------------------------------------------------

REF_API int ref_frontier_new(double l_max, double c_max, void** out) {
    return guard([&] { *out = new ParetoFrontier(l_max, c_max); });
}
REF_API void ref_frontier_free(void* h) { delete static_cast<ParetoFrontier*>(h); }

REF_API int ref_frontier_update(void* h, double l_ms, double cost, int* inserted, int* clamped) {
    return guard([&] {
        auto r = static_cast<ParetoFrontier*>(h)->update(l_ms, cost);
        *inserted = r.inserted;
        *clamped = r.clamped;
    });
}

REF_API int ref_frontier_insert_normalized(void* h, double l, double c) {
    return static_cast<ParetoFrontier*>(h)->insert_normalized({l, c}) ? 1 : 0;
}

REF_API std::size_t ref_frontier_points(void* h, double* l, double* c) {
    const auto& p = static_cast<ParetoFrontier*>(h)->points();
    for (std::size_t i = 0; l && i < p.size(); ++i) {
        l[i] = p[i].latency;
        c[i] = p[i].cost;
    }
    return p.size();
}

REF_API double ref_frontier_hypervolume(void* h) {
    return static_cast<ParetoFrontier*>(h)->hypervolume();
}

REF_API int ref_frontier_contribution(void* h, double l, double c, double* out) {
    return guard([&] { *out = static_cast<ParetoFrontier*>(h)->contribution({l, c}); });
}

REF_API int ref_frontier_strictly_dominated(void* h, double l, double c) {
    return static_cast<ParetoFrontier*>(h)->strictly_dominated({l, c}) ? 1 : 0;
}

REF_API double ref_frontier_distance(void* h, double l, double c) {
    auto d = static_cast<ParetoFrontier*>(h)->distance({l, c});
    return d ? *d : -1.0;
}

REF_API double ref_frontier_reward(void* h, double l, double c) {
    return static_cast<ParetoFrontier*>(h)->reward({l, c});
}

REF_API void ref_frontier_normalize(void* h, double l_ms, double cost, double* l, double* c,
                                    int* clamped) {
    bool cl = false;
    auto p = static_cast<ParetoFrontier*>(h)->normalize(l_ms, cost, &cl);
    *l = p.latency;
    *c = p.cost;
    *clamped = cl;
}

// T reward() calls against the fixed frontier (the scoring half of compute_reward)
REF_API void ref_frontier_reward_batch(void* h, const double* pts, std::size_t T, double* out) {
    auto* f = static_cast<ParetoFrontier*>(h);
    for (std::size_t t = 0; t < T; ++t) out[t] = f->reward({pts[2 * t], pts[2 * t + 1]});
}

// T sequential insert_normalized() calls (the update loop)
REF_API void ref_frontier_insert_batch(void* h, const double* pts, std::size_t T,
                                       uint8_t* inserted) {
    auto* f = static_cast<ParetoFrontier*>(h);
    for (std::size_t t = 0; t < T; ++t) {
        bool ins = f->insert_normalized({pts[2 * t], pts[2 * t + 1]});
        if (inserted) inserted[t] = ins;
    }
}

// ---- reward --------------------------------------------------------------------

// cfg: {t_sla, l_baseline (0 = 4*t_sla), c_budget, w_latency, w_cost, w_proactive, r_max}
// deltas: stages x {replicas, cpu_mc, mem_mb, rate_tenths}
// out: {latency, cost, sla, proactive, pareto, total, clipped}
REF_API int ref_compute_reward(const double* in, const int32_t* deltas, std::size_t stages,
                               void* frontier, const double* cfg, double* out) {
    return guard([&] {
        RewardInputs ri{in[0], in[1], in[2], in[3]};
        ScalingAction a = ScalingAction::noop(stages);
        for (std::size_t s = 0; s < stages; ++s) {
            a.stages[s].replicas = deltas[4 * s];
            a.stages[s].cpu_millicores = deltas[4 * s + 1];
            a.stages[s].memory_mb = deltas[4 * s + 2];
            a.stages[s].rate_ratio_tenths = deltas[4 * s + 3];
        }
        RewardConfig rc;
        rc.t_sla_ms = cfg[0];
        rc.l_baseline_ms = cfg[1];
        rc.c_budget = cfg[2];
        rc.w_latency = cfg[3];
        rc.w_cost = cfg[4];
        rc.w_proactive = cfg[5];
        rc.r_max = cfg[6];
        auto r = compute_reward(ri, a, *static_cast<ParetoFrontier*>(frontier), rc);
        out[0] = r.latency;
        out[1] = r.cost;
        out[2] = r.sla;
        out[3] = r.proactive;
        out[4] = r.pareto;
        out[5] = r.total;
        out[6] = r.clipped ? 1.0 : 0.0;
    });
}

REF_API double ref_action_magnitude(const int32_t* deltas, std::size_t stages) {
    ScalingAction a = ScalingAction::noop(stages);
    for (std::size_t s = 0; s < stages; ++s) {
        a.stages[s].replicas = deltas[4 * s];
        a.stages[s].cpu_millicores = deltas[4 * s + 1];
        a.stages[s].memory_mb = deltas[4 * s + 2];
        a.stages[s].rate_ratio_tenths = deltas[4 * s + 3];
    }
    return action_magnitude(a);
}
