/*
 * sair_oracle.c -- CPU oracle for the SAIR retrieval + Pareto hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker, never the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product path (libsair.so) has no
 * CPU fallback and never links this.
 *
 * A plain-C fp64 restatement of the reference algorithm, statement by
 * statement, so results are bit-identical to the reference's own code
 * (pinned in tests/test_oracle.py against oracle/_ref, which is the reference
 * compiled from /root/reference/proj/src, and against tests/golden/).
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/proj).
 *
 * One deliberate restructuring, bit-identical by construction:
 * ExperienceBuffer::loo_mean re-sums every reward on every call
 * (src/experience.cpp:138-140), making select O(n^2).  The sum is
 * loop-invariant and always accumulated in index order from 0.0, so it is
 * computed once per select here: same additions, same order, same bits.
 *
 * Compile: gcc -O3 -std=c11 -fPIC -shared -pthread (no -ffast-math, no
 * -march flags: x86-64 baseline has no FMA contraction, matching the
 * reference's Release build, CMakeLists.txt:8-12).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------------ */
/* Retrieval                                                                */
/* ------------------------------------------------------------------------ */

/* Running per-dimension sums in append order: src/experience.cpp:55-58. */
ORC_API void orc_stats(const double* ctx, size_t n, int d, double* sum, double* sum_sq) {
    for (int k = 0; k < d; ++k) { sum[k] = 0.0; sum_sq[k] = 0.0; }
    for (size_t i = 0; i < n; ++i) {
        const double* x = ctx + i * (size_t)d;
        for (int k = 0; k < d; ++k) {
            sum[k] += x[k];
            sum_sq[k] += x[k] * x[k];
        }
    }
}

/* Reward total in index order, from 0.0: src/experience.cpp:138-139. */
ORC_API double orc_reward_total(const double* reward, size_t n) {
    double total = 0.0;
    for (size_t i = 0; i < n; ++i) total += reward[i];
    return total;
}

/* ExperienceBuffer::standardize, src/experience.cpp:64-78.  n == 0 copies x. */
ORC_API void orc_standardize(size_t n, int d, const double* sum, const double* sum_sq,
                             const double* x, double* z) {
    if (n == 0) {
        for (int k = 0; k < d; ++k) z[k] = x[k];
        return;
    }
    double nn = (double)n;
    for (int k = 0; k < d; ++k) {
        double mean = sum[k] / nn;
        double var = sum_sq[k] / nn - mean * mean;
        if (var < 0.0) var = 0.0; /* std::max(0.0, v) */
        double sd = sqrt(var);
        if (sd < 1e-12) sd = 1.0;
        z[k] = (x[k] - mean) / sd;
    }
}

/* similarity, src/experience.cpp:30-40 (caller guarantees sigma > 0). */
ORC_API double orc_similarity(const double* a, const double* b, int d, double sigma) {
    double d2 = 0.0;
    for (int k = 0; k < d; ++k) {
        double t = a[k] - b[k];
        d2 += t * t;
    }
    return exp(-d2 / (2.0 * sigma * sigma));
}

static int cmp_double(const void* a, const void* b) {
    double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}

/* refresh_sigma_cache, src/experience.cpp:80-114: median pairwise z-distance
 * over the strided 512-subsample; the element nth_element places at size/2,
 * i.e. the (size/2)-th order statistic.  Returns 1.0 for < 2 rows. */
ORC_API double orc_sigma_median(const double* ctx, size_t n, int d, const double* sum,
                                const double* sum_sq) {
    const size_t cap = 512;
    size_t m = n <= cap ? n : cap;
    size_t* idx = (size_t*)malloc((m ? m : 1) * sizeof(size_t));
    if (n <= cap) {
        for (size_t k = 0; k < n; ++k) idx[k] = k;
    } else {
        double stride = (double)n / (double)cap;
        for (size_t k = 0; k < cap; ++k) idx[k] = (size_t)((double)k * stride);
    }
    double* z = (double*)malloc((m ? m : 1) * (size_t)d * sizeof(double) + 1);
    for (size_t a = 0; a < m; ++a)
        orc_standardize(n, d, sum, sum_sq, ctx + idx[a] * (size_t)d, z + a * (size_t)d);
    size_t np = m * (m - (m ? 1 : 0)) / 2;
    double sigma = 1.0;
    if (np > 0) {
        double* dists = (double*)malloc(np * sizeof(double));
        size_t p = 0;
        for (size_t i = 0; i < m; ++i)
            for (size_t j = i + 1; j < m; ++j) {
                double d2 = 0.0;
                for (int k = 0; k < d; ++k) {
                    double t = z[i * (size_t)d + k] - z[j * (size_t)d + k];
                    d2 += t * t;
                }
                dists[p++] = sqrt(d2);
            }
        /* the order statistic is unique regardless of the selection method */
        qsort(dists, np, sizeof(double), cmp_double);
        double mid = dists[np / 2];
        sigma = mid > 1e-12 ? mid : 1.0;
        free(dists);
    }
    free(z);
    free(idx);
    return sigma;
}

typedef struct {
    const double* ctx;    /* n x d raw contexts (row-major) */
    const double* reward; /* n */
    const int32_t* round; /* n */
    size_t n;
    int d;
    const double* sum;
    const double* sum_sq;
    double total; /* reward total (orc_reward_total) */
    size_t n_loo; /* records of the whole buffer (== n unless this is a shard) */
} orc_store;

/* Per-record surprisal score: src/experience.cpp:163-167 with the global
 * leave-one-out mean of :214-231 (locally_weighted_mean == false). */
static void score_all(const orc_store* s, const double* zq, double sigma, double* score,
                      double* sim_curr, double* ztmp) {
    size_t n = s->n;
    int d = s->d;
    for (size_t i = 0; i < n; ++i) {
        orc_standardize(s->n_loo, d, s->sum, s->sum_sq, s->ctx + i * (size_t)d, ztmp);
        double sim = orc_similarity(ztmp, zq, d, sigma);
        size_t nl = s->n_loo;
        double loo = nl <= 1 ? 0.0 : (s->total - s->reward[i]) / (double)(nl - 1);
        sim_curr[i] = sim;
        score[i] = sim * fabs(s->reward[i] - loo);
    }
}

/* Kernel-weighted leave-one-out mean, src/experience.cpp:125-137, falling back
 * to the global mean when the weights vanish. */
static double loo_local(const orc_store* s, size_t i, double sigma, double* zi, double* zj) {
    size_t n = s->n;
    int d = s->d;
    if (n <= 1) return 0.0;
    orc_standardize(n, d, s->sum, s->sum_sq, s->ctx + i * (size_t)d, zi);
    double wsum = 0.0, acc = 0.0;
    for (size_t j = 0; j < n; ++j) {
        if (j == i) continue;
        orc_standardize(n, d, s->sum, s->sum_sq, s->ctx + j * (size_t)d, zj);
        double w = orc_similarity(zj, zi, d, sigma);
        wsum += w;
        acc += w * s->reward[j];
    }
    if (wsum > 1e-12) return acc / wsum;
    return (s->total - s->reward[i]) / (double)(n - 1);
}

/* ExperienceBuffer::select, src/experience.cpp:151-205.
 * Writes up to min(m, n) picks in curriculum order (stable sort by reward asc,
 * round asc over pick order, :290-294).  Returns the number written. */
static size_t select_one(const orc_store* s, const double* x, size_t m, double lambda,
                         double sigma, int local_mean, int64_t* out_idx, double* out_sim,
                         double* out_score) {
    size_t n = s->n;
    int d = s->d;
    if (n == 0 || m == 0) return 0;
    double* zq = (double*)malloc((size_t)d * sizeof(double));
    double* zi = (double*)malloc((size_t)d * sizeof(double));
    double* zj = (double*)malloc((size_t)d * sizeof(double));
    double* score = (double*)malloc(n * sizeof(double));
    double* sim_curr = (double*)malloc(n * sizeof(double));
    double* penalty = (double*)calloc(n, sizeof(double));
    unsigned char* taken = (unsigned char*)calloc(n, 1);
    orc_standardize(s->n_loo, d, s->sum, s->sum_sq, x, zq);
    score_all(s, zq, sigma, score, sim_curr, zi);
    if (local_mean) {
        for (size_t i = 0; i < n; ++i) {
            double loo = loo_local(s, i, sigma, zi, zj);
            score[i] = sim_curr[i] * fabs(s->reward[i] - loo);
        }
    }
    size_t want = m < n ? m : n;
    int64_t* chosen = (int64_t*)malloc(want * sizeof(int64_t));
    for (size_t step = 0; step < want; ++step) {
        int64_t best = -1;
        double best_gain = 0.0;
        for (size_t i = 0; i < n; ++i) {
            if (taken[i]) continue;
            double gain = score[i] - lambda * penalty[i];
            int better = best < 0 || gain > best_gain ||
                         (gain == best_gain && s->round[i] < s->round[best]);
            if (better) {
                best = (int64_t)i;
                best_gain = gain;
            }
        }
        taken[best] = 1;
        chosen[step] = best;
        /* penalty += sim(z_i, z_b); with lambda == 0 the gain is score - 0 and
         * the (finite) penalties never influence a pick, so skip the update. */
        if (lambda != 0.0) {
            orc_standardize(s->n_loo, d, s->sum, s->sum_sq, s->ctx + (size_t)best * (size_t)d, zj);
            for (size_t i = 0; i < n; ++i) {
                if (taken[i]) continue;
                orc_standardize(s->n_loo, d, s->sum, s->sum_sq, s->ctx + i * (size_t)d, zi);
                penalty[i] += orc_similarity(zi, zj, d, sigma);
            }
        }
    }
    /* stable insertion sort by (reward asc, round asc) over pick order */
    for (size_t a = 1; a < want; ++a) {
        int64_t v = chosen[a];
        size_t b = a;
        while (b > 0) {
            int64_t u = chosen[b - 1];
            int less = s->reward[v] != s->reward[u] ? s->reward[v] < s->reward[u]
                                                    : s->round[v] < s->round[u];
            if (!less) break;
            chosen[b] = u;
            --b;
        }
        chosen[b] = v;
    }
    for (size_t a = 0; a < want; ++a) {
        out_idx[a] = chosen[a];
        if (out_sim) out_sim[a] = sim_curr[chosen[a]];
        if (out_score) out_score[a] = score[chosen[a]];
    }
    free(chosen); free(taken); free(penalty); free(sim_curr); free(score);
    free(zj); free(zi); free(zq);
    return want;
}

ORC_API size_t orc_select(const double* ctx, const double* reward, const int32_t* round,
                          size_t n, int d, const double* sum, const double* sum_sq,
                          const double* x, size_t m, double lambda, double sigma,
                          int local_mean, int64_t* out_idx, double* out_sim, double* out_score) {
    orc_store s = {ctx, reward, round, n, d, sum, sum_sq, orc_reward_total(reward, n), n};
    return select_one(&s, x, m, lambda, sigma, local_mean, out_idx, out_sim, out_score);
}

/* select() restricted to one shard [0, n) of a buffer of n_global records whose
 * sums / reward total are given: the reference's per-record arithmetic with
 * the buffer's n (experience.cpp:68-75, :229-231); indices are shard-local. */
ORC_API size_t orc_select_shard(const double* ctx, const double* reward, const int32_t* round,
                                size_t n, int d, const double* sum, const double* sum_sq,
                                size_t n_global, double total, const double* x, size_t m,
                                double sigma, int64_t* out_idx, double* out_sim,
                                double* out_score) {
    orc_store s = {ctx, reward, round, n, d, sum, sum_sq, total, n_global};
    return select_one(&s, x, m, 0.0, sigma, 0, out_idx, out_sim, out_score);
}

/* refresh_sigma_cache's median over given subsample rows (m x d), standardized
 * with an n-record buffer's sums (experience.cpp:92-112). */
ORC_API double orc_sigma_rows(const double* rows, size_t m, int d, size_t n, const double* sum,
                              const double* sum_sq) {
    double* z = (double*)malloc((m ? m : 1) * (size_t)d * sizeof(double));
    for (size_t a = 0; a < m; ++a) orc_standardize(n, d, sum, sum_sq, rows + a * (size_t)d, z + a * (size_t)d);
    size_t np = m * (m - (m ? 1 : 0)) / 2;
    double sigma = 1.0;
    if (np > 0) {
        double* dists = (double*)malloc(np * sizeof(double));
        size_t p = 0;
        for (size_t i = 0; i < m; ++i)
            for (size_t j = i + 1; j < m; ++j) {
                double d2 = 0.0;
                for (int k = 0; k < d; ++k) {
                    double t = z[i * (size_t)d + k] - z[j * (size_t)d + k];
                    d2 += t * t;
                }
                dists[p++] = sqrt(d2);
            }
        qsort(dists, np, sizeof(double), cmp_double);
        double mid = dists[np / 2];
        sigma = mid > 1e-12 ? mid : 1.0;
        free(dists);
    }
    free(z);
    return sigma;
}

/* ExperienceBuffer::surprisal, src/experience.cpp:143-149. */
ORC_API double orc_surprisal(const double* ctx, const double* reward, size_t n, int d,
                             const double* sum, const double* sum_sq, size_t index,
                             const double* x, double sigma, int local_mean) {
    orc_store s = {ctx, reward, NULL, n, d, sum, sum_sq, orc_reward_total(reward, n), n};
    double* zi = (double*)malloc((size_t)d * sizeof(double));
    double* zq = (double*)malloc((size_t)d * sizeof(double));
    double* zj = (double*)malloc((size_t)d * sizeof(double));
    orc_standardize(n, d, sum, sum_sq, ctx + index * (size_t)d, zi);
    orc_standardize(n, d, sum, sum_sq, x, zq);
    double sim = orc_similarity(zi, zq, d, sigma);
    double loo;
    if (n <= 1)
        loo = 0.0;
    else if (local_mean)
        loo = loo_local(&s, index, sigma, zi, zj);
    else
        loo = (s.total - reward[index]) / (double)(n - 1);
    free(zj); free(zq); free(zi);
    return sim * fabs(reward[index] - loo);
}

/* MockBackend veto scan, src/policy.cpp:140-153: argmax similarity with strict
 * '>' (first index wins ties), best_sim starting at -1.  Returns the index. */
ORC_API int64_t orc_nearest(const double* ctx, size_t n, int d, const double* sum,
                            const double* sum_sq, const double* x, double sigma,
                            double* out_sim) {
    double* zq = (double*)malloc((size_t)d * sizeof(double));
    double* zi = (double*)malloc((size_t)d * sizeof(double));
    orc_standardize(n, d, sum, sum_sq, x, zq);
    double best_sim = -1.0;
    int64_t best = -1;
    for (size_t i = 0; i < n; ++i) {
        orc_standardize(n, d, sum, sum_sq, ctx + i * (size_t)d, zi);
        double s = orc_similarity(zi, zq, d, sigma);
        if (s > best_sim) {
            best_sim = s;
            best = (int64_t)i;
        }
    }
    free(zi); free(zq);
    if (out_sim) *out_sim = best_sim;
    return best;
}

/* Multi-query select on `nthreads` host threads (the CPU baseline leg; queries
 * partitioned like the reference's sweep pool, tools/scalelab_cli.cpp:67-76). */
typedef struct {
    const orc_store* s;
    const double* xq;
    size_t q0, q1, m;
    double lambda, sigma;
    int64_t* out_idx;
    double* out_sim;
    double* out_score;
    size_t* out_count;
} batch_job;

static void* batch_worker(void* p) {
    batch_job* j = (batch_job*)p;
    for (size_t q = j->q0; q < j->q1; ++q)
        j->out_count[q] = select_one(j->s, j->xq + q * (size_t)j->s->d, j->m, j->lambda,
                                     j->sigma, 0, j->out_idx + q * j->m,
                                     j->out_sim ? j->out_sim + q * j->m : NULL,
                                     j->out_score ? j->out_score + q * j->m : NULL);
    return NULL;
}

ORC_API void orc_select_batch(const double* ctx, const double* reward, const int32_t* round,
                              size_t n, int d, const double* sum, const double* sum_sq,
                              const double* xq, size_t nq, size_t m, double lambda,
                              double sigma, int nthreads, int64_t* out_idx, double* out_sim,
                              double* out_score, size_t* out_count) {
    orc_store s = {ctx, reward, round, n, d, sum, sum_sq, orc_reward_total(reward, n), n};
    if (nthreads < 1) nthreads = 1;
    if ((size_t)nthreads > nq) nthreads = (int)(nq ? nq : 1);
    pthread_t* th = (pthread_t*)malloc((size_t)nthreads * sizeof(pthread_t));
    batch_job* jobs = (batch_job*)malloc((size_t)nthreads * sizeof(batch_job));
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = (batch_job){&s, xq, nq * (size_t)t / (size_t)nthreads,
                              nq * (size_t)(t + 1) / (size_t)nthreads, m, lambda, sigma,
                              out_idx, out_sim, out_score, out_count};
        pthread_create(&th[t], NULL, batch_worker, &jobs[t]);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(jobs);
    free(th);
}

/* ------------------------------------------------------------------------ */
/* Synthetic stores at full size (test infrastructure)                       */
/* ------------------------------------------------------------------------ */

/* paper_2601_22397_b200/synth.py contexts()/rewards() restated in C on host
 * threads, so a 16M x 64 host copy of a device-generated store takes seconds
 * (pinned == synth.py in tests/test_oracle.py). */
static uint64_t sm64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static uint64_t synth_key(int64_t seed, uint64_t stream) {
    return (uint64_t)seed * 0x100000001B3ull + stream * 0x9E3779B1ull;
}

typedef struct {
    int64_t seed;
    size_t start, r0, r1;
    int d;
    double* out;
} synth_job;

static void* synth_worker(void* p) {
    synth_job* j = (synth_job*)p;
    uint64_t key = synth_key(j->seed, 1);
    for (size_t r = j->r0; r < j->r1; ++r)
        for (int k = 0; k < j->d; ++k) {
            uint64_t h = sm64(((uint64_t)(j->start + r) * (uint64_t)j->d + (uint64_t)k) ^ key);
            int64_t s = (int64_t)(h & 0xFFF) + (int64_t)((h >> 12) & 0xFFF) +
                        (int64_t)((h >> 24) & 0xFFF) + (int64_t)((h >> 36) & 0xFFF);
            j->out[r * (size_t)j->d + (size_t)k] = (double)(s - 8190) * (1.0 / 2048.0);
        }
    return NULL;
}

ORC_API void orc_synth_contexts(int64_t seed, size_t start, size_t count, int d, int nthreads,
                                double* out) {
    if (nthreads < 1) nthreads = 1;
    pthread_t* th = (pthread_t*)malloc((size_t)nthreads * sizeof(pthread_t));
    synth_job* jobs = (synth_job*)malloc((size_t)nthreads * sizeof(synth_job));
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = (synth_job){seed, start, count * (size_t)t / (size_t)nthreads,
                              count * (size_t)(t + 1) / (size_t)nthreads, d, out};
        pthread_create(&th[t], NULL, synth_worker, &jobs[t]);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(jobs);
    free(th);
}

/* ------------------------------------------------------------------------ */
/* Pareto frontier (2 objectives) -- src/pareto.cpp                         */
/* ------------------------------------------------------------------------ */

/* dominates, src/pareto.cpp:9-12 */
static int dom2(double pl, double pc, double ql, double qc) {
    return pl <= ql && pc <= qc && (pl < ql || pc < qc);
}

/* ParetoFrontier::normalize, src/pareto.cpp:20-29 */
ORC_API void orc_normalize(double l_max, double c_max, double l_ms, double cost, double* pl,
                           double* pc, int* clamped) {
    double l = l_ms / l_max, c = cost / c_max;
    int hit = 0;
    if (l > 1.0) { l = 1.0; hit = 1; }
    if (c > 1.0) { c = 1.0; hit = 1; }
    if (l < 0.0) l = 0.0;
    if (c < 0.0) c = 0.0;
    *pl = l;
    *pc = c;
    if (clamped) *clamped = hit;
}

/* strictly_dominated, src/pareto.cpp:31-34 */
ORC_API int orc_strictly_dominated(const double* fl, const double* fc, size_t F, double pl,
                                   double pc) {
    for (size_t i = 0; i < F; ++i)
        if (dom2(fl[i], fc[i], pl, pc)) return 1;
    return 0;
}

/* insert_normalized, src/pareto.cpp:43-54.  fl/fc have capacity >= *F + 1. */
ORC_API int orc_frontier_insert(double* fl, double* fc, size_t* F, double pl, double pc) {
    size_t n = *F;
    for (size_t i = 0; i < n; ++i)
        if ((fl[i] == pl && fc[i] == pc) || dom2(fl[i], fc[i], pl, pc)) return 0;
    size_t w = 0;
    for (size_t i = 0; i < n; ++i) {
        if (dom2(pl, pc, fl[i], fc[i])) continue;
        fl[w] = fl[i];
        fc[w] = fc[i];
        ++w;
    }
    /* lower_bound by latency */
    size_t pos = 0;
    while (pos < w && fl[pos] < pl) ++pos;
    for (size_t i = w; i > pos; --i) {
        fl[i] = fl[i - 1];
        fc[i] = fc[i - 1];
    }
    fl[pos] = pl;
    fc[pos] = pc;
    *F = w + 1;
    return 1;
}

/* hypervolume, src/pareto.cpp:56-65 */
ORC_API double orc_hypervolume(const double* fl, const double* fc, size_t F) {
    double hv = 0.0;
    for (size_t i = 0; i < F; ++i) {
        double next = (i + 1 < F) ? fl[i + 1] : 1.0;
        hv += (next - fl[i]) * (1.0 - fc[i]);
    }
    return hv;
}

/* contribution, src/pareto.cpp:67-73 (copy, insert, difference of volumes).
 * Returns NAN for a dominated point (the reference throws logic_error). */
ORC_API double orc_contribution(const double* fl, const double* fc, size_t F, double pl,
                                double pc) {
    if (orc_strictly_dominated(fl, fc, F, pl, pc)) return NAN;
    double* wl = (double*)malloc((F + 1) * sizeof(double));
    double* wc = (double*)malloc((F + 1) * sizeof(double));
    memcpy(wl, fl, F * sizeof(double));
    memcpy(wc, fc, F * sizeof(double));
    size_t W = F;
    orc_frontier_insert(wl, wc, &W, pl, pc);
    double r = orc_hypervolume(wl, wc, W) - orc_hypervolume(fl, fc, F);
    free(wc);
    free(wl);
    return r;
}

/* distance, src/pareto.cpp:75-84; returns -1 for an empty frontier (nullopt) */
ORC_API double orc_distance(const double* fl, const double* fc, size_t F, double pl,
                            double pc) {
    if (F == 0) return -1.0;
    double best = INFINITY;
    for (size_t i = 0; i < F; ++i) {
        double dl = pl - fl[i], dc = pc - fc[i];
        double v = dl * dl + dc * dc;
        if (v < best) best = v; /* std::min(best, v) */
    }
    return sqrt(best);
}

/* reward, src/pareto.cpp:86-89 */
ORC_API double orc_pareto_reward(const double* fl, const double* fc, size_t F, double pl,
                                 double pc) {
    if (!orc_strictly_dominated(fl, fc, F, pl, pc))
        return 1.0 + orc_contribution(fl, fc, F, pl, pc);
    return 0.8 / (1.0 + orc_distance(fl, fc, F, pl, pc));
}

/* Batch: score each of T normalized points against the fixed frontier
 * (the scoring half of compute_reward, src/reward.cpp:42-43). */
ORC_API void orc_pareto_reward_batch(const double* fl, const double* fc, size_t F,
                                     const double* pts, size_t T, double* out) {
    for (size_t t = 0; t < T; ++t)
        out[t] = orc_pareto_reward(fl, fc, F, pts[2 * t], pts[2 * t + 1]);
}

/* Batch frontier maintenance: sequential update over T normalized points,
 * exactly the reference's loop (harness.cpp:251 / scalelab_cli.cpp:124-135). */
ORC_API size_t orc_frontier_insert_seq(double* fl, double* fc, size_t F, const double* pts,
                                       size_t T, uint8_t* inserted) {
    for (size_t t = 0; t < T; ++t) {
        int ins = orc_frontier_insert(fl, fc, &F, pts[2 * t], pts[2 * t + 1]);
        if (inserted) inserted[t] = (uint8_t)ins;
    }
    return F;
}

/* ------------------------------------------------------------------------ */
/* K-objective dominance counts (no reference beyond dominates()) */
/* ------------------------------------------------------------------------ */

/* component-wise generalisation of dominates(), src/pareto.cpp:9-12 */
static int domk(const double* p, const double* q, int K) {
    int strict = 0;
    for (int k = 0; k < K; ++k) {
        if (p[k] > q[k]) return 0;
        if (p[k] < q[k]) strict = 1;
    }
    return strict;
}

/* counts[i] = #{j : tuple j dominates tuple i};
 * member[i] = counts[i] == 0 and no equal tuple at a lower index (the
 * first-occurrence rule of tests/test_pareto.cpp:17-33). */
ORC_API void orc_dominance_counts(const double* tuples, size_t T, int K, uint32_t* counts,
                                  uint8_t* member) {
    for (size_t i = 0; i < T; ++i) {
        const double* pi = tuples + i * (size_t)K;
        uint32_t c = 0;
        int dup_before = 0;
        for (size_t j = 0; j < T; ++j) {
            if (j == i) continue;
            const double* pj = tuples + j * (size_t)K;
            if (domk(pj, pi, K)) {
                ++c;
            } else if (j < i && !dup_before) {
                int eq = 1;
                for (int k = 0; k < K; ++k) eq &= pj[k] == pi[k];
                dup_before = eq;
            }
        }
        if (counts) counts[i] = c;
        if (member) member[i] = (uint8_t)(c == 0 && !dup_before);
    }
}

/* The same counts on `nthreads` host threads: tuple i's count is the loop of
 * orc_dominance_counts above, rows of i partitioned across threads (the
 * per-i arithmetic is unchanged, so the result is identical). */
typedef struct {
    const double* t;
    size_t T, i0, i1;
    int K;
    uint32_t* counts;
    uint8_t* member;
} domk_job;

static void* domk_worker(void* p) {
    domk_job* j = (domk_job*)p;
    for (size_t i = j->i0; i < j->i1; ++i) {
        const double* pi = j->t + i * (size_t)j->K;
        uint32_t c = 0;
        int dup_before = 0;
        for (size_t q = 0; q < j->T; ++q) {
            if (q == i) continue;
            const double* pq = j->t + q * (size_t)j->K;
            if (domk(pq, pi, j->K)) {
                ++c;
            } else if (q < i && !dup_before) {
                int eq = 1;
                for (int k = 0; k < j->K; ++k) eq &= pq[k] == pi[k];
                dup_before = eq;
            }
        }
        if (j->counts) j->counts[i] = c;
        if (j->member) j->member[i] = (uint8_t)(c == 0 && !dup_before);
    }
    return NULL;
}

ORC_API void orc_dominance_counts_mt(const double* tuples, size_t T, int K, int nthreads,
                                     uint32_t* counts, uint8_t* member) {
    if (nthreads < 1) nthreads = 1;
    pthread_t* th = (pthread_t*)malloc((size_t)nthreads * sizeof(pthread_t));
    domk_job* jobs = (domk_job*)malloc((size_t)nthreads * sizeof(domk_job));
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = (domk_job){tuples, T, T * (size_t)t / (size_t)nthreads,
                             T * (size_t)(t + 1) / (size_t)nthreads, K, counts, member};
        pthread_create(&th[t], NULL, domk_worker, &jobs[t]);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(jobs);
    free(th);
}

/* Two objectives at millions of tuples, O(T log T) (an independent algorithm
 * from the device's merge counting; pinned == orc_dominance_counts and the
 * sequential insert loop at small T in tests/test_oracle.py):
 *   count_i = #{j : l_j <= l_i and c_j <= c_i} - #{j : (l_j, c_j) == (l_i, c_i)}
 * (dominates(), src/pareto.cpp:9-12: <= on both axes minus exact equals),
 * by a sweep in (l asc, c asc) order with a Fenwick tree over the c-ranks;
 * a whole run of equal l is inserted before any of its members is counted. */
static const double* g_sort_t; /* qsort has no context argument */
static int cmp_lc(const void* a, const void* b) {
    size_t i = *(const size_t*)a, j = *(const size_t*)b;
    const double *p = g_sort_t + 2 * i, *q = g_sort_t + 2 * j;
    if (p[0] != q[0]) return p[0] < q[0] ? -1 : 1;
    if (p[1] != q[1]) return p[1] < q[1] ? -1 : 1;
    return (i > j) - (i < j);
}

static int cmp_dbl(const void* a, const void* b) {
    double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}

ORC_API void orc_dominance_counts2_sorted(const double* t, size_t T, uint32_t* counts,
                                          uint8_t* member) {
    size_t* ord = (size_t*)malloc((T ? T : 1) * sizeof(size_t));
    double* cs = (double*)malloc((T ? T : 1) * sizeof(double));
    uint32_t* fen = (uint32_t*)calloc(T + 1, sizeof(uint32_t));
    for (size_t i = 0; i < T; ++i) { ord[i] = i; cs[i] = t[2 * i + 1]; }
    g_sort_t = t;
    qsort(ord, T, sizeof(size_t), cmp_lc);
    qsort(cs, T, sizeof(double), cmp_dbl);
    size_t a = 0;
    while (a < T) {
        size_t b = a;
        while (b < T && t[2 * ord[b]] == t[2 * ord[a]]) ++b;  /* run of equal l */
        for (size_t r = a; r < b; ++r) {                        /* insert the run */
            double c = t[2 * ord[r] + 1];
            size_t lo = 0, hi = T;                               /* rank = #{c' < c} + 1 */
            while (lo < hi) { size_t md = (lo + hi) / 2; if (cs[md] < c) lo = md + 1; else hi = md; }
            for (size_t k = lo + 1; k <= T; k += k & (~k + 1)) fen[k]++;
        }
        size_t r = a;
        while (r < b) {                                          /* runs of equal (l, c) */
            size_t e = r;
            while (e < b && t[2 * ord[e] + 1] == t[2 * ord[r] + 1]) ++e;
            double c = t[2 * ord[r] + 1];
            size_t lo = 0, hi = T;                               /* #{c' <= c} */
            while (lo < hi) { size_t md = (lo + hi) / 2; if (cs[md] <= c) lo = md + 1; else hi = md; }
            uint32_t le = 0;
            for (size_t k = lo; k > 0; k -= k & (~k + 1)) le += fen[k];
            uint32_t cnt = le - (uint32_t)(e - r);
            for (size_t q = r; q < e; ++q) {
                size_t i = ord[q];
                if (counts) counts[i] = cnt;
                /* the first occurrence (lowest index) of a value: ord is
                 * index-ascending inside an equal run */
                if (member) member[i] = (uint8_t)(cnt == 0 && q == r);
            }
            r = e;
        }
        a = b;
    }
    free(fen);
    free(cs);
    free(ord);
}

/* The frontier the sequential insert loop leaves (src/pareto.cpp:43-54 over
 * every point), for millions of points: insert_normalized keeps exactly the
 * non-dominated distinct values, sorted by latency (the loop's result does not
 * depend on the order, tests/test_pareto.cpp:127-147); here the points with a
 * zero count.  fl/fc have capacity T; returns F. */
ORC_API size_t orc_frontier_sorted(const double* t, size_t T, double* fl, double* fc) {
    uint8_t* member = (uint8_t*)malloc(T ? T : 1);
    orc_dominance_counts2_sorted(t, T, NULL, member);
    size_t F = 0;
    for (size_t i = 0; i < T; ++i)
        if (member[i]) { fl[F] = t[2 * i]; fc[F] = t[2 * i + 1]; ++F; }
    free(member);
    /* sort by latency (distinct frontier points have distinct latencies) */
    size_t* ord = (size_t*)malloc((F ? F : 1) * sizeof(size_t));
    double* tmp = (double*)malloc((F ? F : 1) * 2 * sizeof(double));
    for (size_t i = 0; i < F; ++i) { ord[i] = i; tmp[2 * i] = fl[i]; tmp[2 * i + 1] = fc[i]; }
    g_sort_t = tmp;
    qsort(ord, F, sizeof(size_t), cmp_lc);
    for (size_t i = 0; i < F; ++i) { fl[i] = tmp[2 * ord[i]]; fc[i] = tmp[2 * ord[i] + 1]; }
    free(tmp);
    free(ord);
    return F;
}

/* ------------------------------------------------------------------------ */
/* Reward -- src/reward.cpp                                                  */
/* ------------------------------------------------------------------------ */

/* action_magnitude, src/reward.cpp:9-19; deltas = S x {replicas, cpu_mc,
 * memory_mb, rate_tenths}; kCpuStepMillicores = 500, kMemStepMb = 256
 * (include/scalelab/action.hpp:17-18). */
ORC_API double orc_action_magnitude(const int32_t* deltas, size_t stages) {
    double mu = 0.0;
    int scaled = 0;
    for (size_t s = 0; s < stages; ++s) {
        const int32_t* d = deltas + 4 * s;
        mu += (double)abs(d[0]);
        mu += 0.5 * ((double)abs(d[1]) / (double)500 + (double)abs(d[2]) / (double)256 +
                     (double)abs(d[3]) / 10.0);
        scaled += (d[0] | d[1] | d[2] | d[3]) != 0;
    }
    mu += 0.5 * scaled;
    return mu;
}

/* compute_reward, src/reward.cpp:21-44.  cfg = {t_sla, l_base (resolved),
 * c_budget, w_latency, w_cost, w_proactive, r_max}; in = {l_before, l_after,
 * c_before, c_after}; out = {latency, cost, sla, proactive, pareto, total,
 * clipped}.  The frontier is given normalised; l_max/c_max normalise the
 * outcome.  Returns 0, or -1 on the reference's invalid_argument cases. */
ORC_API int orc_compute_reward(const double* in, double mu, const double* fl, const double* fc,
                               size_t F, double l_max, double c_max, const double* cfg,
                               double* out) {
    double t_sla = cfg[0], l_base = cfg[1], c_budget = cfg[2];
    if (t_sla <= 0.0) return -1;
    if (l_base <= 0.0 || c_budget <= 0.0) return -1;
    double latency = cfg[3] * (in[0] - in[1]) / l_base;
    double cost = -cfg[4] * (in[3] - in[2]) / c_budget;
    double sla = 0.0;
    if (in[1] > t_sla) {
        double ratio = in[1] / t_sla;
        sla = -(ratio * ratio) + 1.0;
    }
    double sg = in[0] / t_sla - 1.0;
    if (sg < 0.0) sg = 0.0;
    double proactive = sg * mu * cfg[5];
    double pl, pc;
    orc_normalize(l_max, c_max, in[1], in[3], &pl, &pc, NULL);
    double pareto = orc_pareto_reward(fl, fc, F, pl, pc);
    double sum = latency + cost + sla + proactive + pareto;
    double total = sum < -cfg[6] ? -cfg[6] : (cfg[6] < sum ? cfg[6] : sum); /* std::clamp */
    out[0] = latency;
    out[1] = cost;
    out[2] = sla;
    out[3] = proactive;
    out[4] = pareto;
    out[5] = total;
    out[6] = total != sum ? 1.0 : 0.0;
    return 0;
}
