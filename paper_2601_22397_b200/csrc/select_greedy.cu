// select_greedy.cu -- the exact select() of many queries over a large store in
// lock-step (the path for lambda_div > 0 above the small-store size, and the
// exact fallback of any uncertified batch).
//
// experience.cpp:151-205 with the reference's rounding order throughout (fp64,
// no contraction): every record's score for every query of a batch of G
// queries, then `want` greedy steps.  State per (query, record): score, penalty
// (fp64) and a taken flag, so a step is one pass:
//   greedy_step_kernel   a CTA holds 128 records' standardized rows in shared
//                        memory (dimension-major) and, four queries at a time
//                        (independent fp64 chains), adds sim(z_i, z_pick) of
//                        the previous step's pick to the penalty (:283-284, in
//                        pick order), forms the gain score - lambda pen (:270)
//                        and reduces each warp's best (gain desc, round asc,
//                        index asc) -- no block barriers per query;
//   greedy_pick_kernel   per query: the best of the warps' bests -> the pick,
//                        marked taken, its row staged for the next step.
// All steps of a batch are enqueued without a host round trip; a finish
// kernel writes the curriculum order (:290-294) and the veto scan's nearest
// record.  Compared with one query at a time (select_exact.cu: 3 + 3m
// launches and m passes per query), the G queries share every pass over the
// rows.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "select_common.cuh"

namespace sair {

namespace {

constexpr int GT = 128;  // records per CTA tile (one per thread), 4 warps
constexpr int GW = GT / 32;
constexpr int GQ = 16;   // pick rows staged in shared memory at a time

struct GreedyArgs {
    const double* z;      // [d][n] standardized rows
    const double* r64;
    const int32_t* rnd;
    const double* loo;    // [n] local LOO means or null (global mean)
    const double* zq;     // [G][d] standardized queries
    size_t n, n_loo;
    int d, G, want;
    double total, two_s2, lambda;
    double* score;        // [G][n]
    double* pen;          // [G][n]
    unsigned char* taken; // [G][n]
    Best* part;           // [G][nwarp] per-warp bests of the current step
    Best* part_nn;        // [G][nwarp] per-warp nearest (step 0)
    int64_t* picks;       // [G][m]
    double* zpick;        // [G][d] the previous pick's row
    int nblk;             // warps over the store (nwarp)
};

// step 0 (score = exact surprisal score, pen = 0) or step t > 0 (penalty update
// with the pick of step t - 1), then each warp's best gain per query
template <bool ZSM>
__global__ void __launch_bounds__(GT) greedy_step_kernel(const GreedyArgs a, int step) {
    extern __shared__ double zt[];  // ZSM: [d][GT] | rows [GQ][d]
    double* rows = zt + (ZSM ? (size_t)a.d * GT : 0);
    const size_t i0 = (size_t)blockIdx.x * GT;
    const size_t i = i0 + threadIdx.x;
    const bool valid = i < a.n;
    const int d = a.d, lane = threadIdx.x & 31;
    const size_t wslot = (size_t)blockIdx.x * GW + (threadIdx.x >> 5);
    if (ZSM)
        for (int e = threadIdx.x; e < d * GT; e += GT) {
            const int k = e / GT, j = e % GT;
            zt[e] = i0 + j < a.n ? a.z[(size_t)k * a.n + i0 + j] : 0.0;
        }
    // ZSM: the CTA's rows staged in shared memory (64 KB at d = 64: three CTAs
    // per SM); otherwise read through L1/L2 -- more CTAs per SM, and faster
    // (1M x 64, lambda 0.1: 8 queries 20.8 -> 15.6 ms, 128 queries 156 -> 149)
    const double* mine = ZSM ? zt + threadIdx.x : a.z + (valid ? i : a.n - 1);
    const size_t kstride = ZSM ? GT : a.n;
    const bool pen_step = step > 0 && a.lambda != 0.0;
    const double* src = step == 0 ? a.zq : a.zpick;
    for (int g0 = 0; g0 < a.G; g0 += GQ) {
        const int gn = min(GQ, a.G - g0);
        __syncthreads();
        if (step == 0 || pen_step)
            for (int e = threadIdx.x; e < gn * d; e += GT) rows[e] = src[(size_t)g0 * d + e];
        __syncthreads();
        for (int gg = 0; gg < gn; gg += 4) {
            // four queries at a time: four independent fp64 chains per record,
            // their state loaded before the chains so the loads overlap them
            int gq[4];
            size_t oq[4];
            bool live[4];
            double scq[4] = {0.0, 0.0, 0.0, 0.0}, pnq[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                gq[h] = g0 + min(gg + h, gn - 1);
                oq[h] = (size_t)gq[h] * a.n + i;
                live[h] = valid && gg + h < gn && (step == 0 || !a.taken[oq[h]]);
                if (step > 0 && live[h]) {
                    scq[h] = a.score[oq[h]];
                    if (pen_step) pnq[h] = a.pen[oq[h]];
                }
            }
            double x[4] = {0.0, 0.0, 0.0, 0.0};
            if ((step == 0 || pen_step) && (live[0] || live[1] || live[2] || live[3])) {
                const double* r0 = rows + (size_t)(gq[0] - g0) * d;
                const double* r1 = rows + (size_t)(gq[1] - g0) * d;
                const double* r2 = rows + (size_t)(gq[2] - g0) * d;
                const double* r3 = rows + (size_t)(gq[3] - g0) * d;
#pragma unroll 2
                for (int k = 0; k < d; ++k) {  // similarity(), :125-130, each in k order
                    const double v = mine[k * kstride];
                    const double t0 = dsub(v, r0[k]), t1 = dsub(v, r1[k]);
                    const double t2 = dsub(v, r2[k]), t3 = dsub(v, r3[k]);
                    x[0] = dadd(x[0], dmul(t0, t0));
                    x[1] = dadd(x[1], dmul(t1, t1));
                    x[2] = dadd(x[2], dmul(t2, t2));
                    x[3] = dadd(x[3], dmul(t3, t3));
                }
            }
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                if (gg + h >= gn) break;
                const int g = gq[h];
                const size_t o = oq[h];
                Best b{0.0, 0, 0, -1};
                if (step == 0) {
                    Best nb{0.0, 0, 0, -1};
                    if (valid) {
                        const double s = sim_from_d2(x[h], a.two_s2);
                        const double r = a.r64[i];
                        const double loo = a.loo ? a.loo[i]
                                                 : (a.n_loo <= 1 ? 0.0
                                                                 : ddiv(dsub(a.total, r),
                                                                        (double)(a.n_loo - 1)));
                        const double sc = dmul(s, fabs(dsub(r, loo)));
                        a.score[o] = sc;
                        a.pen[o] = 0.0;
                        a.taken[o] = 0;
                        b = Best{dsub(sc, dmul(a.lambda, 0.0)), a.rnd[i], (int64_t)i, 1};
                        nb = Best{s, 0, (int64_t)i, 1};
                    }
                    if (a.part_nn) {
                        nb = warp_best(nb);
                        if (lane == 0) a.part_nn[(size_t)g * a.nblk + wslot] = nb;
                    }
                } else if (live[h]) {
                    double pn = 0.0;
                    if (pen_step) {
                        pn = dadd(pnq[h], sim_from_d2(x[h], a.two_s2));  // :283-284
                        a.pen[o] = pn;
                    }
                    b = Best{dsub(scq[h], dmul(a.lambda, pn)), a.rnd[i], (int64_t)i, 1};
                }
                b = warp_best(b);
                if (lane == 0) a.part[(size_t)g * a.nblk + wslot] = b;
            }
        }
    }
}

// per query: the step's pick; marks it taken and stages its row
__global__ void greedy_pick_kernel(const GreedyArgs a, int step) {
    const int g = blockIdx.x;
    __shared__ Best wb[32];
    Best b{0.0, 0, 0, -1};
    for (int t = threadIdx.x; t < a.nblk; t += blockDim.x) {
        const Best c = a.part[(size_t)g * a.nblk + t];
        if (better(c, b)) b = c;
    }
    b = warp_best(b);
    if ((threadIdx.x & 31) == 0) wb[threadIdx.x >> 5] = b;
    __syncthreads();
    if (threadIdx.x < 32) {
        Best c = threadIdx.x < (blockDim.x >> 5) ? wb[threadIdx.x] : Best{0.0, 0, 0, -1};
        c = warp_best(c);
        if (threadIdx.x == 0) wb[0] = c;
    }
    __syncthreads();
    const Best w = wb[0];
    const size_t p = (size_t)w.i;
    if (threadIdx.x == 0) {
        a.picks[(size_t)g * a.want + step] = (int64_t)p;
        a.taken[(size_t)g * a.n + p] = 1;
    }
    for (int k = threadIdx.x; k < a.d; k += blockDim.x)
        a.zpick[(size_t)g * a.d + k] = a.z[(size_t)k * a.n + p];
}

// curriculum order (:290-294) and outputs; the nearest record from step 0
__global__ void greedy_finish_kernel(const GreedyArgs a, int64_t gbase, int m, int64_t* out_idx,
                                     double* out_sim, double* out_score, double* out_rew,
                                     int32_t* out_round, int64_t* out_nn, double* out_nn_sim) {
    const int g = blockIdx.x;
    if (threadIdx.x != 0) return;
    const int64_t* pk = a.picks + (size_t)g * a.want;
    int order[256];
    for (int x = 0; x < a.want; ++x) order[x] = x;
    for (int x = 1; x < a.want; ++x) {
        const int v = order[x];
        const double rv = a.r64[pk[v]];
        const int32_t dv = a.rnd[pk[v]];
        int y = x;
        while (y > 0) {
            const int u = order[y - 1];
            const double ru = a.r64[pk[u]];
            const bool less = rv != ru ? rv < ru : dv < a.rnd[pk[u]];
            if (!less) break;
            order[y] = u;
            --y;
        }
        order[y] = v;
    }
    const double* zq = a.zq + (size_t)g * a.d;
    for (int x = 0; x < a.want; ++x) {
        const size_t p = (size_t)pk[order[x]];
        double d2 = 0.0;  // the pick's similarity, recomputed (same sequence)
        for (int k = 0; k < a.d; ++k) {
            const double t = dsub(a.z[(size_t)k * a.n + p], zq[k]);
            d2 = dadd(d2, dmul(t, t));
        }
        const size_t o = (size_t)g * m + x;
        out_idx[o] = gbase + (int64_t)p;
        out_sim[o] = sim_from_d2(d2, a.two_s2);
        out_score[o] = a.score[(size_t)g * a.n + p];
        out_rew[o] = a.r64[p];
        out_round[o] = a.rnd[p];
    }
    if (out_nn) {
        Best b{0.0, 0, 0, -1};
        for (int t = 0; t < a.nblk; ++t) {
            const Best c = a.part_nn[(size_t)g * a.nblk + t];
            if (better(c, b)) b = c;
        }
        out_nn[g] = b.j < 0 ? -1 : gbase + b.i;
        out_nn_sim[g] = b.j < 0 ? -1.0 : b.g;
    }
}

}  // namespace

// Exact select() of the queries `qidx` over the whole store, G at a time.
// the step kernel's variant (SAIR_GREEDY_ZSM=1: rows staged in shared memory)
bool greedy_zsm() {
    static const bool v = std::getenv("SAIR_GREEDY_ZSM") != nullptr;
    return v;
}

size_t greedy_smem(int d) { return ((greedy_zsm() ? (size_t)d * GT : 0) + (size_t)GQ * d) * 8; }

void greedy_step(int nctas, size_t smem, cudaStream_t st, const GreedyArgs& a, int step) {
    if (greedy_zsm()) {
        SAIR_CUDA(cudaFuncSetAttribute(greedy_step_kernel<true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        greedy_step_kernel<true><<<nctas, GT, smem, st>>>(a, step);
    } else {
        greedy_step_kernel<false><<<nctas, GT, smem, st>>>(a, step);
    }
}

void greedy_select(sair_store_s* s, const QueryPrep& p, const std::vector<size_t>& qidx, size_t m,
                   double lambda, const double* loo, bool want_nn, int64_t* out_idx,
                   double* out_sim, double* out_score, size_t* out_count, int64_t* out_nn,
                   double* out_nn_sim, double* out_reward, int32_t* out_round) {
    const size_t nq = qidx.size();
    if (nq == 0) return;
    const size_t n = s->n;
    const int d = s->d;
    const int want = (int)std::min(m, n);
    // queries per batch: per-(query, record) state of 17 B within ~4 GB
    const size_t G = std::max<size_t>(1, std::min<size_t>({nq, 128, ((size_t)4 << 30) / (17 * n)}));
    const int nctas = (int)((n + GT - 1) / GT);
    const int nblk = nctas * GW;  // per-warp partial bests
    const size_t ob = G * m * (8 * 4 + 4) + G * 16 + 256;
    char* base = static_cast<char*>(s->b_greedy.get(
        n * d * 8 + 2 * (size_t)d * 8 + G * d * 8 * 2 + G * n * 17 + G * nblk * sizeof(Best) * 2 +
        G * want * 8 + ob + 12 * 256));
    size_t off = 0;
    auto take = [&](size_t bytes) {
        char* ptr = base + off;
        off += (bytes + 255) / 256 * 256;
        return ptr;
    };
    double* z = reinterpret_cast<double*>(take(n * d * 8));
    double* msd = reinterpret_cast<double*>(take((2 * (size_t)d + G * d) * 8));
    double* zq = msd + 2 * (size_t)d;
    GreedyArgs a{};
    a.z = z;
    a.r64 = s->r64;
    a.rnd = s->rnd;
    a.loo = loo;
    a.zq = zq;
    a.n = n;
    a.n_loo = eff_n(s);
    a.d = d;
    a.want = want;
    a.total = eff_stats(s).total;
    a.two_s2 = p.two_s2;
    a.lambda = lambda;
    a.score = reinterpret_cast<double*>(take(G * n * 8));
    a.pen = reinterpret_cast<double*>(take(G * n * 8));
    a.taken = reinterpret_cast<unsigned char*>(take(G * n));
    a.part = reinterpret_cast<Best*>(take(G * nblk * sizeof(Best)));
    a.part_nn = want_nn ? reinterpret_cast<Best*>(take(G * nblk * sizeof(Best))) : nullptr;
    a.picks = reinterpret_cast<int64_t*>(take(G * std::max(want, 1) * 8));
    a.zpick = reinterpret_cast<double*>(take(G * d * 8));
    a.nblk = nblk;
    char* dout = take(ob);
    char* hout = static_cast<char*>(s->h_out.get(ob));
    double* hin = s->h_consts.as<double>(2 * (size_t)d + G * d);
    std::copy(p.mean.begin(), p.mean.end(), hin);
    std::copy(p.sd.begin(), p.sd.end(), hin + d);
    SAIR_CUDA(cudaMemcpyAsync(msd, hin, 2 * (size_t)d * 8, cudaMemcpyHostToDevice, s->st));
    zrows_launch(s->x64, msd, msd + d, n, d, z, s->st);
    const size_t smem = greedy_smem(d);
    int64_t* o_idx = reinterpret_cast<int64_t*>(dout);
    double* o_sim = reinterpret_cast<double*>(o_idx + G * m);
    double* o_score = o_sim + G * m;
    double* o_rew = o_score + G * m;
    int64_t* o_nn = reinterpret_cast<int64_t*>(o_rew + G * m);
    double* o_nns = reinterpret_cast<double*>(o_nn + G);
    int32_t* o_round = reinterpret_cast<int32_t*>(o_nns + G);
    for (size_t b0 = 0; b0 < nq; b0 += G) {
        const int g_n = (int)std::min(G, nq - b0);
        a.G = g_n;
        // the host staging of the previous batch was consumed before its sync
        for (int g = 0; g < g_n; ++g)
            std::copy(p.z.begin() + qidx[b0 + g] * d, p.z.begin() + (qidx[b0 + g] + 1) * d,
                      hin + 2 * d + (size_t)g * d);
        SAIR_CUDA(cudaMemcpyAsync(zq, hin + 2 * d, (size_t)g_n * d * 8, cudaMemcpyHostToDevice,
                                  s->st));
        for (int step = 0; step < want; ++step) {
            greedy_step(nctas, smem, s->st, a, step);
            greedy_pick_kernel<<<g_n, 256, 0, s->st>>>(a, step);
        }
        SAIR_LAUNCH("greedy steps");
        GreedyArgs f = a;
        greedy_finish_kernel<<<g_n, 32, 0, s->st>>>(f, s->gbase, (int)m, o_idx, o_sim, o_score,
                                                    o_rew, o_round, want_nn ? o_nn : nullptr,
                                                    o_nns);
        SAIR_LAUNCH("greedy_finish_kernel");
        SAIR_CUDA(cudaMemcpyAsync(hout, dout, ob, cudaMemcpyDeviceToHost, s->st));
        SAIR_CUDA(cudaStreamSynchronize(s->st));
        const int64_t* hidx = reinterpret_cast<const int64_t*>(hout);
        const double* hsim = reinterpret_cast<const double*>(hidx + G * m);
        const double* hsc = hsim + G * m;
        const double* hrw = hsc + G * m;
        const int64_t* hnn = reinterpret_cast<const int64_t*>(hrw + G * m);
        const double* hnns = reinterpret_cast<const double*>(hnn + G);
        const int32_t* hrd = reinterpret_cast<const int32_t*>(hnns + G);
        for (int g = 0; g < g_n; ++g) {
            const size_t q = qidx[b0 + g];
            out_count[q] = (size_t)want;
            std::copy(hidx + g * m, hidx + g * m + want, out_idx + q * m);
            std::copy(hsim + g * m, hsim + g * m + want, out_sim + q * m);
            std::copy(hsc + g * m, hsc + g * m + want, out_score + q * m);
            if (out_reward) std::copy(hrw + g * m, hrw + g * m + want, out_reward + q * m);
            if (out_round) std::copy(hrd + g * m, hrd + g * m + want, out_round + q * m);
            if (out_nn) {
                out_nn[q] = hnn[g];
                out_nn_sim[q] = hnns[g];
            }
        }
    }
}


// ------------------------------------------------- distributed sessions ----
//
// A shard of a buffer spread over ranks runs the same greedy with the global
// pick decided by the caller between steps (sharded.py): greedy_begin scores
// the shard for G queries; greedy_next applies the previous global picks
// (taken where local, their rows added to every penalty) and returns the
// shard's best per query.  A rank's best carries everything the others need:
// gain, round, global index, the pick's similarity, score, reward and row.

namespace {

// the caller's global picks: mark local ones taken, stage every pick's row
__global__ void greedy_apply_kernel(const GreedyArgs a, const int64_t* __restrict__ gpick,
                                    const double* __restrict__ zrows, int64_t gbase) {
    const int g = blockIdx.x;
    const int64_t p = gpick[g] - gbase;
    if (threadIdx.x == 0 && p >= 0 && (size_t)p < a.n) a.taken[(size_t)g * a.n + p] = 1;
    for (int k = threadIdx.x; k < a.d; k += blockDim.x)
        a.zpick[(size_t)g * a.d + k] = zrows[(size_t)g * a.d + k];
}

// per query: the shard's best -> [gain, round, gidx, sim, score, reward, row[d]]
__global__ void greedy_local_best_kernel(const GreedyArgs a, int64_t gbase, double* __restrict__ out) {
    const int g = blockIdx.x;
    __shared__ Best wb[32];
    Best b{0.0, 0, 0, -1};
    for (int t = threadIdx.x; t < a.nblk; t += blockDim.x) {
        const Best c = a.part[(size_t)g * a.nblk + t];
        if (better(c, b)) b = c;
    }
    b = warp_best(b);
    if ((threadIdx.x & 31) == 0) wb[threadIdx.x >> 5] = b;
    __syncthreads();
    if (threadIdx.x < 32) {
        Best c = threadIdx.x < (blockDim.x >> 5) ? wb[threadIdx.x] : Best{0.0, 0, 0, -1};
        c = warp_best(c);
        if (threadIdx.x == 0) wb[0] = c;
    }
    __syncthreads();
    const Best w = wb[0];
    double* o = out + (size_t)g * (6 + a.d);
    if (w.j < 0) {  // no untaken record on this shard
        if (threadIdx.x == 0) {
            o[0] = -INFINITY;
            o[1] = 0.0;
            o[2] = -1.0;
        }
        return;
    }
    const size_t p = (size_t)w.i;
    if (threadIdx.x == 0) {
        const double* zq = a.zq + (size_t)g * a.d;
        double d2 = 0.0;
        for (int k = 0; k < a.d; ++k) {
            const double t = dsub(a.z[(size_t)k * a.n + p], zq[k]);
            d2 = dadd(d2, dmul(t, t));
        }
        o[0] = w.g;
        o[1] = (double)w.r;
        o[2] = (double)(gbase + (int64_t)p);
        o[3] = sim_from_d2(d2, a.two_s2);
        o[4] = a.score[(size_t)g * a.n + p];
        o[5] = a.r64[p];
    }
    for (int k = threadIdx.x; k < a.d; k += blockDim.x) o[6 + k] = a.z[(size_t)k * a.n + p];
}

}  // namespace

struct GreedySession {
    GreedyArgs a{};
    int nctas = 0;
    size_t smem = 0;
    int step = 0;
    double* dout = nullptr;  // [G][6 + d]
    int64_t* dpick = nullptr;
    double* drows = nullptr;
};

static GreedySession& session(sair_store_s* s) {
    if (!s->greedy) s->greedy = std::make_shared<GreedySession>();
    return *s->greedy;
}

void greedy_begin(sair_store_s* s, const double* q, size_t G, int dim,
                  const sair_select_config& cfg, double* out) {
    if (G == 0 || G > 1024) throw Error(SAIR_EINVAL, "greedy session: 1..1024 queries");
    if (s->n == 0) throw Error(SAIR_EINVAL, "greedy session: empty store");
    if (cfg.locally_weighted_mean)
        throw Error(SAIR_EINVAL, "locally_weighted_mean is not supported on a sharded store");
    DeviceGuard dg(s->device);
    const double sigma = store_effective_sigma(s, cfg.sigma_sim);
    if (dim != s->d) throw Error(SAIR_EINVAL, "experience store: feature dimension mismatch");
    const QueryPrep p = prep_queries(s, q, G, sigma);
    const double lambda = cfg.lambda_div;
    GreedySession& ss = session(s);
    const size_t n = s->n;
    const int d = s->d;
    const int nctas = (int)((n + GT - 1) / GT);
    const int nblk = nctas * GW;
    char* base = static_cast<char*>(s->b_greedy.get(
        n * d * 8 + 2 * (size_t)d * 8 + G * d * 8 * 3 + G * n * 17 + G * nblk * sizeof(Best) +
        G * (6 + d) * 8 + G * 8 + 12 * 256));
    size_t off = 0;
    auto take = [&](size_t bytes) {
        char* ptr = base + off;
        off += (bytes + 255) / 256 * 256;
        return ptr;
    };
    double* z = reinterpret_cast<double*>(take(n * d * 8));
    double* msd = reinterpret_cast<double*>(take((2 * (size_t)d + G * d) * 8));
    GreedyArgs& a = ss.a;
    a = GreedyArgs{};
    a.z = z;
    a.r64 = s->r64;
    a.rnd = s->rnd;
    a.zq = msd + 2 * (size_t)d;
    a.n = n;
    a.n_loo = eff_n(s);
    a.d = d;
    a.G = (int)G;
    a.want = 1;
    a.total = eff_stats(s).total;
    a.two_s2 = p.two_s2;
    a.lambda = lambda;
    a.score = reinterpret_cast<double*>(take(G * n * 8));
    a.pen = reinterpret_cast<double*>(take(G * n * 8));
    a.taken = reinterpret_cast<unsigned char*>(take(G * n));
    a.part = reinterpret_cast<Best*>(take(G * nblk * sizeof(Best)));
    a.zpick = reinterpret_cast<double*>(take(G * d * 8));
    a.nblk = nblk;
    ss.dout = reinterpret_cast<double*>(take(G * (6 + d) * 8));
    ss.dpick = reinterpret_cast<int64_t*>(take(G * 8));
    ss.drows = reinterpret_cast<double*>(take(G * d * 8));
    ss.nctas = nctas;
    ss.smem = greedy_smem(d);
    ss.step = 0;
    double* hin = s->h_consts.as<double>(2 * (size_t)d + G * d);
    std::copy(p.mean.begin(), p.mean.end(), hin);
    std::copy(p.sd.begin(), p.sd.end(), hin + d);
    std::copy(p.z.begin(), p.z.begin() + G * d, hin + 2 * d);
    SAIR_CUDA(cudaMemcpyAsync(msd, hin, (2 * (size_t)d + G * d) * 8, cudaMemcpyHostToDevice, s->st));
    zrows_launch(s->x64, msd, msd + d, n, d, z, s->st);
    greedy_step(nctas, ss.smem, s->st, a, 0);
    greedy_local_best_kernel<<<(int)G, 256, 0, s->st>>>(a, s->gbase, ss.dout);
    SAIR_LAUNCH("greedy_begin");
    SAIR_CUDA(cudaMemcpyAsync(out, ss.dout, G * (6 + d) * 8, cudaMemcpyDeviceToHost, s->st));
    SAIR_CUDA(cudaStreamSynchronize(s->st));
}

void greedy_next(sair_store_s* s, const int64_t* gpick, const double* rows, double* out) {
    if (!s->greedy || !s->greedy->a.score) throw Error(SAIR_ELOGIC, "greedy session not begun");
    DeviceGuard dg(s->device);
    GreedySession& ss = *s->greedy;
    GreedyArgs& a = ss.a;
    const size_t G = (size_t)a.G;
    const int d = a.d;
    int64_t* hp = reinterpret_cast<int64_t*>(s->h_consts.as<double>(G * (1 + d)));
    double* hr = reinterpret_cast<double*>(hp + G);
    std::copy(gpick, gpick + G, hp);
    std::copy(rows, rows + G * d, hr);
    SAIR_CUDA(cudaMemcpyAsync(ss.dpick, hp, G * 8, cudaMemcpyHostToDevice, s->st));
    SAIR_CUDA(cudaMemcpyAsync(ss.drows, hr, G * d * 8, cudaMemcpyHostToDevice, s->st));
    greedy_apply_kernel<<<(int)G, 64, 0, s->st>>>(a, ss.dpick, ss.drows, s->gbase);
    ++ss.step;
    greedy_step(ss.nctas, ss.smem, s->st, a, ss.step);
    greedy_local_best_kernel<<<(int)G, 256, 0, s->st>>>(a, s->gbase, ss.dout);
    SAIR_LAUNCH("greedy_next");
    SAIR_CUDA(cudaMemcpyAsync(out, ss.dout, G * (6 + d) * 8, cudaMemcpyDeviceToHost, s->st));
    SAIR_CUDA(cudaStreamSynchronize(s->st));
}

}  // namespace sair
