// select_exact.cu -- the full fp64 pass over the store (x64 rows).
//
// The fallback for a query the fast filter cannot certify, the
// SAIR_SELECT_EXACT mode, locally_weighted_mean (experience.cpp:125-137) and
// surprisal() (:234-240).  Every record's score follows the reference's exact
// rounding sequence (standardize :162-166, similarity :125-130, loo_mean
// :229-231, gain :270); the greedy loop is one arg-max pass per pick and one
// penalty pass per pick (:265-285).
#include <algorithm>
#include <vector>

#include "select_common.cuh"

namespace sair {

// ------------------------------------------------------- exact fallback ----

struct ExactArgs {
    const double* x64;
    const double* r64;
    const int32_t* rnd;
    const double* mean;
    const double* sd;
    const double* zq;  // [d]
    int d;
    size_t n;     // records in this store
    size_t n_loo; // records of the whole buffer (loo_mean's n, experience.cpp:140)
    double total, two_s2, lambda;
    const double* loo;  // locally weighted LOO means (nullable)
    double* score;      // [n]
    double* sim;        // [n]
    double* pen;        // [n]
    unsigned char* taken;
};

__device__ __forceinline__ double zval(const ExactArgs& a, size_t i, int k) {
    return ddiv(dsub(a.x64[i * a.d + k], a.mean[k]), a.sd[k]);
}

__global__ void exact_score_kernel(const ExactArgs a) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < a.n;
         i += (size_t)gridDim.x * blockDim.x) {
        double d2 = 0.0;
        for (int k = 0; k < a.d; ++k) {
            double t = dsub(zval(a, i, k), a.zq[k]);
            d2 = dadd(d2, dmul(t, t));
        }
        double s = sim_from_d2(d2, a.two_s2);
        double r = a.r64[i];
        double loo = a.loo ? a.loo[i]
                           : (a.n_loo <= 1 ? 0.0 : ddiv(dsub(a.total, r), (double)(a.n_loo - 1)));
        a.sim[i] = s;
        a.score[i] = dmul(s, fabs(dsub(r, loo)));
        a.pen[i] = 0.0;
        a.taken[i] = 0;
    }
}

// locally weighted leave-one-out mean, experience.cpp:125-137 (sequential in j
// per record, so the sums round exactly as the reference's loop)
__global__ void local_loo_kernel(const ExactArgs a, double* __restrict__ loo) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < a.n;
         i += (size_t)gridDim.x * blockDim.x) {
        if (a.n_loo <= 1) {
            loo[i] = 0.0;
            continue;
        }
        double wsum = 0.0, acc = 0.0;
        for (size_t j = 0; j < a.n; ++j) {
            if (j == i) continue;
            double d2 = 0.0;
            for (int k = 0; k < a.d; ++k) {
                double t = dsub(zval(a, j, k), zval(a, i, k));
                d2 = dadd(d2, dmul(t, t));
            }
            double w = sim_from_d2(d2, a.two_s2);
            wsum = dadd(wsum, w);
            acc = dadd(acc, dmul(w, a.r64[j]));
        }
        loo[i] = wsum > 1e-12 ? ddiv(acc, wsum)
                              : ddiv(dsub(a.total, a.r64[i]), (double)(a.n_loo - 1));
    }
}

// block-level best of (gain = score - lambda pen, round, index); use_round=0 for
// the veto scan (argmax sim, first index).
__global__ void exact_argmax_kernel(const ExactArgs a, int use_sim, Best* __restrict__ part) {
    Best b{0.0, 0, 0, -1};
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < a.n;
         i += (size_t)gridDim.x * blockDim.x) {
        Best c;
        if (use_sim) {
            c = Best{a.sim[i], 0, (int64_t)i, 1};
        } else {
            if (a.taken[i]) continue;
            c = Best{dsub(a.score[i], dmul(a.lambda, a.pen[i])), a.rnd[i], (int64_t)i, 1};
        }
        if (better(c, b)) b = c;
    }
    __shared__ Best wb[32];
    b = warp_best(b);
    if ((threadIdx.x & 31) == 0) wb[threadIdx.x >> 5] = b;
    __syncthreads();
    if (threadIdx.x < 32) {
        Best c = threadIdx.x < (blockDim.x >> 5) ? wb[threadIdx.x] : Best{0.0, 0, 0, -1};
        c = warp_best(c);
        if (threadIdx.x == 0) part[blockIdx.x] = c;
    }
}

__global__ void exact_pick_kernel(const ExactArgs a, const Best* __restrict__ part, int nparts,
                                  int64_t* __restrict__ picks, int step, int mark) {
    Best b{0.0, 0, 0, -1};
    for (int t = threadIdx.x; t < nparts; t += blockDim.x)
        if (better(part[t], b)) b = part[t];
    __shared__ Best wb[32];
    b = warp_best(b);
    if ((threadIdx.x & 31) == 0) wb[threadIdx.x >> 5] = b;
    __syncthreads();
    if (threadIdx.x < 32) {
        Best c = threadIdx.x < (blockDim.x >> 5) ? wb[threadIdx.x] : Best{0.0, 0, 0, -1};
        c = warp_best(c);
        if (threadIdx.x == 0) {
            picks[step] = c.i;
            if (mark) a.taken[c.i] = 1;
        }
    }
}

__global__ void exact_penalty_kernel(const ExactArgs a, const int64_t* __restrict__ picks,
                                     int step, double* __restrict__ zb_scratch) {
    const int64_t b = picks[step];
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < a.n;
         i += (size_t)gridDim.x * blockDim.x) {
        if (a.taken[i]) continue;
        double d2 = 0.0;
        for (int k = 0; k < a.d; ++k) {
            double t = dsub(zval(a, i, k), zval(a, (size_t)b, k));
            d2 = dadd(d2, dmul(t, t));
        }
        a.pen[i] = dadd(a.pen[i], sim_from_d2(d2, a.two_s2));
    }
    (void)zb_scratch;
}

__global__ void exact_finish_kernel(const ExactArgs a, int64_t* picks, int want, int64_t gbase,
                                    int64_t* out_idx, double* out_sim, double* out_score,
                                    double* out_rew, int32_t* out_round) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int x = 1; x < want; ++x) {
        int64_t v = picks[x];
        int y = x;
        while (y > 0) {
            int64_t u = picks[y - 1];
            bool less = a.r64[v] != a.r64[u] ? a.r64[v] < a.r64[u] : a.rnd[v] < a.rnd[u];
            if (!less) break;
            picks[y] = u;
            --y;
        }
        picks[y] = v;
    }
    for (int x = 0; x < want; ++x) {
        out_idx[x] = gbase + picks[x];
        out_sim[x] = a.sim[picks[x]];
        out_score[x] = a.score[picks[x]];
        out_rew[x] = a.r64[picks[x]];
        out_round[x] = a.rnd[picks[x]];
    }
}

__global__ void surprisal_kernel(const ExactArgs a, size_t index, double* out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double d2 = 0.0;
    for (int k = 0; k < a.d; ++k) {
        double t = dsub(zval(a, index, k), a.zq[k]);
        d2 = dadd(d2, dmul(t, t));
    }
    double s = sim_from_d2(d2, a.two_s2);
    double r = a.r64[index];
    double loo;
    if (a.n_loo <= 1) {
        loo = 0.0;
    } else if (a.loo) {  // local mean computed for this index only
        double wsum = 0.0, acc = 0.0;
        for (size_t j = 0; j < a.n; ++j) {
            if (j == index) continue;
            double e2 = 0.0;
            for (int k = 0; k < a.d; ++k) {
                double t = dsub(zval(a, j, k), zval(a, index, k));
                e2 = dadd(e2, dmul(t, t));
            }
            double w = sim_from_d2(e2, a.two_s2);
            wsum = dadd(wsum, w);
            acc = dadd(acc, dmul(w, a.r64[j]));
        }
        loo = wsum > 1e-12 ? ddiv(acc, wsum) : ddiv(dsub(a.total, r), (double)(a.n_loo - 1));
    } else {
        loo = ddiv(dsub(a.total, r), (double)(a.n_loo - 1));
    }
    *out = dmul(s, fabs(dsub(r, loo)));
}

// --------------------------------------------------------------- host ------

// Exact full-pass answer for one query (fp64 over x64), writing m results.
void exact_one(sair_store_s* s, const QueryPrep& p, const double* zq_host, size_t m,
               double lambda, bool local, int64_t* o_idx, double* o_sim, double* o_score,
               size_t* o_cnt, int64_t* o_nn, double* o_nn_sim, double* o_rew,
               int32_t* o_round, const double* loo_pre) {
    const size_t n = s->n;
    const int d = s->d;
    char* base = static_cast<char*>(
        s->b_exact.get(n * (8 * 4 + 1) + (size_t)d * 8 * 3 + 4096 * sizeof(Best) + 64 * 1024 +
                       m * 8 * 8 + 16 * 256));
    size_t off = 0;
    auto take = [&](size_t bytes) {
        char* ptr = base + off;
        off += (bytes + 255) / 256 * 256;
        return ptr;
    };
    ExactArgs a{};
    a.x64 = s->x64;
    a.r64 = s->r64;
    a.rnd = s->rnd;
    double* dm = reinterpret_cast<double*>(take(3 * (size_t)d * 8));
    a.mean = dm;
    a.sd = dm + d;
    a.zq = dm + 2 * d;
    a.d = d;
    a.n = n;
    a.n_loo = eff_n(s);
    a.total = eff_stats(s).total;
    a.two_s2 = p.two_s2;
    a.lambda = lambda;
    a.score = reinterpret_cast<double*>(take(n * 8));
    a.sim = reinterpret_cast<double*>(take(n * 8));
    a.pen = reinterpret_cast<double*>(take(n * 8));
    double* loo = reinterpret_cast<double*>(take(n * 8));
    a.taken = reinterpret_cast<unsigned char*>(take(n));
    Best* part = reinterpret_cast<Best*>(take(4096 * sizeof(Best)));
    int64_t* picks = reinterpret_cast<int64_t*>(take(m * 8 + 8));
    int64_t* didx = reinterpret_cast<int64_t*>(take(m * 8 + 8));
    double* dsim = reinterpret_cast<double*>(take(m * 8 + 8));
    double* dscore = reinterpret_cast<double*>(take(m * 8 + 8));
    double* drew = reinterpret_cast<double*>(take(m * 8 + 8));
    int32_t* dround = reinterpret_cast<int32_t*>(take(m * 4 + 8));
    std::vector<double> h(3 * (size_t)d);
    std::copy(p.mean.begin(), p.mean.end(), h.begin());
    std::copy(p.sd.begin(), p.sd.end(), h.begin() + d);
    std::copy(zq_host, zq_host + d, h.begin() + 2 * d);
    SAIR_CUDA(cudaMemcpyAsync(dm, h.data(), h.size() * 8, cudaMemcpyHostToDevice, s->st));
    const int threads = 256;
    const int blocks = (int)std::min<size_t>((n + threads - 1) / threads, 4096);
    if (local && loo_pre) {
        a.loo = loo_pre;  // computed once for the whole call (query-independent)
    } else if (local) {
        a.loo = nullptr;
        local_loo_kernel<<<blocks, threads, 0, s->st>>>(a, loo);
        SAIR_LAUNCH("local_loo_kernel");
        a.loo = loo;
    }
    exact_score_kernel<<<blocks, threads, 0, s->st>>>(a);
    SAIR_LAUNCH("exact_score_kernel");
    const size_t want = std::min(m, n);
    for (size_t step = 0; step < want; ++step) {
        exact_argmax_kernel<<<blocks, threads, 0, s->st>>>(a, 0, part);
        exact_pick_kernel<<<1, 1024, 0, s->st>>>(a, part, blocks, picks, (int)step, 1);
        if (lambda != 0.0 && step + 1 < want) {
            exact_penalty_kernel<<<blocks, threads, 0, s->st>>>(a, picks, (int)step, nullptr);
        }
    }
    SAIR_LAUNCH("exact greedy");
    if (want) {
        exact_finish_kernel<<<1, 32, 0, s->st>>>(a, picks, (int)want, s->gbase, didx, dsim, dscore,
                                                 drew, dround);
        SAIR_LAUNCH("exact_finish_kernel");
        SAIR_CUDA(cudaMemcpyAsync(o_idx, didx, want * 8, cudaMemcpyDeviceToHost, s->st));
        SAIR_CUDA(cudaMemcpyAsync(o_sim, dsim, want * 8, cudaMemcpyDeviceToHost, s->st));
        SAIR_CUDA(cudaMemcpyAsync(o_score, dscore, want * 8, cudaMemcpyDeviceToHost, s->st));
        if (o_rew)
            SAIR_CUDA(cudaMemcpyAsync(o_rew, drew, want * 8, cudaMemcpyDeviceToHost, s->st));
        if (o_round)
            SAIR_CUDA(cudaMemcpyAsync(o_round, dround, want * 4, cudaMemcpyDeviceToHost, s->st));
    }
    if (o_nn) {
        exact_argmax_kernel<<<blocks, threads, 0, s->st>>>(a, 1, part);
        exact_pick_kernel<<<1, 1024, 0, s->st>>>(a, part, blocks, picks + want, 0, 0);
        SAIR_LAUNCH("exact nearest");
        int64_t nn = 0;
        SAIR_CUDA(cudaMemcpyAsync(&nn, picks + want, 8, cudaMemcpyDeviceToHost, s->st));
        SAIR_CUDA(cudaStreamSynchronize(s->st));
        double sv = 0.0;
        SAIR_CUDA(cudaMemcpy(&sv, a.sim + nn, 8, cudaMemcpyDeviceToHost));
        *o_nn = s->gbase + nn;
        *o_nn_sim = sv;
    }
    SAIR_CUDA(cudaStreamSynchronize(s->st));
    *o_cnt = want;
}

double store_surprisal(sair_store_s* s, size_t index, const double* x,
                       const sair_select_config& cfg) {
    DeviceGuard g(s->device);
    const double sigma = store_effective_sigma(s, cfg.sigma_sim);
    QueryPrep p = prep_queries(s, x, 1, sigma);
    const int d = s->d;
    double* dm = s->b_consts.as<double>(3 * (size_t)d + 1);
    std::vector<double> h(3 * (size_t)d);
    std::copy(p.mean.begin(), p.mean.end(), h.begin());
    std::copy(p.sd.begin(), p.sd.end(), h.begin() + d);
    std::copy(p.z.begin(), p.z.end(), h.begin() + 2 * d);
    SAIR_CUDA(cudaMemcpyAsync(dm, h.data(), h.size() * 8, cudaMemcpyHostToDevice, s->st));
    ExactArgs a{};
    a.x64 = s->x64;
    a.r64 = s->r64;
    a.rnd = s->rnd;
    a.mean = dm;
    a.sd = dm + d;
    a.zq = dm + 2 * d;
    a.d = d;
    a.n = s->n;
    a.n_loo = eff_n(s);
    a.total = eff_stats(s).total;
    a.two_s2 = p.two_s2;
    a.loo = cfg.locally_weighted_mean ? dm : nullptr;  // non-null flags the local mean
    double* out = dm + 3 * d;
    surprisal_kernel<<<1, 32, 0, s->st>>>(a, index, out);
    SAIR_LAUNCH("surprisal_kernel");
    double v = 0.0;
    SAIR_CUDA(cudaMemcpyAsync(&v, out, 8, cudaMemcpyDeviceToHost, s->st));
    SAIR_CUDA(cudaStreamSynchronize(s->st));
    return v;
}

}  // namespace sair


