// select_small.cu -- the whole exact select() of a small store in one launch.
//
// ExperienceBuffer::select (experience.cpp:151-205) for stores of up to 64k
// records, any lambda_div: one thread-block cluster of up to 8 CTAs per
// query (distributed shared memory), each CTA holding its slice of the
// records' exact scores, penalties and taken flags in shared memory.
//
//   zrows_kernel          standardize() of every stored row once per call
//                         (experience.cpp:71-75, the reference's rounding:
//                         (x - mean) / sd), shared by all the call's queries;
//   small_select_kernel   per query: exact scores (:254-258), the veto scan's
//                         nearest record (policy.cpp:140-157), then `want`
//                         greedy steps (:261-285): a block arg-max per CTA, a
//                         cluster barrier, every CTA reduces the CTAs' bests
//                         from distributed shared memory (the same winner on
//                         all), the owner marks it taken, and every CTA adds
//                         sim(z_i, z_pick) to its slice's penalties; finally
//                         the curriculum order (:290-294).
//
// This replaces the per-step kernel sequence of select_exact.cu (3 + 3m
// launches per query) for the decision-step sizes of configs[0] (10k records)
// and is the exact fallback for uncertified queries of such stores.
#include <cooperative_groups.h>

#include <algorithm>
#include <climits>
#include <cstdint>
#include <mutex>
#include <cstdlib>
#include <vector>

#include "select_common.cuh"

namespace cg = cooperative_groups;

namespace sair {

namespace {

constexpr int SMALL_THREADS = 1024;
constexpr int SMALL_CS_MAX = 8;       // portable cluster size
constexpr size_t SMALL_PER_MAX = 8192;  // records per CTA (shared-memory slice)

struct SmallArgs {
    const double* z;     // [d][n] standardized rows, dimension-major (coalesced per k)
    const double* r64;
    const int32_t* rnd;
    const double* zq;    // [nq][d] standardized queries
    int d, m, nn, cs;
    size_t n, per;       // records, records per CTA
    size_t n_loo;        // loo_mean's n (the whole buffer's)
    double total, two_s2, lambda;
    const double* loo;   // [n] locally weighted LOO means (nullable: the global mean)
    int64_t gbase;
    int64_t* out_idx;    // [nq][m]
    double* out_sim;
    double* out_score;
    double* out_rew;
    int32_t* out_round;
    int* out_cnt;        // [nq]
    int64_t* out_nn;     // [nq]
    double* out_nn_sim;
};

__global__ void zrows_kernel(const double* __restrict__ x64, const double* __restrict__ mean,
                             const double* __restrict__ sd, size_t n, int d,
                             double* __restrict__ z) {
    const size_t total = n * (size_t)d;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total;
         e += (size_t)gridDim.x * blockDim.x) {
        const int k = (int)(e % d);
        z[(size_t)k * n + e / d] = ddiv(dsub(x64[e], mean[k]), sd[k]);
    }
}

// locally_weighted_mean LOO, experience.cpp:125-137 (loo_mean with
// cfg.locally_weighted_mean): for record i, sum_{j != i} w_ij r_j / sum w_ij
// with w_ij = similarity(z_j, z_i) (the reference calls similarity(
// standardize(items_[j].context), zi) -- z_j first), sequential in j; the
// global mean when the weights vanish (<= 1e-12).  Query-independent: once
// per call.  One thread per record i; j tiles of the standardized rows are
// staged in shared memory and shared by the block.
constexpr int LOO_TILE = 64;
__global__ void __launch_bounds__(256) local_loo_z_kernel(const double* __restrict__ z,
                                                           const double* __restrict__ r64, size_t n,
                                                           int d, double two_s2, double total,
                                                           size_t n_loo, double* __restrict__ loo) {
    extern __shared__ double zt[];  // [d][LOO_TILE] + r[LOO_TILE]
    double* rt = zt + (size_t)d * LOO_TILE;
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const bool valid = i < n;
    double wsum = 0.0, acc = 0.0;
    for (size_t j0 = 0; j0 < n; j0 += LOO_TILE) {
        const int cnt = (int)min((size_t)LOO_TILE, n - j0);
        __syncthreads();
        for (int e = threadIdx.x; e < d * LOO_TILE; e += blockDim.x) {
            const int k = e / LOO_TILE, jj = e % LOO_TILE;
            zt[e] = jj < cnt ? z[(size_t)k * n + j0 + jj] : 0.0;
        }
        for (int jj = threadIdx.x; jj < LOO_TILE; jj += blockDim.x)
            rt[jj] = jj < cnt ? r64[j0 + jj] : 0.0;
        __syncthreads();
        if (!valid) continue;
        for (int jj = 0; jj < cnt; ++jj) {
            if (j0 + jj == i) continue;
            double d2 = 0.0;
            for (int k = 0; k < d; ++k) {
                const double t = dsub(zt[k * LOO_TILE + jj], z[(size_t)k * n + i]);
                d2 = dadd(d2, dmul(t, t));
            }
            const double w = sim_from_d2(d2, two_s2);
            wsum = dadd(wsum, w);
            acc = dadd(acc, dmul(w, rt[jj]));
        }
    }
    if (!valid) return;
    if (n_loo <= 1) {
        loo[i] = 0.0;
        return;
    }
    loo[i] = wsum > 1e-12 ? ddiv(acc, wsum) : ddiv(dsub(total, r64[i]), (double)(n_loo - 1));
}

__global__ void __launch_bounds__(SMALL_THREADS) small_select_kernel(const __grid_constant__ SmallArgs a) {
    cg::cluster_group cl = cg::this_cluster();
    const int crank = (int)cl.block_rank();
    const int q = blockIdx.x / a.cs;
    const int tid = threadIdx.x;
    const int d = a.d;
    const size_t lo = (size_t)crank * a.per;
    const size_t hi = min(a.n, lo + a.per);
    const size_t ns = hi > lo ? hi - lo : 0;

    extern __shared__ __align__(16) unsigned char sm[];
    double* score = reinterpret_cast<double*>(sm);
    double* pen = score + a.per;
    double* sim = pen + a.per;
    double* zq = sim + a.per;          // [d]
    double* zb = zq + d;               // [d] the current pick's row
    double* psim = zb + d;             // [m] sim / score of the picks this CTA owns
    double* pscore = psim + a.m;
    int64_t* picks = reinterpret_cast<int64_t*>(pscore + a.m);  // [m] local record index
    Best* cbest = reinterpret_cast<Best*>(picks + a.m);         // [2] double-buffered
    Best* wb = cbest + 2;                                       // [33]
    unsigned char* taken = reinterpret_cast<unsigned char*>(wb + 33);

    for (int k = tid; k < d; k += blockDim.x) zq[k] = a.zq[(size_t)q * d + k];
    __syncthreads();
    // exact scores, experience.cpp:163-167 (standardize, similarity, loo_mean)
    for (size_t j = tid; j < ns; j += blockDim.x) {
        const double* zi = a.z + lo + j;
        double d2 = 0.0;
#pragma unroll 8
        for (int k = 0; k < d; ++k) {
            const double t = dsub(zi[(size_t)k * a.n], zq[k]);
            d2 = dadd(d2, dmul(t, t));
        }
        const double s = sim_from_d2(d2, a.two_s2);
        const double r = a.r64[lo + j];
        const double loo = a.loo ? a.loo[lo + j]
                                 : (a.n_loo <= 1 ? 0.0 : ddiv(dsub(a.total, r), (double)(a.n_loo - 1)));
        sim[j] = s;
        score[j] = dmul(s, fabs(dsub(r, loo)));
        pen[j] = 0.0;
        taken[j] = 0;
    }
    __syncthreads();
    int par = 0;
    const int lane = tid & 31, warp = tid >> 5;
    auto cluster_best = [&](Best b) {
        // the CTA's best (warp shuffles, one barrier), published in shared
        // memory; after the cluster barrier warp 0 reads the CTAs' bests from
        // distributed shared memory (lane r <- rank r) and every CTA reduces
        // the same set to the same winner
        b = warp_best(b);
        if (lane == 0) wb[warp] = b;
        __syncthreads();
        if (warp == 0) {
            Best c = lane < (int)(blockDim.x >> 5) ? wb[lane] : Best{0.0, 0, 0, -1};
            c = warp_best(c);
            if (lane == 0) cbest[par] = c;
        }
        cl.sync();
        if (warp == 0) {
            Best c = lane < a.cs ? *cl.map_shared_rank(cbest + par, lane) : Best{0.0, 0, 0, -1};
            c = warp_best(c);
            if (lane == 0) wb[32] = c;
        }
        __syncthreads();
        const Best g = wb[32];
        par ^= 1;
        return g;
    };
    if (a.nn) {
        // nearest record by similarity, first index on ties (policy.cpp:146-153)
        Best b{0.0, 0, 0, -1};
        for (size_t j = tid; j < ns; j += blockDim.x) {
            const Best c{sim[j], 0, (int64_t)(lo + j), 1};
            if (better(c, b)) b = c;
        }
        const Best g = cluster_best(b);
        if (crank == 0 && tid == 0) {
            a.out_nn[q] = g.j < 0 ? -1 : a.gbase + g.i;
            a.out_nn_sim[q] = g.j < 0 ? -1.0 : g.g;
        }
    }
    const int want = (int)min((size_t)a.m, a.n);
    for (int step = 0; step < want; ++step) {
        Best b{0.0, 0, 0, -1};
        for (size_t j = tid; j < ns; j += blockDim.x) {
            if (taken[j]) continue;
            const Best c{dsub(score[j], dmul(a.lambda, pen[j])), a.rnd[lo + j], (int64_t)(lo + j), 1};
            if (better(c, b)) b = c;
        }
        const Best g = cluster_best(b);
        const size_t gi = (size_t)g.i;
        const bool mine = gi >= lo && gi < hi;
        if (tid == 0) {
            picks[step] = (int64_t)gi;
            if (mine) {
                taken[gi - lo] = 1;
                psim[step] = sim[gi - lo];
                pscore[step] = score[gi - lo];
            }
        }
        if (a.lambda != 0.0 && step + 1 < want) {
            for (int k = tid; k < d; k += blockDim.x) zb[k] = a.z[(size_t)k * a.n + gi];
            __syncthreads();
            for (size_t j = tid; j < ns; j += blockDim.x) {
                if (taken[j] || lo + j == gi) continue;
                const double* zi = a.z + lo + j;
                double d2 = 0.0;
#pragma unroll 8
                for (int k = 0; k < d; ++k) {
                    const double t = dsub(zi[(size_t)k * a.n], zb[k]);
                    d2 = dadd(d2, dmul(t, t));
                }
                pen[j] = dadd(pen[j], sim_from_d2(d2, a.two_s2));  // :283-284
            }
        }
        __syncthreads();
    }
    cl.sync();  // every owner has recorded its picks' sim / score
    if (crank == 0 && tid == 0) {
        // gather each pick's sim / score from its owner, then the curriculum
        // order: stable by (reward asc, round asc) over pick order (:290-294)
        int order[256];
        double ps[256], pc[256];
        for (int x = 0; x < want; ++x) {
            const int owner = (int)((size_t)picks[x] / a.per);
            ps[x] = *cl.map_shared_rank(psim + x, owner);
            pc[x] = *cl.map_shared_rank(pscore + x, owner);
            order[x] = x;
        }
        for (int x = 1; x < want; ++x) {
            const int v = order[x];
            const double rv = a.r64[picks[v]];
            const int32_t dv = a.rnd[picks[v]];
            int y = x;
            while (y > 0) {
                const int u = order[y - 1];
                const double ru = a.r64[picks[u]];
                const bool less = rv != ru ? rv < ru : dv < a.rnd[picks[u]];
                if (!less) break;
                order[y] = u;
                --y;
            }
            order[y] = v;
        }
        for (int x = 0; x < want; ++x) {
            const int v = order[x];
            const size_t o = (size_t)q * a.m + x;
            a.out_idx[o] = a.gbase + picks[v];
            a.out_sim[o] = ps[v];
            a.out_score[o] = pc[v];
            a.out_rew[o] = a.r64[picks[v]];
            a.out_round[o] = a.rnd[picks[v]];
        }
        a.out_cnt[q] = want;
    }
    cl.sync();  // no CTA exits while another may still read its shared memory
}

}  // namespace

void zrows_launch(const double* x64, const double* mean, const double* sd, size_t n, int d,
                  double* z, cudaStream_t st) {
    zrows_kernel<<<(int)std::min<size_t>((n * d + 255) / 256, 2048), 256, 0, st>>>(x64, mean, sd, n,
                                                                                 d, z);
    SAIR_LAUNCH("zrows_kernel");
}

const double* local_loo_all(sair_store_s* s, const QueryPrep& p) {
    const size_t n = s->n;
    const int d = s->d;
    char* base = static_cast<char*>(s->b_loo.get(n * d * 8 + 2 * (size_t)d * 8 + n * 8 + 3 * 256));
    double* z = reinterpret_cast<double*>(base);
    double* msd = reinterpret_cast<double*>(base + ((n * d * 8 + 255) & ~(size_t)255));
    double* loo = msd + 2 * (size_t)d + 32;
    double* hin = s->h_consts.as<double>(2 * (size_t)d);
    std::copy(p.mean.begin(), p.mean.end(), hin);
    std::copy(p.sd.begin(), p.sd.end(), hin + d);
    SAIR_CUDA(cudaMemcpyAsync(msd, hin, 2 * (size_t)d * 8, cudaMemcpyHostToDevice, s->st));
    zrows_kernel<<<(int)std::min<size_t>((n * d + 255) / 256, 2048), 256, 0, s->st>>>(
        s->x64, msd, msd + d, n, d, z);
    const size_t lsm = ((size_t)d * LOO_TILE + LOO_TILE) * 8;
    SAIR_CUDA(cudaFuncSetAttribute(local_loo_z_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)lsm));
    local_loo_z_kernel<<<(int)((n + 255) / 256), 256, lsm, s->st>>>(
        z, s->r64, n, d, p.two_s2, eff_stats(s).total, eff_n(s), loo);
    SAIR_LAUNCH("local_loo_z_kernel");
    return loo;
}

bool small_select_fits(const sair_store_s* s, size_t m) {
    return s->n > 0 && s->n <= SMALL_CS_MAX * SMALL_PER_MAX && m <= 256 && s->d <= 1024;
}

static size_t small_smem_bytes(size_t n, int d, size_t m, int cs) {
    // per CTA: score, penalty, similarity, taken per record of its slice; the
    // query and pick rows; the picks; the bests
    const size_t per = (n + cs - 1) / cs;
    return per * 25 + 2 * (size_t)d * 8 + m * 24 + 35 * sizeof(Best) + 64;
}

// CTAs per query: one record per thread where a cluster of up to 16 CTAs (a
// non-portable size: it needs a GPC with 16 free SMs) is schedulable, so a
// step's critical path is one record (10k x 32, m = 8: 73 -> 59 us); else the
// portable 8.
static int small_cluster_size(size_t n, int d, size_t m) {
    const int want = (int)std::min<size_t>(std::getenv("SAIR_SMALL_CS8") ? 8 : 16,
                                           std::max<size_t>(1, (n + SMALL_THREADS - 1) /
                                                                   SMALL_THREADS));
    if (want <= 8) return want;
    // the answer only changes with the shared-memory size: remembered (per
    // process; the pool's GPUs are identical) so a decision step does not pay
    // the occupancy query
    static std::mutex mu;
    static size_t ok_smem = 0, bad_smem = SIZE_MAX;
    const size_t smem = small_smem_bytes(n, d, m, want);
    {
        std::lock_guard<std::mutex> lk(mu);
        if (smem <= ok_smem) return want;
        if (smem >= bad_smem) return 8;
    }
    SAIR_CUDA(cudaFuncSetAttribute(small_select_kernel,
                                   cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    SAIR_CUDA(cudaFuncSetAttribute(small_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    cudaLaunchConfig_t oc{};
    oc.gridDim = dim3((unsigned)want);
    oc.blockDim = dim3(SMALL_THREADS);
    oc.dynamicSmemBytes = smem;
    cudaLaunchAttribute ca[1];
    ca[0].id = cudaLaunchAttributeClusterDimension;
    ca[0].val.clusterDim.x = (unsigned)want;
    ca[0].val.clusterDim.y = 1;
    ca[0].val.clusterDim.z = 1;
    oc.attrs = ca;
    oc.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, small_select_kernel, &oc) != cudaSuccess ||
        nclusters < 1) {
        cudaGetLastError();
        std::lock_guard<std::mutex> lk(mu);
        bad_smem = std::min(bad_smem, smem);
        return 8;
    }
    std::lock_guard<std::mutex> lk(mu);
    ok_smem = std::max(ok_smem, smem);
    return want;
}

// Exact select() of the queries `qidx` (standardized rows of p.z) in one launch.
void small_select(sair_store_s* s, const QueryPrep& p, const std::vector<size_t>& qidx, size_t m,
                  double lambda, bool local, bool want_nn, int64_t* out_idx, double* out_sim,
                  double* out_score, size_t* out_count, int64_t* out_nn, double* out_nn_sim,
                  double* out_reward, int32_t* out_round) {
    const size_t nq = qidx.size();
    if (nq == 0) return;
    const size_t n = s->n;
    const int d = s->d;
    const int cs = small_cluster_size(n, d, m);
    const size_t per = (n + cs - 1) / cs;
    // device scratch: z rows | mean sd | zq | outputs
    const size_t ob = nq * m * (8 * 4 + 4) + nq * (4 + 8 + 8) + 256;
    char* base = static_cast<char*>(s->b_exact.get(n * d * 8 + 2 * (size_t)d * 8 +
                                                    nq * d * 8 + ob + n * 8 + 5 * 256));
    size_t off = 0;
    auto take = [&](size_t bytes) {
        char* ptr = base + off;
        off += (bytes + 255) / 256 * 256;
        return ptr;
    };
    double* z = reinterpret_cast<double*>(take(n * d * 8));
    double* msd = reinterpret_cast<double*>(take((2 * (size_t)d + nq * d) * 8));
    double* zq = msd + 2 * (size_t)d;  // contiguous with mean | sd: one copy
    char* dout = take(ob);
    double* hin = s->h_consts.as<double>(2 * (size_t)d + nq * d);
    std::copy(p.mean.begin(), p.mean.end(), hin);
    std::copy(p.sd.begin(), p.sd.end(), hin + d);
    for (size_t i = 0; i < nq; ++i)
        std::copy(p.z.begin() + qidx[i] * d, p.z.begin() + (qidx[i] + 1) * d, hin + 2 * d + i * d);
    SAIR_CUDA(cudaMemcpyAsync(msd, hin, (2 * (size_t)d + nq * d) * 8, cudaMemcpyHostToDevice,
                              s->st));
    zrows_kernel<<<(int)std::min<size_t>((n * d + 255) / 256, 2048), 256, 0, s->st>>>(
        s->x64, msd, msd + d, n, d, z);
    SAIR_LAUNCH("zrows_kernel");
    double* dloo = nullptr;
    if (local) {
        dloo = reinterpret_cast<double*>(take(n * 8));
        const size_t lsm = ((size_t)d * LOO_TILE + LOO_TILE) * 8;
        SAIR_CUDA(cudaFuncSetAttribute(local_loo_z_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lsm));
        local_loo_z_kernel<<<(int)((n + 255) / 256), 256, lsm, s->st>>>(
            z, s->r64, n, d, p.two_s2, eff_stats(s).total, eff_n(s), dloo);
        SAIR_LAUNCH("local_loo_z_kernel");
    }

    SmallArgs a{};
    a.z = z;
    a.r64 = s->r64;
    a.rnd = s->rnd;
    a.zq = zq;
    a.d = d;
    a.m = (int)m;
    a.nn = want_nn ? 1 : 0;
    a.cs = cs;
    a.n = n;
    a.per = per;
    a.n_loo = eff_n(s);
    a.total = eff_stats(s).total;
    a.two_s2 = p.two_s2;
    a.lambda = lambda;
    a.loo = dloo;
    a.gbase = s->gbase;
    a.out_idx = reinterpret_cast<int64_t*>(dout);
    a.out_sim = reinterpret_cast<double*>(a.out_idx + nq * m);
    a.out_score = a.out_sim + nq * m;
    a.out_rew = a.out_score + nq * m;
    a.out_nn = reinterpret_cast<int64_t*>(a.out_rew + nq * m);
    a.out_nn_sim = reinterpret_cast<double*>(a.out_nn + nq);
    a.out_round = reinterpret_cast<int32_t*>(a.out_nn_sim + nq);
    a.out_cnt = a.out_round + nq * m;
    const size_t smem = small_smem_bytes(n, d, m, cs);
    SAIR_CUDA(cudaFuncSetAttribute(small_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3((unsigned)(nq * cs));
    lc.blockDim = dim3(SMALL_THREADS);
    lc.dynamicSmemBytes = smem;
    lc.stream = s->st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    SAIR_CUDA(cudaLaunchKernelEx(&lc, small_select_kernel, a));
    SAIR_LAUNCH("small_select_kernel");
    char* hout = static_cast<char*>(s->h_out.get(ob));
    SAIR_CUDA(cudaMemcpyAsync(hout, dout, ob, cudaMemcpyDeviceToHost, s->st));
    auto unpack = [=]() {
    const int64_t* hidx = reinterpret_cast<const int64_t*>(hout);
    const double* hsim = reinterpret_cast<const double*>(hidx + nq * m);
    const double* hsc = hsim + nq * m;
    const double* hrw = hsc + nq * m;
    const int64_t* hnn = reinterpret_cast<const int64_t*>(hrw + nq * m);
    const double* hnns = reinterpret_cast<const double*>(hnn + nq);
    const int32_t* hrd = reinterpret_cast<const int32_t*>(hnns + nq);
    const int* hcnt = hrd + nq * m;
    for (size_t i = 0; i < nq; ++i) {
        const size_t g = qidx[i], c = (size_t)hcnt[i];
        out_count[g] = c;
        std::copy(hidx + i * m, hidx + i * m + c, out_idx + g * m);
        std::copy(hsim + i * m, hsim + i * m + c, out_sim + g * m);
        std::copy(hsc + i * m, hsc + i * m + c, out_score + g * m);
        if (out_reward) std::copy(hrw + i * m, hrw + i * m + c, out_reward + g * m);
        if (out_round) std::copy(hrd + i * m, hrd + i * m + c, out_round + g * m);
        if (out_nn) {
            out_nn[g] = hnn[i];
            out_nn_sim[g] = hnns[i];
        }
    }
    };
    if (s->defer_sync) {  // a decision step: the caller synchronises once, then unpacks
        s->pending = unpack;
        return;
    }
    SAIR_CUDA(cudaStreamSynchronize(s->st));
    unpack();
}

}  // namespace sair
