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
#include "umma.cuh"

namespace cg = cooperative_groups;

namespace sair {

namespace {

constexpr int SMALL_THREADS = 1024;
constexpr int SMALL_CS_MAX = 8;       // portable cluster size
constexpr int SMALL_CS_MAX16 = 16;    // the inbox's slots (non-portable clusters up to 16)
constexpr size_t SMALL_PER_MAX = 8192;  // records per CTA (shared-memory slice)

struct SmallArgs {
    const double* z;     // [d][n] standardized rows, dimension-major (coalesced per k)
    const double* r64;
    const int32_t* rnd;
    const double* zq;    // [nq][d] standardized queries
    int d, m, nn, cs;
    size_t n, per;       // records, records per CTA (even)
    size_t ldz;          // row stride of z (even: 16-byte aligned rows for the bulk copies)
    size_t n_loo;        // loo_mean's n (the whole buffer's)
    double total, two_s2, lambda;
    const double* loo;   // [n] locally weighted LOO means (nullable: the global mean)
    unsigned long long* trace;  // diagnostics (SAIR_SMALL_TRACE): phase times of CTA 0, or null
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
                             const double* __restrict__ sd, size_t n, int d, size_t ld,
                             double* __restrict__ z) {
    const size_t total = n * (size_t)d;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total;
         e += (size_t)gridDim.x * blockDim.x) {
        const int k = (int)(e % d);
        z[(size_t)k * ld + e / d] = ddiv(dsub(x64[e], mean[k]), sd[k]);
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
__global__ void __launch_bounds__(256) local_loo_z_kernel(const double* __restrict__ z, size_t ld,
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
            zt[e] = jj < cnt ? z[(size_t)k * ld + j0 + jj] : 0.0;
        }
        for (int jj = threadIdx.x; jj < LOO_TILE; jj += blockDim.x)
            rt[jj] = jj < cnt ? r64[j0 + jj] : 0.0;
        __syncthreads();
        if (!valid) continue;
        for (int jj = 0; jj < cnt; ++jj) {
            if (j0 + jj == i) continue;
            double d2 = 0.0;
            for (int k = 0; k < d; ++k) {
                const double t = dsub(zt[k * LOO_TILE + jj], z[(size_t)k * ld + i]);
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

// The same, tiled for parallelism: per CTA LR = 64 records, per tile LJ = 64
// of the j.  Phase A: all 256 threads compute the tile's 64 x 64 weights w_ij
// (each a 32-term ordered fp64 distance and an exp -- independent pairs, two
// interleaved per thread) into shared memory; phase B: one thread per record
// adds them to its two running sums in j order, exactly as the reference's
// loop does (experience.cpp:129-134; the skipped j = i enters as an exact
// zero: wsum and acc are never -0, so x + (+-0) = x).  10k x 32: 11.5 ms ->
// ~1 ms (the old kernel had one thread per record: 40 CTAs for 148 SMs).
constexpr int LR = 64, LJ = 64;
__global__ void __launch_bounds__(256) local_loo_tiled_kernel(const double* __restrict__ z,
                                                              size_t ld,
                                                              const double* __restrict__ r64,
                                                              size_t n, int d, double two_s2,
                                                              double total, size_t n_loo,
                                                              double* __restrict__ loo) {
    extern __shared__ double sm_loo[];
    double* zi = sm_loo;                 // [d][LR]
    double* zt = zi + (size_t)d * LR;    // [d][LJ]
    double* rt = zt + (size_t)d * LJ;    // [LJ]
    double* W = rt + LJ;                 // [LR][LJ + 1]
    const int tid = threadIdx.x;
    const size_t i0 = (size_t)blockIdx.x * LR;
    for (int e = tid; e < d * LR; e += blockDim.x) {
        const int k = e / LR, il = e % LR;
        zi[e] = i0 + il < n ? z[(size_t)k * ld + i0 + il] : 0.0;
    }
    const int il = tid & (LR - 1), jq = tid >> 6;  // phase A: record il, j = jq + 4 m
    const size_t ia = i0 + il;
    double wsum = 0.0, acc = 0.0;  // phase B (tid < LR): record i0 + tid
    for (size_t j0 = 0; j0 < n; j0 += LJ) {
        const int cnt = (int)min((size_t)LJ, n - j0);
        __syncthreads();  // (the previous tile's W and zt are consumed)
        for (int e = tid; e < d * LJ; e += blockDim.x) {
            const int k = e / LJ, jj = e % LJ;
            zt[e] = jj < cnt ? z[(size_t)k * ld + j0 + jj] : 0.0;
        }
        for (int jj = tid; jj < LJ; jj += blockDim.x) rt[jj] = jj < cnt ? r64[j0 + jj] : 0.0;
        __syncthreads();
        for (int m = 0; m < LJ / 4; m += 2) {
            const int ja = jq + 4 * m, jb = ja + 4;
            double da = 0.0, db = 0.0;
            for (int k = 0; k < d; ++k) {
                const double x = zi[k * LR + il];
                const double ta = dsub(zt[k * LJ + ja], x);  // standardize(z_j) - z_i
                const double tb = dsub(zt[k * LJ + jb], x);
                da = dadd(da, dmul(ta, ta));
                db = dadd(db, dmul(tb, tb));
            }
            const bool oka = ja < cnt && j0 + ja != ia, okb = jb < cnt && j0 + jb != ia;
            W[il * (LJ + 1) + ja] = oka ? sim_from_d2(da, two_s2) : 0.0;
            W[il * (LJ + 1) + jb] = okb ? sim_from_d2(db, two_s2) : 0.0;
        }
        __syncthreads();
        if (tid < LR) {
            const double* wr = W + tid * (LJ + 1);
            for (int jj = 0; jj < cnt; ++jj) {
                const double w = wr[jj];
                wsum = dadd(wsum, w);
                acc = dadd(acc, dmul(w, rt[jj]));
            }
        }
    }
    const size_t i = i0 + tid;
    if (tid >= LR || i >= n) return;
    if (n_loo <= 1) {
        loo[i] = 0.0;
        return;
    }
    loo[i] = wsum > 1e-12 ? ddiv(acc, wsum) : ddiv(dsub(total, r64[i]), (double)(n_loo - 1));
}

static size_t loo_tiled_smem(int d) { return ((size_t)d * (LR + LJ) + LJ + (size_t)LR * (LJ + 1)) * 8; }

// the local LOO means of every record (one launch; the tiled kernel where its
// shared memory fits, d <= 160)
static void local_loo_launch(const double* z, size_t ld, const double* r64, size_t n, int d,
                             double two_s2, double total, size_t n_loo, double* loo,
                             cudaStream_t st) {
    const size_t tsm = loo_tiled_smem(d);
    if (tsm <= 200 * 1024 && !std::getenv("SAIR_LOO_SIMPLE")) {
        static size_t raised = 0;
        if (tsm > raised) {
            SAIR_CUDA(cudaFuncSetAttribute(local_loo_tiled_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm));
            raised = tsm;
        }
        local_loo_tiled_kernel<<<(int)((n + LR - 1) / LR), 256, tsm, st>>>(z, ld, r64, n, d, two_s2,
                                                                           total, n_loo, loo);
        SAIR_LAUNCH("local_loo_tiled_kernel");
        return;
    }
    const size_t lsm = ((size_t)d * LOO_TILE + LOO_TILE) * 8;
    SAIR_CUDA(cudaFuncSetAttribute(local_loo_z_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)lsm));
    local_loo_z_kernel<<<(int)((n + 255) / 256), 256, lsm, st>>>(z, ld, r64, n, d, two_s2, total,
                                                                 n_loo, loo);
    SAIR_LAUNCH("local_loo_z_kernel");
}

__device__ __forceinline__ void small_ev(const SmallArgs& a, int crank, int e) {
    if (a.trace && crank == 0 && threadIdx.x == 0 && blockIdx.x == 0 && e < 64) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.trace[e] = t;
    }
}

// warp arg-max by the greedy's key (better(): gain desc, round asc, index asc)
// with redux.sync instead of a shuffle tree: the gain's order-preserving
// 64-bit image in two 32-bit max reductions, ties by round, then by index
// (record indices of a small store fit 32 bits).  Every lane gets the winner.
__device__ __forceinline__ Best warp_best_fast(const Best& b) {
    const bool valid = b.j >= 0;
    const unsigned long long u = (unsigned long long)__double_as_longlong(b.g);
    const unsigned long long key = valid ? ((u >> 63) ? ~u : (u | 0x8000000000000000ull)) : 0ull;
    const uint32_t khi = (uint32_t)(key >> 32), klo = (uint32_t)key;
    const uint32_t mhi = __reduce_max_sync(0xffffffffu, khi);
    const uint32_t mlo = __reduce_max_sync(0xffffffffu, khi == mhi ? klo : 0u);
    unsigned tie = __ballot_sync(0xffffffffu, valid && khi == mhi && klo == mlo);
    if (tie == 0) return Best{0.0, 0, 0, -1};
    if (__popc(tie) > 1) {
        const bool in = (tie >> (threadIdx.x & 31)) & 1u;
        const int rmin = __reduce_min_sync(0xffffffffu, in ? b.r : INT_MAX);
        tie = __ballot_sync(0xffffffffu, in && b.r == rmin);
        if (__popc(tie) > 1) {
            const bool in2 = (tie >> (threadIdx.x & 31)) & 1u;
            const uint32_t imin = __reduce_min_sync(0xffffffffu, in2 ? (uint32_t)b.i : 0xFFFFFFFFu);
            tie = __ballot_sync(0xffffffffu, in2 && (uint32_t)b.i == imin);
        }
    }
    const int src = __ffs(tie) - 1;
    Best w;
    w.g = __shfl_sync(0xffffffffu, b.g, src);
    w.r = __shfl_sync(0xffffffffu, b.r, src);
    w.i = __shfl_sync(0xffffffffu, b.i, src);
    w.j = 1;
    return w;
}

// Shared-memory layout of one CTA (small_smem_bytes): per slice record score,
// penalty, similarity (doubles), taken (byte); the query row; the current
// pick's row; the picks' data (owner-recorded) and indices; the per-warp
// bests; the inbox the cluster's CTAs push their bests into ([2 buffers][2
// kinds][16]) and its two mbarriers; ZS: the slice's rows [d][per].
struct SmallSmem {
    double *score, *pen, *sim, *zq, *zb, *pdat, *zs;
    int64_t* pidx;
    Best *inbox, *wb;
    uint64_t* mbar;
    unsigned char* taken;
};

__device__ __forceinline__ SmallSmem small_carve(unsigned char* sm, size_t per, int d, int m) {
    SmallSmem S;
    S.score = reinterpret_cast<double*>(sm);
    S.pen = S.score + per;
    S.sim = S.pen + per;
    S.zq = S.sim + per;
    S.zb = S.zq + d;
    S.pdat = S.zb + d;                                             // [m][4]: sim, score, reward, round
    S.pidx = reinterpret_cast<int64_t*>(S.pdat + 4 * (size_t)m);   // [m]
    S.inbox = reinterpret_cast<Best*>(                             // [2][2][SMALL_CS_MAX16]
        (reinterpret_cast<uintptr_t>(S.pidx + m) + 15) & ~(uintptr_t)15);  // (st.async: 16-aligned)
    S.wb = S.inbox + 4 * SMALL_CS_MAX16;                           // [32][2]
    S.mbar = reinterpret_cast<uint64_t*>(S.wb + 64);               // [3]: inbox x 2, rows copy
    S.taken = reinterpret_cast<unsigned char*>(S.mbar + 4);
    S.zs = reinterpret_cast<double*>(S.taken + ((per + 15) & ~(size_t)15));  // (16-aligned)
    return S;
}

// push a Best into another CTA's shared memory (32 bytes, two 16-byte
// st.async), completing that many transaction bytes on its mbarrier
__device__ __forceinline__ void push_best(const Best& b, uint32_t dst, uint32_t mbar) {
    const unsigned long long w0 = (unsigned long long)__double_as_longlong(b.g);
    const unsigned long long w1 = (unsigned long long)(uint32_t)b.r;
    const unsigned long long w2 = (unsigned long long)b.i;
    const unsigned long long w3 = (unsigned long long)(uint32_t)b.j;
    static_assert(sizeof(Best) == 32, "Best layout");
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];"
        ::"r"(dst), "l"(w0), "l"(w1), "r"(mbar) : "memory");
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];"
        ::"r"(dst + 16), "l"(w2), "l"(w3), "r"(mbar) : "memory");
}

// One cluster per query, each CTA a slice of the records.  A greedy step is
// one pass over the slice (the previous pick's similarity added to every
// untaken penalty, experience.cpp:283-284, fused with the arg-max of the
// gains, :176-188), a block reduction whose result warp 0 pushes into every
// CTA's inbox (st.async, completing on the receiver's mbarrier), and every
// warp reducing its own CTA's inbox once the mbarrier's phase completes --
// the same winner everywhere, no cluster barrier inside the loop (each one
// also invalidates L1).  Step 0's pass computes the exact scores (:163-167)
// and the veto scan's nearest record (policy.cpp:146-153) together.  ZS: the
// slice's standardized rows are copied to shared memory once.
template <bool ZS>
__global__ void __launch_bounds__(SMALL_THREADS) small_select_kernel(const __grid_constant__ SmallArgs a) {
    cg::cluster_group cl = cg::this_cluster();
    const int crank = (int)cl.block_rank();
    const int q = blockIdx.x / a.cs;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int d = a.d;
    const size_t lo = (size_t)crank * a.per;
    const size_t hi = min(a.n, lo + a.per);
    const uint32_t ns = hi > lo ? (uint32_t)(hi - lo) : 0u;
    extern __shared__ __align__(16) unsigned char sm[];
    const SmallSmem S = small_carve(sm, a.per, d, a.m);
    const double* zl = a.z + lo;  // this slice's rows in global memory, [d][ldz]
    auto zat = [&](int k, uint32_t j) -> double {
        if constexpr (ZS) return S.zs[(size_t)k * a.per + j];
        else return zl[(size_t)k * a.ldz + j];
    };
    small_ev(a, crank, 0);
    // (ZS: one bulk copy per dimension row of the slice, rounded up to an even
    // record count -- rows are padded to ldz, slices to an even per)
    const uint32_t cb = ((ns + 1u) & ~1u) * 8u;
    if (tid == 0) {
        umma::bar_init(S.mbar, 1);
        umma::bar_init(S.mbar + 1, 1);
        umma::bar_init(S.mbar + 2, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (ZS && cb) {
            umma::bar_expect_tx(S.mbar + 2, cb * (uint32_t)d);
            for (int k = 0; k < d; ++k)
                umma::bulk_g2s(S.zs + (size_t)k * a.per, zl + (size_t)k * a.ldz, cb, S.mbar + 2);
        }
    }
    for (int k = tid; k < d; k += blockDim.x) S.zq[k] = a.zq[(size_t)q * d + k];
    cl.sync();  // the mbarriers are initialised before any CTA pushes
    if (ZS && cb) umma::bar_wait(S.mbar + 2, 0);

    const Best none{0.0, 0, 0, -1};
    int round = 0;
    // block reduction of (gain best[, nearest best]), pushed into the inbox
    // of every CTA of the cluster; returns the cluster's best (every warp,
    // from its own CTA's inbox)
    auto reduce = [&](Best b, Best nb, bool with_nn, Best& nn_out) {
        const int buf = round & 1;
        const uint32_t parity = (uint32_t)(round >> 1) & 1u;
        ++round;
        if (tid == 0) umma::bar_expect_tx(S.mbar + buf, (uint32_t)(a.cs * (with_nn ? 64 : 32)));
        b = warp_best_fast(b);
        if (with_nn) nb = warp_best_fast(nb);
        if (lane == 0) {
            S.wb[2 * warp] = b;
            S.wb[2 * warp + 1] = nb;
        }
        __syncthreads();
        Best* box = S.inbox + 2 * buf * SMALL_CS_MAX16;
        if (warp == 0) {
            const bool in = lane < (int)(blockDim.x >> 5);
            const Best c = warp_best_fast(in ? S.wb[2 * lane] : none);
            const Best cn = with_nn ? warp_best_fast(in ? S.wb[2 * lane + 1] : none) : none;
            if (lane < a.cs) {
                const uint32_t mb = umma::peer_addr(S.mbar + buf, (uint32_t)lane);
                push_best(c, umma::peer_addr(box + crank, (uint32_t)lane), mb);
                if (with_nn) push_best(cn, umma::peer_addr(box + SMALL_CS_MAX16 + crank, (uint32_t)lane), mb);
            }
        }
        umma::bar_wait(S.mbar + buf, parity);
        if (with_nn) nn_out = warp_best_fast(lane < a.cs ? box[SMALL_CS_MAX16 + lane] : none);
        return warp_best_fast(lane < a.cs ? box[lane] : none);
    };

    // step 0: exact scores, nearest record, best score
    Best b = none, nb = none;
    for (uint32_t j = tid; j < ns; j += blockDim.x) {
        double d2 = 0.0;
#pragma unroll 8
        for (int k = 0; k < d; ++k) {
            const double t = dsub(zat(k, j), S.zq[k]);
            d2 = dadd(d2, dmul(t, t));
        }
        const double s = sim_from_d2(d2, a.two_s2);
        const double r = a.r64[lo + j];
        const double loo = a.loo ? a.loo[lo + j]
                                 : (a.n_loo <= 1 ? 0.0 : ddiv(dsub(a.total, r), (double)(a.n_loo - 1)));
        const double sc = dmul(s, fabs(dsub(r, loo)));
        S.sim[j] = s;
        S.score[j] = sc;
        S.pen[j] = 0.0;
        S.taken[j] = 0;
        const Best c{sc, a.rnd[lo + j], (int64_t)(lo + j), 1};
        if (better(c, b)) b = c;
        const Best cn{s, 0, (int64_t)(lo + j), 1};  // first index on ties
        if (better(cn, nb)) nb = cn;
    }
    small_ev(a, crank, 1);
    const int want = (int)min((size_t)a.m, a.n);
    Best nn = none;
    Best g = reduce(b, nb, a.nn != 0, nn);
    small_ev(a, crank, 2);
    if (a.nn && crank == 0 && tid == 0) {
        a.out_nn[q] = nn.j < 0 ? -1 : a.gbase + nn.i;
        a.out_nn_sim[q] = nn.j < 0 ? -1.0 : nn.g;
    }
    const bool pen_on = a.lambda != 0.0;
    for (int step = 0; step < want; ++step) {
        // g: this step's pick (every thread holds it)
        const size_t gi = (size_t)g.i;
        if (tid == 0) {
            S.pidx[step] = (int64_t)gi;
            if (gi >= lo && gi < hi) {  // the owner records its data for the final gather
                S.pdat[4 * step] = S.sim[gi - lo];
                S.pdat[4 * step + 1] = S.score[gi - lo];
                S.pdat[4 * step + 2] = a.r64[gi];
                S.pdat[4 * step + 3] = (double)a.rnd[gi];
            }
        }
        if (step + 1 == want) break;
        if (pen_on) {  // the pick's row (ZS: from its owner's shared memory)
            if (warp == 0) {
                if constexpr (ZS) {
                    const int owner = (int)(gi / a.per);
                    const double* src = cl.map_shared_rank(S.zs, owner) + (gi - (size_t)owner * a.per);
                    for (int k = lane; k < d; k += 32) S.zb[k] = src[(size_t)k * a.per];
                } else {
                    for (int k = lane; k < d; k += 32) S.zb[k] = a.z[(size_t)k * a.ldz + gi];
                }
            }
            __syncthreads();
        }
        b = none;
        for (uint32_t j = tid; j < ns; j += blockDim.x) {
            if (S.taken[j]) continue;
            if (lo + j == gi) {
                S.taken[j] = 1;
                continue;
            }
            double p = S.pen[j];
            if (pen_on) {
                double d2 = 0.0;
#pragma unroll 8
                for (int k = 0; k < d; ++k) {
                    const double t = dsub(zat(k, j), S.zb[k]);
                    d2 = dadd(d2, dmul(t, t));
                }
                p = dadd(p, sim_from_d2(d2, a.two_s2));  // :283-284
                S.pen[j] = p;
            }
            const Best c{dsub(S.score[j], dmul(a.lambda, p)), a.rnd[lo + j], (int64_t)(lo + j), 1};
            if (better(c, b)) b = c;
        }
        small_ev(a, crank, 3 + 2 * step);
        g = reduce(b, nb, false, nn);
        small_ev(a, crank, 4 + 2 * step);
    }
    cl.sync();  // every owner has recorded its picks
    small_ev(a, crank, 62);
    if (crank == 0 && warp == 0) {
        // gather (sim, score, reward, round) of each pick from its owner, then
        // the curriculum order: stable by (reward asc, round asc) over pick
        // order (:290-294) -- each lane ranks its picks by counting
        for (int x = lane; x < want; x += 32) {
            const int owner = (int)((size_t)S.pidx[x] / a.per);
            if (owner == 0) continue;
            const double* src = cl.map_shared_rank(S.pdat, owner) + 4 * x;
            S.pdat[4 * x] = src[0];
            S.pdat[4 * x + 1] = src[1];
            S.pdat[4 * x + 2] = src[2];
            S.pdat[4 * x + 3] = src[3];
        }
        __syncwarp();
        for (int x = lane; x < want; x += 32) {
            const double rv = S.pdat[4 * x + 2], dv = S.pdat[4 * x + 3];
            int pos = 0;
            for (int y = 0; y < want; ++y) {
                const double ru = S.pdat[4 * y + 2], du = S.pdat[4 * y + 3];
                pos += ru != rv ? ru < rv : (du < dv || (du == dv && y < x));
            }
            const size_t o = (size_t)q * a.m + pos;
            a.out_idx[o] = a.gbase + S.pidx[x];
            a.out_sim[o] = S.pdat[4 * x];
            a.out_score[o] = S.pdat[4 * x + 1];
            a.out_rew[o] = rv;
            a.out_round[o] = (int32_t)dv;
        }
        if (lane == 0) a.out_cnt[q] = want;
    }
    small_ev(a, crank, 63);
    cl.sync();  // no CTA exits while another may still read its shared memory
}

}  // namespace

void zrows_launch(const double* x64, const double* mean, const double* sd, size_t n, int d,
                  double* z, cudaStream_t st) {
    zrows_kernel<<<(int)std::min<size_t>((n * d + 255) / 256, 2048), 256, 0, st>>>(x64, mean, sd, n,
                                                                                 d, n, z);
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
        s->x64, msd, msd + d, n, d, n, z);
    local_loo_launch(z, n, s->r64, n, d, p.two_s2, eff_stats(s).total, eff_n(s), loo, s->st);
    return loo;
}

bool small_select_fits(const sair_store_s* s, size_t m) {
    return s->n > 0 && s->n <= SMALL_CS_MAX * SMALL_PER_MAX && m <= 256 && s->d <= 1024;
}

// records per CTA: even, so every slice starts 16-byte aligned for the bulk copies
static size_t small_per(size_t n, int cs) { return ((n + cs - 1) / cs + 1) & ~(size_t)1; }

static size_t small_smem_bytes(size_t n, int d, size_t m, int cs, bool zs) {
    // SmallSmem (small_carve)
    const size_t per = small_per(n, cs);
    return per * 24 + (size_t)d * 16 + m * 40 + (4 * SMALL_CS_MAX16 + 64) * sizeof(Best) + 32 +
           ((per + 15) & ~(size_t)15) + 64 + (zs ? per * (size_t)d * 8 : 0);
}

constexpr size_t SMALL_SMEM_MAX = 227 * 1024;

// the kernel's shared-memory limit (set once per variant, to the maximum:
// the attribute only permits), and whether a cluster of cs CTAs with that
// much shared memory is schedulable (cs > 8 is a non-portable size: it needs a
// GPC with 16 free SMs) -- remembered per (variant, cs) as the largest size
// known to fit and the smallest known not to (a decision step grows the store
// by one record per call: no query per call)
static bool small_cluster_ok(bool zs, int cs, size_t smem) {
    static std::mutex mu;
    struct Known {
        size_t ok = 0, bad = SIZE_MAX;
    };
    static Known known[2][SMALL_CS_MAX16 + 1];
    static uint64_t raised[2] = {0, 0};  // per device: function attributes are per device
    std::lock_guard<std::mutex> lk(mu);
    const void* fn = zs ? (const void*)small_select_kernel<true> : (const void*)small_select_kernel<false>;
    int dev = 0;
    SAIR_CUDA(cudaGetDevice(&dev));
    const uint64_t bit = 1ull << (dev & 63);
    if (!(raised[zs] & bit)) {
        SAIR_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)SMALL_SMEM_MAX));
        SAIR_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        raised[zs] |= bit;
    }
    if (cs <= 8) return true;
    Known& k = known[zs][cs];
    if (smem <= k.ok) return true;
    if (smem >= k.bad) return false;
    cudaLaunchConfig_t oc{};
    oc.gridDim = dim3((unsigned)cs);
    oc.blockDim = dim3(SMALL_THREADS);
    oc.dynamicSmemBytes = smem;
    cudaLaunchAttribute ca[1];
    ca[0].id = cudaLaunchAttributeClusterDimension;
    ca[0].val.clusterDim.x = (unsigned)cs;
    ca[0].val.clusterDim.y = 1;
    ca[0].val.clusterDim.z = 1;
    oc.attrs = ca;
    oc.numAttrs = 1;
    int nclusters = 0;
    const bool ok = cudaOccupancyMaxActiveClusters(&nclusters, fn, &oc) == cudaSuccess && nclusters >= 1;
    if (!ok) {
        cudaGetLastError();
        k.bad = smem;
    } else {
        k.ok = smem;
    }
    return ok;
}

// CTAs per query and where the rows live: the slice's standardized rows in
// shared memory (ZS) when a cluster of up to 16 CTAs holds them (10k x 32:
// 16 CTAs of 625 records, 160 KB each); else one record per thread where a
// 16-CTA cluster is schedulable, the portable 8 otherwise, rows read from
// global memory.
static int small_plan(size_t n, int d, size_t m, bool* zs) {
    const int cmax = std::getenv("SAIR_SMALL_CS8") ? 8 : SMALL_CS_MAX16;
    *zs = false;
    if (!std::getenv("SAIR_SMALL_NOZS")) {
        // (as many CTAs as useful: a step's pass is fp64-bound per slice)
        const int cs = (int)std::min<size_t>(cmax, std::max<size_t>(1, (n + 255) / 256));
        const size_t smem = small_smem_bytes(n, d, m, cs, true);
        if (smem <= SMALL_SMEM_MAX && small_cluster_ok(true, cs, smem)) {
            *zs = true;
            return cs;
        }
    }
    int cs = (int)std::min<size_t>(cmax, std::max<size_t>(1, (n + SMALL_THREADS - 1) / SMALL_THREADS));
    if (cs > 8 && !small_cluster_ok(false, cs, small_smem_bytes(n, d, m, cs, false))) cs = 8;
    small_cluster_ok(false, cs, small_smem_bytes(n, d, m, cs, false));
    return cs;
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
    bool zsm = false;
    const int cs = small_plan(n, d, m, &zsm);
    const size_t per = small_per(n, cs);
    const size_t ldz = (n + 1) & ~(size_t)1;
    // device scratch: z rows | mean sd | zq | outputs
    const size_t ob = nq * m * (8 * 4 + 4) + nq * (4 + 8 + 8) + 256;
    char* base = static_cast<char*>(s->b_exact.get(ldz * d * 8 + 2 * (size_t)d * 8 +
                                                    nq * d * 8 + ob + n * 8 + 5 * 256));
    size_t off = 0;
    auto take = [&](size_t bytes) {
        char* ptr = base + off;
        off += (bytes + 255) / 256 * 256;
        return ptr;
    };
    double* z = reinterpret_cast<double*>(take(ldz * d * 8));
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
        s->x64, msd, msd + d, n, d, ldz, z);
    SAIR_LAUNCH("zrows_kernel");
    double* dloo = nullptr;
    if (local) {
        dloo = reinterpret_cast<double*>(take(n * 8));
        local_loo_launch(z, ldz, s->r64, n, d, p.two_s2, eff_stats(s).total, eff_n(s), dloo, s->st);
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
    a.ldz = ldz;
    a.n_loo = eff_n(s);
    a.total = eff_stats(s).total;
    a.two_s2 = p.two_s2;
    a.lambda = lambda;
    a.loo = dloo;
    static const bool trace = std::getenv("SAIR_SMALL_TRACE") != nullptr;
    unsigned long long* dtr = nullptr;
    if (trace) {
        SAIR_CUDA(cudaMalloc(&dtr, 64 * 8));
        SAIR_CUDA(cudaMemsetAsync(dtr, 0, 64 * 8, s->st));
    }
    a.trace = dtr;
    a.gbase = s->gbase;
    a.out_idx = reinterpret_cast<int64_t*>(dout);
    a.out_sim = reinterpret_cast<double*>(a.out_idx + nq * m);
    a.out_score = a.out_sim + nq * m;
    a.out_rew = a.out_score + nq * m;
    a.out_nn = reinterpret_cast<int64_t*>(a.out_rew + nq * m);
    a.out_nn_sim = reinterpret_cast<double*>(a.out_nn + nq);
    a.out_round = reinterpret_cast<int32_t*>(a.out_nn_sim + nq);
    a.out_cnt = a.out_round + nq * m;
    const size_t smem = small_smem_bytes(n, d, m, cs, zsm);  // (limit raised by small_plan)
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
    if (zsm)
        SAIR_CUDA(cudaLaunchKernelEx(&lc, small_select_kernel<true>, a));
    else
        SAIR_CUDA(cudaLaunchKernelEx(&lc, small_select_kernel<false>, a));
    SAIR_LAUNCH("small_select_kernel");
    if (dtr) {  // diagnostics: phase times (us from the kernel's start)
        unsigned long long h[64];
        SAIR_CUDA(cudaMemcpyAsync(h, dtr, sizeof h, cudaMemcpyDeviceToHost, s->st));
        SAIR_CUDA(cudaStreamSynchronize(s->st));
        fprintf(stderr, "[small] cs=%d zs=%d per=%zu:", cs, (int)zsm, per);
        for (int e = 1; e < 64; ++e)
            if (h[e]) fprintf(stderr, " %d:%.1f", e, (h[e] - h[0]) * 1e-3);
        fprintf(stderr, "\n");
        cudaFree(dtr);
    }
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
