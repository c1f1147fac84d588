// pareto.cu -- Pareto-dominance reward shaping on the device.
//
// Restates ParetoFrontier (pareto.cpp:9-89) and compute_reward
// (reward.cpp:9-44):
//   K6  batch frontier maintenance: T sequential insert_normalized() calls are
//       order-independent (the result is the non-dominated set of F u P with
//       first occurrences of duplicates kept), so the batch is a radix sort by
//       (latency, cost, arrival) + an exclusive prefix-min of cost + compaction.
//   K8  per-tuple scoring against a sorted frontier: binary search for the
//       dominance test, pruned bidirectional scan for the distance, the
//       reference's own hypervolume sequence for the contribution.
//   K7  k-objective dominance counts: per-objective dense ranks (exact
//       comparisons on integers), sort by rank sum (a dominator has a strictly
//       smaller sum), tiled pairwise tests with shared-memory j-tiles.
//   reward: the five-term compute_reward per row, fused with K8.
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>

#include "internal.hpp"


namespace sair {

// dominates, pareto.cpp:9-12
__device__ __forceinline__ bool dom2(double pl, double pc, double ql, double qc) {
    return pl <= ql && pc <= qc && (pl < ql || pc < qc);
}

// ------------------------------------------------------------- K8 helpers --

struct FrontierView {
    const double* l;
    const double* c;
    size_t F;
    double hv;  // hypervolume of the view (reference sequence)
    // K8 on frontiers too large for shared memory: li[j] = l[j S] (j < nli),
    // a coarse index in shared memory that narrows each search to S entries
    const double* li = nullptr;
    uint32_t S = 1, nli = 0;
    // K8 on bucketed tuples: frontier points [wbase, wbase + wlen) staged in
    // shared memory (wl, wc); every other index reads l / c
    const double* wl = nullptr;
    const double* wc = nullptr;
    uint32_t wbase = 0, wlen = 0;
};
// point i of the view (W: through the staged window where it covers i)
template <bool W>
__device__ __forceinline__ double at_l(const FrontierView& f, uint32_t i) {
    return W && i - f.wbase < f.wlen ? f.wl[i - f.wbase] : f.l[i];
}
template <bool W>
__device__ __forceinline__ double at_c(const FrontierView& f, uint32_t i) {
    return W && i - f.wbase < f.wlen ? f.wc[i - f.wbase] : f.c[i];
}

// first index with l[i] > x (gt) / l[i] >= x (!gt), within [lo, hi)
// (32-bit indices: a frontier holds < 2^32 points)
template <bool GT>
__device__ __forceinline__ uint32_t bound_l(const double* l, double x, uint32_t lo, uint32_t hi) {
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (GT ? l[mid] > x : !(l[mid] < x)) hi = mid; else lo = mid + 1;
    }
    return lo;
}
template <bool GT>
__device__ __forceinline__ uint32_t bound_lv(const FrontierView& f, double x) {
    const uint32_t F = (uint32_t)f.F;
    if (!f.li) return bound_l<GT>(f.l, x, 0, F);
    // coarse: first index entry past x; the answer lies in ((j - 1) S, j S]
    const uint32_t j = bound_l<GT>(f.li, x, 0, f.nli);
    if (j == 0) return 0;
    return bound_l<GT>(f.l, x, (j - 1) * f.S + 1, min(j * f.S, F));
}
// first index with l[i] > x
__device__ __forceinline__ uint32_t upper_bound_l(const FrontierView& f, double x) {
    return bound_lv<true>(f, x);
}
// first index with l[i] >= x
__device__ __forceinline__ uint32_t lower_bound_l(const FrontierView& f, double x) {
    return bound_lv<false>(f, x);
}

// strictly_dominated, pareto.cpp:31-34: the candidate dominator is the point
// with the largest latency <= pl (the cheapest among those, costs descend).
template <bool W = false>
__device__ __forceinline__ bool f_dominated_u(const FrontierView& f, uint32_t u, double pl,
                                              double pc) {
    if (u == 0) return false;
    return dom2(at_l<W>(f, u - 1), at_c<W>(f, u - 1), pl, pc);
}
__device__ __forceinline__ bool f_dominated(const FrontierView& f, double pl, double pc) {
    return f_dominated_u(f, upper_bound_l(f, pl), pl, pc);
}

// distance, pareto.cpp:75-84: min over points of dl^2 + dc^2, then sqrt.
// Latencies ascend and costs descend along the frontier, so scanning outwards
// from pl can stop once no further point can come closer: backwards when
// dl^2 alone reaches the best value, or once c >= pc (from there both |dl|
// and |dc| only grow); forwards (l > pl, and c < pc for a dominated p) as
// soon as a point is no closer (both grow from there on).  The minimum is
// the same value as the reference's full scan.
template <bool W = false>
__device__ __forceinline__ double f_distance_u(const FrontierView& f, uint32_t u, double pl,
                                               double pc) {
    double best = INFINITY;
    const uint32_t F = (uint32_t)f.F;
    if (F >= 256) {
        // Blocks of 32 points: a block's box is [l_first, l_last] x [c_last,
        // c_first] (l ascends, c descends), and the distance to it bounds every
        // point inside from below -- in rounded arithmetic too, rounding being
        // monotone -- so a block whose bound reaches `best` is skipped whole.
        // Same exits as the point scan below; the same minimum.
        auto box_lb = [&](uint32_t a, uint32_t b) {  // points a..b (a <= b)
            const double l0 = at_l<W>(f, a), l1 = at_l<W>(f, b);
            const double c0 = at_c<W>(f, a), c1 = at_c<W>(f, b);  // c0 >= c1
            const double dx = pl < l0 ? dsub(l0, pl) : (pl > l1 ? dsub(pl, l1) : 0.0);
            const double dy = pc < c1 ? dsub(c1, pc) : (pc > c0 ? dsub(pc, c0) : 0.0);
            return dadd(dmul(dx, dx), dmul(dy, dy));
        };
        // backwards: blocks [s, e] with e from u - 1 down
        for (uint32_t e = u; e > 0;) {
            const uint32_t hi = e - 1, lo = hi >= 31 ? hi - 31 : 0;
            e = lo;
            {
                const double dl = dsub(pl, at_l<W>(f, hi));
                if (dmul(dl, dl) >= best) break;  // the block's nearest latency already too far
            }
            if (box_lb(lo, hi) >= best) continue;
            bool stop = false;
            for (uint32_t i = hi + 1; i-- > lo;) {
                double dl = dsub(pl, at_l<W>(f, i));
                double dl2 = dmul(dl, dl);
                if (dl2 >= best) { stop = true; break; }
                double dc = dsub(pc, at_c<W>(f, i));
                double v = dadd(dl2, dmul(dc, dc));
                best = fmin(best, v);
                if (dc <= 0.0 && v >= best) { stop = true; break; }
            }
            if (stop) break;
        }
        for (uint32_t s0 = u; s0 < F;) {
            const uint32_t lo = s0, hi = min(F - 1, s0 + 31);
            s0 = hi + 1;
            {
                const double dl = dsub(pl, at_l<W>(f, lo));
                if (dmul(dl, dl) >= best) break;
            }
            if (box_lb(lo, hi) >= best) continue;
            bool stop = false;
            for (uint32_t i = lo; i <= hi; ++i) {
                double dl = dsub(pl, at_l<W>(f, i));
                double dl2 = dmul(dl, dl);
                if (dl2 >= best) { stop = true; break; }
                double dc = dsub(pc, at_c<W>(f, i));
                double v = dadd(dl2, dmul(dc, dc));
                best = fmin(best, v);
                if (dc >= 0.0 && v >= best) { stop = true; break; }
            }
            if (stop) break;
        }
        return sqrt(best);
    }
    for (uint32_t i = u; i-- > 0;) {
        double dl = dsub(pl, at_l<W>(f, i));
        double dl2 = dmul(dl, dl);
        if (dl2 >= best) break;
        double dc = dsub(pc, at_c<W>(f, i));
        double v = dadd(dl2, dmul(dc, dc));
        best = fmin(best, v);
        if (dc <= 0.0 && v >= best) break;
    }
    for (uint32_t i = u; i < F; ++i) {
        double dl = dsub(pl, at_l<W>(f, i));
        double dl2 = dmul(dl, dl);
        if (dl2 >= best) break;
        double dc = dsub(pc, at_c<W>(f, i));
        double v = dadd(dl2, dmul(dc, dc));
        best = fmin(best, v);
        if (dc >= 0.0 && v >= best) break;
    }
    return sqrt(best);
}
__device__ __forceinline__ double f_distance(const FrontierView& f, double pl, double pc) {
    return f_distance_u(f, upper_bound_l(f, pl), pl, pc);
}

// contribution, pareto.cpp:67-73, for a non-dominated p.  For small frontiers
// the reference's exact sequence is replayed (copy, insert, hypervolume of the
// result minus hypervolume()), so the value is bit-identical; for large ones
// the exclusive area is summed locally over p's dominated run.
template <bool W = false>
__device__ double f_contribution_a(const FrontierView& f, uint32_t a, double pl, double pc) {
    const uint32_t F = (uint32_t)f.F;
    if (a < F && at_l<W>(f, a) == pl && at_c<W>(f, a) == pc) return 0.0;  // duplicate: no-op insert
    if (F <= 64) {
        // hypervolume (pareto.cpp:56-65) of: survivors l < pl, p, survivors l > pl
        double hv = 0.0;
        bool placed = false;
        double cur_l = 0.0, cur_c = 0.0;
        bool have = false;
        auto emit = [&](double l, double c) {
            if (have) hv = dadd(hv, dmul(dsub(l, cur_l), dsub(1.0, cur_c)));
            cur_l = l;
            cur_c = c;
            have = true;
        };
        for (uint32_t i = 0; i < F; ++i) {
            double l = at_l<W>(f, i), c = at_c<W>(f, i);
            if (dom2(pl, pc, l, c)) continue;  // erased by insert_normalized
            if (!placed && !(l < pl)) {
                emit(pl, pc);
                placed = true;
            }
            emit(l, c);
        }
        if (!placed) emit(pl, pc);
        if (have) hv = dadd(hv, dmul(dsub(1.0, cur_l), dsub(1.0, cur_c)));
        return dsub(hv, f.hv);
    }
    // exclusive area of [pl,1]x[pc,1] not covered by the frontier's boxes
    double c_prev = a > 0 ? at_c<W>(f, a - 1) : 1.0;
    double l_next = a < F ? at_l<W>(f, a) : 1.0;
    double area = dmul(dsub(l_next, pl), dsub(fmin(c_prev, 1.0), pc));
    for (uint32_t j = a; j < F && at_c<W>(f, j) >= pc; ++j) {
        double ln = j + 1 < F ? at_l<W>(f, j + 1) : 1.0;
        area = dadd(area, dmul(dsub(ln, at_l<W>(f, j)), dsub(at_c<W>(f, j), pc)));
    }
    return area;
}
__device__ double f_contribution(const FrontierView& f, double pl, double pc) {
    return f_contribution_a(f, lower_bound_l(f, pl), pl, pc);
}

// reward, pareto.cpp:86-89
// (u = upper_bound of pl: the one binary search every branch shares;
// lower_bound differs only on points with l == pl, just before u)
template <bool W = false>
__device__ double f_reward_u(const FrontierView& f, uint32_t u, double pl, double pc,
                             bool* dominated) {
    bool dm = f_dominated_u<W>(f, u, pl, pc);
    if (dominated) *dominated = dm;
    if (!dm) {
        uint32_t a = u;
        while (a > 0 && !(at_l<W>(f, a - 1) < pl)) --a;
        return dadd(1.0, f_contribution_a<W>(f, a, pl, pc));
    }
    return ddiv(0.8, dadd(1.0, f_distance_u<W>(f, u, pl, pc)));
}
__device__ double f_reward(const FrontierView& f, double pl, double pc, bool* dominated) {
    return f_reward_u(f, upper_bound_l(f, pl), pl, pc, dominated);
}

// normalize, pareto.cpp:20-29
__device__ __forceinline__ void f_normalize(double l_max, double c_max, double l_ms,
                                            double cost, double* pl, double* pc, bool* clamped) {
    double l = ddiv(l_ms, l_max), c = ddiv(cost, c_max);
    bool hit = false;
    if (l > 1.0) { l = 1.0; hit = true; }
    if (c > 1.0) { c = 1.0; hit = true; }
    if (l < 0.0) l = 0.0;
    if (c < 0.0) c = 0.0;
    *pl = l;
    *pc = c;
    if (clamped) *clamped = hit;
}

// ----------------------------------------------------------------- kernels --

// K8: one tuple per thread, tuples read as one 16-byte load.  The frontier
// goes to shared memory as far as SCORE_SMEM_B allows (every tuple's binary
// search and scans hit it): both coordinates (F <= 6144), the latencies only
// (F <= 12288; costs from L2), or a coarse index of every S-th latency (each
// search finishes within S entries in L2) -- an anti-correlated 4M-tuple set
// has F ~ 17.6k, which used to fall back to global-memory searches entirely.
constexpr size_t SCORE_SMEM_B = 96 * 1024;
constexpr uint32_t SCORE_SMEM_F = SCORE_SMEM_B / 16;
// larger frontiers: a coarse index of at most SCORE_IDX latencies (16 KB, so
// four 512-thread blocks fit an SM: the searches' L2 latency needs the warps)
constexpr uint32_t SCORE_IDX = 2048;
__global__ void __launch_bounds__(512) score_batch_kernel(FrontierView f, const double* __restrict__ pts,
                                                          size_t T, double* __restrict__ out,
                                                          uint8_t* __restrict__ dom_out) {
    extern __shared__ double fs[];
    const double2* p2 = reinterpret_cast<const double2*>(pts);
    // (each branch inlines its own loop, so the staged arrays are addressed as
    // shared memory, not through generic loads)
    auto run = [&](const FrontierView& v) {
        for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < T;
             t += (size_t)gridDim.x * blockDim.x) {
            const double2 q = p2[t];
            bool dm;
            out[t] = f_reward(v, q.x, q.y, &dm);
            if (dom_out) dom_out[t] = dm;
        }
    };
    const uint32_t F = (uint32_t)f.F;
    if (F <= SCORE_SMEM_F) {  // [F] l | [F] c
        for (uint32_t i = threadIdx.x; i < F; i += blockDim.x) {
            fs[i] = f.l[i];
            fs[F + i] = f.c[i];
        }
        __syncthreads();
        FrontierView v = f;
        v.l = fs;
        v.c = fs + F;
        run(v);
    } else {  // [nli] every S-th l (S = 1: all of them), costs and the fine search from L2
        FrontierView v = f;
        v.S = (F + SCORE_IDX - 1) / SCORE_IDX;
        v.nli = (F + v.S - 1) / v.S;
        for (uint32_t j = threadIdx.x; j < v.nli; j += blockDim.x) fs[j] = f.l[(size_t)j * v.S];
        __syncthreads();
        v.li = fs;
        run(v);
    }
}

// K8 on frontiers beyond shared memory (anti-correlated sets: F ~ 17.6k at
// 4M tuples): the tuples are bucketed by their position on the frontier
// (upper_bound of the latency, SCORE_NB buckets over the frontier's indices),
// so a block's tuples need only a window of the frontier -- their positions
// plus the scans' reach -- which it stages in shared memory; a scan that
// leaves the window reads L2.  Results go back to the tuples' own slots.
constexpr int SCORE_WIN = 6144;  // staged points per block (96 KB)
constexpr int SCORE_CH = 1024;   // sorted tuples per block

__global__ void __launch_bounds__(512) score_bucket_kernel(FrontierView f, const double* __restrict__ pts,
                                                           size_t T, uint32_t NB, uint32_t* __restrict__ upos,
                                                           uint32_t* __restrict__ hist) {
    extern __shared__ double fs[];
    uint32_t* sh = reinterpret_cast<uint32_t*>(fs + SCORE_IDX);
    const uint32_t F = (uint32_t)f.F;
    FrontierView v = f;
    v.S = (F + SCORE_IDX - 1) / SCORE_IDX;
    v.nli = (F + v.S - 1) / v.S;
    for (uint32_t j = threadIdx.x; j < v.nli; j += blockDim.x) fs[j] = f.l[(size_t)j * v.S];
    for (uint32_t b = threadIdx.x; b < NB; b += blockDim.x) sh[b] = 0;
    __syncthreads();
    v.li = fs;
    const double2* p2 = reinterpret_cast<const double2*>(pts);
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < T;
         t += (size_t)gridDim.x * blockDim.x) {
        const uint32_t u = upper_bound_l(v, p2[t].x);
        upos[t] = u;
        atomicAdd(&sh[(uint32_t)((uint64_t)u * NB / (F + 1))], 1u);
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < NB; b += blockDim.x)
        if (sh[b]) atomicAdd(&hist[b], sh[b]);
}

// one block per SCATTER_CH tuples: counts per bucket in shared memory, one
// global reservation per (block, bucket), then the scatter
constexpr int SCATTER_CH = 8192;
__global__ void __launch_bounds__(512) score_scatter_kernel(const double* __restrict__ pts,
                                                            const uint32_t* __restrict__ upos, size_t T,
                                                            uint32_t F, uint32_t NB,
                                                            uint32_t* __restrict__ cursor,
                                                            double2* __restrict__ spts,
                                                            uint32_t* __restrict__ su,
                                                            uint32_t* __restrict__ sidx) {
    extern __shared__ uint32_t scnt[];  // [NB] counts, then bases
    const double2* p2 = reinterpret_cast<const double2*>(pts);
    const size_t t0 = (size_t)blockIdx.x * SCATTER_CH, t1 = min(t0 + SCATTER_CH, T);
    for (uint32_t b = threadIdx.x; b < NB; b += blockDim.x) scnt[b] = 0;
    __syncthreads();
    for (size_t t = t0 + threadIdx.x; t < t1; t += blockDim.x)
        atomicAdd(&scnt[(uint32_t)((uint64_t)upos[t] * NB / (F + 1))], 1u);
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < NB; b += blockDim.x)
        if (scnt[b]) scnt[b] = atomicAdd(&cursor[b], scnt[b]);
    __syncthreads();
    for (size_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
        const uint32_t u = upos[t];
        const uint32_t pos = atomicAdd(&scnt[(uint32_t)((uint64_t)u * NB / (F + 1))], 1u);
        spts[pos] = p2[t];
        su[pos] = u;
        sidx[pos] = (uint32_t)t;
    }
}

__global__ void __launch_bounds__(512) score_window_kernel(FrontierView f, const double2* __restrict__ spts,
                                                           const uint32_t* __restrict__ su,
                                                           const uint32_t* __restrict__ sidx, size_t T,
                                                           double* __restrict__ out,
                                                           uint8_t* __restrict__ dom_out) {
    extern __shared__ double fs[];  // [SCORE_WIN] l | [SCORE_WIN] c
    __shared__ uint32_t s_lo, s_hi;
    const uint32_t F = (uint32_t)f.F;
    for (size_t c0 = (size_t)blockIdx.x * SCORE_CH; c0 < T; c0 += (size_t)gridDim.x * SCORE_CH) {
        const size_t c1 = min(c0 + SCORE_CH, T);
        if (threadIdx.x == 0) {
            s_lo = 0xFFFFFFFFu;
            s_hi = 0;
        }
        __syncthreads();
        uint32_t lo = 0xFFFFFFFFu, hi = 0;
        for (size_t p = c0 + threadIdx.x; p < c1; p += blockDim.x) {
            lo = min(lo, su[p]);
            hi = max(hi, su[p]);
        }
        atomicMin(&s_lo, lo);
        atomicMax(&s_hi, hi);
        __syncthreads();
        // the window: the chunk's positions with a margin each side for the scans
        const uint32_t span = s_hi - s_lo + 1;
        const uint32_t margin = span >= SCORE_WIN ? 0 : (SCORE_WIN - span) / 2;
        const uint32_t wb = s_lo > margin ? s_lo - margin : 0;
        const uint32_t we = min(F, wb + SCORE_WIN);
        FrontierView v = f;
        v.wl = fs;
        v.wc = fs + SCORE_WIN;
        v.wbase = wb;
        v.wlen = we - wb;
        for (uint32_t i = threadIdx.x; i < v.wlen; i += blockDim.x) {
            fs[i] = f.l[wb + i];
            fs[SCORE_WIN + i] = f.c[wb + i];
        }
        __syncthreads();
        for (size_t p = c0 + threadIdx.x; p < c1; p += blockDim.x) {
            const double2 q = spts[p];
            bool dm;
            const double r = f_reward_u<true>(v, su[p], q.x, q.y, &dm);
            const uint32_t t = sidx[p];
            out[t] = r;
            if (dom_out) dom_out[t] = dm;
        }
        __syncthreads();
    }
}

// op codes for the single-point query kernel

__global__ void point_query_kernel(FrontierView f, double pl, double pc, int op,
                                   double* __restrict__ out) {
    if (blockIdx.x) return;
    if (op == Q_HV) {
        // pareto.cpp:56-65: the slab terms in parallel (coalesced loads), their
        // sum in the reference's order -- every lane runs the same chain over
        // the terms shuffled in 32 at a time (one thread re-loading the
        // frontier from global memory term by term took 2 ms at F = 17.7k)
        const int lane = threadIdx.x & 31;
        double hv = 0.0;
        for (size_t i0 = 0; i0 < f.F; i0 += 32) {
            const size_t i = i0 + lane;
            double term = 0.0;
            if (i < f.F) {
                const double nl = i + 1 < f.F ? f.l[i + 1] : 1.0;
                term = dmul(dsub(nl, f.l[i]), dsub(1.0, f.c[i]));
            }
            const int cnt = (int)min((size_t)32, f.F - i0);
            for (int j = 0; j < cnt; ++j) hv = dadd(hv, __shfl_sync(0xffffffffu, term, j));
        }
        if (threadIdx.x == 0) out[0] = hv;
        return;
    }
    if (threadIdx.x) return;
    switch (op) {
        case Q_DOMINATED: out[0] = f_dominated(f, pl, pc) ? 1.0 : 0.0; break;
        case Q_CONTRIB:
            out[1] = f_dominated(f, pl, pc) ? 1.0 : 0.0;
            out[0] = out[1] != 0.0 ? 0.0 : f_contribution(f, pl, pc);
            break;
        case Q_DISTANCE: out[0] = f.F ? f_distance(f, pl, pc) : -1.0; break;
        case Q_REWARD: out[0] = f_reward(f, pl, pc, nullptr); break;
    }
}

// insert_normalized, pareto.cpp:43-54, one point, one CTA: reject test, then
// survivors (not dominated by p) compacted around p's lower_bound slot.
__device__ void insert_one_block(const double* __restrict__ fl, const double* __restrict__ fc,
                                 size_t F, double pl, double pc, double* __restrict__ ol,
                                 double* __restrict__ oc,
                                 unsigned long long* __restrict__ res /* [0]=inserted, [1]=newF */) {
    __shared__ int s_reject;
    __shared__ unsigned s_wsum[32];
    __shared__ size_t s_base;
    if (threadIdx.x == 0) {
        s_reject = 0;
        s_base = 0;
    }
    __syncthreads();
    for (size_t i = threadIdx.x; i < F; i += blockDim.x)
        if ((fl[i] == pl && fc[i] == pc) || dom2(fl[i], fc[i], pl, pc)) s_reject = 1;
    __syncthreads();
    if (s_reject) {
        if (threadIdx.x == 0) {
            res[0] = 0;
            res[1] = F;
        }
        return;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    bool placed_total = false;
    for (size_t c0 = 0; c0 < F; c0 += blockDim.x) {
        size_t i = c0 + threadIdx.x;
        bool keep = i < F && !dom2(pl, pc, fl[i], fc[i]);
        bool before = keep && fl[i] < pl;
        unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) s_wsum[warp] = __popc(bal);
        __syncthreads();
        unsigned off = 0, tot = 0;
        for (int w = 0; w < nw; ++w) {
            if (w < warp) off += s_wsum[w];
            tot += s_wsum[w];
        }
        size_t rank = s_base + off + __popc(bal & ((1u << lane) - 1u));
        if (keep) {
            size_t pos = before ? rank : rank + 1;
            ol[pos] = fl[i];
            oc[pos] = fc[i];
        }
        // p goes right after the last survivor with l < pl
        int nbefore = __syncthreads_count(before);
        if (!placed_total && (size_t)nbefore < (size_t)tot) {
            // survivors are sorted, so the first survivor with l >= pl is in this chunk
            if (threadIdx.x == 0) {
                ol[s_base + nbefore] = pl;
                oc[s_base + nbefore] = pc;
            }
            placed_total = true;
        }
        __syncthreads();
        if (threadIdx.x == 0) s_base += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        if (!placed_total) {
            ol[s_base] = pl;
            oc[s_base] = pc;
        }
        res[0] = 1;
        res[1] = s_base + 1;
    }
}

__global__ void __launch_bounds__(1024)
    insert_one_kernel(const double* __restrict__ fl, const double* __restrict__ fc, size_t F,
                      double pl, double pc, double* __restrict__ ol, double* __restrict__ oc,
                      unsigned long long* __restrict__ res) {
    insert_one_block(fl, fc, F, pl, pc, ol, oc, res);
}

// ---- K6 batch insert --------------------------------------------------------

__device__ __forceinline__ uint64_t ord64(double v) {
    if (v == 0.0) v = 0.0;  // -0 and +0 compare equal in the reference
    uint64_t u = (uint64_t)__double_as_longlong(v);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

__global__ void batch_keys_kernel(const double* __restrict__ l, const double* __restrict__ c,
                                  size_t n, uint64_t* __restrict__ kl, uint64_t* __restrict__ kc,
                                  uint32_t* __restrict__ pos) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        kl[i] = ord64(l[i]);
        kc[i] = ord64(c[i]);
        pos[i] = (uint32_t)i;
    }
}

__global__ void gather_key_kernel(const uint64_t* __restrict__ key, const uint32_t* __restrict__ perm,
                                  size_t n, uint64_t* __restrict__ out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x)
        out[i] = key[perm[i]];
}

// sorted cost (by lexicographic order) for the prefix-min scan
__global__ void sorted_cost_kernel(const double* __restrict__ c, const uint32_t* __restrict__ perm,
                                   size_t n, double* __restrict__ out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x)
        out[i] = c[perm[i]];
}

struct MinOp {
    __device__ __forceinline__ double operator()(double a, double b) const { return a < b ? a : b; }
};

// member = first of its duplicate run && cost < min cost of every
// lexicographically smaller point
__global__ void member_kernel(const double* __restrict__ l, const double* __restrict__ c,
                              const uint32_t* __restrict__ perm, const double* __restrict__ pmin,
                              size_t n, uint32_t* __restrict__ flag) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        uint32_t p = perm[i];
        bool first = i == 0 || !(l[perm[i - 1]] == l[p] && c[perm[i - 1]] == c[p]);
        flag[i] = first && c[p] < pmin[i] ? 1u : 0u;
    }
}

__global__ void compact_kernel(const double* __restrict__ l, const double* __restrict__ c,
                               const uint32_t* __restrict__ perm, const uint32_t* __restrict__ flag,
                               const uint32_t* __restrict__ slot, size_t n,
                               double* __restrict__ ol, double* __restrict__ oc) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        if (!flag[i]) continue;
        uint32_t p = perm[i];
        ol[slot[i]] = l[p];
        oc[slot[i]] = c[p];
    }
}

// K6 pre-filter: one CTA per PF_B arriving tuples, read once from the caller's
// interleaved (l, c) layout.  The CTA sorts its tuples by the high 32 bits of
// the latency's order key in shared memory (block radix sort, 8 passes) and
// drops a tuple when the minimum cost over the tuples of strictly smaller key
// is strictly below its cost -- such a tuple q has q.l < p.l and q.c < p.c,
// i.e. dominates(q, p) (pareto.cpp:9-12), so p cannot be on the final
// frontier and, lying above its dominator's cost, cannot change any other
// tuple's prefix-min in the sort path either.  Survivors are a superset of the
// CTA's local frontier (latency ties and duplicates are left to the exact
// path), written in arrival order so the exact path still keeps the first
// occurrence of a duplicate.  Uniform 4M tuples: ~10 survivors per 4096.
// A NaN coordinate anywhere sets *nan_seen: the host then takes the unfiltered
// path (the filter's order argument needs totally ordered coordinates).
constexpr int PF_THREADS = 512, PF_ITEMS = 8, PF_B = PF_THREADS * PF_ITEMS;

using PfSort = cub::BlockRadixSort<uint32_t, PF_THREADS, PF_ITEMS, uint16_t>;
using PfScanD = cub::BlockScan<double, PF_THREADS>;
using PfScanU = cub::BlockScan<uint32_t, PF_THREADS>;
union PfTemp {
    typename PfSort::TempStorage sort;
    typename PfScanD::TempStorage sd;
    typename PfScanU::TempStorage su;
};
// shared: scan/sort temp | c by arrival [PF_B] | inclusive prefix-min by rank [PF_B] | keep [PF_B]
constexpr size_t PF_SMEM = sizeof(PfTemp) + PF_B * 16 + PF_B + 64;

__global__ void __launch_bounds__(PF_THREADS, 2)  // two CTAs per SM (88 KB shared each)
    prefilter_kernel(const double2* __restrict__ pts, size_t T, double* __restrict__ rl,
                     double* __restrict__ rc, uint32_t* __restrict__ cnt,
                     unsigned int* __restrict__ nan_seen) {
    extern __shared__ __align__(16) unsigned char pf_smem[];
    PfTemp& tmp = *reinterpret_cast<PfTemp*>(pf_smem);
    double* s_c = reinterpret_cast<double*>(pf_smem + sizeof(PfTemp));
    double* s_pm = s_c + PF_B;
    uint8_t* s_keep = reinterpret_cast<uint8_t*>(s_pm + PF_B);
    const int tid = threadIdx.x;
    const size_t base = (size_t)blockIdx.x * PF_B;
    const int nb = (int)min((size_t)PF_B, T - base);
    uint32_t key[PF_ITEMS];
    uint16_t li[PF_ITEMS];
    bool nan = false;
#pragma unroll
    for (int i = 0; i < PF_ITEMS; ++i) {  // striped: coalesced 16-byte loads
        const int j = i * PF_THREADS + tid;
        li[i] = (uint16_t)j;
        if (j < nb) {
            const double2 p = pts[base + j];
            nan |= isnan(p.x) || isnan(p.y);
            key[i] = (uint32_t)(ord64(p.x) >> 32);
            s_c[j] = p.y;
        } else {
            key[i] = ~0u;  // padding sorts last and is never written
        }
    }
    if (__syncthreads_or(nan)) {
        if (tid == 0) atomicOr(nan_seen, 1u);
        return;
    }
    PfSort(tmp.sort).Sort(key, li);  // blocked: thread t holds sorted ranks t*8 .. t*8+7
    __syncthreads();
    double cv[PF_ITEMS], pm[PF_ITEMS];
#pragma unroll
    for (int i = 0; i < PF_ITEMS; ++i) cv[i] = li[i] < nb ? s_c[li[i]] : INFINITY;
    PfScanD(tmp.sd).InclusiveScan(cv, pm, MinOp());
    const int r0 = tid * PF_ITEMS;
#pragma unroll
    for (int i = 0; i < PF_ITEMS; ++i) s_pm[r0 + i] = pm[i];
    __syncthreads();  // every cv read of s_c is done: its space takes the sorted keys
    uint32_t* s_key = reinterpret_cast<uint32_t*>(s_c);
#pragma unroll
    for (int i = 0; i < PF_ITEMS; ++i) s_key[r0 + i] = key[i];
    __syncthreads();
    // the rank where each key's run starts (inclusive max-scan of the run
    // heads); the rank before it holds the minimum cost over every strictly
    // smaller key
    uint32_t hs[PF_ITEMS], rs[PF_ITEMS];
#pragma unroll
    for (int i = 0; i < PF_ITEMS; ++i) {
        const int r = r0 + i;
        const uint32_t pk = i ? key[i - 1] : (r ? s_key[r - 1] : ~key[0]);
        hs[i] = pk != key[i] ? (uint32_t)r : 0u;
    }
    PfScanU(tmp.su).InclusiveScan(hs, rs, cub::Max());
#pragma unroll
    for (int i = 0; i < PF_ITEMS; ++i) {
        if (li[i] >= nb) continue;
        const double m = rs[i] ? s_pm[rs[i] - 1] : INFINITY;
        s_keep[li[i]] = m < cv[i] ? 0 : 1;
    }
    __syncthreads();
    // arrival order: thread t owns local tuples t*8 .. t*8+7
    uint32_t k[PF_ITEMS], pos[PF_ITEMS], tot = 0;
#pragma unroll
    for (int i = 0; i < PF_ITEMS; ++i) {
        const int j = tid * PF_ITEMS + i;
        k[i] = j < nb ? s_keep[j] : 0u;
    }
    PfScanU(tmp.su).ExclusiveSum(k, pos, tot);
#pragma unroll
    for (int i = 0; i < PF_ITEMS; ++i)
        if (k[i]) {
            const double2 p = pts[base + tid * PF_ITEMS + i];
            rl[base + pos[i]] = p.x;
            rc[base + pos[i]] = p.y;
        }
    if (tid == 0) cnt[blockIdx.x] = tot;
}

// the CTAs' survivors, in CTA (= arrival) order, behind the existing frontier
__global__ void __launch_bounds__(256)
    prefilter_gather_kernel(const double* __restrict__ rl, const double* __restrict__ rc,
                            const uint32_t* __restrict__ cnt, const uint32_t* __restrict__ off,
                            int nblk, double* __restrict__ l, double* __restrict__ c,
                            uint32_t* __restrict__ total) {
    const int b = blockIdx.x;
    const uint32_t n = cnt[b], o = off[b];
    const size_t base = (size_t)b * PF_B;
    for (uint32_t k = threadIdx.x; k < n; k += blockDim.x) {
        l[o + k] = rl[base + k];
        c[o + k] = rc[base + k];
    }
    if (b == nblk - 1 && threadIdx.x == 0) *total = o + n;
}

__global__ void deinterleave_kernel(const double2* __restrict__ pts, size_t T,
                                    double* __restrict__ l, double* __restrict__ c) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < T;
         i += (size_t)gridDim.x * blockDim.x) {
        const double2 p = pts[i];
        l[i] = p.x;
        c[i] = p.y;
    }
}

// ---- K7 k-objective dominance counts ----------------------------------------

__global__ void col_keys_kernel(const double* __restrict__ t, size_t T, int K, int k,
                                uint64_t* __restrict__ key, uint32_t* __restrict__ pos) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < T;
         i += (size_t)gridDim.x * blockDim.x) {
        key[i] = ord64(t[i * K + k]);
        pos[i] = (uint32_t)i;
    }
}

__global__ void new_value_kernel(const uint64_t* __restrict__ skey, size_t T,
                                 uint32_t* __restrict__ flag) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < T;
         i += (size_t)gridDim.x * blockDim.x)
        flag[i] = (i > 0 && skey[i] != skey[i - 1]) ? 1u : 0u;
}

__global__ void scatter_rank_kernel(const uint32_t* __restrict__ rank_sorted,
                                    const uint32_t* __restrict__ perm, size_t T, int K, int k,
                                    uint32_t* __restrict__ ranks, uint32_t* __restrict__ rsum) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < T;
         i += (size_t)gridDim.x * blockDim.x) {
        uint32_t p = perm[i];
        ranks[(size_t)p * K + k] = rank_sorted[i];
        if (k == 0) rsum[p] = rank_sorted[i];
        else rsum[p] += rank_sorted[i];
    }
}

__global__ void pack_sorted_kernel(const uint32_t* __restrict__ ranks, const uint32_t* __restrict__ perm,
                                   size_t T, int K, uint32_t* __restrict__ sranks) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < T;
         i += (size_t)gridDim.x * blockDim.x) {
        uint32_t p = perm[i];
        for (int k = 0; k < K; ++k) sranks[i * K + k] = ranks[(size_t)p * K + k];
    }
}

// Tuples are sorted by rank sum.  j dominates i => sum_j < sum_i, and equal
// tuples have equal sums, so every j that matters lies before the first
// position whose sum exceeds the i-tile's largest sum.  One thread per i;
// j-tiles staged in shared memory; dominance is `all(rj <= ri) && rj != ri`.
template <int K>
__global__ void __launch_bounds__(256)
    dominance_kernel(const uint32_t* __restrict__ sr, const uint32_t* __restrict__ ssum,
                     const uint32_t* __restrict__ perm, size_t T, size_t i_begin, int members_only,
                     uint32_t* __restrict__ counts, uint8_t* __restrict__ member) {
    constexpr int TILE = 256;
    __shared__ uint32_t tj[TILE * K];
    __shared__ uint32_t tp[TILE];
    const size_t i0 = i_begin + (size_t)blockIdx.x * TILE;
    const size_t i = i0 + threadIdx.x;
    const bool valid = i < T;
    uint32_t ri[K];
#pragma unroll
    for (int k = 0; k < K; ++k) ri[k] = valid ? sr[i * K + k] : 0xFFFFFFFFu;
    const uint32_t pi = valid ? perm[i] : 0xFFFFFFFFu;
    // j range: [0, first position with sum > max sum of this tile)
    const size_t ilast = min(i0 + TILE, T) - 1;
    const uint32_t smax = ssum[ilast];
    size_t lo = ilast, hi = T;  // first index with ssum > smax
    while (lo < hi) {
        size_t mid = (lo + hi) >> 1;
        if (ssum[mid] > smax) hi = mid; else lo = mid + 1;
    }
    const size_t jend = lo;
    uint32_t cnt = 0;
    bool dup = false;
    for (size_t j0 = 0; j0 < jend; j0 += TILE) {
        __syncthreads();
        for (int t = threadIdx.x; t < TILE; t += blockDim.x) {
            size_t j = j0 + t;
#pragma unroll
            for (int k = 0; k < K; ++k) tj[t * K + k] = j < jend ? sr[j * K + k] : 0xFFFFFFFFu;
            tp[t] = j < jend ? perm[j] : 0xFFFFFFFFu;
        }
        __syncthreads();
        const int lim = (int)min((size_t)TILE, jend - j0);
        for (int t = 0; t < lim; ++t) {
            bool le = true, eq = true;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                uint32_t v = tj[t * K + k];
                le &= v <= ri[k];
                eq &= v == ri[k];
            }
            cnt += (le && !eq) ? 1u : 0u;
            dup |= eq && tp[t] < pi;
        }
        if (members_only && __syncthreads_and(!valid || cnt > 0 || dup)) break;
    }
    if (valid) {
        if (counts) counts[pi] = cnt;
        if (member) member[pi] = (cnt == 0 && !dup) ? 1 : 0;
    }
}


// K <= 4: the same counts with a leaner inner loop.  A j-tile is staged as
// one 16-byte word per tuple (its ranks, padded with 0), so each (i, j) pair
// is one broadcast LDS.128 and K unsigned compares folded into one predicate.
// Tuples are sorted by rank sum: every j before the first position whose sum
// reaches the tile's smallest sum has a strictly smaller sum than every i of
// the tile, so there dominance is just `all(r_j <= r_i)` (equal vectors have
// equal sums); only the j with sums in the tile's own range -- a handful --
// take the exact test with the duplicate rule (pareto.cpp:43-54 keeps the
// first of equal points).  A warp vote ends the scan early when only
// frontier membership is wanted.
template <int K>
__global__ void __launch_bounds__(256)
    dominance4_kernel(const uint32_t* __restrict__ sr, const uint32_t* __restrict__ ssum,
                      const uint32_t* __restrict__ perm, size_t T, size_t i_begin, int members_only,
                      uint32_t* __restrict__ counts, uint8_t* __restrict__ member) {
    static_assert(K >= 1 && K <= 4, "packed ranks: K <= 4");
    constexpr int TILE = 256;
    __shared__ uint4 tj[TILE];
    __shared__ uint32_t tsum[TILE], tp[TILE];
    const size_t i0 = i_begin + (size_t)blockIdx.x * TILE;
    const size_t i = i0 + threadIdx.x;
    const bool valid = i < T;
    uint32_t rr[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int k = 0; k < K; ++k) rr[k] = valid ? sr[i * K + k] : 0xFFFFFFFFu;
    const uint4 ri = make_uint4(rr[0], rr[1], rr[2], rr[3]);
    const uint32_t pi = valid ? perm[i] : 0xFFFFFFFFu;
    const uint32_t sumi = valid ? ssum[i] : 0xFFFFFFFFu;
    const size_t ilast = min(i0 + TILE, T) - 1;
    const uint32_t smax = ssum[ilast], smin = ssum[i0];
    auto first_above = [&](uint32_t v, size_t lo) {  // first index with ssum > v
        size_t hi = T;
        while (lo < hi) {
            const size_t mid = (lo + hi) >> 1;
            if (ssum[mid] > v) hi = mid; else lo = mid + 1;
        }
        return lo;
    };
    const size_t jend = first_above(smax, ilast);
    // first index with ssum >= smin (= first_above(smin - 1)): before it, sums are < every sum_i
    const size_t jsame = smin == 0 ? 0 : min(first_above(smin - 1, 0), jend);
    uint32_t cnt = 0;
    bool dup = false;
    for (size_t j0 = 0; j0 < jend; j0 += TILE) {
        __syncthreads();
        {
            const size_t j = j0 + threadIdx.x;
            uint32_t v[4] = {0u, 0u, 0u, 0u};
            if (j < jend) {
#pragma unroll
                for (int k = 0; k < K; ++k) v[k] = sr[j * K + k];
            } else {
                v[0] = 0xFFFFFFFFu;  // never <= a valid rank vector ... (ranks < T)
            }
            tj[threadIdx.x] = make_uint4(v[0], v[1], v[2], v[3]);
            tsum[threadIdx.x] = j < jend ? ssum[j] : 0xFFFFFFFFu;
            tp[threadIdx.x] = j < jend ? perm[j] : 0xFFFFFFFFu;
        }
        __syncthreads();
        const int lim = (int)min((size_t)TILE, jend - j0);
        // [0, lim_strict): sums strictly below the whole i-tile
        const int lim_strict = j0 >= jsame ? 0 : (int)min((size_t)lim, jsame - j0);
        int t = 0;
#pragma unroll 8
        for (; t < lim_strict; ++t) {
            const uint4 v = tj[t];
            bool le = v.x <= ri.x;
            if (K > 1) le &= v.y <= ri.y;
            if (K > 2) le &= v.z <= ri.z;
            if (K > 3) le &= v.w <= ri.w;
            cnt += le ? 1u : 0u;
        }
        for (; t < lim; ++t) {
            const uint4 v = tj[t];
            bool le = v.x <= ri.x;
            if (K > 1) le &= v.y <= ri.y;
            if (K > 2) le &= v.z <= ri.z;
            if (K > 3) le &= v.w <= ri.w;
            const uint32_t sj = tsum[t];
            cnt += (le && sj < sumi) ? 1u : 0u;
            dup |= le && sj == sumi && tp[t] < pi;  // an equal vector seen earlier
        }
        if (members_only && __syncthreads_and(!valid || cnt > 0 || dup)) break;
    }
    if (valid) {
        if (counts) counts[pi] = cnt;
        if (member) member[pi] = (cnt == 0 && !dup) ? 1 : 0;
    }
}

// ---- K7b: K = 3, 4 over Morton-ordered tiles with bounding boxes ----------
//
// The rank-sum order above makes every i-tile scan about half the store.  Here
// the tuples are sorted by the Morton (bit-interleaved) key of their dense
// ranks, so 256 consecutive tuples -- a tile -- sit in a compact box of rank
// space, and 32 consecutive tiles form a super-tile with its own box.  For the
// j-tile J of a CTA, a box A (all its tuples i) is
//   NONE    if min_A[k] > max_J[k] for some k: no i is <= any j in k;
//   FULL    if max_A <= min_J in every k and < in some k: every i dominates
//           every j (a strict coordinate: no equal vectors);
//   PARTIAL otherwise: the pairs are tested one by one.
// FULL boxes add their tuple count to every j of the tile at once; only
// PARTIAL tiles (the ones whose box touches J's "lower orthant" boundary) are
// staged in shared memory for the pairwise test `all(r_i <= r_j) && r_i != r_j`
// plus the duplicate rule (an equal vector with a smaller original index makes
// j a non-member: pareto.cpp:43-54 keeps the first of equal points).
constexpr int BX_TILE = 256, BX_SUP = 32, BX_SUB = 64, BX_JT = 128, BX_LCAP = BX_JT * BX_SUP;

template <int K>
__global__ void morton_key_kernel(const uint32_t* __restrict__ ranks, size_t T, int shift,
                                  uint64_t* __restrict__ key, uint32_t* __restrict__ pos) {
    constexpr int B = 64 / K;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < T;
         i += (size_t)gridDim.x * blockDim.x) {
        uint32_t r[K];
#pragma unroll
        for (int k = 0; k < K; ++k) r[k] = ranks[i * K + k] >> shift;
        uint64_t m = 0;
#pragma unroll
        for (int b = B - 1; b >= 0; --b)
#pragma unroll
            for (int k = 0; k < K; ++k) m = (m << 1) | ((r[k] >> b) & 1u);
        key[i] = m;
        pos[i] = (uint32_t)i;
    }
}

template <int K>
__global__ void pack4_kernel(const uint32_t* __restrict__ ranks, const uint32_t* __restrict__ perm,
                             size_t T, uint4* __restrict__ rv) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < T;
         i += (size_t)gridDim.x * blockDim.x) {
        const size_t p = perm[i];
        uint32_t v[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int k = 0; k < K; ++k) v[k] = ranks[p * K + k];
        rv[i] = make_uint4(v[0], v[1], v[2], v[3]);
    }
}

__device__ __forceinline__ uint4 umin4(uint4 a, uint4 b) {
    return make_uint4(min(a.x, b.x), min(a.y, b.y), min(a.z, b.z), min(a.w, b.w));
}
__device__ __forceinline__ uint4 umax4(uint4 a, uint4 b) {
    return make_uint4(max(a.x, b.x), max(a.y, b.y), max(a.z, b.z), max(a.w, b.w));
}

// one thread per tile (level 0: tuples -> tile boxes) or per super-tile
// (level 1: tile boxes -> super boxes)
__global__ void box_kernel(const uint4* __restrict__ lo_in, const uint4* __restrict__ hi_in,
                           size_t n_in, int group, size_t n_out, uint4* __restrict__ lo,
                           uint4* __restrict__ hi) {
    const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (t >= n_out) return;
    const size_t a = t * group, e = min(a + group, n_in);
    uint4 mn = lo_in[a], mx = hi_in ? hi_in[a] : lo_in[a];
    for (size_t i = a + 1; i < e; ++i) {
        mn = umin4(mn, lo_in[i]);
        mx = umax4(mx, hi_in ? hi_in[i] : lo_in[i]);
    }
    lo[t] = mn;
    hi[t] = mx;
}

template <int K>
__device__ __forceinline__ int box_class(uint4 amin, uint4 amax, uint4 jmin, uint4 jmax) {
    bool none = amin.x > jmax.x, le = amax.x <= jmin.x, lt = amax.x < jmin.x;
    if (K > 1) { none |= amin.y > jmax.y; le &= amax.y <= jmin.y; lt |= amax.y < jmin.y; }
    if (K > 2) { none |= amin.z > jmax.z; le &= amax.z <= jmin.z; lt |= amax.z < jmin.z; }
    if (K > 3) { none |= amin.w > jmax.w; le &= amax.w <= jmin.w; lt |= amax.w < jmin.w; }
    return none ? 0 : (le && lt ? 1 : 2);
}

template <int K>
__global__ void __launch_bounds__(BX_JT)
    dominance_box_kernel(const uint4* __restrict__ rv, const uint32_t* __restrict__ perm, size_t T,
                         const uint4* __restrict__ bmin64, const uint4* __restrict__ bmax64,
                         const uint4* __restrict__ tmin, const uint4* __restrict__ tmax,
                         const uint4* __restrict__ smin, const uint4* __restrict__ smax,
                         uint32_t ntiles, uint32_t nsup, uint32_t tile_begin, int members_only,
                         uint32_t* __restrict__ counts, uint8_t* __restrict__ member,
                         unsigned long long* __restrict__ stats) {
    __shared__ uint4 ti[BX_TILE];
    __shared__ uint32_t tp[BX_TILE];
    __shared__ uint32_t list[BX_LCAP];
    __shared__ uint32_t nlist, full_add;
    // one CTA per BX_JT = 128 j (two 64-tuple boxes: a tighter box than the
    // 256-tuple i-tiles' -- fewer PARTIAL tiles per j)
    const uint32_t J = tile_begin + blockIdx.x;
    const size_t j = (size_t)J * BX_JT + threadIdx.x;
    const bool valid = j < T;
    const uint4 rj = valid ? rv[j] : make_uint4(0u, 0u, 0u, 0u);
    const uint32_t pj = valid ? perm[j] : 0xFFFFFFFFu;
    const size_t n64 = (T + BX_SUB - 1) / BX_SUB, jb = (size_t)J * (BX_JT / BX_SUB);
    uint4 jmin = bmin64[jb], jmax = bmax64[jb];
    if (jb + 1 < n64) {
        jmin = umin4(jmin, bmin64[jb + 1]);
        jmax = umax4(jmax, bmax64[jb + 1]);
    }
    if (threadIdx.x == 0) {
        nlist = 0;
        full_add = 0;
    }
    uint32_t cnt = 0;
    bool dup = false;
    __syncthreads();
    for (uint32_t s0 = 0; s0 < nsup; s0 += blockDim.x) {
        // 1. the CTA's tile box against super-tile boxes, then tile boxes
        const uint32_t sidx = s0 + threadIdx.x;
        if (sidx < nsup) {
            const int c = box_class<K>(smin[sidx], smax[sidx], jmin, jmax);
            const uint32_t t0 = sidx * BX_SUP, t1 = min(t0 + BX_SUP, ntiles);
            if (c == 1) {
                atomicAdd(&full_add,
                          (uint32_t)(min((size_t)t1 * BX_TILE, T) - (size_t)t0 * BX_TILE));
            } else if (c == 2) {
                uint32_t add = 0;
                for (uint32_t t = t0; t < t1; ++t) {
                    const uint4 amin = tmin[t], amax = tmax[t];
                    const int ct = box_class<K>(amin, amax, jmin, jmax);
                    if (ct == 1) {
                        add += (uint32_t)(min((size_t)(t + 1) * BX_TILE, T) - (size_t)t * BX_TILE);
                    } else if (ct == 2) {
                        // equal vectors need overlapping boxes in every coordinate
                        bool below = amax.x < jmin.x;
                        if (K > 1) below |= amax.y < jmin.y;
                        if (K > 2) below |= amax.z < jmin.z;
                        if (K > 3) below |= amax.w < jmin.w;
                        list[atomicAdd(&nlist, 1u)] = t | (below ? 0u : 0x80000000u);
                    }
                }
                if (add) atomicAdd(&full_add, add);
            }
        }
        __syncthreads();
        if (members_only && full_add > 0) break;  // every j of the tile is dominated
        // 2. PARTIAL tiles, pairwise.  A tile whose box lies strictly below
        // J's in some coordinate holds no vector equal to any j: there the
        // test is `all(r_i <= r_j)` alone (one LDS.128 and K compares a pair)
        const uint32_t nl = nlist;
        if (stats && threadIdx.x == 0) atomicAdd(&stats[0], (unsigned long long)nl);
        for (uint32_t e = 0; e < nl; ++e) {
            const uint32_t I = list[e] & 0x7FFFFFFFu;
            const bool exact = (list[e] >> 31) != 0;
            for (int k = threadIdx.x; k < BX_TILE; k += blockDim.x) {
                const size_t i = (size_t)I * BX_TILE + k;
                ti[k] = i < T ? rv[i] : make_uint4(0xFFFFFFFFu, 0u, 0u, 0u);
                if (exact) tp[k] = i < T ? perm[i] : 0xFFFFFFFFu;
            }
            __syncthreads();
            const int lim = (int)min((size_t)BX_TILE, T - (size_t)I * BX_TILE);
            // each warp's own 32 j (Morton-consecutive: a compact box) against
            // the tile's box: a warp whose j all see it NONE skips the tile, one
            // whose j all see it FULL adds its size -- warp-uniform branches
            const int pcl = valid ? box_class<K>(tmin[I], tmax[I], rj, rj) : 0;
            if (!exact && __all_sync(0xffffffffu, pcl == 0)) {
            } else if (!exact && __all_sync(0xffffffffu, pcl == 1 || !valid)) {
                if (valid) cnt += (uint32_t)lim;
            } else if (!exact) {
                // the same warp-uniform test per 64-tuple quarter of the tile
                uint32_t c2 = 0;
#pragma unroll 1
                for (int q0 = 0; q0 < lim; q0 += BX_SUB) {
                    const size_t sb = (size_t)I * (BX_TILE / BX_SUB) + (size_t)(q0 / BX_SUB);
                    const int qn = min(BX_SUB, lim - q0);
                    const int qc = valid ? box_class<K>(bmin64[sb], bmax64[sb], rj, rj) : 0;
                    if (__all_sync(0xffffffffu, qc == 0)) continue;
                    if (__all_sync(0xffffffffu, qc == 1 || !valid)) {
                        c2 += (uint32_t)qn;
                        continue;
                    }
#pragma unroll 8
                    for (int t = q0; t < q0 + qn; ++t) {
                        const uint4 v = ti[t];
                        bool le = v.x <= rj.x;
                        if (K > 1) le &= v.y <= rj.y;
                        if (K > 2) le &= v.z <= rj.z;
                        if (K > 3) le &= v.w <= rj.w;
                        c2 += le ? 1u : 0u;
                    }
                }
                if (valid) cnt += c2;
            } else {
                if (stats && threadIdx.x == 0) atomicAdd(&stats[1], 1ull);
#pragma unroll 4
                for (int t = 0; t < lim; ++t) {
                    const uint4 v = ti[t];
                    bool le = v.x <= rj.x, eq = v.x == rj.x;
                    if (K > 1) { le &= v.y <= rj.y; eq &= v.y == rj.y; }
                    if (K > 2) { le &= v.z <= rj.z; eq &= v.z == rj.z; }
                    if (K > 3) { le &= v.w <= rj.w; eq &= v.w == rj.w; }
                    cnt += (le && !eq) ? 1u : 0u;
                    dup |= eq && tp[t] < pj;
                }
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) nlist = 0;
        __syncthreads();
        if (members_only && __syncthreads_and(!valid || cnt > 0 || dup)) break;
    }
    if (valid) {
        const uint32_t tot = cnt + full_add;
        if (counts) counts[pj] = tot;
        if (member) member[pj] = (tot == 0 && !dup) ? 1 : 0;
    }
}

// ---- K7 for two objectives: O(T log T) counting ----------------------------
//
// Sort by (rank_l, rank_c, arrival): j dominates i iff j sits before i with
// rank_c(j) <= rank_c(i), except exact duplicates (equal pair), which form a
// contiguous run.  #{earlier, c <= c_i} is counted by a bottom-up merge sort
// of the c-ranks in that order: at the level where j (left block) and i (right
// block) separate, i's upper_bound in the sorted left block counts every such
// j exactly once.  count_i = that total - (duplicates before i); member_i =
// count 0 and first of its duplicate run (pareto.cpp:36-54 keeps the first).

__global__ void pair_key_kernel(const uint32_t* __restrict__ ranks, size_t T, int K,
                                uint64_t* __restrict__ key, uint32_t* __restrict__ pos) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < T;
         i += (size_t)gridDim.x * blockDim.x) {
        const uint64_t rl = ranks[i * K], rc = K > 1 ? ranks[i * K + 1] : 0u;
        key[i] = (rl << 32) | rc;
        pos[i] = (uint32_t)i;
    }
}

// v[p] = c-rank in sorted order, id[p] = p, first[p] = start of p's run of equal keys
__global__ void pair_init_kernel(const uint64_t* __restrict__ skey, size_t T,
                                 uint32_t* __restrict__ v, uint32_t* __restrict__ id,
                                 uint32_t* __restrict__ first, uint32_t* __restrict__ acc) {
    for (size_t p = blockIdx.x * (size_t)blockDim.x + threadIdx.x; p < T;
         p += (size_t)gridDim.x * blockDim.x) {
        v[p] = (uint32_t)(skey[p] & 0xFFFFFFFFull);
        id[p] = (uint32_t)p;
        acc[p] = 0;
        first[p] = (p == 0 || skey[p] != skey[p - 1]) ? (uint32_t)p : 0u;
    }
}

// one merge level: blocks of w sorted values; right-block elements count the
// left block's values <= theirs; both write their merged position (left first
// on ties)
__global__ void merge_count_kernel(const uint32_t* __restrict__ v, const uint32_t* __restrict__ id,
                                   size_t T, size_t w, uint32_t* __restrict__ v2,
                                   uint32_t* __restrict__ id2, uint32_t* __restrict__ acc) {
    for (size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x < T;
         x += (size_t)gridDim.x * blockDim.x) {
        const size_t blk = x / w, base = (blk & ~(size_t)1) * w;
        const bool right = blk & 1;
        const size_t lo = right ? base : base + w;  // the sibling block
        const size_t hi = min(lo + w, T);
        const uint32_t val = v[x];
        size_t a = lo, b = hi;  // right: upper_bound (<= val); left: lower_bound (< val)
        while (a < b) {
            const size_t mid = (a + b) >> 1;
            if (right ? v[mid] <= val : v[mid] < val) a = mid + 1; else b = mid;
        }
        const size_t in_sib = a - lo, own = x - (right ? base + w : base);
        if (right) acc[id[x]] += (uint32_t)in_sib;
        const size_t out = base + own + in_sib;
        v2[out] = val;
        id2[out] = id[x];
    }
}

__global__ void pair_finish_kernel(const uint32_t* __restrict__ acc, const uint32_t* __restrict__ first,
                                   const uint32_t* __restrict__ perm, size_t T,
                                   uint32_t* __restrict__ counts, uint8_t* __restrict__ member) {
    for (size_t p = blockIdx.x * (size_t)blockDim.x + threadIdx.x; p < T;
         p += (size_t)gridDim.x * blockDim.x) {
        const uint32_t f = first[p];
        const uint32_t c = acc[p] - (uint32_t)(p - f);
        counts[perm[p]] = c;
        member[perm[p]] = (c == 0 && f == p) ? 1 : 0;
    }
}

// ---- reward ---------------------------------------------------------------

struct RewardCfg {
    double t_sla, l_base, c_budget, w_l, w_c, w_p, r_max;
};

// action_magnitude, reward.cpp:9-19
__device__ double action_mu(const int32_t* d, size_t S) {
    double mu = 0.0;
    int scaled = 0;
    for (size_t s = 0; s < S; ++s) {
        const int32_t* x = d + 4 * s;
        mu = dadd(mu, (double)abs(x[0]));
        double inner = dadd(dadd(ddiv((double)abs(x[1]), 500.0), ddiv((double)abs(x[2]), 256.0)),
                            ddiv((double)abs(x[3]), 10.0));
        mu = dadd(mu, dmul(0.5, inner));
        scaled += (x[0] | x[1] | x[2] | x[3]) != 0;
    }
    return dadd(mu, dmul(0.5, (double)scaled));
}

__global__ void action_mu_kernel(const int32_t* __restrict__ d, size_t S, double* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = action_mu(d, S);
}

// compute_reward, reward.cpp:21-44 (config validity checked on the host)
__global__ void reward_kernel(const double* __restrict__ in, const int32_t* __restrict__ deltas,
                              size_t S, size_t T, FrontierView f, double l_max, double c_max,
                              RewardCfg cfg, double* __restrict__ out) {
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < T;
         t += (size_t)gridDim.x * blockDim.x) {
        const double lb = in[4 * t], la = in[4 * t + 1], cb = in[4 * t + 2], ca = in[4 * t + 3];
        double latency = ddiv(dmul(cfg.w_l, dsub(lb, la)), cfg.l_base);
        double cost = ddiv(dmul(-cfg.w_c, dsub(ca, cb)), cfg.c_budget);
        double sla = 0.0;
        if (la > cfg.t_sla) {
            double ratio = ddiv(la, cfg.t_sla);
            sla = dadd(-dmul(ratio, ratio), 1.0);
        }
        double sg = dsub(ddiv(lb, cfg.t_sla), 1.0);
        if (sg < 0.0) sg = 0.0;  // std::max(0.0, .)
        double proactive = dmul(dmul(sg, action_mu(deltas + t * S * 4, S)), cfg.w_p);
        double pl, pc;
        f_normalize(l_max, c_max, la, ca, &pl, &pc, nullptr);
        double pareto = f_reward(f, pl, pc, nullptr);
        double sum = dadd(dadd(dadd(dadd(latency, cost), sla), proactive), pareto);
        double total = sum < -cfg.r_max ? -cfg.r_max : (cfg.r_max < sum ? cfg.r_max : sum);
        double* o = out + 7 * t;
        o[0] = latency;
        o[1] = cost;
        o[2] = sla;
        o[3] = proactive;
        o[4] = pareto;
        o[5] = total;
        o[6] = total != sum ? 1.0 : 0.0;
    }
}

// ---- prefix-sequential replay ----------------------
//
// Round t's reward is scored against the frontier of the rows s < t flagged
// for update (scalelab_cli.cpp:118-147 cmd_replay; harness.cpp:250-251), then
// row t is inserted when flagged.  The rounds are cut into R blocks, one
// replayer thread each:
//   replay_local_kernel   block b's own frontier L_b (its flagged rows only);
//   replay_prefix_kernel  G_0 = the frontier before the replay, G_{b+1} =
//                         G_b (+) L_b -- the frontier of a union is the
//                         frontier of the union of frontiers, and the batch
//                         result is order-independent -- stored as the start
//                         state S_b of every block;
//   replay_block_kernel   replayer b walks its rounds from S_b exactly as the
//                         sequential loop does: the five-term reward against
//                         the current frontier, then insert_normalized.
// Frontiers live in per-replayer global scratch of `cap` points; a replayer
// that would exceed it raises a flag and the host re-runs with one replayer.

// insert_normalized, pareto.cpp:43-54, on a sorted array (sequential)
__device__ bool fr_insert(double* l, double* c, size_t& F, size_t cap, double pl, double pc,
                          int* overflow) {
    size_t u = 0, hi = F;  // upper_bound(pl)
    while (u < hi) {
        const size_t mid = (u + hi) >> 1;
        if (l[mid] > pl) hi = mid; else u = mid + 1;
    }
    if (u > 0 && (dom2(l[u - 1], c[u - 1], pl, pc) || (l[u - 1] == pl && c[u - 1] == pc)))
        return false;  // equal to or dominated by a member
    size_t a = u;      // members with l == pl sit before u; with c > pc they are dominated
    while (a > 0 && l[a - 1] == pl) --a;
    size_t e = a;      // members p dominates: l >= pl and c >= pc, a contiguous run
    while (e < F && c[e] >= pc) ++e;
    const size_t nF = F - (e - a) + 1;
    if (nF > cap) {
        atomicExch(overflow, 1);
        return false;
    }
    if (e - a != 1) {  // shift the tail [e, F) to a + 1
        if (e > a + 1) {
            for (size_t i = e; i < F; ++i) {
                l[i - (e - a) + 1] = l[i];
                c[i - (e - a) + 1] = c[i];
            }
        } else {
            for (size_t i = F; i-- > e;) {
                l[i + 1] = l[i];
                c[i + 1] = c[i];
            }
        }
    }
    l[a] = pl;
    c[a] = pc;
    F = nF;
    return true;
}

__device__ double fr_hv(const double* l, const double* c, size_t F) {  // pareto.cpp:56-65
    double hv = 0.0;
    for (size_t i = 0; i < F; ++i) {
        const double nl = i + 1 < F ? l[i + 1] : 1.0;
        hv = dadd(hv, dmul(dsub(nl, l[i]), dsub(1.0, c[i])));
    }
    return hv;
}

struct ReplayArgs {
    const double* in;        // [T][4] l_before, l_after, c_before, c_after
    const int32_t* deltas;   // [T][S][4]
    const uint8_t* update;   // [T]
    size_t T, S, B, R, cap;
    double l_max, c_max;
    RewardCfg cfg;
    double* fl;              // [R][cap] working frontiers
    double* fc;
    size_t* fn;              // [R]
    double* sl;              // [R][cap] block start states
    double* sc;
    size_t* sn;              // [R]
    const double* f0l;       // the frontier before the replay
    const double* f0c;
    size_t f0n;
    double* gl;              // [gcap] running prefix frontier (its final state is the result)
    double* gc;
    size_t* gn;
    size_t gcap;
    double* out;             // [T][7]
    int* overflow;
};

// compute_reward, reward.cpp:21-44, of one row against a frontier view;
// returns the normalized (l_after, c_after) for the caller's update()
__device__ void reward_row(const double* in, const int32_t* deltas, size_t S, const FrontierView& v,
                           double l_max, double c_max, const RewardCfg& cfg, double* o, double* pl,
                           double* pc) {
    const double lb = in[0], la = in[1], cb = in[2], ca = in[3];
    double latency = ddiv(dmul(cfg.w_l, dsub(lb, la)), cfg.l_base);
    double cost = ddiv(dmul(-cfg.w_c, dsub(ca, cb)), cfg.c_budget);
    double sla = 0.0;
    if (la > cfg.t_sla) {
        double ratio = ddiv(la, cfg.t_sla);
        sla = dadd(-dmul(ratio, ratio), 1.0);
    }
    double sg = dsub(ddiv(lb, cfg.t_sla), 1.0);
    if (sg < 0.0) sg = 0.0;
    double proactive = dmul(dmul(sg, action_mu(deltas, S)), cfg.w_p);
    f_normalize(l_max, c_max, la, ca, pl, pc, nullptr);
    double pareto = f_reward(v, *pl, *pc, nullptr);
    double sum = dadd(dadd(dadd(dadd(latency, cost), sla), proactive), pareto);
    double total = sum < -cfg.r_max ? -cfg.r_max : (cfg.r_max < sum ? cfg.r_max : sum);
    o[0] = latency;
    o[1] = cost;
    o[2] = sla;
    o[3] = proactive;
    o[4] = pareto;
    o[5] = total;
    o[6] = total != sum ? 1.0 : 0.0;
}

__global__ void replay_local_kernel(const ReplayArgs a) {
    const size_t b = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (b >= a.R) return;
    double* l = a.fl + b * a.cap;
    double* c = a.fc + b * a.cap;
    size_t F = 0;
    const size_t t1 = min(a.T, (b + 1) * a.B);
    for (size_t t = b * a.B; t < t1; ++t) {
        if (!a.update[t]) continue;
        double pl, pc;
        f_normalize(a.l_max, a.c_max, a.in[4 * t + 1], a.in[4 * t + 3], &pl, &pc, nullptr);
        fr_insert(l, c, F, a.cap, pl, pc, a.overflow);
    }
    a.fn[b] = F;
}

__global__ void replay_prefix_kernel(const ReplayArgs a) {
    if (threadIdx.x || blockIdx.x) return;
    size_t G = a.f0n;
    for (size_t i = 0; i < G; ++i) {
        a.gl[i] = a.f0l[i];
        a.gc[i] = a.f0c[i];
    }
    for (size_t b = 0; b < a.R; ++b) {
        if (G > a.cap) {
            atomicExch(a.overflow, 1);
            return;
        }
        for (size_t i = 0; i < G; ++i) {
            a.sl[b * a.cap + i] = a.gl[i];
            a.sc[b * a.cap + i] = a.gc[i];
        }
        a.sn[b] = G;
        for (size_t i = 0; i < a.fn[b]; ++i)
            fr_insert(a.gl, a.gc, G, a.gcap, a.fl[b * a.cap + i], a.fc[b * a.cap + i], a.overflow);
    }
    *a.gn = G;
}

__global__ void replay_block_kernel(const ReplayArgs a) {
    const size_t b = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (b >= a.R) return;
    double* l = a.fl + b * a.cap;
    double* c = a.fc + b * a.cap;
    size_t F = a.sn[b];
    for (size_t i = 0; i < F; ++i) {
        l[i] = a.sl[b * a.cap + i];
        c[i] = a.sc[b * a.cap + i];
    }
    double hv = fr_hv(l, c, F);
    const size_t t1 = min(a.T, (b + 1) * a.B);
    for (size_t t = b * a.B; t < t1; ++t) {
        double pl, pc;
        reward_row(a.in + 4 * t, a.deltas + t * a.S * 4, a.S, FrontierView{l, c, F, hv}, a.l_max,
                   a.c_max, a.cfg, a.out + 7 * t, &pl, &pc);
        // update(l_after, c_after), pareto.cpp:36-41: normalize, then insert
        if (a.update[t] && fr_insert(l, c, F, a.cap, pl, pc, a.overflow)) hv = fr_hv(l, c, F);
    }
}

// ---- a set of independent frontiers (config 5: one per pipeline) ----------
//
// P small frontiers in one allocation ([P][cap] latencies / costs, sizes,
// cached hypervolumes).  One decision step scores every pipeline's outcome
// against its own frontier and applies its update() (harness.cpp:250-251),
// one thread per pipeline (frontiers stay small: tens of points).

struct SetArgs {
    const double* in;       // [P][4]
    const int32_t* deltas;  // [P][S][4]
    const uint8_t* update;  // [P]
    size_t P, S, cap;
    double l_max, c_max;
    RewardCfg cfg;
    double* fl;
    double* fc;
    size_t* fn;
    double* hv;
    double* out;            // [P][7]
    unsigned long long* maxf;
    int* overflow;
};

__global__ void frontier_set_step_kernel(const SetArgs a) {
    for (size_t p = blockIdx.x * (size_t)blockDim.x + threadIdx.x; p < a.P;
         p += (size_t)gridDim.x * blockDim.x) {
        double* l = a.fl + p * a.cap;
        double* c = a.fc + p * a.cap;
        size_t F = a.fn[p];
        double pl, pc;
        reward_row(a.in + 4 * p, a.deltas + p * a.S * 4, a.S, FrontierView{l, c, F, a.hv[p]},
                   a.l_max, a.c_max, a.cfg, a.out + 7 * p, &pl, &pc);
        if (a.update[p] && fr_insert(l, c, F, a.cap, pl, pc, a.overflow)) {
            a.fn[p] = F;
            a.hv[p] = fr_hv(l, c, F);
        }
        atomicMax(a.maxf, (unsigned long long)F);
    }
}

// ------------------------------------------------------------------- host --

static int grid_for(size_t n, int threads = 256) {
    return (int)std::max<size_t>(1, std::min<size_t>((n + threads - 1) / threads, 148 * 32));
}

static FrontierView view(const sair_frontier_s* f) { return FrontierView{f->fl, f->fc, f->F, f->hv}; }

static size_t score_smem(size_t F) {
    const size_t b = F <= SCORE_SMEM_F ? F * 16 : (size_t)SCORE_IDX * 8;
    if (b > 48 * 1024) cudaFuncSetAttribute(score_batch_kernel,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b);
    return b;
}
// K8 grid: persistent, several 512-thread blocks per SM (two at the largest
// shared-memory footprint)
static int score_grid(size_t T, size_t F) {
    const int per_sm = score_smem(F) > 64 * 1024 ? 2 : 4;
    return (int)std::max<size_t>(1, std::min<size_t>((T + 511) / 512, (size_t)148 * per_sm));
}

void frontier_init(sair_frontier_s* f, double l_max, double c_max, int device) {
    // pareto.cpp:14-18
    if (l_max <= 0.0 || c_max <= 0.0)
        throw Error(SAIR_EINVAL, "ParetoFrontier: normalizers must be positive");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        throw Error(SAIR_ECUDA, "no CUDA device (libsair has no CPU fallback)");
    if (device < 0 || device >= ndev) throw Error(SAIR_EINVAL, "device ordinal out of range");
    f->device = device;
    f->l_max = l_max;
    f->c_max = c_max;
    DeviceGuard g(device);
    SAIR_CUDA(cudaStreamCreateWithFlags(&f->st, cudaStreamNonBlocking));
}

void frontier_free(sair_frontier_s* f) {
    DeviceGuard g(f->device);
    if (f->st) cudaStreamSynchronize(f->st);
    cudaFree(f->fl);
    cudaFree(f->fc);
    f->fl = f->fc = nullptr;
    f->b_tmp.release();
    f->b_in.release();
    f->b_out.release();
    f->b_sort.release();
    if (f->ev_tail) cudaEventDestroy(f->ev_tail);
    f->ev_tail = nullptr;
    if (f->st) cudaStreamDestroy(f->st);
    f->st = nullptr;
}

static void reserve(sair_frontier_s* f, size_t need) {
    if (need <= f->cap) return;
    size_t cap = std::max<size_t>({need, f->cap * 2, 64});
    double *l, *c;
    SAIR_CUDA(cudaMalloc(&l, cap * 8));
    SAIR_CUDA(cudaMalloc(&c, cap * 8));
    if (f->F) {
        SAIR_CUDA(cudaMemcpyAsync(l, f->fl, f->F * 8, cudaMemcpyDeviceToDevice, f->st));
        SAIR_CUDA(cudaMemcpyAsync(c, f->fc, f->F * 8, cudaMemcpyDeviceToDevice, f->st));
    }
    SAIR_CUDA(cudaStreamSynchronize(f->st));
    cudaFree(f->fl);
    cudaFree(f->fc);
    f->fl = l;
    f->fc = c;
    f->cap = cap;
}

// refresh the host mirror and the cached hypervolume after a change
static void sync_mirror(sair_frontier_s* f) {
    f->hl.resize(f->F);
    f->hc.resize(f->F);
    if (f->F) {
        SAIR_CUDA(cudaMemcpyAsync(f->hl.data(), f->fl, f->F * 8, cudaMemcpyDeviceToHost, f->st));
        SAIR_CUDA(cudaMemcpyAsync(f->hc.data(), f->fc, f->F * 8, cudaMemcpyDeviceToHost, f->st));
    }
    double* d = f->b_tmp.as<double>(4);
    point_query_kernel<<<1, 32, 0, f->st>>>(view(f), 0.0, 0.0, Q_HV, d);
    SAIR_LAUNCH("point_query_kernel(hv)");
    SAIR_CUDA(cudaMemcpyAsync(&f->hv, d, 8, cudaMemcpyDeviceToHost, f->st));
    SAIR_CUDA(cudaStreamSynchronize(f->st));
}

void frontier_clone(const sair_frontier_s* f, sair_frontier_s* o) {
    frontier_init(o, f->l_max, f->c_max, f->device);
    DeviceGuard g(f->device);
    SAIR_CUDA(cudaStreamSynchronize(f->st));
    reserve(o, std::max<size_t>(f->F, 1));
    if (f->F) {
        SAIR_CUDA(cudaMemcpyAsync(o->fl, f->fl, f->F * 8, cudaMemcpyDeviceToDevice, o->st));
        SAIR_CUDA(cudaMemcpyAsync(o->fc, f->fc, f->F * 8, cudaMemcpyDeviceToDevice, o->st));
    }
    SAIR_CUDA(cudaStreamSynchronize(o->st));
    o->F = f->F;
    o->hv = f->hv;
    o->hl = f->hl;
    o->hc = f->hc;
}

bool frontier_insert_one(sair_frontier_s* f, double pl, double pc) {
    DeviceGuard g(f->device);
    reserve(f, f->F + 1);
    double* ol = f->b_out.as<double>(2 * (f->F + 1) + 4);
    double* oc = ol + (f->F + 1);
    auto* res = reinterpret_cast<unsigned long long*>(f->b_tmp.as<double>(4));
    insert_one_kernel<<<1, 1024, 0, f->st>>>(f->fl, f->fc, f->F, pl, pc, ol, oc, res);
    SAIR_LAUNCH("insert_one_kernel");
    unsigned long long h[2];
    SAIR_CUDA(cudaMemcpyAsync(h, res, 16, cudaMemcpyDeviceToHost, f->st));
    SAIR_CUDA(cudaStreamSynchronize(f->st));
    if (!h[0]) return false;
    size_t nF = (size_t)h[1];
    SAIR_CUDA(cudaMemcpyAsync(f->fl, ol, nF * 8, cudaMemcpyDeviceToDevice, f->st));
    SAIR_CUDA(cudaMemcpyAsync(f->fc, oc, nF * 8, cudaMemcpyDeviceToDevice, f->st));
    f->F = nF;
    sync_mirror(f);
    return true;
}

// The arriving tuples land on the device in the caller's interleaved layout
// (one H2D copy), K6's pre-filter drops the tuples its CTA proves dominated,
// and the exact sort path below runs on the existing frontier + the survivors.
// Returns the number of tuples behind the frontier in l / c (at l + F).
static size_t stage_batch(sair_frontier_s* f, const double* pts, size_t T, double* l, double* c) {
    const size_t nblk = (T + PF_B - 1) / PF_B;
    // raw[T] double2 | rl[T] | rc[T] | cnt[nblk] | off[nblk] | total, nan
    size_t scan_b = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan_b, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (int)nblk);
    const size_t o_rl = T * 16, o_rc = o_rl + T * 8, o_cnt = o_rc + T * 8,
                 o_off = o_cnt + ((nblk * 4 + 255) & ~(size_t)255),
                 o_misc = o_off + ((nblk * 4 + 255) & ~(size_t)255), o_scan = o_misc + 256;
    char* b = static_cast<char*>(f->b_sort.get(o_scan + scan_b + 256));
    auto* raw = reinterpret_cast<double2*>(b);
    auto* cnt = reinterpret_cast<uint32_t*>(b + o_cnt);
    auto* off = reinterpret_cast<uint32_t*>(b + o_off);
    auto* misc = reinterpret_cast<uint32_t*>(b + o_misc);  // [0] total, [1] nan seen
    copy_h2d_staged(raw, pts, T * 16, f->st);
    static const bool nofilter = std::getenv("SAIR_K6_NOFILTER") != nullptr;
    if (nofilter || T < 2 * PF_B) {
        deinterleave_kernel<<<grid_for(T), 256, 0, f->st>>>(raw, T, l, c);
        SAIR_LAUNCH("deinterleave_kernel");
        SAIR_CUDA(cudaStreamSynchronize(f->st));  // raw lives in b_sort, which the sort reuses
        return T;
    }
    // the dynamic shared-memory limit is a per-device function attribute (a
    // sharded insert runs this on several GPUs of the process)
    static std::atomic<uint64_t> attr_set{0};
    const uint64_t bit = 1ull << (f->device & 63);
    if (!(attr_set.load() & bit)) {
        SAIR_CUDA(cudaFuncSetAttribute(prefilter_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PF_SMEM));
        attr_set.fetch_or(bit);
    }
    SAIR_CUDA(cudaMemsetAsync(misc, 0, 8, f->st));
    prefilter_kernel<<<(unsigned)nblk, PF_THREADS, PF_SMEM, f->st>>>(
        raw, T, reinterpret_cast<double*>(b + o_rl), reinterpret_cast<double*>(b + o_rc), cnt,
        misc + 1);
    SAIR_LAUNCH("prefilter_kernel");
    size_t tb = scan_b;
    SAIR_CUDA(cub::DeviceScan::ExclusiveSum(b + o_scan, tb, cnt, off, (int)nblk, f->st));
    prefilter_gather_kernel<<<(unsigned)nblk, 256, 0, f->st>>>(
        reinterpret_cast<double*>(b + o_rl), reinterpret_cast<double*>(b + o_rc), cnt, off,
        (int)nblk, l, c, misc);
    SAIR_LAUNCH("prefilter_gather_kernel");
    uint32_t h[2];
    SAIR_CUDA(cudaMemcpyAsync(h, misc, 8, cudaMemcpyDeviceToHost, f->st));
    SAIR_CUDA(cudaStreamSynchronize(f->st));
    if (h[1]) {  // a NaN coordinate: every tuple goes to the exact path
        deinterleave_kernel<<<grid_for(T), 256, 0, f->st>>>(raw, T, l, c);
        SAIR_LAUNCH("deinterleave_kernel");
        SAIR_CUDA(cudaStreamSynchronize(f->st));  // raw lives in b_sort, which the sort reuses
        return T;
    }
    return h[0];
}

size_t frontier_insert_batch(sair_frontier_s* f, const double* pts, size_t T) {
    if (T == 0) return f->F;
    DeviceGuard g(f->device);
    if (f->F + T >= 0xFFFFFFFFull) throw Error(SAIR_EINVAL, "batch too large");
    // the tuples land first (l / c at F .. F+T), the sort arrays behind them
    // (sized for the worst case: every tuple survives the pre-filter)
    const size_t N = f->F + T, lc_bytes = ((N + 31) & ~(size_t)31) * 8 + N * 8;
    // 1/16 headroom: the next batch of the same size into the grown frontier
    // must not reallocate (a free + malloc of ~300 MB per 4M batch)
    const size_t need = ((lc_bytes + 255) & ~(size_t)255) + N * (8 * 4 + 4 * 5) + 4096;
    char* base = static_cast<char*>(f->b_in.get(need > f->b_in.bytes ? need + need / 16 : need));
    double* l = reinterpret_cast<double*>(base);
    double* c = l + ((N + 31) & ~(size_t)31);
    const size_t n = f->F + stage_batch(f, pts, T, l + f->F, c + f->F);
    // layout: l, c (staged above), kl[n], kc[n], kt[n], pmin[n], pos[n], perm[n], perm2[n], flag[n], slot[n]
    size_t off = (lc_bytes + 255) & ~(size_t)255;
    auto take = [&](size_t b) {
        char* p = base + off;
        off += (b + 255) / 256 * 256;
        return p;
    };
    uint64_t* kl = reinterpret_cast<uint64_t*>(take(n * 8));
    uint64_t* kc = reinterpret_cast<uint64_t*>(take(n * 8));
    uint64_t* kt = reinterpret_cast<uint64_t*>(take(n * 8));
    double* pmin = reinterpret_cast<double*>(take(n * 8));
    uint32_t* pos = reinterpret_cast<uint32_t*>(take(n * 4));
    uint32_t* perm = reinterpret_cast<uint32_t*>(take(n * 4));
    uint32_t* perm2 = reinterpret_cast<uint32_t*>(take(n * 4));
    uint32_t* flag = reinterpret_cast<uint32_t*>(take(n * 4));
    uint32_t* slot = reinterpret_cast<uint32_t*>(take(n * 4));
    // existing frontier first: it is the earliest arrival
    if (f->F) {
        SAIR_CUDA(cudaMemcpyAsync(l, f->fl, f->F * 8, cudaMemcpyDeviceToDevice, f->st));
        SAIR_CUDA(cudaMemcpyAsync(c, f->fc, f->F * 8, cudaMemcpyDeviceToDevice, f->st));
    }
    batch_keys_kernel<<<grid_for(n), 256, 0, f->st>>>(l, c, n, kl, kc, pos);
    SAIR_LAUNCH("batch_keys_kernel");
    // LSD: stable by cost, then stable by latency -> (l, c, arrival)
    size_t tmp = 0, tmp2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, kc, kt, pos, perm, (int)n);
    cub::DeviceRadixSort::SortPairs(nullptr, tmp2, kl, kt, perm2, perm, (int)n);
    size_t tmp3 = 0;
    cub::DeviceScan::ExclusiveScan(nullptr, tmp3, pmin, reinterpret_cast<double*>(kt), MinOp(), (double)INFINITY, (int)n);
    size_t tmp4 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp4, flag, slot, (int)n);
    void* dtmp = f->b_sort.get(std::max({tmp, tmp2, tmp3, tmp4}) + 256);
    size_t tb = f->b_sort.bytes;
    SAIR_CUDA(cub::DeviceRadixSort::SortPairs(dtmp, tb, kc, kt, pos, perm2, (int)n, 0, 64, f->st));
    gather_key_kernel<<<grid_for(n), 256, 0, f->st>>>(kl, perm2, n, kc);  // kc := l-key in c-order
    SAIR_LAUNCH("gather_key_kernel");
    tb = f->b_sort.bytes;
    SAIR_CUDA(cub::DeviceRadixSort::SortPairs(dtmp, tb, kc, kt, perm2, perm, (int)n, 0, 64, f->st));
    sorted_cost_kernel<<<grid_for(n), 256, 0, f->st>>>(c, perm, n, pmin);
    SAIR_LAUNCH("sorted_cost_kernel");
    tb = f->b_sort.bytes;
    SAIR_CUDA(cub::DeviceScan::ExclusiveScan(dtmp, tb, pmin, reinterpret_cast<double*>(kt), MinOp(),
                                             (double)INFINITY, (int)n, f->st));
    member_kernel<<<grid_for(n), 256, 0, f->st>>>(l, c, perm, reinterpret_cast<double*>(kt), n,
                                                  flag);
    SAIR_LAUNCH("member_kernel");
    tb = f->b_sort.bytes;
    SAIR_CUDA(cub::DeviceScan::ExclusiveSum(dtmp, tb, flag, slot, (int)n, f->st));
    uint32_t last[2];
    SAIR_CUDA(cudaMemcpyAsync(&last[0], slot + n - 1, 4, cudaMemcpyDeviceToHost, f->st));
    SAIR_CUDA(cudaMemcpyAsync(&last[1], flag + n - 1, 4, cudaMemcpyDeviceToHost, f->st));
    SAIR_CUDA(cudaStreamSynchronize(f->st));
    const size_t nF = (size_t)last[0] + last[1];
    reserve(f, nF);
    compact_kernel<<<grid_for(n), 256, 0, f->st>>>(l, c, perm, flag, slot, n, f->fl, f->fc);
    SAIR_LAUNCH("compact_kernel");
    f->F = nF;
    sync_mirror(f);
    return nF;
}

double frontier_point_query(sair_frontier_s* f, double pl, double pc, int op, double* aux) {
    DeviceGuard g(f->device);
    double* d = f->b_tmp.as<double>(4);
    point_query_kernel<<<1, 32, 0, f->st>>>(view(f), pl, pc, op, d);
    SAIR_LAUNCH("point_query_kernel");
    double h[2] = {0.0, 0.0};
    SAIR_CUDA(cudaMemcpyAsync(h, d, 16, cudaMemcpyDeviceToHost, f->st));
    SAIR_CUDA(cudaStreamSynchronize(f->st));
    if (aux) *aux = h[1];
    return h[0];
}

// K8 launch: the frontier in shared memory when it fits, else bucketed tuples
// against staged frontier windows (score_window_kernel)
static void score_launch(sair_frontier_s* f, const double* dp, size_t T, double* dout,
                         uint8_t* ddom, cudaStream_t st) {
    if (f->F <= SCORE_SMEM_F || T < 65536) {
        score_batch_kernel<<<score_grid(T, f->F), 512, score_smem(f->F), st>>>(view(f), dp, T, dout,
                                                                             ddom);
        SAIR_LAUNCH("score_batch_kernel");
        return;
    }
    const uint32_t F = (uint32_t)f->F;
    const uint32_t NB = std::min<uint32_t>(16384u, std::max<uint32_t>(64u, F / 32));
    size_t off = 0;
    auto take = [&](size_t b) { const size_t o = off; off += (b + 255) & ~(size_t)255; return o; };
    const size_t o_u = take(T * 4), o_su = take(T * 4), o_si = take(T * 4), o_sp = take(T * 16),
                 o_h = take((size_t)NB * 4), o_c = take((size_t)NB * 4);
    size_t scan_b = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan_b, (uint32_t*)nullptr, (uint32_t*)nullptr, (int)NB);
    const size_t o_t = take(scan_b);
    char* b = static_cast<char*>(f->b_sort.get(off + 256));
    uint32_t* upos = reinterpret_cast<uint32_t*>(b + o_u);
    uint32_t* su = reinterpret_cast<uint32_t*>(b + o_su);
    uint32_t* sidx = reinterpret_cast<uint32_t*>(b + o_si);
    double2* spts = reinterpret_cast<double2*>(b + o_sp);
    uint32_t* hist = reinterpret_cast<uint32_t*>(b + o_h);
    uint32_t* cursor = reinterpret_cast<uint32_t*>(b + o_c);
    SAIR_CUDA(cudaMemsetAsync(hist, 0, (size_t)NB * 4, st));
    const size_t bsm = SCORE_IDX * 8 + (size_t)NB * 4;
    if (bsm > 48 * 1024)
        SAIR_CUDA(cudaFuncSetAttribute(score_bucket_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)bsm));
    const int gb = (int)std::min<size_t>((T + 511) / 512, 148 * 2);
    score_bucket_kernel<<<gb, 512, bsm, st>>>(view(f), dp, T, NB, upos, hist);
    SAIR_LAUNCH("score_bucket_kernel");
    size_t tb = scan_b;
    SAIR_CUDA(cub::DeviceScan::ExclusiveSum(b + o_t, tb, hist, cursor, (int)NB, st));
    if (NB * 4 > 48 * 1024)
        SAIR_CUDA(cudaFuncSetAttribute(score_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(NB * 4)));
    score_scatter_kernel<<<(int)((T + SCATTER_CH - 1) / SCATTER_CH), 512, NB * 4, st>>>(
        dp, upos, T, F, NB, cursor, spts, su, sidx);
    SAIR_LAUNCH("score_scatter_kernel");
    const size_t wsm = (size_t)SCORE_WIN * 16;
    SAIR_CUDA(cudaFuncSetAttribute(score_window_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)wsm));
    const int gw = (int)std::min<size_t>((T + SCORE_CH - 1) / SCORE_CH, 148 * 2);
    score_window_kernel<<<gw, 512, wsm, st>>>(view(f), spts, su, sidx, T, dout, ddom);
    SAIR_LAUNCH("score_window_kernel");
}

void frontier_score_batch(sair_frontier_s* f, const double* pts, size_t T, double* out,
                          uint8_t* dom) {
    if (T == 0) return;
    DeviceGuard g(f->device);
    char* base = static_cast<char*>(f->b_in.get(T * (16 + 8 + 1) + 1024));
    double* dp = reinterpret_cast<double*>(base);
    double* dout = dp + 2 * T;
    uint8_t* ddom = reinterpret_cast<uint8_t*>(dout + T);
    copy_h2d_staged(dp, pts, T * 16, f->st);
    score_launch(f, dp, T, dout, ddom, f->st);
    SAIR_CUDA(cudaMemcpyAsync(out, dout, T * 8, cudaMemcpyDeviceToHost, f->st));
    if (dom) SAIR_CUDA(cudaMemcpyAsync(dom, ddom, T, cudaMemcpyDeviceToHost, f->st));
    SAIR_CUDA(cudaStreamSynchronize(f->st));
}

// device-pointer variant (bench: tuples resident in HBM)
void frontier_score_batch_device(sair_frontier_s* f, const double* dpts, size_t T, double* dout,
                                 uint8_t* ddom, cudaStream_t st) {
    score_launch(f, dpts, T, dout, ddom, st);
}

void dominance_counts(const double* tuples, size_t T, int K, int device, uint32_t* counts,
                      uint8_t* member, int part, int nparts) {
    if (T == 0) return;
    if (nparts < 1 || part < 0 || part >= nparts)
        throw Error(SAIR_EINVAL, "dominance: part must be in [0, nparts)");
    if (K < 1 || K > 8) throw Error(SAIR_EINVAL, "dominance: K must be in 1..8");
    if (T >= 0xFFFFFFF0ull) throw Error(SAIR_EINVAL, "dominance: too many tuples");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        throw Error(SAIR_ECUDA, "no CUDA device (libsair has no CPU fallback)");
    DeviceGuard g(device);
    cudaStream_t st;
    SAIR_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    DBuf b_all, b_tmp;
    char* base = static_cast<char*>(
        b_all.get(T * (size_t)K * 8 + T * 8 * 2 + T * 4 * 7 + T * (size_t)K * 4 * 2 + T +
                  16 * 256));
    size_t off = 0;
    auto take = [&](size_t b) {
        char* p = base + off;
        off += (b + 255) / 256 * 256;
        return p;
    };
    double* dt = reinterpret_cast<double*>(take(T * K * 8));
    uint64_t* key = reinterpret_cast<uint64_t*>(take(T * 8));
    uint64_t* skey = reinterpret_cast<uint64_t*>(take(T * 8));
    uint32_t* pos = reinterpret_cast<uint32_t*>(take(T * 4));
    uint32_t* perm = reinterpret_cast<uint32_t*>(take(T * 4));
    uint32_t* flag = reinterpret_cast<uint32_t*>(take(T * 4));
    uint32_t* rk = reinterpret_cast<uint32_t*>(take(T * 4));
    uint32_t* rsum = reinterpret_cast<uint32_t*>(take(T * 4));
    uint32_t* ssum = reinterpret_cast<uint32_t*>(take(T * 4));
    uint32_t* ranks = reinterpret_cast<uint32_t*>(take(T * K * 4));
    uint32_t* sranks = reinterpret_cast<uint32_t*>(take(T * K * 4));
    uint32_t* dcnt = reinterpret_cast<uint32_t*>(take(T * 4));
    uint8_t* dmem = reinterpret_cast<uint8_t*>(take(T));
    copy_h2d_staged(dt, tuples, T * K * 8, st);
    size_t t1 = 0, t2 = 0, t3 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, t1, key, skey, pos, perm, (int)T);
    cub::DeviceScan::InclusiveSum(nullptr, t2, flag, rk, (int)T);
    cub::DeviceRadixSort::SortPairs(nullptr, t3, rsum, ssum, pos, perm, (int)T);
    void* tmp = b_tmp.get(std::max({t1, t2, t3}) + 256);
    const int gr = grid_for(T);
    // dense ranks per objective: equal values share a rank, so comparisons on
    // ranks are the exact fp64 comparisons of dominates()
    for (int k = 0; k < K; ++k) {
        col_keys_kernel<<<gr, 256, 0, st>>>(dt, T, K, k, key, pos);
        size_t tb = b_tmp.bytes;
        SAIR_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, key, skey, pos, perm, (int)T, 0, 64, st));
        new_value_kernel<<<gr, 256, 0, st>>>(skey, T, flag);
        tb = b_tmp.bytes;
        SAIR_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb, flag, rk, (int)T, st));
        scatter_rank_kernel<<<gr, 256, 0, st>>>(rk, perm, T, K, k, ranks, rsum);
    }
    SAIR_LAUNCH("rank kernels");
    if (K <= 2 && std::getenv("SAIR_DOM_TILES") == nullptr) {
        // two objectives: O(T log T) merge counting (the pairwise tiles are for K >= 3)
        if (part == 0) {
            pair_key_kernel<<<gr, 256, 0, st>>>(ranks, T, K, key, pos);
            size_t tb = b_tmp.bytes;
            SAIR_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, key, skey, pos, perm, (int)T, 0, 64,
                                                      st));
            uint32_t* first = flag;    // reuse: run starts (max-scan below)
            uint32_t* va = rk;
            uint32_t* ida = rsum;
            uint32_t* vb = ssum;
            uint32_t* idb = sranks;   // >= T entries
            pair_init_kernel<<<gr, 256, 0, st>>>(skey, T, va, ida, first, dcnt);
            tb = b_tmp.bytes;
            SAIR_CUDA(cub::DeviceScan::InclusiveScan(tmp, tb, first, first, cub::Max(), (int)T, st));
            for (size_t w = 1; w < T; w <<= 1) {
                merge_count_kernel<<<gr, 256, 0, st>>>(va, ida, T, w, vb, idb, dcnt);
                std::swap(va, vb);
                std::swap(ida, idb);
            }
            pair_finish_kernel<<<gr, 256, 0, st>>>(dcnt, first, perm, T, reinterpret_cast<uint32_t*>(ranks),
                                                   dmem);
            SAIR_LAUNCH("pair counting");
            if (counts)
                SAIR_CUDA(cudaMemcpyAsync(counts, ranks, T * 4, cudaMemcpyDeviceToHost, st));
        } else {
            SAIR_CUDA(cudaMemsetAsync(dmem, 0, T, st));
            if (counts) std::memset(counts, 0, T * 4);
        }
        if (member) SAIR_CUDA(cudaMemcpyAsync(member, dmem, T, cudaMemcpyDeviceToHost, st));
        SAIR_CUDA(cudaStreamSynchronize(st));
        cudaStreamDestroy(st);
        return;
    }
    static const bool pairwise = std::getenv("SAIR_DOM_PAIRWISE") != nullptr;
    if ((K == 3 || K == 4) && !pairwise) {
        // K7b: Morton-ordered tiles, box-pruned (FULL / NONE / PARTIAL)
        int bits = 1;
        while (((size_t)1 << bits) < T) ++bits;
        const int B = 64 / K, shift = bits > B ? bits - B : 0;
        if (K == 3) morton_key_kernel<3><<<gr, 256, 0, st>>>(ranks, T, shift, key, pos);
        else morton_key_kernel<4><<<gr, 256, 0, st>>>(ranks, T, shift, key, pos);
        size_t tb = b_tmp.bytes;
        SAIR_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, key, skey, pos, perm, (int)T, 0, 64, st));
        // rank vectors in Morton order (16 B each) reuse key | skey (16 B per tuple)
        uint4* rv = reinterpret_cast<uint4*>(key);
        if (K == 3) pack4_kernel<3><<<gr, 256, 0, st>>>(ranks, perm, T, rv);
        else pack4_kernel<4><<<gr, 256, 0, st>>>(ranks, perm, T, rv);
        const size_t ntiles = (T + BX_TILE - 1) / BX_TILE, nsup = (ntiles + BX_SUP - 1) / BX_SUP;
        const size_t n64 = (T + BX_SUB - 1) / BX_SUB;
        DBuf b_box;
        uint4* bx = static_cast<uint4*>(b_box.get((n64 + ntiles + nsup) * 32 + 256));
        uint4 *b64n = bx, *b64x = bx + n64;
        uint4 *tmn = bx + 2 * n64, *tmx = tmn + ntiles, *smn = tmx + ntiles, *smx = smn + nsup;
        box_kernel<<<(int)((n64 + 255) / 256), 256, 0, st>>>(rv, nullptr, T, BX_SUB, n64, b64n,
                                                            b64x);
        box_kernel<<<(int)((ntiles + 255) / 256), 256, 0, st>>>(b64n, b64x, n64, BX_TILE / BX_SUB,
                                                               ntiles, tmn, tmx);
        box_kernel<<<(int)((nsup + 255) / 256), 256, 0, st>>>(tmn, tmx, ntiles, BX_SUP, nsup, smn,
                                                             smx);
        SAIR_LAUNCH("morton tiles");
        // part p of n: an equal share of the j-tiles (BX_JT tuples each; the
        // work per tile is about uniform); tuples outside the part get count 0
        // / member 0
        const size_t njt = (T + BX_JT - 1) / BX_JT;
        const size_t t_lo = njt * (size_t)part / nparts, t_hi = njt * (size_t)(part + 1) / nparts;
        if (nparts > 1) {
            SAIR_CUDA(cudaMemsetAsync(dcnt, 0, T * 4, st));
            SAIR_CUDA(cudaMemsetAsync(dmem, 0, T, st));
        }
        const int members_only = counts == nullptr;
        static const bool dstats = std::getenv("SAIR_DOM_STATS") != nullptr;
        unsigned long long* dst = nullptr;
        if (dstats) {
            SAIR_CUDA(cudaMalloc(&dst, 64));
            SAIR_CUDA(cudaMemsetAsync(dst, 0, 64, st));
        }
        if (t_hi > t_lo) {
            if (K == 3)
                dominance_box_kernel<3><<<(int)(t_hi - t_lo), BX_JT, 0, st>>>(
                    rv, perm, T, b64n, b64x, tmn, tmx, smn, smx, (uint32_t)ntiles, (uint32_t)nsup,
                    (uint32_t)t_lo, members_only, dcnt, dmem, dst);
            else
                dominance_box_kernel<4><<<(int)(t_hi - t_lo), BX_JT, 0, st>>>(
                    rv, perm, T, b64n, b64x, tmn, tmx, smn, smx, (uint32_t)ntiles, (uint32_t)nsup,
                    (uint32_t)t_lo, members_only, dcnt, dmem, dst);
        }
        SAIR_LAUNCH("dominance_box_kernel");
        if (dst) {  // diagnostics: partial tiles per CTA, of which exact-test tiles
            unsigned long long h[3];
            SAIR_CUDA(cudaMemcpyAsync(h, dst, 24, cudaMemcpyDeviceToHost, st));
            SAIR_CUDA(cudaStreamSynchronize(st));
            fprintf(stderr, "[dom] T=%zu K=%d tiles=%zu partial tiles/CTA %.1f (exact-test tiles/CTA %.1f)\n",
                    T, K, ntiles, (double)h[0] / (double)(t_hi - t_lo),
                    (double)h[1] / (double)(t_hi - t_lo));
            cudaFree(dst);
        }
        if (counts) SAIR_CUDA(cudaMemcpyAsync(counts, dcnt, T * 4, cudaMemcpyDeviceToHost, st));
        if (member) SAIR_CUDA(cudaMemcpyAsync(member, dmem, T, cudaMemcpyDeviceToHost, st));
        SAIR_CUDA(cudaStreamSynchronize(st));
        cudaStreamDestroy(st);
        return;
    }
    // order by rank sum
    {
        batch_keys_kernel<<<gr, 256, 0, st>>>(dt, dt, T, key, skey, pos);  // pos = iota
        size_t tb = b_tmp.bytes;
        SAIR_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, rsum, ssum, pos, perm, (int)T, 0, 32, st));
        pack_sorted_kernel<<<gr, 256, 0, st>>>(ranks, perm, T, K, sranks);
    }
    const int members_only = counts == nullptr;
    // Part p of n: the sorted positions [T sqrt(p/n), T sqrt((p+1)/n)) in whole
    // tiles.  Tile i scans ~i earlier tuples (sorted by rank sum), so the
    // pairwise work up to position x grows as x^2 and these parts carry equal
    // shares of it.  Tuples outside the part get count 0 / member 0, so the
    // parts of all n ranks combine by a sum.
    const size_t tiles = (T + 255) / 256;
    auto bound = [&](int q) {
        return std::min(tiles, (size_t)std::ceil((double)tiles * std::sqrt((double)q / nparts)));
    };
    const size_t t_lo = nparts == 1 ? 0 : bound(part), t_hi = nparts == 1 ? tiles : bound(part + 1);
    if (nparts > 1) {
        SAIR_CUDA(cudaMemsetAsync(dcnt, 0, T * 4, st));
        SAIR_CUDA(cudaMemsetAsync(dmem, 0, T, st));
    }
    const int blocks = (int)(t_hi - t_lo);
    const size_t i_begin = t_lo * 256;
    if (blocks > 0) switch (K) {
#define DK(KK) case KK: dominance_kernel<KK><<<blocks, 256, 0, st>>>(sranks, ssum, perm, T, i_begin, members_only, dcnt, dmem); break;
#define DK4(KK) case KK: dominance4_kernel<KK><<<blocks, 256, 0, st>>>(sranks, ssum, perm, T, i_begin, members_only, dcnt, dmem); break;
        DK4(1) DK4(2) DK4(3) DK4(4) DK(5) DK(6) DK(7) DK(8)
#undef DK4
#undef DK
    }
    SAIR_LAUNCH("dominance_kernel");
    if (counts) SAIR_CUDA(cudaMemcpyAsync(counts, dcnt, T * 4, cudaMemcpyDeviceToHost, st));
    if (member) SAIR_CUDA(cudaMemcpyAsync(member, dmem, T, cudaMemcpyDeviceToHost, st));
    SAIR_CUDA(cudaStreamSynchronize(st));
    cudaStreamDestroy(st);
}

static RewardCfg check_cfg(const sair_reward_config* c) {
    // reward.cpp:22-26 (resolved_l_baseline: reward.hpp:17-19)
    if (c->t_sla_ms <= 0.0) throw Error(SAIR_EINVAL, "reward: t_sla_ms must be positive");
    double l_base = c->l_baseline_ms > 0.0 ? c->l_baseline_ms : 4.0 * c->t_sla_ms;
    if (l_base <= 0.0 || c->c_budget <= 0.0)
        throw Error(SAIR_EINVAL, "reward: normalizers must be positive");
    return RewardCfg{c->t_sla_ms, l_base, c->c_budget, c->w_latency, c->w_cost, c->w_proactive,
                     c->r_max};
}

void compute_reward_batch(const sair_reward_inputs* in, const int32_t* deltas, size_t S, size_t T,
                          sair_frontier_s* f, const sair_reward_config* cfg,
                          sair_reward_breakdown* out) {
    RewardCfg rc = check_cfg(cfg);
    if (T == 0) return;
    DeviceGuard g(f->device);
    // one pinned staging buffer: inputs | deltas in, breakdowns out (a decision
    // step scores one row: one copy each way, no pageable staging)
    const size_t dbytes = T * S * 4 * 4;
    const size_t inb = T * 32 + ((dbytes + 255) & ~(size_t)255);
    char* base = static_cast<char*>(f->b_in.get(inb + T * 56 + 1024));
    char* hb = static_cast<char*>(f->h_io.get(inb + T * 56 + 1024));
    std::memcpy(hb, in, T * 32);
    if (dbytes) std::memcpy(hb + T * 32, deltas, dbytes);
    double* din = reinterpret_cast<double*>(base);
    int32_t* dd = reinterpret_cast<int32_t*>(base + T * 32);
    double* dout = reinterpret_cast<double*>(base + inb);
    SAIR_CUDA(cudaMemcpyAsync(base, hb, T * 32 + dbytes, cudaMemcpyHostToDevice, f->st));
    reward_kernel<<<grid_for(T), 256, 0, f->st>>>(din, dd, S, T, view(f), f->l_max, f->c_max, rc,
                                                  dout);
    SAIR_LAUNCH("reward_kernel");
    const double* h = reinterpret_cast<const double*>(hb + inb);
    SAIR_CUDA(cudaMemcpyAsync(hb + inb, dout, T * 56, cudaMemcpyDeviceToHost, f->st));
    SAIR_CUDA(cudaStreamSynchronize(f->st));
    for (size_t t = 0; t < T; ++t) {
        const double* o = h + 7 * t;
        out[t] = sair_reward_breakdown{o[0], o[1], o[2], o[3], o[4], o[5], o[6] != 0.0};
    }
}

void compute_reward_replay(const sair_reward_inputs* in, const int32_t* deltas, size_t S,
                           size_t T, const uint8_t* update, sair_frontier_s* f,
                           const sair_reward_config* cfg, sair_reward_breakdown* out) {
    RewardCfg rc = check_cfg(cfg);
    if (T == 0) return;
    DeviceGuard g(f->device);
    size_t nupd = 0;
    for (size_t t = 0; t < T; ++t) nupd += update[t] != 0;
    // replayers: >= 32 rounds each, <= 4096; frontier scratch of `cap` points
    size_t R = std::max<size_t>(1, std::min<size_t>(4096, T / 32));
    for (int attempt = 0; attempt < 2; ++attempt) {
        const size_t B = (T + R - 1) / R;
        R = (T + B - 1) / B;
        const size_t cap = R == 1 ? f->F + nupd + 1 : std::min<size_t>(f->F + nupd + 1, 1024);
        const size_t gcap = f->F + nupd + 1;
        const size_t dbytes = T * S * 16;
        const size_t bytes = T * 32 + dbytes + T + T * 56 + 4 * R * cap * 8 + 2 * R * 8 +
                             2 * gcap * 8 + 64 + 16 * 256;
        char* base = static_cast<char*>(f->b_in.get(bytes));
        size_t off = 0;
        auto take = [&](size_t n) {
            char* ptr = base + off;
            off += (n + 255) / 256 * 256;
            return ptr;
        };
        ReplayArgs a{};
        double* din = reinterpret_cast<double*>(take(T * 32));
        int32_t* dd = reinterpret_cast<int32_t*>(take(dbytes + 16));
        uint8_t* du = reinterpret_cast<uint8_t*>(take(T));
        a.in = din;
        a.deltas = dd;
        a.update = du;
        a.T = T;
        a.S = S;
        a.B = B;
        a.R = R;
        a.cap = cap;
        a.l_max = f->l_max;
        a.c_max = f->c_max;
        a.cfg = rc;
        a.out = reinterpret_cast<double*>(take(T * 56));
        a.fl = reinterpret_cast<double*>(take(R * cap * 8));
        a.fc = reinterpret_cast<double*>(take(R * cap * 8));
        a.sl = reinterpret_cast<double*>(take(R * cap * 8));
        a.sc = reinterpret_cast<double*>(take(R * cap * 8));
        a.fn = reinterpret_cast<size_t*>(take(R * 8));
        a.sn = reinterpret_cast<size_t*>(take(R * 8));
        a.gl = reinterpret_cast<double*>(take(gcap * 8));
        a.gc = reinterpret_cast<double*>(take(gcap * 8));
        a.gn = reinterpret_cast<size_t*>(take(8));
        a.overflow = reinterpret_cast<int*>(take(8));
        a.gcap = gcap;
        a.f0l = f->fl;
        a.f0c = f->fc;
        a.f0n = f->F;
        SAIR_CUDA(cudaMemcpyAsync(din, in, T * 32, cudaMemcpyHostToDevice, f->st));
        if (dbytes) SAIR_CUDA(cudaMemcpyAsync(dd, deltas, dbytes, cudaMemcpyHostToDevice, f->st));
        SAIR_CUDA(cudaMemcpyAsync(du, update, T, cudaMemcpyHostToDevice, f->st));
        SAIR_CUDA(cudaMemsetAsync(a.overflow, 0, 4, f->st));
        const int blocks = (int)((R + 127) / 128);
        replay_local_kernel<<<blocks, 128, 0, f->st>>>(a);
        replay_prefix_kernel<<<1, 32, 0, f->st>>>(a);
        replay_block_kernel<<<blocks, 128, 0, f->st>>>(a);
        SAIR_LAUNCH("replay kernels");
        int ovf = 0;
        size_t G = 0;
        SAIR_CUDA(cudaMemcpyAsync(&ovf, a.overflow, 4, cudaMemcpyDeviceToHost, f->st));
        SAIR_CUDA(cudaMemcpyAsync(&G, a.gn, 8, cudaMemcpyDeviceToHost, f->st));
        SAIR_CUDA(cudaStreamSynchronize(f->st));
        if (ovf) {  // a frontier outgrew its scratch: one replayer, full capacity
            R = 1;
            continue;
        }
        std::vector<double> h(7 * T);
        SAIR_CUDA(cudaMemcpyAsync(h.data(), a.out, T * 56, cudaMemcpyDeviceToHost, f->st));
        // the frontier after every flagged row (the prefix kernel's final state)
        reserve(f, std::max<size_t>(G, 1));
        if (G) {
            SAIR_CUDA(cudaMemcpyAsync(f->fl, a.gl, G * 8, cudaMemcpyDeviceToDevice, f->st));
            SAIR_CUDA(cudaMemcpyAsync(f->fc, a.gc, G * 8, cudaMemcpyDeviceToDevice, f->st));
        }
        SAIR_CUDA(cudaStreamSynchronize(f->st));
        f->F = G;
        sync_mirror(f);
        for (size_t t = 0; t < T; ++t) {
            const double* o = h.data() + 7 * t;
            out[t] = sair_reward_breakdown{o[0], o[1], o[2], o[3], o[4], o[5], o[6] != 0.0};
        }
        return;
    }
    throw Error(SAIR_EINVAL, "replay: frontier scratch overflow");
}

void frontier_set_init(sair_frontier_set_s* s, size_t P, double l_max, double c_max, int device) {
    if (l_max <= 0.0 || c_max <= 0.0)
        throw Error(SAIR_EINVAL, "ParetoFrontier: normalizers must be positive");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        throw Error(SAIR_ECUDA, "no CUDA device (libsair has no CPU fallback)");
    if (device < 0 || device >= ndev) throw Error(SAIR_EINVAL, "device ordinal out of range");
    s->device = device;
    s->P = P;
    s->l_max = l_max;
    s->c_max = c_max;
    DeviceGuard g(device);
    SAIR_CUDA(cudaStreamCreateWithFlags(&s->st, cudaStreamNonBlocking));
    s->cap = 16;
    SAIR_CUDA(cudaMalloc(&s->fl, std::max<size_t>(P, 1) * s->cap * 8));
    SAIR_CUDA(cudaMalloc(&s->fc, std::max<size_t>(P, 1) * s->cap * 8));
    SAIR_CUDA(cudaMalloc(&s->fn, std::max<size_t>(P, 1) * 8));
    SAIR_CUDA(cudaMalloc(&s->hv, std::max<size_t>(P, 1) * 8));
    SAIR_CUDA(cudaMemsetAsync(s->fn, 0, std::max<size_t>(P, 1) * 8, s->st));
    SAIR_CUDA(cudaMemsetAsync(s->hv, 0, std::max<size_t>(P, 1) * 8, s->st));
    SAIR_CUDA(cudaStreamSynchronize(s->st));
}

void frontier_set_free(sair_frontier_set_s* s) {
    DeviceGuard g(s->device);
    if (s->st) cudaStreamSynchronize(s->st);
    cudaFree(s->fl);
    cudaFree(s->fc);
    cudaFree(s->fn);
    cudaFree(s->hv);
    s->b_in.release();
    if (s->st) cudaStreamDestroy(s->st);
    s->st = nullptr;
}

// grow every frontier's capacity (strided copy: [P][cap] -> [P][ncap])
static void set_grow(sair_frontier_set_s* s, size_t ncap) {
    double *l, *c;
    SAIR_CUDA(cudaMalloc(&l, s->P * ncap * 8));
    SAIR_CUDA(cudaMalloc(&c, s->P * ncap * 8));
    SAIR_CUDA(cudaMemcpy2DAsync(l, ncap * 8, s->fl, s->cap * 8, s->cap * 8, s->P,
                                cudaMemcpyDeviceToDevice, s->st));
    SAIR_CUDA(cudaMemcpy2DAsync(c, ncap * 8, s->fc, s->cap * 8, s->cap * 8, s->P,
                                cudaMemcpyDeviceToDevice, s->st));
    SAIR_CUDA(cudaStreamSynchronize(s->st));
    cudaFree(s->fl);
    cudaFree(s->fc);
    s->fl = l;
    s->fc = c;
    s->cap = ncap;
}

void frontier_set_step(sair_frontier_set_s* s, const sair_reward_inputs* in, const int32_t* deltas,
                       size_t S, const uint8_t* update, const sair_reward_config* cfg,
                       sair_reward_breakdown* out) {
    RewardCfg rc = check_cfg(cfg);
    const size_t P = s->P;
    if (P == 0) return;
    DeviceGuard g(s->device);
    if (s->maxf + 1 > s->cap) set_grow(s, std::max(2 * s->cap, s->maxf + 1));
    const size_t dbytes = P * S * 16;
    char* base = static_cast<char*>(s->b_in.get(P * 32 + dbytes + P + P * 56 + 64 + 5 * 256));
    size_t off = 0;
    auto take = [&](size_t n) {
        char* ptr = base + off;
        off += (n + 255) / 256 * 256;
        return ptr;
    };
    SetArgs a{};
    double* din = reinterpret_cast<double*>(take(P * 32));
    int32_t* dd = reinterpret_cast<int32_t*>(take(dbytes + 16));
    uint8_t* du = reinterpret_cast<uint8_t*>(take(P));
    a.out = reinterpret_cast<double*>(take(P * 56));
    a.maxf = reinterpret_cast<unsigned long long*>(take(16));
    a.overflow = reinterpret_cast<int*>(a.maxf + 1);
    a.in = din;
    a.deltas = dd;
    a.update = du;
    a.P = P;
    a.S = S;
    a.cap = s->cap;
    a.l_max = s->l_max;
    a.c_max = s->c_max;
    a.cfg = rc;
    a.fl = s->fl;
    a.fc = s->fc;
    a.fn = s->fn;
    a.hv = s->hv;
    SAIR_CUDA(cudaMemcpyAsync(din, in, P * 32, cudaMemcpyHostToDevice, s->st));
    if (dbytes) SAIR_CUDA(cudaMemcpyAsync(dd, deltas, dbytes, cudaMemcpyHostToDevice, s->st));
    SAIR_CUDA(cudaMemcpyAsync(du, update, P, cudaMemcpyHostToDevice, s->st));
    SAIR_CUDA(cudaMemsetAsync(a.maxf, 0, 16, s->st));
    frontier_set_step_kernel<<<grid_for(P, 128), 128, 0, s->st>>>(a);
    SAIR_LAUNCH("frontier_set_step_kernel");
    std::vector<double> h(7 * P);
    unsigned long long mf[2] = {0, 0};
    SAIR_CUDA(cudaMemcpyAsync(h.data(), a.out, P * 56, cudaMemcpyDeviceToHost, s->st));
    SAIR_CUDA(cudaMemcpyAsync(mf, a.maxf, 16, cudaMemcpyDeviceToHost, s->st));
    SAIR_CUDA(cudaStreamSynchronize(s->st));
    // capacity was ensured up front (>= max F + 1), so an insert never overflows
    if (mf[1] & 0xFFFFFFFFull) throw Error(SAIR_ECUDA, "frontier set: capacity overflow");
    s->maxf = (size_t)mf[0];
    for (size_t p = 0; p < P; ++p) {
        const double* o = h.data() + 7 * p;
        out[p] = sair_reward_breakdown{o[0], o[1], o[2], o[3], o[4], o[5], o[6] != 0.0};
    }
}

size_t frontier_set_points(sair_frontier_set_s* s, size_t p, double* l, double* c, size_t cap,
                           double* hv) {
    if (p >= s->P) throw Error(SAIR_ERANGE, "frontier set: pipeline index out of range");
    DeviceGuard g(s->device);
    size_t F = 0;
    SAIR_CUDA(cudaMemcpyAsync(&F, s->fn + p, 8, cudaMemcpyDeviceToHost, s->st));
    if (hv) SAIR_CUDA(cudaMemcpyAsync(hv, s->hv + p, 8, cudaMemcpyDeviceToHost, s->st));
    SAIR_CUDA(cudaStreamSynchronize(s->st));
    const size_t k = std::min(F, cap);
    if (k && l) SAIR_CUDA(cudaMemcpy(l, s->fl + p * s->cap, k * 8, cudaMemcpyDeviceToHost));
    if (k && c) SAIR_CUDA(cudaMemcpy(c, s->fc + p * s->cap, k * 8, cudaMemcpyDeviceToHost));
    return F;
}

// ---------------------------------------------------------- decision step --
struct DecisionTail {
    const double* in;      // [4] RewardInputs | deltas [S][4] int32 | x [d]
    const int32_t* deltas;
    const double* x;
    size_t S;
    double* fl;            // the frontier (device), F0 points, capacity >= F0 + 1
    double* fc;
    size_t F0;
    double hv, l_max, c_max;
    RewardCfg rc;
    int update;
    double pl, pc;         // the outcome, normalized (host normalize(), pareto.cpp:20-29)
    double* ol;            // [F0 + 1] insert scratch
    double* oc;
    // the store row
    double r_min;
    int32_t round;
    size_t rec;
    int d, dp;
    float* pages;
    float* r32;
    double* r64;
    int32_t* rnd;
    double* x64;
    const double* shift;
    double* out;           // [7] breakdown | [2] insert result | hv | pad | fl [F0+1] | fc [F0+1]
};

// The decision's reward side, one CTA on the frontier's stream (it does not
// depend on the select, so it runs beside it): compute_reward against the
// frontier before the update (reward.cpp:21-44), insert_normalized
// (pareto.cpp:43-54) and its commit, hypervolume() (pareto.cpp:56-65).
__global__ void __launch_bounds__(1024) decision_reward_kernel(const DecisionTail a) {
    __shared__ double srw[7];
    __shared__ unsigned long long sres[2];
    const int tid = threadIdx.x;
    if (tid == 0) {
        double pl, pc;
        reward_row(a.in, a.deltas, a.S, FrontierView{a.fl, a.fc, a.F0, a.hv}, a.l_max, a.c_max,
                   a.rc, srw, &pl, &pc);
        sres[0] = 0;
        sres[1] = a.F0;
    }
    __syncthreads();
    if (tid < 7) a.out[tid] = srw[tid];
    if (a.update) {
        insert_one_block(a.fl, a.fc, a.F0, a.pl, a.pc, a.ol, a.oc, sres);
        __syncthreads();
        const size_t F = (size_t)sres[1];
        if (sres[0])
            for (size_t i = tid; i < F; i += blockDim.x) {
                a.fl[i] = a.ol[i];
                a.fc[i] = a.oc[i];
            }
        __syncthreads();
        double* ml = a.out + 10;
        double* mc = ml + a.F0 + 1;
        for (size_t i = tid; i < F; i += blockDim.x) {
            ml[i] = a.fl[i];
            mc[i] = a.fc[i];
        }
        if (tid == 0) {
            double hv = 0.0;
            for (size_t i = 0; i < F; ++i) {
                double nl = i + 1 < F ? a.fl[i + 1] : 1.0;
                hv = dadd(hv, dmul(dsub(nl, a.fl[i]), dsub(1.0, a.fc[i])));
            }
            a.out[9] = hv;
            reinterpret_cast<unsigned long long*>(a.out)[7] = sres[0];
            reinterpret_cast<unsigned long long*>(a.out)[8] = sres[1];
        }
    }
}

// The store() row behind the r_min gate on the reward total (experience.cpp:
// 45-48), on the store's stream after the select (which must not see it).
__global__ void __launch_bounds__(128) decision_append_kernel(const DecisionTail a) {
    const int tid = threadIdx.x;
    const double r = a.out[5];
    if (!(r > a.r_min)) return;
    const int w = a.d > a.dp ? a.d : a.dp;  // x64 takes all d columns, the page dp
    for (int k = tid; k < w; k += blockDim.x) {
        const double v = k < a.d ? a.x[k] : 0.0;
        if (k < a.dp) a.pages[page_index(a.rec, k, a.dp)] = k < a.d ? to_tf32(v - a.shift[k]) : 0.f;
        if (k < a.d) a.x64[a.rec * a.d + k] = v;
    }
    if (tid == 0) {
        a.r64[a.rec] = r;
        a.r32[a.rec] = (float)r;
        a.rnd[a.rec] = a.round;
    }
}

// One decision of the reference's loop (harness.cpp:197-261), replayed with the
// step's outcome known: select(x) + veto scan
// (:205, policy.cpp:140-157), compute_reward against the pre-update frontier
// (:250), update (:251), store() (:253-261) -- enqueued on the store's stream
// back to back with one host synchronisation; results identical to the four
// calls in that order.  A store that is empty or of another dimension (store()
// would fix or reject the dimension) takes the four calls.
void decision_step(sair_store_s* s, sair_frontier_s* f, const double* x, int dim,
                   const sair_select_config& cfg, const sair_reward_inputs* in,
                   const int32_t* deltas, size_t S, const sair_reward_config* rcfg, bool update,
                   double pl, double pc, int32_t round, int64_t* o_idx, double* o_sim,
                   double* o_score, size_t* o_count, int64_t* o_nn, double* o_nn_sim,
                   sair_reward_breakdown* o_rw, int* o_inserted, int* o_stored) {
    const RewardCfg rc = check_cfg(rcfg);
    if (s->device != f->device)
        throw Error(SAIR_EINVAL, "decision step: store and frontier on different devices");
    if (s->n == 0 || dim != s->d) {
        store_select(s, x, 1, dim, cfg, o_idx, o_sim, o_score, o_count, o_nn, o_nn_sim, nullptr,
                     nullptr);
        compute_reward_batch(in, deltas, S, 1, f, rcfg, o_rw);
        *o_inserted = update ? frontier_insert_one(f, pl, pc) : 0;
        uint8_t acc = 0;
        store_append(s, x, 1, dim, &o_rw->total, &round, &acc);
        *o_stored = acc;
        return;
    }
    static const bool trace = std::getenv("SAIR_TRACE_DECISION") != nullptr;
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    DeviceGuard g(s->device);
    SAIR_CUDA(cudaStreamSynchronize(f->st));
    // capacity first: a reallocation synchronises, and must not move arrays
    // under work already enqueued
    store_reserve(s, s->n + 1);
    if (update) reserve(f, f->F + 1);
    const size_t F0 = f->F;
    // the reward side first, on the frontier's stream: one input copy, one
    // kernel -- it overlaps the select
    const int d = s->d;
    const size_t dbytes = S * 4 * 4;
    const size_t xo = (32 + dbytes + 7) & ~(size_t)7;
    const size_t inb = xo + (size_t)d * 8;
    const size_t outn = 10 + 2 * (F0 + 1);
    char* dbase = static_cast<char*>(f->b_in.get(((inb + 255) & ~(size_t)255) + outn * 8 + 64));
    char* hb = static_cast<char*>(f->h_io.get(((inb + 255) & ~(size_t)255) + outn * 8 + 64));
    std::memcpy(hb, in, 32);
    if (dbytes) std::memcpy(hb + 32, deltas, dbytes);
    std::memcpy(hb + xo, x, (size_t)d * 8);
    double* dout = reinterpret_cast<double*>(dbase + ((inb + 255) & ~(size_t)255));
    double* hout = reinterpret_cast<double*>(hb + ((inb + 255) & ~(size_t)255));
    SAIR_CUDA(cudaMemcpyAsync(dbase, hb, inb, cudaMemcpyHostToDevice, f->st));
    DecisionTail t{};
    t.in = reinterpret_cast<const double*>(dbase);
    t.deltas = reinterpret_cast<const int32_t*>(dbase + 32);
    t.x = reinterpret_cast<const double*>(dbase + xo);
    t.S = S;
    t.fl = f->fl;
    t.fc = f->fc;
    t.F0 = F0;
    t.hv = f->hv;
    t.l_max = f->l_max;
    t.c_max = f->c_max;
    t.rc = rc;
    t.update = update ? 1 : 0;
    t.pl = pl;
    t.pc = pc;
    double* ol = update ? f->b_out.as<double>(2 * (F0 + 1) + 4) : nullptr;
    t.ol = ol;
    t.oc = ol ? ol + (F0 + 1) : nullptr;
    t.r_min = s->r_min;
    t.round = round;
    t.rec = s->n;
    t.d = d;
    t.dp = s->dp;
    t.pages = s->pages;
    t.r32 = s->r32;
    t.r64 = s->r64;
    t.rnd = s->rnd;
    t.x64 = s->x64;
    t.shift = s->d_shift;
    t.out = dout;
    decision_reward_kernel<<<1, 1024, 0, f->st>>>(t);
    SAIR_LAUNCH("decision_reward_kernel");
    if (!f->ev_tail) SAIR_CUDA(cudaEventCreateWithFlags(&f->ev_tail, cudaEventDisableTiming));
    SAIR_CUDA(cudaEventRecord(f->ev_tail, f->st));
    s->defer_sync = true;
    try {
        store_select(s, x, 1, dim, cfg, o_idx, o_sim, o_score, o_count, o_nn, o_nn_sim, nullptr,
                     nullptr);
    } catch (...) {
        s->defer_sync = false;
        s->pending = nullptr;
        SAIR_CUDA(cudaStreamSynchronize(f->st));
        throw;
    }
    s->defer_sync = false;
    const auto t1 = clk::now();
    cudaStream_t st = s->st;
    // then, after the select on the store's stream: the new row
    SAIR_CUDA(cudaStreamWaitEvent(st, f->ev_tail, 0));
    decision_append_kernel<<<1, 128, 0, st>>>(t);
    SAIR_LAUNCH("decision_append_kernel");
    SAIR_CUDA(cudaMemcpyAsync(hout, dout, (update ? outn : 7) * 8, cudaMemcpyDeviceToHost, st));
    const auto t2 = clk::now();
    SAIR_CUDA(cudaStreamSynchronize(st));
    const auto t3 = clk::now();
    if (s->pending) {  // the select's outputs
        auto unpack = std::move(s->pending);
        s->pending = nullptr;
        unpack();
        float tot = 0.f;
        cudaEventElapsedTime(&tot, s->ev[0], s->ev[3]);
        s->last.total_ms = tot;
    }
    const double* h_rw = hout;
    *o_rw = sair_reward_breakdown{h_rw[0], h_rw[1], h_rw[2], h_rw[3], h_rw[4], h_rw[5],
                                  h_rw[6] != 0.0};
    *o_inserted = 0;
    if (update) {
        unsigned long long res[2];
        std::memcpy(res, hout + 7, 16);
        if (res[0]) {
            f->F = (size_t)res[1];
            f->hl.assign(hout + 10, hout + 10 + f->F);
            f->hc.assign(hout + 10 + F0 + 1, hout + 10 + F0 + 1 + f->F);
            f->hv = hout[9];
            *o_inserted = 1;
        }
    }
    *o_stored = store_append_one_commit(s, x, h_rw[5]);
    if (trace) {
        auto us = [](clk::duration d) { return std::chrono::duration<double, std::micro>(d).count(); };
        fprintf(stderr, "[decision] select enqueue %.1f  rest enqueue %.1f  sync wait %.1f  after %.1f us\n",
                us(t1 - t0), us(t2 - t1), us(t3 - t2), us(clk::now() - t3));
    }
}

double action_magnitude(const int32_t* deltas, size_t S, int device) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        throw Error(SAIR_ECUDA, "no CUDA device (libsair has no CPU fallback)");
    DeviceGuard g(device);
    DBuf b;
    char* base = static_cast<char*>(b.get(S * 16 + 256));
    double* dout = reinterpret_cast<double*>(base);
    int32_t* dd = reinterpret_cast<int32_t*>(base + 64);
    if (S) SAIR_CUDA(cudaMemcpy(dd, deltas, S * 16, cudaMemcpyHostToDevice));
    action_mu_kernel<<<1, 32>>>(dd, S, dout);
    SAIR_LAUNCH("action_mu_kernel");
    double v = 0.0;
    SAIR_CUDA(cudaMemcpy(&v, dout, 8, cudaMemcpyDeviceToHost));
    return v;
}

}  // namespace sair
