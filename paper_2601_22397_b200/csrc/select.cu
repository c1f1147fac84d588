// select.cu -- surprisal-guided retrieval on the device (the fast path).
//
// Restates ExperienceBuffer::select (experience.cpp:151-205) and the
// MockBackend veto scan (policy.cpp:140-157) as three kernels per group of up
// to 8 queries:
//
//   K3 stream_kernel  one HBM pass over the fp32 page copy of the store.  A
//                     persistent CTA per SM walks chunks of 2 pages (256
//                     records); an elected thread keeps a 3-deep ring of
//                     cp.async.bulk copies (TMA bulk engine, mbarrier
//                     complete_tx) in flight.  Each thread owns one record:
//                     y_k = x_k / sd_k once, then ||y - c_q||^2 by the norm
//                     expansion P + C_q - 2 <y, c_q> -- one FFMA per
//                     (query, dimension) with c_q in the constant bank.  The
//                     record's upper-bound log2 surprisal score is thresholded
//                     into per-CTA candidate lists (warp-aggregated inserts; a
//                     warp-level radix select compacts a list to its K' best
//                     and raises the threshold).  Records never leave the chip.
//   merge_kernel      global top-K' per list across CTAs (block radix select on
//                     (key, index), bitonic sort of the survivors).
//   refine_kernel     fp64 re-score of the K' candidates with the reference's
//                     exact rounding sequence, the greedy max-marginal-gain
//                     loop (rank-selection when lambda == 0), certification
//                     against the filter's bound, the curriculum order and the
//                     veto scan's nearest record.
// Queries that cannot be certified are answered by the full fp64 pass
// (select_exact.cu).  The exactness argument is DESIGN.md "Exactness".
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cfloat>
#include <cstring>
#include <vector>

#include "select_common.cuh"
#include "topk_select.cuh"
#include "warp_topk.cuh"

namespace sair {

// ------------------------------------------------------------ PTX helpers --

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
// TMA bulk engine: global -> shared, completion counted on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra LAB_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// ------------------------------------------------------------ K3 stream --
//
// Warp-specialised persistent kernel, one CTA per SM:
//   warp 8 (producer)   one elected lane streams the CTA's rounds through an
//                       NST-deep ring of shared-memory stages with the TMA
//                       bulk engine; a stage is the same DH-dimension slice of
//                       4 consecutive pages (512 records, 64 KB at DH = 32);
//                       `full` mbarriers complete on the byte count, `empty`
//                       mbarriers collect one arrival per consumer warp.
//   warps 0-7 (consumers) two adjacent records per thread (one LDS.64 per
//                       dimension), y = x / sd once, P = |y|^2 and
//                       D_q = <y, -2 c_q> with the query constants broadcast
//                       from shared memory (LDS.128), then the per-record keys
//                       and the threshold inserts.  Consumers synchronise
//                       among themselves only at round ends (named barrier 1).
constexpr int CONS_WARPS = 8;
constexpr int CONS_THREADS = CONS_WARPS * 32;
constexpr int STREAM_THREADS = CONS_THREADS + 32;
constexpr int ROUND_PAGES = 4;  // 512 records per round: 2 per consumer thread

template <int DP, int QB>
struct StreamArgs {
    const float* pages;  // [npages][DP][PAGE] fp32 (x - shift)
    const float* r32;
    uint32_t n, npages;
    float c1, c0, rdelta, alpha;  // resid32 = |r c1 - c0|; key = log2(resid32 + rdelta) - d2 alpha
    int kp, knn, nst, cap_sel, cap_nn, kmax;
    float* out_key;  // [grid][2*QB][kmax]
    uint32_t* out_idx;
    unsigned int* pmax;  // max over records of P = |y|^2 (float bits; E_q bound)
    float s[DP];         // 1 / sd (0 on padding)
    float cc[QB];        // sum_k c_qk^2
    float c2[DP][QB];    // -2 c_qk, c_qk = (mean - shift) / sd + z_qk (0 on padding)
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void consumer_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(CONS_THREADS) : "memory");
}

template <int QB>
__device__ __forceinline__ void load_consts(const float* c, float (&v)[QB]) {
    if constexpr (QB % 4 == 0) {
#pragma unroll
        for (int q = 0; q < QB; q += 4) {
            const float4 t = *reinterpret_cast<const float4*>(c + q);
            v[q] = t.x;
            v[q + 1] = t.y;
            v[q + 2] = t.z;
            v[q + 3] = t.w;
        }
    } else if constexpr (QB == 2) {
        const float2 t = *reinterpret_cast<const float2*>(c);
        v[0] = t.x;
        v[1] = t.y;
    } else {
        v[0] = c[0];
    }
}

template <int DP, int QB>
__global__ void __launch_bounds__(STREAM_THREADS, 1)
    stream_kernel(const __grid_constant__ StreamArgs<DP, QB> a) {
    constexpr int DH = DP < 16 ? DP : 16;  // dimensions per stage
    constexpr int NH = DP / DH;            // stages per round
    constexpr int STAGE_FLOATS = ROUND_PAGES * DH * PAGE;
    extern __shared__ __align__(128) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nl = a.knn ? 2 * QB : QB;
    float* stage = reinterpret_cast<float*>(smem);
    float* cs = stage + (size_t)a.nst * STAGE_FLOATS;  // [DP][QB]
    float* ss = cs + DP * QB;                           // [DP]
    uint64_t* full = reinterpret_cast<uint64_t*>(ss + DP);
    uint64_t* empty = full + 8;
    // (8 slots each: nst goes up to 8 -- racecheck caught empty[4..7] overlapping thr)
    float* thr = reinterpret_cast<float*>(empty + 8);
    int* cnt = reinterpret_cast<int*>(thr + 2 * QB);
    uint32_t* hist = reinterpret_cast<uint32_t*>(cnt + 2 * QB);
    float* lkey = reinterpret_cast<float*>(hist + CONS_WARPS * 256);
    const int total_cap = QB * a.cap_sel + (a.knn ? QB * a.cap_nn : 0);
    uint32_t* lidx = reinterpret_cast<uint32_t*>(lkey + total_cap);
    auto lbase = [&](int L) { return L < QB ? L * a.cap_sel : QB * a.cap_sel + (L - QB) * a.cap_nn; };
    auto lcap = [&](int L) { return L < QB ? a.cap_sel : a.cap_nn; };
    auto lk = [&](int L) { return L < QB ? a.kp : a.knn; };

    for (int i = tid; i < DP * QB; i += STREAM_THREADS) cs[i] = (&a.c2[0][0])[i];
    for (int i = tid; i < DP; i += STREAM_THREADS) ss[i] = a.s[i];
    if (tid < 2 * QB) {
        thr[tid] = -FLT_MAX;
        cnt[tid] = 0;
    }
    if (tid == 0) {
        for (int s = 0; s < a.nst; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CONS_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const uint32_t nrounds = (a.npages + ROUND_PAGES - 1) / ROUND_PAGES;
    const uint32_t G = gridDim.x, r0 = blockIdx.x;
    const uint32_t mine = r0 < nrounds ? (nrounds - 1 - r0) / G + 1 : 0;

    if (warp == CONS_WARPS) {
        // ---------------- producer ----------------
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (uint32_t it = 0; it < mine; ++it) {
                const uint32_t p0 = (r0 + it * G) * ROUND_PAGES;
                const uint32_t np = min((uint32_t)ROUND_PAGES, a.npages - p0);
                for (int h = 0; h < NH; ++h) {
                    if (it * NH + h >= (uint32_t)a.nst) mbar_wait(&empty[s], ph ^ 1u);
                    mbar_expect_tx(&full[s], np * DH * PAGE * 4);
                    for (uint32_t p = 0; p < np; ++p)
                        for (int b = 0; b < 4; ++b)  // rows h*DH.. of each 32-record block
                            bulk_g2s(stage + (size_t)s * STAGE_FLOATS + p * DH * PAGE + b * DH * 32,
                                     a.pages + (size_t)(p0 + p) * DP * PAGE + b * DP * 32 + h * DH * 32,
                                     DH * 32 * 4, &full[s]);
                    if (++s == a.nst) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
            }
        }
        return;
    }

    // ---------------- consumers ----------------
    const int pg = tid >> 6;          // page within the round
    const int slot = (tid & 63) * 2;  // two adjacent records
    float thr_r[2 * QB];
#pragma unroll
    for (int L = 0; L < 2 * QB; ++L) thr_r[L] = -FLT_MAX;
    float pmax = 0.f;
    int s = 0;
    uint32_t ph = 0;

    auto insert = [&](const float (&key)[2 * QB], uint32_t pm, uint32_t rec) {
        if (!__any_sync(0xffffffffu, pm)) return;
#pragma unroll
        for (int L = 0; L < 2 * QB; ++L) {
            const bool pass = (pm >> L) & 1u;
            const unsigned bal = __ballot_sync(0xffffffffu, pass);
            if (bal) {
                const int leader = __ffs(bal) - 1;
                int base = 0;
                if (lane == leader) base = atomicAdd(&cnt[L], __popc(bal));
                base = __shfl_sync(0xffffffffu, base, leader);
                if (pass) {
                    const int pos = lbase(L) + base + __popc(bal & ((1u << lane) - 1u));
                    lkey[pos] = key[L];
                    lidx[pos] = rec;
                }
            }
        }
    };
    auto maybe_compact = [&]() {
        consumer_sync();
        bool need = false;
        for (int L = 0; L < nl; ++L) need |= cnt[L] > lcap(L) - 2 * CONS_THREADS;
        // every consumer has read the counts before any compaction rewrites
        // one (racecheck: a warp could otherwise see a rewritten count and
        // skip the barriers below while the others take them)
        consumer_sync();
        if (need) {
            for (int L = warp; L < nl; L += CONS_WARPS) {
                if (cnt[L] > lcap(L) - 2 * CONS_THREADS) {
                    const uint32_t T = warp_keep_topk(lkey + lbase(L), lidx + lbase(L), cnt[L],
                                                      lk(L), hist + warp * 256, lane);
                    if (lane == 0) {
                        cnt[L] = lk(L);
                        thr[L] = ord2f(T);
                    }
                }
            }
            consumer_sync();
#pragma unroll
            for (int L = 0; L < 2 * QB; ++L) thr_r[L] = thr[L];
        }
    };

    for (uint32_t it = 0; it < mine; ++it) {
        const uint32_t rec = ((r0 + it * G) * ROUND_PAGES + pg) * PAGE + slot;
        const bool v0 = rec < a.n, v1 = rec + 1 < a.n;
        const float rw0 = v0 ? __ldg(a.r32 + rec) : 0.f;
        const float rw1 = v1 ? __ldg(a.r32 + rec + 1) : 0.f;
        float P0 = 0.f, P1 = 0.f, D0[QB], D1[QB];
#pragma unroll
        for (int q = 0; q < QB; ++q) D0[q] = D1[q] = 0.f;
#pragma unroll 1
        for (int h = 0; h < NH; ++h) {
            mbar_wait(&full[s], ph);
            // pre-swizzled block rows (page_index): records t, t+1 share a chunk
            const float* xp = stage + (size_t)s * STAGE_FLOATS + pg * DH * PAGE + (slot >> 5) * DH * 32;
            const int t8 = (slot & 31) >> 3, t7 = slot & 7;
            const float* ch = cs + h * DH * QB;
            const float* sh = ss + h * DH;
#pragma unroll
            for (int k = 0; k < DH; ++k) {
                const float2 x = *reinterpret_cast<const float2*>(
                    xp + k * 32 + (((t8 ^ (k & 3)) << 3) | t7));
                float c[QB];
                load_consts<QB>(ch + k * QB, c);
                const float sk = sh[k];
                const float y0 = __fmul_rn(x.x, sk);  // not contracted
                const float y1 = __fmul_rn(x.y, sk);
                P0 = fmaf(y0, y0, P0);
                P1 = fmaf(y1, y1, P1);
#pragma unroll
                for (int q = 0; q < QB; ++q) {
                    D0[q] = fmaf(y0, c[q], D0[q]);
                    D1[q] = fmaf(y1, c[q], D1[q]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == a.nst) {
                s = 0;
                ph ^= 1u;
            }
        }
        if (v0) pmax = fmaxf(pmax, P0);
        if (v1) pmax = fmaxf(pmax, P1);
        const float lg0 = log2f(fabsf(fmaf(rw0, a.c1, -a.c0)) + a.rdelta);
        const float lg1 = log2f(fabsf(fmaf(rw1, a.c1, -a.c0)) + a.rdelta);
        float k0[2 * QB], k1[2 * QB];
        uint32_t pm0 = 0, pm1 = 0;
#pragma unroll
        for (int q = 0; q < QB; ++q) {
            const float d0 = (P0 + a.cc[q]) + D0[q];
            const float d1 = (P1 + a.cc[q]) + D1[q];
            k0[q] = fmaf(-d0, a.alpha, lg0);
            k1[q] = fmaf(-d1, a.alpha, lg1);
            k0[QB + q] = -d0;
            k1[QB + q] = -d1;
            pm0 |= (k0[q] > thr_r[q] ? 1u : 0u) << q;
            pm1 |= (k1[q] > thr_r[q] ? 1u : 0u) << q;
            pm0 |= (k0[QB + q] > thr_r[QB + q] ? 1u : 0u) << (QB + q);
            pm1 |= (k1[QB + q] > thr_r[QB + q] ? 1u : 0u) << (QB + q);
        }
        const uint32_t lmask = a.knn ? 0xFFFFFFFFu : ((1u << QB) - 1u);
        insert(k0, v0 ? pm0 & lmask : 0u, rec);
        insert(k1, v1 ? pm1 & lmask : 0u, rec + 1);
        maybe_compact();
    }
    for (int L = warp; L < nl; L += CONS_WARPS) {
        if (cnt[L] > lk(L)) {
            warp_keep_topk(lkey + lbase(L), lidx + lbase(L), cnt[L], lk(L), hist + warp * 256,
                           lane);
            if (lane == 0) cnt[L] = lk(L);
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) pmax = fmaxf(pmax, __shfl_xor_sync(0xffffffffu, pmax, o));
    if (lane == 0) atomicMax(a.pmax, __float_as_uint(pmax));
    consumer_sync();
    for (int L = 0; L < nl; ++L) {
        const size_t row = ((size_t)blockIdx.x * 2 * QB + L) * a.kmax;
        for (int j = tid; j < lk(L); j += CONS_THREADS) {
            const bool have = j < cnt[L];
            a.out_key[row + j] = have ? lkey[lbase(L) + j] : -INFINITY;
            // padding indices are unique and >= n (n < 2^31), so merged
            // composites stay unique; the refine kernel skips idx >= n
            a.out_idx[row + j] = have ? lidx[lbase(L) + j] : 0xFFFFFFFFu - (uint32_t)(row + j);
        }
    }
}

// ------------------------------------------------------------ merge --------


// Global top-K (key desc, idx asc) of list L across all CTAs, sorted, plus the
// K-th key (the filter threshold U of every record outside the pool).  Padding
// entries (key -inf) are skipped; histogram updates are warp-aggregated
// because the keys of one list share their leading digits.
__global__ void __launch_bounds__(1024)
    merge_kernel(const float* __restrict__ in_key, const uint32_t* __restrict__ in_idx, int G,
                 int lists_stride, int kmax, int kout, int QB, int kp, int knn, float* __restrict__ out_key,
                 uint32_t* __restrict__ out_idx, float* __restrict__ out_thr, size_t in_g,
                 size_t out_g) {
    // blockIdx.y: a query group (in_g / out_g: its input / output strides)
    in_key += blockIdx.y * in_g;
    in_idx += blockIdx.y * in_g;
    out_key += blockIdx.y * out_g;
    out_idx += blockIdx.y * out_g;
    out_thr += blockIdx.y * (size_t)lists_stride;
    const int L = blockIdx.x;
    const int K = L < QB ? kp : knn;
    const int total = G * K;
    __shared__ uint32_t hist[256];
    __shared__ uint32_t sh_bin, sh_r, sh_pop, sh_cnt, sh_valid;
    constexpr int FAST = 2048;  // >= kp, knn (<= 512)
    __shared__ unsigned long long skey[FAST];
    const int tid = threadIdx.x, lane = tid & 31;
    auto comp = [&](int e) {
        const int g = e / K, j = e - g * K;
        const size_t off = ((size_t)g * lists_stride + L) * kmax + j;
        return ((unsigned long long)f2ord(in_key[off]) << 32) | (unsigned long long)(~in_idx[off]);
    };
    if (tid == 0) {
        sh_cnt = 0;
        sh_valid = 0;
    }
    __syncthreads();
    // Fast path: the CTAs' lists are mostly padding (a pass's start threshold
    // admits a few K' records per query over the whole store) and every
    // producer writes a list's valid entries first: one thread per CTA list
    // reads up to its first padding entry, the valid ones are gathered into
    // shared memory and sorted there when they fit.
    for (int g = tid; g < G; g += blockDim.x) {
        for (int j = 0; j < K; ++j) {
            const unsigned long long u = comp(g * K + j);
            if ((u >> 32) <= PAD_TOP) break;
            const uint32_t p = atomicAdd(&sh_valid, 1u);
            if (p < (uint32_t)FAST) skey[p] = u;
        }
    }
    __syncthreads();
    const uint32_t nvf = sh_valid;
    int P = 1;
    while (P < K) P <<= 1;
    if (nvf <= (uint32_t)FAST) {
        while (P < (int)nvf) P <<= 1;
        for (int j = (int)nvf + tid; j < P; j += blockDim.x)
            skey[j] = j < K ? ((PAD_TOP << 32) | (unsigned long long)(uint32_t)j) : 0ull;
        __syncthreads();
    } else {
    __syncthreads();  // (every thread has read nvf before the counter is reused)
    if (tid == 0) sh_valid = 0;
    __syncthreads();
    unsigned long long prefix = 0, pmask = 0;
    uint32_t r = (uint32_t)K;
    bool all_valid = false;
    for (int shift = 56; shift >= 0; shift -= 8) {
        for (int b = tid; b < 256; b += blockDim.x) hist[b] = 0;
        __syncthreads();
        uint32_t nvalid = 0;
        for (int e0 = tid - lane; e0 < total; e0 += blockDim.x) {
            const int e = e0 + lane;
            uint32_t bin = 256;
            if (e < total) {
                const unsigned long long u = comp(e);
                if ((u >> 32) > PAD_TOP && (u & pmask) == prefix) bin = (uint32_t)(u >> shift) & 255u;
            }
            const unsigned peers = __match_any_sync(0xffffffffu, bin);
            if (bin < 256 && lane == __ffs(peers) - 1) atomicAdd(&hist[bin], __popc(peers));
            nvalid += bin < 256;
        }
        if (shift == 56) {
            for (int o = 16; o; o >>= 1) nvalid += __shfl_xor_sync(0xffffffffu, nvalid, o);
            if (lane == 0 && nvalid) atomicAdd(&sh_valid, nvalid);
        }
        __syncthreads();
        if (shift == 56 && sh_valid <= (uint32_t)K) {  // every valid entry is kept
            all_valid = true;
            break;
        }
        if (tid < 32) {
            uint32_t loc[8], sum = 0;
            for (int j = 0; j < 8; ++j) {
                loc[j] = hist[255 - (lane * 8 + j)];
                sum += loc[j];
            }
            uint32_t incl = sum;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            const uint32_t excl = incl - sum;
            const unsigned own = __ballot_sync(0xffffffffu, excl < r && r <= incl);
            if (lane == __ffs(own) - 1) {
                uint32_t c = excl;
                for (int j = 0; j < 8; ++j) {
                    if (c + loc[j] >= r) {
                        sh_bin = 255 - (lane * 8 + j);
                        sh_r = r - c;
                        sh_pop = loc[j];
                        break;
                    }
                    c += loc[j];
                }
            }
        }
        __syncthreads();
        prefix |= (unsigned long long)sh_bin << shift;
        pmask |= 255ull << shift;
        r = sh_r;
        const bool done = sh_pop == r;  // the whole bin is kept: lower digits do not matter
        __syncthreads();
        if (done) {
            pmask = ~((1ull << shift) - 1ull);
            break;
        }
    }
    // composites are unique: exactly K entries (or every valid one) qualify
    for (int j = tid; j < P; j += blockDim.x) skey[j] = 0ull;
    __syncthreads();
    for (int e = tid; e < total; e += blockDim.x) {
        const unsigned long long u = comp(e);
        if ((u >> 32) > PAD_TOP && (all_valid || (u & pmask) >= prefix))
            skey[atomicAdd(&sh_cnt, 1u)] = u;
    }
    __syncthreads();
    // short lists: unique padding composites (key -inf, idx >= n, skipped by refine)
    for (int j = (int)sh_cnt + tid; j < K; j += blockDim.x)
        skey[j] = (PAD_TOP << 32) | (unsigned long long)(uint32_t)j;
    __syncthreads();
    }  // radix path
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = tid; t < P / 2; t += blockDim.x) {
                const int pos = 2 * stride * (t / stride) + (t % stride);
                const int partner = pos + stride;
                const bool desc = (pos & size) == 0;
                const unsigned long long x = skey[pos], y = skey[partner];
                if ((x < y) == desc) {
                    skey[pos] = y;
                    skey[partner] = x;
                }
            }
            __syncthreads();
        }
    }
    for (int j = tid; j < K; j += blockDim.x) {
        const unsigned long long u = skey[j];
        out_key[(size_t)L * kout + j] = ord2f((uint32_t)(u >> 32));
        out_idx[(size_t)L * kout + j] = ~(uint32_t)(u & 0xffffffffu);
    }
    if (tid == 0) out_thr[L] = ord2f((uint32_t)(skey[K - 1] >> 32));
}

template <int ITEMS>
__global__ void __launch_bounds__(1024)
    merge_reg_kernel(const float* __restrict__ in_key, const uint32_t* __restrict__ in_idx, int G,
                     int lists_stride, int kmax, int kout, int QB, int kp, int knn,
                     float* __restrict__ out_key, uint32_t* __restrict__ out_idx,
                     float* __restrict__ out_thr, size_t in_g, size_t out_g) {
    in_key += blockIdx.y * in_g;
    in_idx += blockIdx.y * in_g;
    out_key += blockIdx.y * out_g;
    out_idx += blockIdx.y * out_g;
    out_thr += blockIdx.y * (size_t)lists_stride;
    const int L = blockIdx.x;
    const int K = L < QB ? kp : knn;
    auto load = [&](int e, float& key, uint32_t& idx) {
        const int g = e / K, j = e - g * K;
        const size_t off = ((size_t)g * lists_stride + L) * kmax + j;
        key = in_key[off];
        idx = in_idx[off];
        return true;
    };
    block_topk<ITEMS>(load, G * K, K, out_key + (size_t)L * kout, out_idx + (size_t)L * kout,
                      out_thr + L);
}

// one merge launch: the register kernel when every list fits, else the global
// one.  Inputs [G][lists][kmax] with K entries per CTA list; outputs
// [2 qb][kout] (kout = kmax unless the caller's input stride is larger).
void launch_merge(cudaStream_t st, const float* ck, const uint32_t* ci, int G, int lists, int kmax,
                  int qb, int kp, int knn, float* mk, uint32_t* mi, float* mthr, int kout,
                  int ngroups, size_t in_g, size_t out_g) {
    if (kout <= 0) kout = kmax;
    const dim3 nb((unsigned)(knn ? 2 * qb : qb), (unsigned)ngroups);
    const size_t total = (size_t)G * std::max(kp, knn);
    // (above 4k entries the global kernel: its fast path reads only each CTA
    // list's valid prefix -- 2M records x 4096 queries: 413 -> ~ 50 us)
    if (total <= 4 * 1024)
        merge_reg_kernel<4><<<nb, 1024, 0, st>>>(ck, ci, G, lists, kmax, kout, qb, kp, knn, mk, mi,
                                                 mthr, in_g, out_g);
    else
        merge_kernel<<<nb, 1024, 0, st>>>(ck, ci, G, lists, kmax, kout, qb, kp, knn, mk, mi, mthr,
                                          in_g, out_g);
    SAIR_LAUNCH("merge_kernel");
}

// ------------------------------------------------------------ refine -------

struct RefineArgs {
    const double* x64;
    const double* r64;
    const int32_t* rnd;
    const double* mean;  // [d]
    const double* sd;    // [d]
    const double* zq;    // [QB][d]
    const double* cc;    // [QB] sum_k c_qk^2 (fp64 of the fp32 constants)
    const unsigned int* pmax;
    int d, m, kp, knn, QB, kmax;
    size_t n;      // records in this store (candidate validity)
    size_t n_loo;  // records of the whole buffer (loo_mean's n)
    double total, two_s2, lambda, beta, gamma, key_slack_abs;
    double bq_rel;  // relative rounding of the MMA's query operand (wide pass), else 0
    double bias_rel;  // wide pass: D = D' - B_q from an accumulator that also held B_q
    double rec_rel;   // relative rounding of the stored records (TF32 2^-11; bf16 pass)
    int has_excl, has_excl_nn;
    int nq;                // queries of this group (<= QB)
    const float* ckey;
    const uint32_t* cidx;  // merged, sorted [2QB][kmax]
    const float* cthr;     // [2QB]
    const float* t0;                // [2QB] stream-pass start thresholds (MMA path) or null
    const float* t0safe;            // [2QB] wide pass: the sample's guaranteed ones (retry), or null
    const unsigned int* dropped;    // [2QB] max ordinal key dropped on a full list, or null
    double* zs;            // scratch [QB][kp][d]
    int64_t gbase;
    int64_t* out_idx;  // [QB][m]
    double* out_sim;
    double* out_score;
    int* out_count;
    int* out_cert;
    int64_t* out_nn;
    double* out_nn_sim;
    int* out_nn_cert;
    float* out_thr;     // [4][QB]: merged K'-th key (sel, veto), start threshold (sel, veto)
    double* out_rew;    // [QB][m] reward of each pick (shard merge)
    int32_t* out_round; // [QB][m]
};

// Largest key any record outside list L's pool can have: the merged K'-th key,
// the stream pass's start threshold (records at or below it were never
// listed) and the largest key dropped on a full list.
__device__ __forceinline__ double excl_bound(const RefineArgs& a, int L, float kth) {
    double U = (double)kth;
    if (a.t0) U = fmax(U, (double)a.t0[L]);
    if (a.dropped && a.dropped[L]) U = fmax(U, (double)ord2f(a.dropped[L]));
    return U;
}

// One launch refines every query group of a call: blockIdx.y = group (its
// own argument block), blockIdx.x = query within the group.
__global__ void __launch_bounds__(256) refine_kernel(const RefineArgs* __restrict__ args) {
    __shared__ RefineArgs sa;
    if (threadIdx.x == 0) sa = args[blockIdx.y];
    __syncthreads();
    const RefineArgs& a = sa;
    const int q = blockIdx.x;
    if (q >= a.nq) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    extern __shared__ __align__(16) unsigned char sm[];
    double* score = reinterpret_cast<double*>(sm);
    double* simc = score + a.kp;
    double* pen = simc + a.kp;
    double* rew = pen + a.kp;
    int32_t* rr = reinterpret_cast<int32_t*>(rew + a.kp);
    int* taken = rr + a.kp;
    int* picks = taken + a.kp;
    int* order = picks + a.kp;
    double* nnsim = reinterpret_cast<double*>(order + a.kp + (a.kp & 1));  // [knn]
    double* sqbuf = nnsim + a.knn;  // [warps][8][d + 1]
    uint32_t* sidx = reinterpret_cast<uint32_t*>(sqbuf + (blockDim.x >> 5) * 8 * (a.d + 1));
    __shared__ Best wb[8];
    __shared__ int s_cert, s_valid;
    const int d = a.d;
    const double* zq = a.zq + (size_t)q * d;
    double* zs = a.zs + (size_t)q * a.kp * d;
    __shared__ float s_thr[2];
    const uint32_t* ci = sidx;           // select candidates, merged (smem)
    const uint32_t* ni = sidx + a.kp;    // veto candidates
    {
        for (int j = tid; j < a.kp; j += blockDim.x) sidx[j] = a.cidx[(size_t)q * a.kmax + j];
        for (int j = tid; j < a.knn; j += blockDim.x)
            sidx[a.kp + j] = a.cidx[(size_t)(a.QB + q) * a.kmax + j];
        if (tid == 0) s_thr[0] = a.cthr[q];
        if (tid == 1 && a.knn) s_thr[1] = a.cthr[a.QB + q];
    }
    __syncthreads();

    // d2 error bound of the filter: E_q = gamma (sqrt(Pmax) + sqrt(C_q))^2
    const double pmx = (double)__uint_as_float(*a.pmax);
    const double sq = sqrt(pmx) + sqrt(a.cc[q]);
    // + the TF32 rounding of the stored records: d2_true >= d2 (1 - 2^-11) - 2^-11 P
    // + the rounded query operand: |<x, b' - b>| <= bq_rel sqrt(P C_q)
    // + (wide pass) the accumulator also summed B_q = t0_q / alpha + cc_q (the
    //   pre-test constant, select_wide.cu): D = D' - B_q carries the fp32
    //   rounding of partial sums up to |D| + |B_q| <= Pmax + 2 cc_q + |B_q|
    double Eq = a.gamma * sq * sq + a.rec_rel * pmx * (1.0 + 1e-6) +
                a.bq_rel * sqrt(pmx * a.cc[q]) + 1e-30;
    if (a.bias_rel != 0.0 && a.t0) {
        const double tq = (double)a.t0[q];
        const double Bq = fabs(tq) < 1e30 ? fabs(tq) / (a.beta * (1.0 - a.rec_rel)) + a.cc[q] : 0.0;
        Eq += a.bias_rel * (pmx + 2.0 * a.cc[q] + Bq);
    }

    // exact score of every candidate: experience.cpp:163-167 with the
    // reference's rounding sequence (standardize :162-166, similarity
    // :125-130, loo_mean :229-231).  Select and veto candidates form one work
    // list; a warp takes 8 at a time: its lanes compute the squared
    // differences of all 8 rows in parallel, then 8 lanes each sum one row in
    // k order (the order the reference's loop rounds in).
    const int nwarps = blockDim.x >> 5;
    const int nitems = a.kp + a.knn;
    const int ld = d + 1;  // padded row: lanes summing different rows hit distinct banks
    double* sqw = sqbuf + (size_t)warp * 8 * ld;
    for (int base = warp * 8; base < nitems; base += 8 * nwarps) {
        const int nb = min(8, nitems - base);
        // UN loads in flight per lane before any of the dependent fp64 math
        constexpr int UN = 8;
        for (int e0 = lane; e0 < nb * d; e0 += 32 * UN) {
            double xv[UN];
#pragma unroll
            for (int u = 0; u < UN; ++u) {
                const int e = e0 + 32 * u;
                xv[u] = 0.0;
                if (e < nb * d) {
                    const int b = e / d, k = e - b * d;
                    const uint32_t i = sidx[base + b];
                    if (i < a.n) xv[u] = a.x64[(size_t)i * d + k];
                }
            }
#pragma unroll
            for (int u = 0; u < UN; ++u) {
                const int e = e0 + 32 * u;
                if (e >= nb * d) break;
                const int b = e / d, k = e - b * d;
                const int it = base + b;
                double v = 0.0;
                if (sidx[it] < a.n) {
                    const double z = ddiv(dsub(xv[u], a.mean[k]), a.sd[k]);
                    if (it < a.kp) zs[(size_t)it * d + k] = z;
                    const double t = dsub(z, zq[k]);
                    v = dmul(t, t);
                }
                sqw[b * ld + k] = v;
            }
        }
        __syncwarp();
        if (lane < nb) {
            const int it = base + lane;
            const bool sel = it < a.kp;
            const uint32_t i = sidx[it];
            double d2 = 0.0;
            for (int k = 0; k < d; ++k) d2 = dadd(d2, sqw[lane * ld + k]);
            if (sel) {
                const int j = it;
                pen[j] = 0.0;
                if (i >= a.n) {
                    score[j] = -INFINITY;
                    rr[j] = INT32_MAX;
                    taken[j] = 1;
                } else {
                    const double sim = sim_from_d2(d2, a.two_s2);
                    const double r = a.r64[i];
                    const double loo =
                        a.n_loo <= 1 ? 0.0 : ddiv(dsub(a.total, r), (double)(a.n_loo - 1));
                    taken[j] = 0;
                    simc[j] = sim;
                    score[j] = dmul(sim, fabs(dsub(r, loo)));
                    rew[j] = r;
                    rr[j] = a.rnd[i];
                }
            } else {
                nnsim[it - a.kp] = i < a.n ? sim_from_d2(d2, a.two_s2) : -1.0;
            }
        }
        __syncwarp();
    }
    if (tid == 0) {
        s_cert = 1;
        s_valid = 0;
    }
    __syncthreads();
    for (int j = tid; j < a.kp; j += blockDim.x)
        if (!taken[j]) atomicAdd(&s_valid, 1);
    __syncthreads();

    // every record outside the pool has score <= 2^(U + E_q beta + slack)
    double bound = -1.0;
    if (a.has_excl) {
        const double U = excl_bound(a, q, s_thr[0]);
        bound = exp2(U + Eq * a.beta + 1e-5 * (fabs(U) + a.key_slack_abs));
    }
    // the pool always holds min(K', n) >= min(m, n) valid records; the cap
    // only guards against an inconsistent pool (no pick may index past it)
    const int want = (int)min(min((size_t)a.m, a.n), (size_t)s_valid);
    if (want < (int)min((size_t)a.m, a.n) && tid == 0) s_cert = 0;
    if (a.lambda == 0.0) {
        // gain == score: the greedy picks are the top-`want` by (score desc,
        // round asc, index asc) -- one rank per candidate, no loop
        for (int j = tid; j < a.kp; j += blockDim.x) {
            if (taken[j]) continue;
            const Best bj{score[j], rr[j], (int64_t)ci[j], j};
            int rank = 0;
            for (int i = 0; i < a.kp; ++i) {
                if (taken[i] || i == j) continue;
                rank += better(Best{score[i], rr[i], (int64_t)ci[i], i}, bj);
            }
            if (rank < want) {
                picks[rank] = j;
                if (rank == want - 1 && a.has_excl && !(score[j] > bound)) s_cert = 0;
            }
        }
        __syncthreads();
    } else {
        for (int step = 0; step < want; ++step) {
            Best b{0.0, 0, 0, -1};
            for (int j = tid; j < a.kp; j += blockDim.x) {
                if (taken[j]) continue;
                const Best c{dsub(score[j], dmul(a.lambda, pen[j])), rr[j], (int64_t)ci[j], j};
                if (better(c, b)) b = c;
            }
            b = warp_best(b);
            if (lane == 0) wb[warp] = b;
            __syncthreads();
            if (warp == 0) {
                Best c = lane < (int)(blockDim.x >> 5) ? wb[lane] : Best{0.0, 0, 0, -1};
                c = warp_best(c);
                if (lane == 0) {
                    picks[step] = c.j;
                    taken[c.j] = 1;
                    if (a.has_excl && !(c.g > bound)) s_cert = 0;
                }
            }
            __syncthreads();
            const int jb = picks[step];
            const double* zb = zs + (size_t)jb * d;
            for (int j = tid; j < a.kp; j += blockDim.x) {
                if (taken[j]) continue;
                const double* zj = zs + (size_t)j * d;
                double d2 = 0.0;
                for (int k = 0; k < d; ++k) {
                    const double t = dsub(zj[k], zb[k]);
                    d2 = dadd(d2, dmul(t, t));
                }
                pen[j] = dadd(pen[j], sim_from_d2(d2, a.two_s2));  // :283-284
            }
            __syncthreads();
        }
    }
    // curriculum order, :290-294: stable by (reward asc, round asc) over pick order
    for (int x = tid; x < want; x += blockDim.x) {
        const int v = picks[x];
        int pos = 0;
        for (int y = 0; y < want; ++y) {
            const int u = picks[y];
            const bool less = rew[u] != rew[v] ? rew[u] < rew[v] : rr[u] < rr[v];
            const bool same = rew[u] == rew[v] && rr[u] == rr[v];
            pos += less || (same && y < x);
        }
        order[pos] = v;
    }
    __syncthreads();
    for (int x = tid; x < want; x += blockDim.x) {
        const int j = order[x];
        a.out_idx[(size_t)q * a.m + x] = a.gbase + (int64_t)ci[j];
        a.out_sim[(size_t)q * a.m + x] = simc[j];
        a.out_score[(size_t)q * a.m + x] = score[j];
        a.out_rew[(size_t)q * a.m + x] = rew[j];
        a.out_round[(size_t)q * a.m + x] = rr[j];
    }
    if (tid == 0) {
        a.out_count[q] = want;
        a.out_cert[q] = s_cert;
        if (a.out_thr) {
            a.out_thr[q] = s_thr[0];
            a.out_thr[a.QB + q] = a.knn ? s_thr[1] : -INFINITY;
            // the retry's start: the guaranteed threshold where the pass used an estimate
            const float* ts = a.t0safe ? a.t0safe : a.t0;
            a.out_thr[2 * a.QB + q] = ts ? ts[q] : -INFINITY;
            a.out_thr[3 * a.QB + q] = ts && a.knn ? ts[a.QB + q] : -INFINITY;
        }
    }
    if (a.knn == 0) return;
    // nearest record by exact similarity; first index wins ties (policy.cpp:146-153)
    Best b{0.0, 0, 0, -1};
    for (int j = tid; j < a.knn; j += blockDim.x) {
        const uint32_t i = ni[j];
        if (i >= a.n) continue;
        const Best c{nnsim[j], 0, (int64_t)i, j};
        if (better(c, b)) b = c;
    }
    b = warp_best(b);
    __syncthreads();
    if (lane == 0) wb[warp] = b;
    __syncthreads();
    if (tid == 0) {
        Best c = wb[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
            if (better(wb[w], c)) c = wb[w];
        int cert = 1;
        if (a.has_excl_nn) {
            // excluded records have d2_32 >= D = -U_nn, so true d2 >= D - E_q
            const double D = -excl_bound(a, a.QB + q, s_thr[1]);
            const double lo = fmax(D * (1.0 - a.rec_rel) - Eq, 0.0);
            cert = c.g > exp(-lo / a.two_s2) * (1.0 + 1e-12);
        }
        a.out_nn[q] = a.gbase + c.i;
        a.out_nn_sim[q] = c.g;
        a.out_nn_cert[q] = cert;
    }
}

// --------------------------------------------------------------- host ------

namespace {

struct StreamPlan {
    int dp, qb, kp, knn, kmax, nst, cap_sel, cap_nn, grid;
    size_t smem;
};

template <int DP, int QB>
void fill_and_launch(sair_store_s* s, const StreamPlan& pl, const QueryPrep& p, const double* zgrp,
                     int nqg, float c1, float c0, float rdelta, float alpha, float* ck,
                     uint32_t* ci, unsigned int* pmax, std::vector<double>& cc_out) {
    StreamArgs<DP, QB> a{};
    a.pages = s->pages;
    a.r32 = s->r32;
    a.n = (uint32_t)s->n;
    a.npages = (uint32_t)((s->n + PAGE - 1) / PAGE);
    a.c1 = c1;
    a.c0 = c0;
    a.rdelta = rdelta;
    a.alpha = alpha;
    a.kp = pl.kp;
    a.knn = pl.knn;
    a.nst = pl.nst;
    a.cap_sel = pl.cap_sel;
    a.cap_nn = pl.cap_nn;
    a.kmax = pl.kmax;
    a.out_key = ck;
    a.out_idx = ci;
    a.pmax = pmax;
    const int d = s->d;
    for (int k = 0; k < DP; ++k) a.s[k] = k < d ? (float)(1.0 / p.sd[k]) : 0.f;
    cc_out.assign(QB, 0.0);
    for (int q = 0; q < QB; ++q) {
        // padded query slots repeat query 0 (their lists are never read)
        const double* z = zgrp + (size_t)(q < nqg ? q : 0) * d;
        double cc = 0.0;
        for (int k = 0; k < DP; ++k) {
            float c = 0.f;
            if (k < d) c = (float)((p.mean[k] - s->shift[k]) / p.sd[k] + z[k]);
            a.c2[k][q] = -2.f * c;
            cc += (double)c * (double)c;
        }
        a.cc[q] = (float)cc;
        cc_out[q] = cc;
    }
    SAIR_CUDA(cudaFuncSetAttribute(stream_kernel<DP, QB>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
    stream_kernel<DP, QB><<<pl.grid, STREAM_THREADS, pl.smem, s->st>>>(a);
    SAIR_LAUNCH("stream_kernel");
}

using FillFn = void (*)(sair_store_s*, const StreamPlan&, const QueryPrep&, const double*, int,
                        float, float, float, float, float*, uint32_t*, unsigned int*,
                        std::vector<double>&);

template <int DP>
FillFn pick_qb(int qb) {
    switch (qb) {
        case 1: return fill_and_launch<DP, 1>;
        case 2: return fill_and_launch<DP, 2>;
        case 4: return fill_and_launch<DP, 4>;
        default: return fill_and_launch<DP, 8>;
    }
}
FillFn pick_fill(int dp, int qb) {
    switch (dp) {
        case 8: return pick_qb<8>(qb);
        case 16: return pick_qb<16>(qb);
        case 32: return pick_qb<32>(qb);
        case 64: return pick_qb<64>(qb);
        case 128: return pick_qb<128>(qb);
        default: return nullptr;
    }
}

StreamPlan make_plan(const sair_store_s* s, size_t nq, size_t m, double lambda, bool nn) {
    StreamPlan pl{};
    pl.dp = s->dp;
    pl.qb = nq >= 8 ? 8 : (nq >= 4 ? 4 : (nq >= 2 ? 2 : 1));
    // candidate pool sizes
    pl.kp = 32;
    const size_t want_pool = lambda != 0.0 ? 4 * m : 2 * m;
    while ((size_t)pl.kp < want_pool && pl.kp < 512) pl.kp <<= 1;
    pl.knn = nn ? 16 : 0;
    pl.kmax = std::max(pl.kp, pl.knn);
    // a list takes at most 2 * CONS_THREADS inserts between two compaction checks
    pl.cap_sel = pl.kp + 2 * CONS_THREADS + 64;
    pl.cap_nn = pl.knn + 2 * CONS_THREADS + 64;
    const int dh = pl.dp < 16 ? pl.dp : 16;
    const size_t stage_bytes = (size_t)ROUND_PAGES * dh * PAGE * 4;
    const size_t fixed = (size_t)pl.dp * pl.qb * 4 + pl.dp * 4 + 16 * 8 + 2 * 16 * 4 +
                         CONS_WARPS * 256 * 4 + (size_t)pl.qb * pl.cap_sel * 8 +
                         (nn ? (size_t)pl.qb * pl.cap_nn * 8 : 0);
    const size_t limit = 227 * 1024;
    // deep ring of small stages: up to 160 KB in flight per SM
    pl.nst = (int)std::min<size_t>(8, std::max<size_t>(2, 160 * 1024 / stage_bytes + 1));
    while (pl.nst > 2 && fixed + pl.nst * stage_bytes > limit) --pl.nst;
    if (fixed + pl.nst * stage_bytes > limit)
        throw Error(SAIR_EINVAL, "select: candidate lists do not fit in shared memory");
    pl.smem = fixed + pl.nst * stage_bytes;
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, s->device);
    const size_t npages = (s->n + PAGE - 1) / PAGE;
    const size_t nrounds = (npages + ROUND_PAGES - 1) / ROUND_PAGES;
    pl.grid = (int)std::max<size_t>(1, std::min<size_t>(nrounds, (size_t)nsm));
    return pl;
}

}  // namespace

void store_select(sair_store_s* s, const double* q, size_t nq, int dim,
                  const sair_select_config& cfg, int64_t* out_idx, double* out_sim,
                  double* out_score, size_t* out_count, int64_t* out_nn, double* out_nn_sim,
                  double* out_reward, int32_t* out_round) {
    s->last = sair_select_stats{};
    s->last.queries = nq;
    if (nq == 0) return;
    const size_t m = cfg.m;
    if (s->n == 0 || m == 0) {  // experience.cpp:154
        for (size_t i = 0; i < nq; ++i) out_count[i] = 0;
        if (out_nn)
            for (size_t i = 0; i < nq; ++i) {
                out_nn[i] = -1;
                out_nn_sim[i] = -1.0;
            }
        return;
    }
    DeviceGuard g(s->device);
    // SAIR_TRACE_SELECT=1: host-side phase times of the call (us), to stderr
    static const bool trace = std::getenv("SAIR_TRACE_SELECT") != nullptr;
    std::vector<std::pair<const char*, std::chrono::steady_clock::time_point>> marks;
    auto mark = [&](const char* what) {
        if (trace) marks.emplace_back(what, std::chrono::steady_clock::now());
    };
    struct TraceOut {
        decltype(marks)& m;
        ~TraceOut() {
            if (m.size() < 2) return;
            fprintf(stderr, "[select]");
            for (size_t i = 1; i < m.size(); ++i)
                fprintf(stderr, " %s %.1f", m[i].first,
                        std::chrono::duration<double, std::micro>(m[i].second - m[i - 1].second).count());
            fprintf(stderr, "\n");
        }
    } trace_out{marks};
    mark("start");
    const double sigma = store_effective_sigma(s, cfg.sigma_sim);  // :246
    if (dim != s->d)  // standardize(x_curr) throws after the sigma refresh (:157-158)
        throw Error(SAIR_EINVAL, "experience store: feature dimension mismatch");
    mark("sigma");
    QueryPrep p = prep_queries(s, q, nq, sigma);
    mark("prep");
    const int d = s->d;
    const size_t n = s->n;
    SAIR_CUDA(cudaEventRecord(s->ev[0], s->st));

    std::vector<int> done(nq, 0);
    if (s->sharded && cfg.locally_weighted_mean)
        throw Error(SAIR_EINVAL, "locally_weighted_mean is not supported on a sharded store");
    // Small stores (<= 64k records): the whole exact select in one clustered
    // launch (select_small.cu) when the filter cannot pay off -- lambda > 0
    // (the greedy's diversity penalties defeat a fixed candidate pool), the
    // exact mode, or a store small enough that one exact pass is the cheaper
    // launch sequence.
    const bool small_ok = small_select_fits(s, m) &&
                          std::getenv("SAIR_NO_SMALL") == nullptr;
    if (small_ok && (cfg.lambda_div != 0.0 || cfg.mode == SAIR_SELECT_EXACT ||
                     cfg.locally_weighted_mean || n <= SMALL_DIRECT_N)) {
        std::vector<size_t> all(nq);
        for (size_t i = 0; i < nq; ++i) all[i] = i;
        small_select(s, p, all, m, cfg.lambda_div, cfg.locally_weighted_mean != 0, out_nn != nullptr,
                     out_idx, out_sim, out_score,
                     out_count, out_nn, out_nn_sim, out_reward, out_round);
        s->last.exact_fallbacks = 0;
        s->last.small = 1;
        SAIR_CUDA(cudaEventRecord(s->ev[3], s->st));
        if (s->defer_sync) return;  // the decision step synchronises (and times) later
        SAIR_CUDA(cudaEventSynchronize(s->ev[3]));
        float tot = 0.f;
        cudaEventElapsedTime(&tot, s->ev[0], s->ev[3]);
        s->last.total_ms = tot;
        return;
    }
    // the filter's certification bounds an outside record's gain by its score,
    // which needs lambda_div >= 0 (a negative lambda rewards similarity; the
    // reference accepts it, scenario.cpp:197): those queries take the exact paths
    const bool lam_pos = cfg.lambda_div > 0.0;
    const bool force_pool = lam_pos && std::getenv("SAIR_LAM_POOL") != nullptr;  // (tests: always try)
    const bool skip_pool =
        lam_pos && !force_pool && s->lam_pool_fail && (++s->lam_probe % 16u) != 0u;
    const bool fast = cfg.mode != SAIR_SELECT_EXACT && !cfg.locally_weighted_mean && d <= 128 &&
                      n < (size_t)1 << 31 && m <= 256 && cfg.lambda_div >= 0.0 && !skip_pool;
    float stream_ms = 0.f, prepass_ms = 0.f;
    if (fast) {
        // tensor-core streaming kernel when the shape fits,
        // the CUDA-core kernel otherwise or when SAIR_NO_MMA is set
        MmaPlan mp{};
        WidePlan wp{};
        const bool no_tc = std::getenv("SAIR_NO_MMA") != nullptr;
        const bool use_wide =
            !no_tc && make_wide_plan(s, nq, m, cfg.lambda_div, out_nn != nullptr, &wp);
        const bool use_mma = !no_tc && !use_wide &&
                             make_mma_plan(s, nq, m, cfg.lambda_div, out_nn != nullptr, &mp);
        StreamPlan pl = make_plan(s, nq, m, cfg.lambda_div, out_nn != nullptr);
        if (use_wide) {
            pl.dp = wp.dp;
            pl.qb = wp.qw;
            pl.kp = wp.kp;
            pl.knn = wp.knn;
            pl.kmax = wp.kmax;
            pl.grid = wp.grid;
        } else if (use_mma) {
            pl.dp = mp.dp;
            pl.qb = mp.qb;
            pl.kp = mp.kp;
            pl.knn = mp.knn;
            pl.kmax = mp.kmax;
            pl.grid = mp.grid;
        }
        const int qb = pl.qb, kp = pl.kp, knn = pl.knn, kmax = pl.kmax;
        FillFn fill = use_wide ? nullptr : pick_fill(pl.dp, qb);
        MmaFillFn mfill = use_mma ? pick_mma_fill(mp.dp, qb) : nullptr;
        WideFn wfill = use_wide ? pick_wide(wp.dp, qb) : nullptr;

        // filter constants
        const double u = 0x1p-24;
        const StoreStats& est = eff_stats(s);
        const uint64_t nb = eff_n(s);
        double c1d = 1.0, c0d = 0.0;
        if (nb >= 2) {
            c1d = (double)nb / (double)(nb - 1);
            c0d = est.total / (double)(nb - 1);
        }
        const float c1 = (float)c1d, c0 = (float)c0d;
        const double rdel = 4.0 * u * (est.rabs * c1d + std::fabs(c0d)) * 1.01 + 1e-30;
        const float rdelta = (float)rdel;
        const double beta = 1.4426950408889634 / p.two_s2;  // log2(e) / (2 sigma^2)
        // TF32 (or, the bf16 wide pass, bf16) storage of the records, see Eq
        const double rec_rel = use_wide ? wide_rec_rel(wp) : 0x1p-11;
        const float alpha = (float)(beta * (1.0 - rec_rel));
        const double lg_hi = std::log2(est.rabs * c1d + std::fabs(c0d) + rdel);
        const double key_slack_abs = 1.0 + 2.0 * (std::fabs(std::log2(rdel)) + std::fabs(lg_hi));

        const size_t lists = use_wide ? 1 : (size_t)pl.grid * 2 * qb * kmax;
        float* ck = s->b_cand.as<float>(lists * 2);
        uint32_t* ci = reinterpret_cast<uint32_t*>(ck + lists);
        // One batch: the queries ql (indices into the call's queries), in groups
        // of qb; t0o (wide pass only) overrides the sampled start thresholds,
        // 2 qb floats per group (selection lists, then veto lists).
        std::vector<float> thr_of(nq * 4, -INFINITY);
        bool pl_ready = false;  // the (P, lg) cache holds this call's values
        uint32_t nhot = 0;
        mark("plan");
        const uint32_t* hot = use_wide ? wide_hot_pages(s, wp, c1, c0, &nhot) : nullptr;
        mark("hot");
        auto run_batch = [&](const std::vector<size_t>& ql, const std::vector<float>* t0o) {
        const size_t nbq = ql.size();
        const size_t ngroups = (nbq + qb - 1) / qb;
        std::vector<double> zc(nbq * d);
        for (size_t i = 0; i < nbq; ++i)
            std::copy(p.z.begin() + ql[i] * d, p.z.begin() + (ql[i] + 1) * d, zc.begin() + i * d);
        // Every group's kernels are enqueued back to back on the store's stream
        // (device scratch is reused in stream order); each group has its own
        // pinned staging, output slice and events, and the host synchronises
        // once, after one device-to-host copy of all outputs.
        const size_t ob = ((size_t)qb * m * 8 * 4 + (size_t)qb * m * 4 + (size_t)qb * 8 * 2 +
                           (size_t)qb * 4 * 4 + (size_t)qb * 4 * 4 + 64 + 255) & ~(size_t)255;
        char* dout = static_cast<char*>(s->b_out.get(ob * ngroups));
        char* hout = static_cast<char*>(s->h_out.get(ob * ngroups));
        struct O {
            int64_t* idx;
            double* sim;
            double* score;
            int64_t* nn;
            double* nn_sim;
            int* cnt;
            int* cert;
            int* nn_cert;
            double* rew;
            int32_t* round;
            float* thr;  // [4][qb]: K'-th merged key (sel, veto), start threshold (sel, veto)
        };
        auto carve = [&](char* b) {
            O o;
            o.idx = reinterpret_cast<int64_t*>(b);
            o.sim = reinterpret_cast<double*>(o.idx + qb * m);
            o.score = o.sim + qb * m;
            o.nn = reinterpret_cast<int64_t*>(o.score + qb * m);
            o.nn_sim = reinterpret_cast<double*>(o.nn + qb);
            o.cnt = reinterpret_cast<int*>(o.nn_sim + qb);
            o.cert = o.cnt + qb;
            o.nn_cert = o.cert + qb;
            o.rew = reinterpret_cast<double*>(o.nn_cert + qb + (qb & 1));
            o.round = reinterpret_cast<int32_t*>(o.rew + qb * m);
            o.thr = reinterpret_cast<float*>(o.round + qb * m);
            return o;
        };
        // pinned, so the copies never stage through pageable memory
        const size_t nhc = 2 * (size_t)d + (size_t)qb * d + qb;
        double* hc_all = s->h_consts.as<double>(nhc * ngroups);
        const size_t hstride = ((size_t)3 * pl.dp * qb + pl.dp + 4 * (size_t)qb + 256 + 63) & ~(size_t)63;
        float* hstage_all = use_mma || use_wide ? s->h_mmab.as<float>(hstride * ngroups) : nullptr;
        while (s->gev.size() < 3 * ngroups) {
            cudaEvent_t e;
            SAIR_CUDA(cudaEventCreate(&e));
            s->gev.push_back(e);
        }
        // per-group device state read by the one refine launch at the end:
        // merged lists, start thresholds, dropped keys, Pmax, refine constants,
        // the refine's standardized-row scratch
        const size_t mstride = (size_t)2 * qb * kmax;
        const size_t zstride = (size_t)qb * kp * d;
        char* gbase_p = static_cast<char*>(s->b_grp.get(
            ngroups * (mstride * 8 + 2 * qb * 4 + 2 * qb * 8 + 8 + nhc * 8 + zstride * 8) +
            8 * 256 + ngroups * sizeof(RefineArgs) +
            (use_wide ? ngroups * (hstride * 4 + 4 * (size_t)qb * 4) + 2 * 256 : 0)));
        size_t goff = 0;
        auto gtake = [&](size_t bytes) {
            char* ptr = gbase_p + goff;
            goff += (bytes + 255) / 256 * 256;
            return ptr;
        };
        float* mk_g = reinterpret_cast<float*>(gtake(ngroups * mstride * 4));
        uint32_t* mi_g = reinterpret_cast<uint32_t*>(gtake(ngroups * mstride * 4));
        float* mthr_g = reinterpret_cast<float*>(gtake(ngroups * 2 * qb * 4));
        float* t0_g = reinterpret_cast<float*>(gtake(ngroups * 2 * qb * 4));
        unsigned int* drop_g = reinterpret_cast<unsigned int*>(gtake(ngroups * 2 * qb * 4));
        unsigned int* pmax_g = reinterpret_cast<unsigned int*>(gtake(ngroups * 4));
        double* dc_g = reinterpret_cast<double*>(gtake(ngroups * nhc * 8));
        double* zs_g = reinterpret_cast<double*>(gtake(ngroups * zstride * 8));
        RefineArgs* ra_dev = reinterpret_cast<RefineArgs*>(gtake(ngroups * sizeof(RefineArgs)));
        // wide pass: every group's constants (hstride floats each, the host
        // staging's image) and list counters [2][2 qb], uploaded / zeroed once
        float* wc_g = use_wide ? reinterpret_cast<float*>(gtake(ngroups * hstride * 4)) : nullptr;
        uint32_t* wcnt_g =
            use_wide ? reinterpret_cast<uint32_t*>(gtake(ngroups * 4 * (size_t)qb * 4)) : nullptr;
        // the wide pass's compacted CTA lists of every group (merged in one launch)
        const size_t lstride = use_wide ? (size_t)wp.grid * 2 * qb * kmax : 0;
        float* lk_g = use_wide ? s->b_wlists.as<float>(ngroups * lstride * 2) : nullptr;
        // (P, log residual) per record: the same for every group of the call
        // (one standardization, one set of reward constants) -- computed by the
        // first stream pass, read by every later launch
        float* pl_cache = use_wide ? s->b_pl.as<float>(((n + PAGE - 1) / PAGE) * PAGE * 2) : nullptr;
        float* pl16_cache =
            use_wide && wp.bf16 ? s->b_pl16.as<float>(((n + PAGE - 1) / PAGE) * PAGE * 2) : nullptr;
        uint32_t* li_g = use_wide ? reinterpret_cast<uint32_t*>(lk_g + ngroups * lstride) : nullptr;
        RefineArgs* ra_host = reinterpret_cast<RefineArgs*>(
            s->h_ra.get(ngroups * sizeof(RefineArgs) + 64));
        SAIR_CUDA(cudaMemsetAsync(pmax_g, 0, ngroups * 4, s->st));
        std::vector<double> cc;
        const size_t refine_smem = (size_t)kp * (8 * 4 + 4 * 4) + 16 + (size_t)knn * 8 +
                                   (size_t)8 * 8 * (d + 1) * 8 + (size_t)(kp + knn) * 4 + 64;
        SAIR_CUDA(cudaFuncSetAttribute(refine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)refine_smem));
        s->last.candidates = kp;
        s->last.qb = qb;
        s->last.tensor_core = use_wide ? (wp.bf16 ? 3 : 2) : (use_mma ? 1 : 0);
        // wide pass: a group's constants on the host (phase 1 of wfill) and the
        // refine's cc; group 0's go up before its passes, each later group's
        // are prepared while the device runs the group before it and copied
        // on the copy stream (the group's passes wait on that copy's event)
        auto wide_prep = [&](size_t g) {
            const size_t g0 = g * qb;
            GroupIo io{};
            io.hstage = hstage_all + g * hstride;
            io.t0_override = t0o ? t0o->data() + g * 2 * qb : nullptr;
            io.phase = 1;
            wfill(s, wp, p, zc.data() + g0 * d, (int)std::min<size_t>(qb, nbq - g0), c1, c0,
                  rdelta, alpha, nullptr, nullptr, nullptr, nullptr, cc, io);
            double* hc = hc_all + g * nhc;
            for (int qq = 0; qq < qb; ++qq) hc[2 * (size_t)d + (size_t)qb * d + qq] = cc[qq];
        };
        mark("setup");
        if (use_wide) {
            wide_prep(0);
            mark("prep0");
            SAIR_CUDA(cudaMemcpyAsync(wc_g, hstage_all, hstride * 4, cudaMemcpyHostToDevice, s->st));
            SAIR_CUDA(cudaMemsetAsync(wcnt_g, 0, ngroups * 4 * (size_t)qb * 4, s->st));
        }
        for (size_t g = 0; g < ngroups; ++g) {
            const size_t g0 = g * qb;
            const int nqg = (int)std::min<size_t>(qb, nbq - g0);
            const double* zgrp = zc.data() + g0 * d;
            double* hc = hc_all + g * nhc;
            std::copy(p.mean.begin(), p.mean.end(), hc);
            std::copy(p.sd.begin(), p.sd.end(), hc + d);
            for (int qq = 0; qq < qb; ++qq) {
                const double* z = zgrp + (size_t)(qq < nqg ? qq : 0) * d;
                for (int k = 0; k < d; ++k) hc[2 * (size_t)d + (size_t)qq * d + k] = z[k];
            }
            GroupIo io{hstage_all ? hstage_all + g * hstride : nullptr, s->gev[3 * g + 1],
                             s->gev[3 * g + 2], t0o ? t0o->data() + g * 2 * qb : nullptr,
                             use_wide ? lk_g + g * lstride : nullptr,
                             use_wide ? li_g + g * lstride : nullptr,
                             use_wide && pl_ready ? pl_cache : nullptr,
                             use_wide && !pl_ready ? pl_cache : nullptr, hot, nhot,
                             use_wide ? 2 : 0, use_wide ? wc_g + g * hstride : nullptr,
                             use_wide ? wcnt_g + g * 4 * (size_t)qb : nullptr};
            io.pl16_in = pl16_cache && pl_ready ? pl16_cache : nullptr;
            io.pl16_out = pl16_cache && !pl_ready ? pl16_cache : nullptr;
            if (use_wide) pl_ready = true;
            const O D = carve(dout + g * ob);
            float* mk = mk_g + g * mstride;
            uint32_t* mi = mi_g + g * mstride;
            float* mthr = mthr_g + g * 2 * qb;
            unsigned int* dpmax = pmax_g + g;
            double* dc = dc_g + g * nhc;
            if (use_wide && g > 0) SAIR_CUDA(cudaStreamWaitEvent(s->st, s->cev[g], 0));
            SAIR_CUDA(cudaEventRecord(s->gev[3 * g], s->st));
            mark("grp");
            if (use_wide)  // sample + stream + per-list top-K' (records e_mid, e_end)
                wfill(s, wp, p, zgrp, nqg, c1, c0, rdelta, alpha, mk, mi, mthr, dpmax, cc, io);
            else if (use_mma)
                mfill(s, mp, p, zgrp, nqg, c1, c0, rdelta, alpha, ck, ci, dpmax, cc, io);
            else
                fill(s, pl, p, zgrp, nqg, c1, c0, rdelta, alpha, ck, ci, dpmax, cc);
            mark("launch");
            if (!use_wide) SAIR_CUDA(cudaEventRecord(io.e_end, s->st));
            if (use_wide && g + 1 < ngroups) {
                // the next group's constants, prepared while the device runs
                // this group's passes and copied on the copy stream beside
                // them (one copy for all later groups made the device wait for
                // the host's whole preparation: 2M records x 4096 queries, ~1 ms)
                wide_prep(g + 1);
                while (s->cev.size() < ngroups) {
                    cudaEvent_t e;
                    SAIR_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                    s->cev.push_back(e);
                }
                SAIR_CUDA(cudaMemcpyAsync(wc_g + (g + 1) * hstride, hstage_all + (g + 1) * hstride,
                                          hstride * 4, cudaMemcpyHostToDevice, s->cst));
                SAIR_CUDA(cudaEventRecord(s->cev[g + 1], s->cst));
            }
            s->last.stream_launches++;
            if (!use_wide)  // (the wide pass's were written by its first loop)
                for (int qq = 0; qq < qb; ++qq) hc[2 * (size_t)d + (size_t)qb * d + qq] = cc[qq];
            // (the refine constants of every group go up in one copy after the loop)
            if (!use_wide)
                launch_merge(s->st, ck, ci, pl.grid, 2 * qb, kmax, qb, kp, knn, mk, mi, mthr);
            if (use_mma) {  // keep this group's thresholds past the next group (the wide
                            // pass's stay in the group's own constants / counters)
                SAIR_CUDA(cudaMemcpyAsync(t0_g + g * 2 * qb, s->mma_t0, 2 * qb * 4,
                                          cudaMemcpyDeviceToDevice, s->st));
                SAIR_CUDA(cudaMemcpyAsync(drop_g + g * 2 * qb, s->mma_dropped, 2 * qb * 4,
                                          cudaMemcpyDeviceToDevice, s->st));
            }
            RefineArgs ra{};
            ra.nq = nqg;
            ra.x64 = s->x64;
            ra.r64 = s->r64;
            ra.rnd = s->rnd;
            ra.mean = dc;
            ra.sd = dc + d;
            ra.zq = dc + 2 * d;
            ra.cc = dc + 2 * d + (size_t)qb * d;
            ra.pmax = dpmax;
            ra.d = d;
            ra.m = (int)m;
            ra.kp = kp;
            ra.knn = knn;
            ra.QB = qb;
            ra.kmax = kmax;
            ra.n = n;
            ra.n_loo = nb;
            ra.total = est.total;
            ra.two_s2 = p.two_s2;
            ra.lambda = cfg.lambda_div;
            ra.beta = beta;
            // fp32 error of the filter's d2; the wide pass
            // accumulates the hi and lo products in one chain of 2 dp / 8 MMAs
            ra.gamma = use_wide ? (2 * pl.dp + 32) * u + 0x1p-20
                                : (use_mma ? (pl.dp + 24) * u + 0x1p-20 : (pl.dp + 16) * u);
            ra.key_slack_abs = key_slack_abs;
            ra.bq_rel = use_wide ? wide_bq_rel(wp) : 0.0;
            ra.bias_rel = use_wide ? 0x1p-19 : 0.0;
            ra.rec_rel = rec_rel;
            ra.has_excl = n > (size_t)kp;
            ra.has_excl_nn = n > (size_t)knn;
            ra.ckey = mk;
            ra.cidx = mi;
            ra.cthr = mthr;
            ra.t0 = use_wide ? s->mma_t0 : (use_mma ? t0_g + g * 2 * qb : nullptr);
            ra.t0safe = use_wide ? s->mma_t0safe : nullptr;
            ra.dropped = use_wide ? s->mma_dropped : (use_mma ? drop_g + g * 2 * qb : nullptr);
            ra.zs = zs_g + g * zstride;
            ra.gbase = s->gbase;
            ra.out_idx = D.idx;
            ra.out_sim = D.sim;
            ra.out_score = D.score;
            ra.out_count = D.cnt;
            ra.out_cert = D.cert;
            ra.out_nn = D.nn;
            ra.out_nn_sim = D.nn_sim;
            ra.out_nn_cert = D.nn_cert;
            ra.out_rew = D.rew;
            ra.out_round = D.round;
            ra.out_thr = D.thr;
            ra_host[g] = ra;
        }
        if (use_wide)  // every group's per-query top-K' across its CTA lists, one launch
            launch_merge(s->st, lk_g, li_g, wp.grid, 2 * qb, kmax, qb, kp, knn, mk_g, mi_g, mthr_g,
                         kmax, (int)ngroups, lstride, mstride);
        // every group's refine in one launch
        SAIR_CUDA(cudaMemcpyAsync(dc_g, hc_all, ngroups * nhc * 8, cudaMemcpyHostToDevice, s->st));
        SAIR_CUDA(cudaMemcpyAsync(ra_dev, ra_host, ngroups * sizeof(RefineArgs),
                                  cudaMemcpyHostToDevice, s->st));
        refine_kernel<<<dim3((unsigned)qb, (unsigned)ngroups), 256, refine_smem, s->st>>>(ra_dev);
        SAIR_LAUNCH("refine_kernel");
        SAIR_CUDA(cudaMemcpyAsync(hout, dout, ob * ngroups, cudaMemcpyDeviceToHost, s->st));
        mark("tail");
        SAIR_CUDA(cudaStreamSynchronize(s->st));
        mark("sync");
        for (size_t g = 0; g < ngroups; ++g) {
            const size_t g0 = g * qb;
            const int nqg = (int)std::min<size_t>(qb, nbq - g0);
            const O H = carve(hout + g * ob);
            float ms = 0.f;
            if (use_mma || use_wide) {
                float pre = 0.f;
                cudaEventElapsedTime(&pre, s->gev[3 * g], s->gev[3 * g + 1]);
                cudaEventElapsedTime(&ms, s->gev[3 * g + 1], s->gev[3 * g + 2]);
                prepass_ms += pre;
            } else {
                cudaEventElapsedTime(&ms, s->gev[3 * g], s->gev[3 * g + 2]);
            }
            stream_ms += ms;
            for (int qq = 0; qq < nqg; ++qq) {
                const size_t gq = ql[g0 + qq];
                for (int k = 0; k < 4; ++k) thr_of[gq * 4 + k] = H.thr[k * qb + qq];
                if (!(H.cert[qq] && (!out_nn || H.nn_cert[qq]))) continue;
                done[gq] = 1;
                out_count[gq] = (size_t)H.cnt[qq];
                std::memcpy(out_idx + gq * m, H.idx + (size_t)qq * m, H.cnt[qq] * 8);
                std::memcpy(out_sim + gq * m, H.sim + (size_t)qq * m, H.cnt[qq] * 8);
                std::memcpy(out_score + gq * m, H.score + (size_t)qq * m, H.cnt[qq] * 8);
                if (out_reward)
                    std::memcpy(out_reward + gq * m, H.rew + (size_t)qq * m, H.cnt[qq] * 8);
                if (out_round)
                    std::memcpy(out_round + gq * m, H.round + (size_t)qq * m, H.cnt[qq] * 4);
                if (out_nn) {
                    out_nn[gq] = H.nn[qq];
                    out_nn_sim[gq] = H.nn_sim[qq];
                }
                s->last.certified++;
            }
        }
        };
        std::vector<size_t> all_q(nq);
        for (size_t i = 0; i < nq; ++i) all_q[i] = i;
        run_batch(all_q, nullptr);
        if (use_wide && cfg.lambda_div == 0.0) {
            // Second chance before the exact pass: a list that overflowed its
            // per-CTA capacity (records with high keys concentrated in a few
            // pages: a freshly appended batch) still kept >= K' keys above the
            // start threshold, so its K'-th kept key is a valid, higher start
            // threshold.  One more wide pass with it usually certifies.
            std::vector<size_t> rest;
            for (size_t i = 0; i < nq; ++i)
                if (!done[i]) rest.push_back(i);
            if (!rest.empty()) {
                const size_t ng = (rest.size() + qb - 1) / qb;
                // padding slots of the last group never admit a record (a -inf
                // start there would send every record down the slow path)
                std::vector<float> t0r(ng * 2 * qb, FLT_MAX);
                for (size_t j = 0; j < rest.size(); ++j) {
                    const size_t i = rest[j], g = j / qb, qq = j % qb;
                    t0r[g * 2 * qb + qq] = std::max(thr_of[i * 4 + 2], thr_of[i * 4 + 0]);
                    t0r[g * 2 * qb + qb + qq] = std::max(thr_of[i * 4 + 3], thr_of[i * 4 + 1]);
                }
                run_batch(rest, &t0r);
                s->last.retried = rest.size();
            }
        }
        if (lam_pos) s->lam_pool_fail = s->last.certified * 20 < nq ? 1 : 0;
    }
    if (small_ok) {  // the uncertified queries of a small store: one clustered launch
        std::vector<size_t> rest;
        for (size_t i = 0; i < nq; ++i)
            if (!done[i]) rest.push_back(i);
        small_select(s, p, rest, m, cfg.lambda_div, cfg.locally_weighted_mean != 0,
                     out_nn != nullptr, out_idx, out_sim,
                     out_score, out_count, out_nn, out_nn_sim, out_reward, out_round);
        s->last.exact_fallbacks += rest.size();
        for (size_t i : rest) done[i] = 1;
    }
    const double* loo_pre = nullptr;
    for (size_t i = 0; i < nq && cfg.locally_weighted_mean && !loo_pre; ++i)
        if (!done[i]) loo_pre = local_loo_all(s, p);  // once for every remaining query
    if (m <= 256 && std::getenv("SAIR_NO_GREEDY") == nullptr) {
        // the remaining queries (lambda > 0 on a large store, the exact mode,
        // uncertified ones): the batched exact greedy, G queries per pass
        std::vector<size_t> rest;
        for (size_t i = 0; i < nq; ++i)
            if (!done[i]) rest.push_back(i);
        if (!rest.empty()) {
            // fp32-filtered, fp64-decided steps (select_greedy32.cu); the fp64
            // greedy for what that path declines (SAIR_GREEDY64=1: always)
            std::vector<size_t> fb;
            const bool g32 = std::getenv("SAIR_GREEDY64") == nullptr &&
                             greedy32_select(s, p, rest, m, cfg.lambda_div, loo_pre, out_nn != nullptr,
                                             out_idx, out_sim, out_score, out_count, out_nn,
                                             out_nn_sim, out_reward, out_round, &fb);
            if (g32) {
                s->last.greedy32 = rest.size() - fb.size();
                for (size_t i : rest) done[i] = 1;
                rest.swap(fb);
            }
            if (!rest.empty())
                greedy_select(s, p, rest, m, cfg.lambda_div, loo_pre, out_nn != nullptr, out_idx,
                              out_sim, out_score, out_count, out_nn, out_nn_sim, out_reward,
                              out_round);
            s->last.exact_fallbacks += (g32 ? s->last.greedy32 : 0) + rest.size();
            for (size_t i : rest) done[i] = 1;
        }
    }
    for (size_t i = 0; i < nq; ++i) {
        if (done[i]) continue;
        exact_one(s, p, p.z.data() + i * d, m, cfg.lambda_div, cfg.locally_weighted_mean != 0,
                  out_idx + i * m, out_sim + i * m, out_score + i * m, &out_count[i],
                  out_nn ? out_nn + i : nullptr, out_nn ? out_nn_sim + i : nullptr,
                  out_reward ? out_reward + i * m : nullptr, out_round ? out_round + i * m : nullptr,
                  loo_pre);
        s->last.exact_fallbacks++;
    }
    SAIR_CUDA(cudaEventRecord(s->ev[3], s->st));
    SAIR_CUDA(cudaEventSynchronize(s->ev[3]));
    float tot = 0.f;
    cudaEventElapsedTime(&tot, s->ev[0], s->ev[3]);
    s->last.stream_ms = stream_ms;
    s->last.prepass_ms = prepass_ms;
    s->last.total_ms = tot;
}

// ------------------------------------------------------- shard merge ------

// Per query: the union of the shards' top-m (exact fp64 scores over the
// buffer's global statistics) holds the buffer's top-m when lambda_div == 0;
// pick it by (score desc, round asc, global index asc) -- experience.cpp:177-187
// -- then order it by (reward asc, round asc, pick order) -- :290-294.
__global__ void merge_topk_kernel(const double* __restrict__ score, const double* __restrict__ sim,
                                  const double* __restrict__ rew, const int32_t* __restrict__ rnd,
                                  const int64_t* __restrict__ gidx, const size_t* __restrict__ cnt,
                                  int nshards, int nq, int m, int64_t* __restrict__ o_idx,
                                  double* __restrict__ o_sim, double* __restrict__ o_score,
                                  size_t* __restrict__ o_cnt) {
    extern __shared__ int picks_sh[];  // [m] pick order, then [m] curriculum order
    int* order = picks_sh + m;
    const int q = blockIdx.x;
    const int total = nshards * m;
    auto at = [&](int e) { return (size_t)(e / m) * nq * m + (size_t)q * m + (e % m); };
    auto valid = [&](int e) { return (size_t)(e % m) < cnt[(size_t)(e / m) * nq + q]; };
    int want = 0;
    for (int sh = 0; sh < nshards; ++sh) want += (int)cnt[(size_t)sh * nq + q];
    want = min(want, m);
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
        if (!valid(e)) continue;
        const size_t ie = at(e);
        const Best be{score[ie], rnd[ie], gidx[ie], 1};
        int rank = 0;
        for (int f = 0; f < total; ++f) {
            if (f == e || !valid(f)) continue;
            const size_t jf = at(f);
            rank += better(Best{score[jf], rnd[jf], gidx[jf], 1}, be);
        }
        if (rank < want) picks_sh[rank] = e;
    }
    __syncthreads();
    for (int x = threadIdx.x; x < want; x += blockDim.x) {
        const size_t v = at(picks_sh[x]);
        int pos = 0;
        for (int y = 0; y < want; ++y) {
            const size_t u = at(picks_sh[y]);
            const bool less = rew[u] != rew[v] ? rew[u] < rew[v] : rnd[u] < rnd[v];
            const bool same = rew[u] == rew[v] && rnd[u] == rnd[v];
            pos += less || (same && y < x);
        }
        order[pos] = picks_sh[x];
    }
    __syncthreads();
    for (int x = threadIdx.x; x < want; x += blockDim.x) {
        const size_t v = at(order[x]);
        o_idx[(size_t)q * m + x] = gidx[v];
        o_sim[(size_t)q * m + x] = sim[v];
        o_score[(size_t)q * m + x] = score[v];
    }
    if (threadIdx.x == 0) o_cnt[q] = want;
}

// The same merge on an all-gathered device buffer (sharded.py, NCCL):
// parts [nshards][nq][5m + 1] doubles per rank -- score[m], sim[m], reward[m],
// global index[m], round[m], count -- into out [nq][3m + 1]: index[m], sim[m],
// score[m], count.
__global__ void merge_packed_kernel(const double* __restrict__ parts, int nshards, int nq, int m,
                                    double* __restrict__ out) {
    extern __shared__ int picks_sh[];  // [m] pick order, then [m] curriculum order
    int* order = picks_sh + m;
    const int q = blockIdx.x;
    const int W = 5 * m + 1, total = nshards * m;
    auto row = [&](int sh) { return parts + ((size_t)sh * nq + q) * W; };
    auto cnt = [&](int sh) { return (int)row(sh)[5 * m]; };
    auto valid = [&](int e) { return e % m < cnt(e / m); };
    auto best_of = [&](int e) {
        const double* r = row(e / m);
        const int j = e % m;
        return Best{r[j], (int32_t)r[4 * m + j], (int64_t)r[3 * m + j], 1};
    };
    int want = 0;
    for (int sh = 0; sh < nshards; ++sh) want += cnt(sh);
    want = min(want, m);
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
        if (!valid(e)) continue;
        const Best be = best_of(e);
        int rank = 0;
        for (int f = 0; f < total; ++f) {
            if (f == e || !valid(f)) continue;
            rank += better(best_of(f), be);
        }
        if (rank < want) picks_sh[rank] = e;
    }
    __syncthreads();
    auto rw = [&](int e) { return row(e / m)[2 * m + e % m]; };
    auto rd = [&](int e) { return row(e / m)[4 * m + e % m]; };
    for (int x = threadIdx.x; x < want; x += blockDim.x) {
        const int v = picks_sh[x];
        int pos = 0;
        for (int y = 0; y < want; ++y) {
            const int u = picks_sh[y];
            const bool less = rw(u) != rw(v) ? rw(u) < rw(v) : rd(u) < rd(v);
            const bool same = rw(u) == rw(v) && rd(u) == rd(v);
            pos += less || (same && y < x);
        }
        order[pos] = v;
    }
    __syncthreads();
    double* o = out + (size_t)q * (3 * m + 1);
    for (int x = threadIdx.x; x < want; x += blockDim.x) {
        const double* r = row(order[x] / m);
        const int j = order[x] % m;
        o[x] = r[3 * m + j];
        o[m + x] = r[m + j];
        o[2 * m + x] = r[j];
    }
    if (threadIdx.x == 0) o[3 * m] = (double)want;
}

void merge_packed(const double* parts, size_t nshards, size_t nq, size_t m, int device,
                  cudaStream_t st, double* out) {
    if (nq == 0 || m == 0) return;
    DeviceGuard g(device);
    merge_packed_kernel<<<(int)nq, 256, 2 * m * sizeof(int), st>>>(parts, (int)nshards, (int)nq,
                                                                  (int)m, out);
    SAIR_LAUNCH("merge_packed_kernel");
}

void merge_topk(const double* score, const double* sim, const double* reward,
                const int32_t* round, const int64_t* gidx, const size_t* count, size_t nshards,
                size_t nq, size_t m, int device, int64_t* out_idx, double* out_sim,
                double* out_score, size_t* out_count) {
    if (nq == 0 || m == 0) {
        for (size_t q = 0; q < nq; ++q) out_count[q] = 0;
        return;
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        throw Error(SAIR_ECUDA, "no CUDA device (libsair has no CPU fallback)");
    DeviceGuard g(device);
    const size_t e = nshards * nq * m;
    DBuf b;
    char* base = static_cast<char*>(b.get(e * (8 * 4 + 4) + nshards * nq * 8 + nq * m * 24 +
                                          nq * 8 + 16 * 256));
    size_t off = 0;
    auto take = [&](size_t bytes) {
        char* ptr = base + off;
        off += (bytes + 255) / 256 * 256;
        return ptr;
    };
    auto* dsc = reinterpret_cast<double*>(take(e * 8));
    auto* dsi = reinterpret_cast<double*>(take(e * 8));
    auto* drw = reinterpret_cast<double*>(take(e * 8));
    auto* dgi = reinterpret_cast<int64_t*>(take(e * 8));
    auto* drd = reinterpret_cast<int32_t*>(take(e * 4));
    auto* dct = reinterpret_cast<size_t*>(take(nshards * nq * 8));
    auto* oi = reinterpret_cast<int64_t*>(take(nq * m * 8));
    auto* os = reinterpret_cast<double*>(take(nq * m * 8));
    auto* oc = reinterpret_cast<double*>(take(nq * m * 8));
    auto* on = reinterpret_cast<size_t*>(take(nq * 8));
    SAIR_CUDA(cudaMemcpy(dsc, score, e * 8, cudaMemcpyHostToDevice));
    SAIR_CUDA(cudaMemcpy(dsi, sim, e * 8, cudaMemcpyHostToDevice));
    SAIR_CUDA(cudaMemcpy(drw, reward, e * 8, cudaMemcpyHostToDevice));
    SAIR_CUDA(cudaMemcpy(dgi, gidx, e * 8, cudaMemcpyHostToDevice));
    SAIR_CUDA(cudaMemcpy(drd, round, e * 4, cudaMemcpyHostToDevice));
    SAIR_CUDA(cudaMemcpy(dct, count, nshards * nq * 8, cudaMemcpyHostToDevice));
    merge_topk_kernel<<<(int)nq, 256, 2 * m * sizeof(int)>>>(dsc, dsi, drw, drd, dgi, dct,
                                                            (int)nshards, (int)nq, (int)m, oi, os,
                                                            oc, on);
    SAIR_LAUNCH("merge_topk_kernel");
    SAIR_CUDA(cudaMemcpy(out_idx, oi, nq * m * 8, cudaMemcpyDeviceToHost));
    SAIR_CUDA(cudaMemcpy(out_sim, os, nq * m * 8, cudaMemcpyDeviceToHost));
    SAIR_CUDA(cudaMemcpy(out_score, oc, nq * m * 8, cudaMemcpyDeviceToHost));
    SAIR_CUDA(cudaMemcpy(out_count, on, nq * 8, cudaMemcpyDeviceToHost));
}

}  // namespace sair
