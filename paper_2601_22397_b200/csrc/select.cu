// select.cu -- surprisal-guided retrieval on the device.
//
// Restates ExperienceBuffer::select (experience.cpp:242-296), surprisal
// (:234-240) and the MockBackend veto scan (policy.cpp:140-157) as:
//
//   K3  stream_kernel   one HBM pass over the fp32 page copy of the store for a
//                       group of up to 8 queries: TMA bulk copies (cp.async.bulk
//                       + mbarrier ring) stage pages in shared memory, CUDA-core
//                       FFMAs compute d2 with the query constants in the
//                       constant bank, and every record's *upper-bound* log2
//                       score is thresholded into per-CTA candidate lists
//                       (warp-aggregated inserts, warp-level radix-select
//                       compaction).  Records never leave the chip.
//   merge_kernel        global top-K' per list across CTAs (block radix select).
//   refine_kernel       fp64 re-score of the K' candidates with the reference's
//                       exact rounding sequence, the greedy max-marginal-gain
//                       loop, certification against the filter's bound, the
//                       curriculum sort and the nearest-neighbour veto answer.
//   exact_*             full fp64 pass (fallback when a query cannot be
//                       certified, SAIR_SELECT_EXACT, locally_weighted_mean).
//
// Exactness argument: DESIGN.md "Exactness".
#include <algorithm>
#include <cfloat>
#include <cstring>
#include <vector>

#include "internal.hpp"

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

constexpr uint32_t NOIDX = 0xFFFFFFFFu;

// ------------------------------------------------- warp radix-select (smem) --
// Among the `cnt` entries (key, idx) of one candidate list, keep the K
// largest by (key desc, idx asc), compacted in place to [0, K).  Returns the
// ordinal f2ord() of the K-th kept key.  One warp; `hist` is 256 words.
__device__ uint32_t warp_keep_topk(float* key, uint32_t* idx, int cnt, int K, uint32_t* hist,
                                   int lane) {
    // pass A: radix select on the key ordinal (descending)
    uint32_t prefix = 0, pmask = 0;
    int r = K;
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int b = lane; b < 256; b += 32) hist[b] = 0;
        __syncwarp();
        for (int i = lane; i < cnt; i += 32) {
            uint32_t u = f2ord(key[i]);
            if ((u & pmask) == prefix) atomicAdd(&hist[(u >> shift) & 255u], 1u);
        }
        __syncwarp();
        uint32_t loc[8], sum = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            loc[j] = hist[255 - (lane * 8 + j)];
            sum += loc[j];
        }
        uint32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        uint32_t excl = incl - sum;
        unsigned own = __ballot_sync(0xffffffffu, excl < (uint32_t)r && (uint32_t)r <= incl);
        int owner = __ffs(own) - 1;
        int bin = 0;
        uint32_t above = 0;
        if (lane == owner) {
            uint32_t c = excl;
            for (int j = 0; j < 8; ++j) {
                if (c + loc[j] >= (uint32_t)r) {
                    bin = 255 - (lane * 8 + j);
                    above = c;
                    break;
                }
                c += loc[j];
            }
        }
        bin = __shfl_sync(0xffffffffu, bin, owner);
        above = __shfl_sync(0xffffffffu, above, owner);
        r -= (int)above;
        prefix |= (uint32_t)bin << shift;
        pmask |= 255u << shift;
        __syncwarp();
    }
    const uint32_t T = prefix;
    // r = how many entries equal to T are kept; count them
    int eq = 0;
    for (int i = lane; i < cnt; i += 32) eq += f2ord(key[i]) == T;
#pragma unroll
    for (int o = 16; o; o >>= 1) eq += __shfl_xor_sync(0xffffffffu, eq, o);
    // pass B (rare): among ties keep the r smallest idx -> threshold on ~idx
    uint32_t TI = 0;  // keep ties with ~idx >= TI
    if (eq > r) {
        uint32_t pre = 0, pm = 0;
        int rr = r;
        for (int shift = 24; shift >= 0; shift -= 8) {
            for (int b = lane; b < 256; b += 32) hist[b] = 0;
            __syncwarp();
            for (int i = lane; i < cnt; i += 32) {
                if (f2ord(key[i]) != T) continue;
                uint32_t u = ~idx[i];
                if ((u & pm) == pre) atomicAdd(&hist[(u >> shift) & 255u], 1u);
            }
            __syncwarp();
            uint32_t loc[8], sum = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                loc[j] = hist[255 - (lane * 8 + j)];
                sum += loc[j];
            }
            uint32_t incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            uint32_t excl = incl - sum;
            unsigned own = __ballot_sync(0xffffffffu, excl < (uint32_t)rr && (uint32_t)rr <= incl);
            int owner = __ffs(own) - 1;
            int bin = 0;
            uint32_t above = 0;
            if (lane == owner) {
                uint32_t c = excl;
                for (int j = 0; j < 8; ++j) {
                    if (c + loc[j] >= (uint32_t)rr) {
                        bin = 255 - (lane * 8 + j);
                        above = c;
                        break;
                    }
                    c += loc[j];
                }
            }
            bin = __shfl_sync(0xffffffffu, bin, owner);
            above = __shfl_sync(0xffffffffu, above, owner);
            rr -= (int)above;
            pre |= (uint32_t)bin << shift;
            pm |= 255u << shift;
            __syncwarp();
        }
        TI = pre;
    }
    // in-place compaction (writes never pass the read position)
    int w = 0;
    for (int base = 0; base < cnt; base += 32) {
        int i = base + lane;
        float kk = 0.f;
        uint32_t ii = 0;
        bool keep = false;
        if (i < cnt) {
            kk = key[i];
            ii = idx[i];
            uint32_t u = f2ord(kk);
            keep = u > T || (u == T && ~ii >= TI);
        }
        unsigned bal = __ballot_sync(0xffffffffu, keep);
        __syncwarp();
        if (keep) {
            int pos = w + __popc(bal & ((1u << lane) - 1u));
            key[pos] = kk;
            idx[pos] = ii;
        }
        w += __popc(bal);
        __syncwarp();
    }
    return T;
}

// ------------------------------------------------------------ K3 stream --

template <int DP, int QB>
struct StreamArgs {
    const float* pages;
    const float* r32;
    uint32_t n, npages;
    float c1, c0, rdelta, alpha;  // resid32 = |r c1 - c0|; key = log2(resid32+rdelta) - d2 alpha
    int kp, knn, nstage, cap_sel, cap_nn, kmax;
    float* out_key;  // [grid][2*QB][kmax]
    uint32_t* out_idx;
    float s[DP];      // 1/sd (0 on padding)
    float c[QB][DP];  // mean/sd + z_q (0 on padding)
};

template <int DP, int QB>
__global__ void __launch_bounds__(PAGE, 2)
    stream_kernel(const __grid_constant__ StreamArgs<DP, QB> a) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nl = a.knn ? 2 * QB : QB;
    const size_t stage_floats = (size_t)DP * PAGE;
    float* stage = reinterpret_cast<float*>(smem);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + a.nstage * stage_floats * 4);
    float* thr = reinterpret_cast<float*>(bars + 4);
    int* cnt = reinterpret_cast<int*>(thr + 2 * QB);
    uint32_t* hist = reinterpret_cast<uint32_t*>(cnt + 2 * QB);
    float* lkey = reinterpret_cast<float*>(hist + 4 * 256);
    const int total_cap = QB * a.cap_sel + (a.knn ? QB * a.cap_nn : 0);
    uint32_t* lidx = reinterpret_cast<uint32_t*>(lkey + total_cap);
    auto lbase = [&](int L) { return L < QB ? L * a.cap_sel : QB * a.cap_sel + (L - QB) * a.cap_nn; };
    auto lcap = [&](int L) { return L < QB ? a.cap_sel : a.cap_nn; };
    auto lk = [&](int L) { return L < QB ? a.kp : a.knn; };

    if (tid < 2 * QB) {
        thr[tid] = -INFINITY;
        cnt[tid] = 0;
    }
    if (tid == 0) {
        for (int s = 0; s < a.nstage; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const uint32_t G = gridDim.x, p0 = blockIdx.x;
    const uint32_t count = p0 < a.npages ? (a.npages - 1 - p0) / G + 1 : 0;
    const uint32_t bytes = (uint32_t)(stage_floats * 4);
    if (tid == 0) {
        for (int s = 0; s < a.nstage && (uint32_t)s < count; ++s) {
            mbar_expect_tx(&bars[s], bytes);
            bulk_g2s(stage + s * stage_floats, a.pages + (size_t)(p0 + s * G) * stage_floats,
                     bytes, &bars[s]);
        }
    }

    for (uint32_t it = 0; it < count; ++it) {
        const int s = it % a.nstage;
        const uint32_t page = p0 + it * G;
        const uint32_t rec = page * PAGE + tid;
        const bool valid = rec < a.n;
        const float r = valid ? __ldg(a.r32 + rec) : 0.f;
        mbar_wait(&bars[s], (it / a.nstage) & 1u);
        const float* buf = stage + s * stage_floats;
        float acc[QB];
#pragma unroll
        for (int q = 0; q < QB; ++q) acc[q] = 0.f;
#pragma unroll
        for (int k = 0; k < DP; ++k) {
            // y = x / sd once per record (not contracted), then one FADD with
            // the query constant as a constant-bank operand and one FFMA
            const float y = __fmul_rn(buf[k * PAGE + tid], a.s[k]);
#pragma unroll
            for (int q = 0; q < QB; ++q) {
                const float t = y - a.c[q][k];
                acc[q] = fmaf(t, t, acc[q]);
            }
        }
        const float lg = log2f(fabsf(fmaf(r, a.c1, -a.c0)) + a.rdelta);
#pragma unroll
        for (int q = 0; q < QB; ++q) {
            const float key = fmaf(-acc[q], a.alpha, lg);
            bool pass = valid && (key > thr[q] || thr[q] == -INFINITY);
            unsigned bal = __ballot_sync(0xffffffffu, pass);
            if (bal) {
                int leader = __ffs(bal) - 1, base = 0;
                if (lane == leader) base = atomicAdd(&cnt[q], __popc(bal));
                base = __shfl_sync(0xffffffffu, base, leader);
                if (pass) {
                    int pos = lbase(q) + base + __popc(bal & ((1u << lane) - 1u));
                    lkey[pos] = key;
                    lidx[pos] = rec;
                }
            }
        }
        if (a.knn) {
#pragma unroll
            for (int q = 0; q < QB; ++q) {
                const int L = QB + q;
                const float key = -acc[q];
                bool pass = valid && (key > thr[L] || thr[L] == -INFINITY);
                unsigned bal = __ballot_sync(0xffffffffu, pass);
                if (bal) {
                    int leader = __ffs(bal) - 1, base = 0;
                    if (lane == leader) base = atomicAdd(&cnt[L], __popc(bal));
                    base = __shfl_sync(0xffffffffu, base, leader);
                    if (pass) {
                        int pos = lbase(L) + base + __popc(bal & ((1u << lane) - 1u));
                        lkey[pos] = key;
                        lidx[pos] = rec;
                    }
                }
            }
        }
        __syncthreads();  // stage s consumed; list counters settled
        if (tid == 0 && it + a.nstage < count) {
            mbar_expect_tx(&bars[s], bytes);
            bulk_g2s(stage + s * stage_floats,
                     a.pages + (size_t)(p0 + (it + a.nstage) * G) * stage_floats, bytes, &bars[s]);
        }
        bool need = false;
        for (int L = 0; L < nl; ++L) need |= cnt[L] > lcap(L) - PAGE;
        if (need) {
            for (int L = warp; L < nl; L += 4) {
                if (cnt[L] > lcap(L) - PAGE) {
                    uint32_t T = warp_keep_topk(lkey + lbase(L), lidx + lbase(L), cnt[L], lk(L),
                                                hist + warp * 256, lane);
                    if (lane == 0) {
                        cnt[L] = lk(L);
                        thr[L] = ord2f(T);
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int L = warp; L < nl; L += 4) {
        if (cnt[L] > lk(L)) {
            uint32_t T = warp_keep_topk(lkey + lbase(L), lidx + lbase(L), cnt[L], lk(L),
                                        hist + warp * 256, lane);
            if (lane == 0) {
                cnt[L] = lk(L);
                thr[L] = ord2f(T);
            }
        }
    }
    __syncthreads();
    for (int L = 0; L < nl; ++L) {
        float* ok = a.out_key + ((size_t)blockIdx.x * 2 * QB + L) * a.kmax;
        uint32_t* oi = a.out_idx + ((size_t)blockIdx.x * 2 * QB + L) * a.kmax;
        for (int j = tid; j < lk(L); j += PAGE) {
            bool have = j < cnt[L];
            ok[j] = have ? lkey[lbase(L) + j] : -INFINITY;
            oi[j] = have ? lidx[lbase(L) + j] : NOIDX;
        }
    }
}

// ------------------------------------------------------------ merge --------
// Global top-K (key desc, idx asc) of list L across all CTAs; output sorted.
// Also returns the K-th key (the filter threshold U) per list.
__global__ void __launch_bounds__(512)
    merge_kernel(const float* __restrict__ in_key, const uint32_t* __restrict__ in_idx, int G,
                 int lists_stride, int kmax, int QB, int kp, int knn, float* __restrict__ out_key,
                 uint32_t* __restrict__ out_idx, float* __restrict__ out_thr) {
    const int L = blockIdx.x;
    const int K = L < QB ? kp : knn;
    const int total = G * K;
    __shared__ uint32_t hist[256];
    __shared__ uint32_t sh_prefix, sh_r, sh_cnt;
    __shared__ unsigned long long skey[1024];  // K <= 512 -> pow2 <= 1024
    const int tid = threadIdx.x;
    auto get = [&](int e, float& k, uint32_t& i) {
        int g = e / K, j = e % K;
        size_t off = ((size_t)g * lists_stride + L) * kmax + j;
        k = in_key[off];
        i = in_idx[off];
    };
    // radix select on (ordinal key) then (~idx): a 64-bit composite, 8 digits
    uint64_t prefix = 0, pmask = 0;
    uint32_t r = (uint32_t)min(K, total);
    for (int shift = 56; shift >= 0; shift -= 8) {
        for (int b = tid; b < 256; b += blockDim.x) hist[b] = 0;
        __syncthreads();
        for (int e = tid; e < total; e += blockDim.x) {
            float k;
            uint32_t i;
            get(e, k, i);
            uint64_t u = ((uint64_t)f2ord(k) << 32) | (uint64_t)(~i);
            if ((u & pmask) == prefix) atomicAdd(&hist[(u >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (tid < 32) {
            int lane = tid;
            uint32_t loc[8], sum = 0;
            for (int j = 0; j < 8; ++j) {
                loc[j] = hist[255 - (lane * 8 + j)];
                sum += loc[j];
            }
            uint32_t incl = sum;
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            uint32_t excl = incl - sum;
            unsigned own = __ballot_sync(0xffffffffu, excl < r && r <= incl);
            int owner = __ffs(own) - 1;
            if (lane == owner) {
                uint32_t c = excl;
                for (int j = 0; j < 8; ++j) {
                    if (c + loc[j] >= r) {
                        sh_prefix = 255 - (lane * 8 + j);
                        sh_r = r - c;
                        break;
                    }
                    c += loc[j];
                }
            }
        }
        __syncthreads();
        prefix |= (uint64_t)sh_prefix << shift;
        pmask |= 255ull << shift;
        r = sh_r;
        __syncthreads();
    }
    // composite keys are unique -> exactly K entries are >= prefix
    if (tid == 0) sh_cnt = 0;
    int P = 1;
    while (P < K) P <<= 1;
    for (int j = tid; j < P; j += blockDim.x) skey[j] = 0ull;
    __syncthreads();
    for (int e = tid; e < total; e += blockDim.x) {
        float k;
        uint32_t i;
        get(e, k, i);
        uint64_t u = ((uint64_t)f2ord(k) << 32) | (uint64_t)(~i);
        if (u > prefix) skey[atomicAdd(&sh_cnt, 1u)] = u;  // fewer than K by definition
    }
    __syncthreads();
    // the K-th composite is unique for a real entry; only padding repeats
    for (int j = sh_cnt + tid; j < K; j += blockDim.x) skey[j] = prefix;
    __syncthreads();
    // bitonic sort descending
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = tid; t < P / 2; t += blockDim.x) {
                int pos = 2 * stride * (t / stride) + (t % stride);
                int partner = pos + stride;
                bool desc = ((pos & size) == 0);
                unsigned long long x = skey[pos], y = skey[partner];
                if ((x < y) == desc) {
                    skey[pos] = y;
                    skey[partner] = x;
                }
            }
            __syncthreads();
        }
    }
    for (int j = tid; j < K; j += blockDim.x) {
        unsigned long long u = skey[j];
        out_key[(size_t)L * kmax + j] = ord2f((uint32_t)(u >> 32));
        out_idx[(size_t)L * kmax + j] = ~(uint32_t)(u & 0xffffffffu);
    }
    if (tid == 0) out_thr[L] = ord2f((uint32_t)(prefix >> 32));
}

// ------------------------------------------------------------ refine -------

struct RefineArgs {
    const double* x64;
    const double* r64;
    const int32_t* rnd;
    const double* mean;  // [d]
    const double* sd;    // [d]
    const double* zq;    // [QB][d]
    const double* eq;    // [QB] additive d2 error bound E_q
    int d, m, kp, knn, QB, kmax;
    size_t n;
    double total, two_s2, lambda, log2e_over_2s2, d2_rel;
    int has_excl, has_excl_nn;
    const float* ckey;
    const uint32_t* cidx;  // merged, sorted [2QB][kmax]
    const float* cthr;     // [2QB]
    double* zs;            // scratch [QB][kp][d]
    int64_t gbase;
    // outputs per query (group-local q)
    int64_t* out_idx;  // [QB][m]
    double* out_sim;
    double* out_score;
    int* out_count;
    int* out_cert;
    int64_t* out_nn;
    double* out_nn_sim;
    int* out_nn_cert;
};

struct Best {
    double g;
    int32_t r;
    int64_t i;
    int j;
};
__device__ __forceinline__ bool better(const Best& a, const Best& b) {
    // (gain desc, round asc, index asc): experience.cpp:268-278
    if (a.j < 0) return false;
    if (b.j < 0) return true;
    if (a.g > b.g) return true;
    if (a.g < b.g) return false;
    if (a.r != b.r) return a.r < b.r;
    return a.i < b.i;
}
__device__ Best warp_best(Best b) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        Best c;
        c.g = __shfl_xor_sync(0xffffffffu, b.g, o);
        c.r = __shfl_xor_sync(0xffffffffu, b.r, o);
        c.i = __shfl_xor_sync(0xffffffffu, b.i, o);
        c.j = __shfl_xor_sync(0xffffffffu, b.j, o);
        if (better(c, b)) b = c;
    }
    return b;
}

__global__ void __launch_bounds__(256) refine_kernel(const RefineArgs a) {
    const int q = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    extern __shared__ __align__(16) unsigned char sm[];
    double* score = reinterpret_cast<double*>(sm);
    double* simc = score + a.kp;
    double* pen = simc + a.kp;
    int32_t* rr = reinterpret_cast<int32_t*>(pen + a.kp);
    int* taken = rr + a.kp;
    int* picks = taken + a.kp;
    __shared__ Best wb[8];
    __shared__ int s_cert;
    const int d = a.d;
    const double* zq = a.zq + (size_t)q * d;
    double* zs = a.zs + (size_t)q * a.kp * d;
    const uint32_t* ci = a.cidx + (size_t)q * a.kmax;

    // exact score of every candidate: experience.cpp:254-258 with the
    // reference's rounding sequence (standardize :162-166, similarity :125-130,
    // loo_mean :229-231)
    for (int j = tid; j < a.kp; j += blockDim.x) {
        uint32_t i = ci[j];
        taken[j] = 0;
        pen[j] = 0.0;
        if (i == NOIDX) {
            score[j] = -INFINITY;
            rr[j] = INT32_MAX;
            taken[j] = 1;
            continue;
        }
        double d2 = 0.0;
        for (int k = 0; k < d; ++k) {
            double z = ddiv(dsub(a.x64[(size_t)i * d + k], a.mean[k]), a.sd[k]);
            zs[(size_t)j * d + k] = z;
            double t = dsub(z, zq[k]);
            d2 = dadd(d2, dmul(t, t));
        }
        double sim = sim_from_d2(d2, a.two_s2);
        double r = a.r64[i];
        double loo = a.n <= 1 ? 0.0 : ddiv(dsub(a.total, r), (double)(a.n - 1));
        simc[j] = sim;
        score[j] = dmul(sim, fabs(dsub(r, loo)));
        rr[j] = a.rnd[i];
    }
    if (tid == 0) s_cert = 1;
    __syncthreads();

    // any record outside the pool has score <= 2^(U + slack)
    double bound = -1.0;
    if (a.has_excl) {
        double U = (double)a.cthr[q];
        double key = U + a.eq[q] * a.log2e_over_2s2 + 1e-5 * (fabs(U) + 1.0) + 1e-6;
        bound = exp2(key);
    }
    const int want = (int)min((size_t)a.m, a.n);
    for (int step = 0; step < want; ++step) {
        Best b{0.0, 0, 0, -1};
        for (int j = tid; j < a.kp; j += blockDim.x) {
            if (taken[j]) continue;
            Best c{dsub(score[j], dmul(a.lambda, pen[j])), rr[j], (int64_t)ci[j], j};
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
        if (a.lambda != 0.0) {
            const int jb = picks[step];
            const double* zb = zs + (size_t)jb * d;
            for (int j = tid; j < a.kp; j += blockDim.x) {
                if (taken[j]) continue;
                const double* zj = zs + (size_t)j * d;
                double d2 = 0.0;
                for (int k = 0; k < d; ++k) {
                    double t = dsub(zj[k], zb[k]);
                    d2 = dadd(d2, dmul(t, t));
                }
                pen[j] = dadd(pen[j], sim_from_d2(d2, a.two_s2));
            }
            __syncthreads();
        }
    }
    if (tid == 0) {
        // curriculum order: stable sort by (reward asc, round asc), :290-294
        for (int x = 1; x < want; ++x) {
            int v = picks[x], y = x;
            double rv = a.r64[ci[v]];
            while (y > 0) {
                int u = picks[y - 1];
                double ru = a.r64[ci[u]];
                bool less = rv != ru ? rv < ru : rr[v] < rr[u];
                if (!less) break;
                picks[y] = u;
                --y;
            }
            picks[y] = v;
        }
        for (int x = 0; x < want; ++x) {
            int j = picks[x];
            a.out_idx[(size_t)q * a.m + x] = a.gbase + (int64_t)ci[j];
            a.out_sim[(size_t)q * a.m + x] = simc[j];
            a.out_score[(size_t)q * a.m + x] = score[j];
        }
        a.out_count[q] = want;
        a.out_cert[q] = s_cert;
    }
    if (a.knn == 0) return;
    __syncthreads();
    // nearest neighbour by exact similarity; first index wins ties (policy.cpp:146-153)
    const uint32_t* ni = a.cidx + (size_t)(a.QB + q) * a.kmax;
    Best b{0.0, 0, 0, -1};
    for (int j = tid; j < a.knn; j += blockDim.x) {
        uint32_t i = ni[j];
        if (i == NOIDX) continue;
        double d2 = 0.0;
        for (int k = 0; k < d; ++k) {
            double z = ddiv(dsub(a.x64[(size_t)i * d + k], a.mean[k]), a.sd[k]);
            double t = dsub(z, zq[k]);
            d2 = dadd(d2, dmul(t, t));
        }
        Best c{sim_from_d2(d2, a.two_s2), 0, (int64_t)i, j};
        if (better(c, b)) b = c;
    }
    b = warp_best(b);
    if (lane == 0) wb[warp] = b;
    __syncthreads();
    if (tid == 0) {
        Best c = wb[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
            if (better(wb[w], c)) c = wb[w];
        int cert = 1;
        if (a.has_excl_nn) {
            // excluded records have d2_32 >= D = -U_nn; true d2 >= D (1 - rel) - E_q
            double D = -(double)a.cthr[a.QB + q];
            double lo = D * (1.0 - a.d2_rel) - a.eq[q];
            if (lo < 0.0) lo = 0.0;
            double bnd = exp(-lo / a.two_s2) * (1.0 + 1e-12);
            cert = c.g > bnd;
        }
        a.out_nn[q] = a.gbase + c.i;
        a.out_nn_sim[q] = c.g;
        a.out_nn_cert[q] = cert;
    }
}

// ------------------------------------------------------- exact fallback ----

struct ExactArgs {
    const double* x64;
    const double* r64;
    const int32_t* rnd;
    const double* mean;
    const double* sd;
    const double* zq;  // [d]
    int d;
    size_t n;
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
                           : (a.n <= 1 ? 0.0 : ddiv(dsub(a.total, r), (double)(a.n - 1)));
        a.sim[i] = s;
        a.score[i] = dmul(s, fabs(dsub(r, loo)));
        a.pen[i] = 0.0;
        a.taken[i] = 0;
    }
}

// locally weighted leave-one-out mean, experience.cpp:216-228 (sequential in j
// per record, so the sums round exactly as the reference's loop)
__global__ void local_loo_kernel(const ExactArgs a, double* __restrict__ loo) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < a.n;
         i += (size_t)gridDim.x * blockDim.x) {
        if (a.n <= 1) {
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
                              : ddiv(dsub(a.total, a.r64[i]), (double)(a.n - 1));
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
                                    int64_t* out_idx, double* out_sim, double* out_score) {
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
    if (a.n <= 1) {
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
        loo = wsum > 1e-12 ? ddiv(acc, wsum) : ddiv(dsub(a.total, r), (double)(a.n - 1));
    } else {
        loo = ddiv(dsub(a.total, r), (double)(a.n - 1));
    }
    *out = dmul(s, fabs(dsub(r, loo)));
}

// --------------------------------------------------------------- host ------

namespace {

struct QueryPrep {
    std::vector<double> mean, sd, z;  // z: [nq][d]
    double sigma = 1.0, two_s2 = 2.0;
};

QueryPrep prep_queries(sair_store_s* s, const double* q, size_t nq, double sigma) {
    QueryPrep p;
    int d = s->d;
    p.mean.resize(d);
    p.sd.resize(d);
    store_mean_sd(s, p.mean.data(), p.sd.data());
    p.z.resize(nq * d);
    for (size_t i = 0; i < nq; ++i)
        for (int k = 0; k < d; ++k)  // standardize, experience.cpp:166
            p.z[i * d + k] = (q[i * d + k] - p.mean[k]) / p.sd[k];
    p.sigma = sigma;
    p.two_s2 = 2.0 * sigma * sigma;  // experience.cpp:130
    return p;
}

// Exact full-pass answer for one query (fp64 over x64), writing m results.
void exact_one(sair_store_s* s, const QueryPrep& p, const double* zq_host, size_t m,
               double lambda, bool local, int64_t* o_idx, double* o_sim, double* o_score,
               size_t* o_cnt, int64_t* o_nn, double* o_nn_sim) {
    const size_t n = s->n;
    const int d = s->d;
    char* base = static_cast<char*>(
        s->b_exact.get(n * (8 * 4 + 1) + (size_t)d * 8 * 3 + 4096 * sizeof(Best) + 64 * 1024 +
                       m * 8 * 4 + 256));
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
    a.total = s->stats.total;
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
    std::vector<double> h(3 * (size_t)d);
    std::copy(p.mean.begin(), p.mean.end(), h.begin());
    std::copy(p.sd.begin(), p.sd.end(), h.begin() + d);
    std::copy(zq_host, zq_host + d, h.begin() + 2 * d);
    SAIR_CUDA(cudaMemcpyAsync(dm, h.data(), h.size() * 8, cudaMemcpyHostToDevice, s->st));
    const int threads = 256;
    const int blocks = (int)std::min<size_t>((n + threads - 1) / threads, 4096);
    if (local) {
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
        exact_finish_kernel<<<1, 32, 0, s->st>>>(a, picks, (int)want, s->gbase, didx, dsim, dscore);
        SAIR_LAUNCH("exact_finish_kernel");
        SAIR_CUDA(cudaMemcpyAsync(o_idx, didx, want * 8, cudaMemcpyDeviceToHost, s->st));
        SAIR_CUDA(cudaMemcpyAsync(o_sim, dsim, want * 8, cudaMemcpyDeviceToHost, s->st));
        SAIR_CUDA(cudaMemcpyAsync(o_score, dscore, want * 8, cudaMemcpyDeviceToHost, s->st));
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

template <int DP, int QB>
void launch_stream(sair_store_s* s, const QueryPrep& p, const double* zgrp, int nqg, int kp,
                   int knn, int nstage, int grid, size_t smem, float c1, float c0, float rdelta,
                   float alpha, float* ck, uint32_t* ci, int kmax, int cap_sel, int cap_nn) {
    StreamArgs<DP, QB> a{};
    a.pages = s->pages;
    a.r32 = s->r32;
    a.n = (uint32_t)s->n;
    a.npages = (uint32_t)((s->n + PAGE - 1) / PAGE);
    a.c1 = c1;
    a.c0 = c0;
    a.rdelta = rdelta;
    a.alpha = alpha;
    a.kp = kp;
    a.knn = knn;
    a.nstage = nstage;
    a.cap_sel = cap_sel;
    a.cap_nn = cap_nn;
    a.kmax = kmax;
    a.out_key = ck;
    a.out_idx = ci;
    const int d = s->d;
    for (int k = 0; k < DP; ++k) a.s[k] = k < d ? (float)(1.0 / p.sd[k]) : 0.f;
    for (int q = 0; q < QB; ++q)
        for (int k = 0; k < DP; ++k) {
            // padded query slots repeat query 0 (their lists are ignored)
            const double* z = zgrp + (size_t)(q < nqg ? q : 0) * d;
            a.c[q][k] = k < d ? (float)(p.mean[k] / p.sd[k] + z[k]) : 0.f;
        }
    static bool attr_set[1] = {false};
    (void)attr_set;
    SAIR_CUDA(cudaFuncSetAttribute(stream_kernel<DP, QB>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    stream_kernel<DP, QB><<<grid, PAGE, smem, s->st>>>(a);
    SAIR_LAUNCH("stream_kernel");
}

using LaunchFn = void (*)(sair_store_s*, const QueryPrep&, const double*, int, int, int, int, int,
                          size_t, float, float, float, float, float*, uint32_t*, int, int, int);

template <int DP>
LaunchFn pick_qb(int qb) {
    switch (qb) {
        case 1: return launch_stream<DP, 1>;
        case 2: return launch_stream<DP, 2>;
        case 4: return launch_stream<DP, 4>;
        default: return launch_stream<DP, 8>;
    }
}
LaunchFn pick_launch(int dp, int qb) {
    switch (dp) {
        case 8: return pick_qb<8>(qb);
        case 16: return pick_qb<16>(qb);
        case 32: return pick_qb<32>(qb);
        case 64: return pick_qb<64>(qb);
        case 128: return pick_qb<128>(qb);
        default: return nullptr;
    }
}

}  // namespace

void store_select(sair_store_s* s, const double* q, size_t nq, int dim,
                  const sair_select_config& cfg, int64_t* out_idx, double* out_sim, double* out_score, size_t* out_count,
                  int64_t* out_nn, double* out_nn_sim) {
    s->last = sair_select_stats{};
    s->last.queries = nq;
    if (nq == 0) return;
    const size_t m = cfg.m;
    if (s->n == 0 || m == 0) {  // experience.cpp:245
        for (size_t i = 0; i < nq; ++i) out_count[i] = 0;
        if (out_nn)
            for (size_t i = 0; i < nq; ++i) {
                out_nn[i] = -1;
                out_nn_sim[i] = -1.0;
            }
        return;
    }
    DeviceGuard g(s->device);
    const double sigma = store_effective_sigma(s, cfg.sigma_sim);  // :246
    if (dim != s->d)  // standardize(x_curr) throws after the sigma refresh (:157-158)
        throw Error(SAIR_EINVAL, "experience store: feature dimension mismatch");
    QueryPrep p = prep_queries(s, q, nq, sigma);
    const int d = s->d;
    const size_t n = s->n;
    SAIR_CUDA(cudaEventRecord(s->ev[0], s->st));

    std::vector<int> done(nq, 0);
    const bool fast = cfg.mode != SAIR_SELECT_EXACT && !cfg.locally_weighted_mean && d <= 128 &&
                      n < (size_t)UINT32_MAX - PAGE && m <= 256;
    float stream_ms = 0.f;
    if (fast) {
        // candidate pool sizes
        int kp = 32;
        size_t want_pool = cfg.lambda_div != 0.0 ? 4 * m : 2 * m;
        while ((size_t)kp < want_pool && kp < 512) kp <<= 1;
        const int knn = out_nn ? 16 : 0;
        const int kmax = std::max(kp, knn);
        const int qb = nq >= 8 ? 8 : (nq >= 4 ? 4 : (nq >= 2 ? 2 : 1));
        const int dp = s->dp;
        const int cap_sel = kp + 2 * PAGE, cap_nn = knn + 2 * PAGE;
        const size_t stage_bytes = (size_t)dp * PAGE * 4;
        int nstage = (int)std::max<size_t>(2, std::min<size_t>(4, 65536 / stage_bytes));
        const size_t list_bytes =
            (size_t)qb * cap_sel * 8 + (knn ? (size_t)qb * cap_nn * 8 : 0);
        size_t smem = nstage * stage_bytes + 4 * 8 + 2 * 16 * 4 + 4 * 256 * 4 + list_bytes;
        if (smem > 200 * 1024) {
            nstage = 2;
            smem = nstage * stage_bytes + 4 * 8 + 2 * 16 * 4 + 4 * 256 * 4 + list_bytes;
        }
        int nsm = 148;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, s->device);
        const int per_sm = smem <= 110 * 1024 ? 2 : 1;
        const size_t npages = (n + PAGE - 1) / PAGE;
        const int grid = (int)std::max<size_t>(1, std::min<size_t>(npages, (size_t)nsm * per_sm));
        LaunchFn launch = pick_launch(dp, qb);

        // filter constants
        const double u = 0x1p-24;
        float c1 = 1.f, c0 = 0.f;
        double c1d = 1.0, c0d = 0.0;
        if (n >= 2) {
            c1d = (double)n / (double)(n - 1);
            c0d = s->stats.total / (double)(n - 1);
            c1 = (float)c1d;
            c0 = (float)c0d;
        }
        const float rdelta =
            (float)(4.0 * u * (s->stats.rabs * c1d + std::fabs(c0d)) * 1.01) + 1e-30f;
        const double log2e_over_2s2 = 1.4426950408889634 / p.two_s2;
        const double d2_rel = (dp + 3) * u;
        const float alpha = (float)(log2e_over_2s2 * (1.0 - d2_rel));

        // device buffers
        float* ck = s->b_cand.as<float>((size_t)grid * 2 * qb * kmax * 2);
        uint32_t* ci = reinterpret_cast<uint32_t*>(ck + (size_t)grid * 2 * qb * kmax);
        float* mk = s->b_merged.as<float>((size_t)2 * qb * kmax * 2 + 2 * qb);
        uint32_t* mi = reinterpret_cast<uint32_t*>(mk + (size_t)2 * qb * kmax);
        float* mthr = reinterpret_cast<float*>(mi + (size_t)2 * qb * kmax);
        double* zs = s->b_z.as<double>((size_t)qb * kp * d);
        // consts: mean, sd, zq[qb][d], eq[qb]
        double* dc = s->b_consts.as<double>(2 * (size_t)d + (size_t)qb * d + qb);
        // outputs
        const size_t ob = (size_t)qb * m * 8 * 3 + (size_t)qb * 8 * 2 + (size_t)qb * 4 * 4 + 64;
        char* dout = static_cast<char*>(s->b_out.get(ob));
        char* hout = static_cast<char*>(s->h_out.get(ob));
        auto carve = [&](char* b) {
            struct O {
                int64_t* idx;
                double* sim;
                double* score;
                int64_t* nn;
                double* nn_sim;
                int* cnt;
                int* cert;
                int* nn_cert;
            } o;
            o.idx = reinterpret_cast<int64_t*>(b);
            o.sim = reinterpret_cast<double*>(o.idx + qb * m);
            o.score = o.sim + qb * m;
            o.nn = reinterpret_cast<int64_t*>(o.score + qb * m);
            o.nn_sim = reinterpret_cast<double*>(o.nn + qb);
            o.cnt = reinterpret_cast<int*>(o.nn_sim + qb);
            o.cert = o.cnt + qb;
            o.nn_cert = o.cert + qb;
            return o;
        };
        auto D = carve(dout);
        auto H = carve(hout);
        std::vector<double> hc(2 * (size_t)d + (size_t)qb * d + qb);
        std::copy(p.mean.begin(), p.mean.end(), hc.begin());
        std::copy(p.sd.begin(), p.sd.end(), hc.begin() + d);
        const size_t refine_smem = (size_t)kp * (8 * 3 + 4 * 3) + 64;
        const int smem_refine_limit = (int)refine_smem;
        SAIR_CUDA(cudaFuncSetAttribute(refine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       smem_refine_limit));

        s->last.candidates = kp;
        s->last.qb = qb;
        for (size_t g0 = 0; g0 < nq; g0 += qb) {
            const int nqg = (int)std::min<size_t>(qb, nq - g0);
            const double* zgrp = p.z.data() + g0 * d;
            // per-query d2 error bound E_q = 6.01 u sum_k A_k^2 (+ slack)
            for (int qq = 0; qq < qb; ++qq) {
                const double* z = zgrp + (size_t)(qq < nqg ? qq : 0) * d;
                double sa = 0.0;
                for (int k = 0; k < d; ++k) {
                    double sk = 1.0 / p.sd[k];
                    double ck2 = std::fabs(p.mean[k] / p.sd[k] + z[k]);
                    double A = s->stats.xabs[k] * sk * (1.0 + 2 * u) + ck2 * (1.0 + 2 * u);
                    sa += A * A;
                }
                hc[2 * (size_t)d + (size_t)qb * d + qq] = 6.02 * u * sa * (1.0 + 1e-6) + 1e-300;
                for (int k = 0; k < d; ++k) hc[2 * (size_t)d + (size_t)qq * d + k] = z[k];
            }
            SAIR_CUDA(cudaMemcpyAsync(dc, hc.data(), hc.size() * 8, cudaMemcpyHostToDevice, s->st));
            SAIR_CUDA(cudaEventRecord(s->ev[1], s->st));
            launch(s, p, zgrp, nqg, kp, knn, nstage, grid, smem, c1, c0, rdelta, alpha, ck, ci,
                   kmax, cap_sel, cap_nn);
            SAIR_CUDA(cudaEventRecord(s->ev[2], s->st));
            s->last.stream_launches++;
            merge_kernel<<<knn ? 2 * qb : qb, 512, 0, s->st>>>(ck, ci, grid, 2 * qb, kmax, qb, kp,
                                                              knn, mk, mi, mthr);
            SAIR_LAUNCH("merge_kernel");
            RefineArgs ra{};
            ra.x64 = s->x64;
            ra.r64 = s->r64;
            ra.rnd = s->rnd;
            ra.mean = dc;
            ra.sd = dc + d;
            ra.zq = dc + 2 * d;
            ra.eq = dc + 2 * d + (size_t)qb * d;
            ra.d = d;
            ra.m = (int)m;
            ra.kp = kp;
            ra.knn = knn;
            ra.QB = qb;
            ra.kmax = kmax;
            ra.n = n;
            ra.total = s->stats.total;
            ra.two_s2 = p.two_s2;
            ra.lambda = cfg.lambda_div;
            ra.log2e_over_2s2 = log2e_over_2s2;
            ra.d2_rel = d2_rel;
            ra.has_excl = n > (size_t)kp;
            ra.has_excl_nn = n > (size_t)knn;
            ra.ckey = mk;
            ra.cidx = mi;
            ra.cthr = mthr;
            ra.zs = zs;
            ra.gbase = s->gbase;
            ra.out_idx = D.idx;
            ra.out_sim = D.sim;
            ra.out_score = D.score;
            ra.out_count = D.cnt;
            ra.out_cert = D.cert;
            ra.out_nn = D.nn;
            ra.out_nn_sim = D.nn_sim;
            ra.out_nn_cert = D.nn_cert;
            refine_kernel<<<nqg, 256, refine_smem, s->st>>>(ra);
            SAIR_LAUNCH("refine_kernel");
            SAIR_CUDA(cudaMemcpyAsync(hout, dout, ob, cudaMemcpyDeviceToHost, s->st));
            SAIR_CUDA(cudaStreamSynchronize(s->st));
            float ms = 0.f;
            cudaEventElapsedTime(&ms, s->ev[1], s->ev[2]);
            stream_ms += ms;
            for (int qq = 0; qq < nqg; ++qq) {
                size_t gq = g0 + qq;
                bool ok = H.cert[qq] && (!out_nn || H.nn_cert[qq]);
                if (!ok) continue;
                done[gq] = 1;
                out_count[gq] = (size_t)H.cnt[qq];
                std::memcpy(out_idx + gq * m, H.idx + (size_t)qq * m, H.cnt[qq] * 8);
                std::memcpy(out_sim + gq * m, H.sim + (size_t)qq * m, H.cnt[qq] * 8);
                std::memcpy(out_score + gq * m, H.score + (size_t)qq * m, H.cnt[qq] * 8);
                if (out_nn) {
                    out_nn[gq] = H.nn[qq];
                    out_nn_sim[gq] = H.nn_sim[qq];
                }
                s->last.certified++;
            }
        }
    }
    for (size_t i = 0; i < nq; ++i) {
        if (done[i]) continue;
        exact_one(s, p, p.z.data() + i * d, m, cfg.lambda_div, cfg.locally_weighted_mean != 0,
                  out_idx + i * m, out_sim + i * m, out_score + i * m, &out_count[i],
                  out_nn ? out_nn + i : nullptr, out_nn ? out_nn_sim + i : nullptr);
        s->last.exact_fallbacks++;
    }
    SAIR_CUDA(cudaEventRecord(s->ev[3], s->st));
    SAIR_CUDA(cudaEventSynchronize(s->ev[3]));
    float tot = 0.f;
    cudaEventElapsedTime(&tot, s->ev[0], s->ev[3]);
    s->last.stream_ms = stream_ms;
    s->last.total_ms = tot;
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
    a.total = s->stats.total;
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
