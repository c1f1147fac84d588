// select_mma.cu -- K3 on the 5th-generation tensor cores.
//
// The streaming filter's dominant work is the contraction
//   D[record][q] = sum_k x[record][k] * b[k][q],   b[k][q] = -2 c_qk / sd_k
// (the cross term of ||y - c_q||^2).  Here it runs as tcgen05.mma kind::tf32:
//
//   warp 8 (producer)  one bulk copy (cp.async.bulk, the TMA engine) per page
//                      into a 5-deep shared-memory ring.  Pages are stored
//                      pre-swizzled (common.cuh page_index): a page is four
//                      32-record blocks, each exactly the MN-major
//                      SWIZZLE_128B_BASE32B operand image tcgen05 requires for
//                      TF32, so the copy lands a ready UMMA operand.
//   warp 9 (MMA)       allocates TMEM, and one elected lane issues
//                      M=128 (records) x N=16 x K=8 MMAs per page: A = the
//                      page tile (MN-major, records contiguous), B = the query
//                      constants split hi/lo in TF32 (K-major, 16 columns: 8
//                      hi + 8 lo), D accumulates in TMEM; tcgen05.commit
//                      signals the consumers.
//   warps 0-7          P = ||y||^2 on the CUDA cores from the same shared tile
//   (consumers)        (one record per thread), D from TMEM (tcgen05.ld
//                      32x32b.x16, lane = record), then keys, thresholds and
//                      candidate lists exactly as the CUDA-core kernel.
//
// Records are stored rounded to TF32 (cvt.rna at append), so the MMA sees the
// stored values exactly and P, D describe the same vector; the rounding is a
// bounded input perturbation the certification accounts for.
#include <algorithm>
#include <cstdlib>
#include <cfloat>
#include <cstring>
#include <vector>

#include "select_common.cuh"
#include "umma.cuh"
#include "warp_topk.cuh"

namespace sair {


using namespace umma;

namespace {

constexpr int MW = 8;                  // consumer warps
constexpr int MMA_THREADS = MW * 32 + 64;  // + producer warp + MMA warp
constexpr int PAGES_PER_STAGE = 1;
constexpr int TMEM_COLS = 128;
// instruction descriptor: D f32, A/B tf32, A MN-major, B K-major, N=16, M=128
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | ((16u >> 3) << 17) |
                           ((128u >> 4) << 24);

}  // namespace

template <int DP, int QB>
struct MmaArgs {
    const float* pages;
    const float* r32;
    uint32_t n, npages;
    float c1, c0, rdelta, alpha;
    int kp, knn, nst, cap_sel, cap_nn, kmax;
    int probe;       // diagnostics only (SAIR_PROBE): 1 = skip inserts/barriers
    float* out_key;  // [grid][2*QB][kmax]
    uint32_t* out_idx;
    unsigned int* pmax;
    const float* t0;        // [2QB] starting thresholds (sample pre-pass)
    unsigned int* dropped;  // [2QB] max ordinal of a key dropped on a full list
    const float* b;   // [2][DP][QB] hi / lo TF32 parts of -2 c_qk / sd_k (device)
    float s[DP];      // 1 / sd (0 on padding)
    float cc[QB];     // sum_k c_qk^2
};

template <int DP, int QB>
__global__ void __launch_bounds__(MMA_THREADS, 1)
    stream_mma_kernel(const __grid_constant__ MmaArgs<DP, QB> a) {
    constexpr int BOX_BYTES = 32 * DP * 4;              // 32 records x DP dims
    constexpr int PAGE_BYTES = 4 * BOX_BYTES;           // 4 boxes = 128 records
    constexpr int STAGE_BYTES = PAGES_PER_STAGE * PAGE_BYTES;
    constexpr int KSTEPS = DP / 8;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte alignment for the SWIZZLE_128B atoms
    // (offsetting smem_raw keeps the pointer in the shared window: LDS, not LD)
    unsigned char* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nl = a.knn ? 2 * QB : QB;
    unsigned char* stage = smem;
    float* btile = reinterpret_cast<float*>(stage + (size_t)a.nst * STAGE_BYTES);  // KSTEPS x 512 B
    float* ss = btile + KSTEPS * 128;
    uint64_t* full = reinterpret_cast<uint64_t*>(ss + DP);
    uint64_t* empty = full + 8;
    uint64_t* tfull = empty + 8;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 8);
    float* thr = reinterpret_cast<float*>(tmem_slot + 4);
    int* cnt = reinterpret_cast<int*>(thr + 2 * QB);
    uint32_t* hist = reinterpret_cast<uint32_t*>(cnt + 2 * QB);
    float* lkey = reinterpret_cast<float*>(hist + MW * 256);
    const int total_cap = QB * a.cap_sel + (a.knn ? QB * a.cap_nn : 0);
    uint32_t* lidx = reinterpret_cast<uint32_t*>(lkey + total_cap);
    auto lbase = [&](int L) { return L < QB ? L * a.cap_sel : QB * a.cap_sel + (L - QB) * a.cap_nn; };
    auto lcap = [&](int L) { return L < QB ? a.cap_sel : a.cap_nn; };
    auto lk = [&](int L) { return L < QB ? a.kp : a.knn; };

    // B operand: K-major, no swizzle; per K-step a 16 (N) x 8 (K) tile of four
    // 8x16B core matrices: (n%8)*16 + (n/8)*256 + (k%4)*4 + (k/4)*128 bytes
    for (int i = tid; i < KSTEPS * 16 * 8; i += MMA_THREADS) {
        const int ks = i / 128, n = (i / 8) % 16, k = i % 8;
        const int dim = ks * 8 + k;
        float v = 0.f;
        if (n < QB) v = a.b[dim * QB + n];
        else if (n >= 8 && n - 8 < QB) v = a.b[(DP + dim) * QB + n - 8];
        const int off = ks * 512 + (n % 8) * 16 + (n / 8) * 256 + (k % 4) * 4 + (k / 4) * 128;
        btile[off / 4] = v;
    }
    for (int i = tid; i < DP; i += MMA_THREADS) ss[i] = a.s[i];
    if (tid < 2 * QB) {
        thr[tid] = -FLT_MAX;
        cnt[tid] = 0;
    }
    if (tid == 0) {
        for (int s = 0; s < a.nst; ++s) {
            bar_init(&full[s], 1);
            bar_init(&empty[s], MW / 2);  // one half of the consumers reads each stage
            bar_init(&tfull[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // generic-proxy writes of the B tiles must be visible to the tensor core
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == MW + 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         su32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    const uint32_t nrounds = (a.npages + PAGES_PER_STAGE - 1) / PAGES_PER_STAGE;
    const uint32_t G = gridDim.x, r0 = blockIdx.x;
    const uint32_t mine = r0 < nrounds ? (nrounds - 1 - r0) / G + 1 : 0;

    if (warp == MW) {
        // ---------------- producer: TMA tensor loads ----------------
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (uint32_t it = 0; it < mine; ++it) {
                const uint32_t p0 = (r0 + it * G) * PAGES_PER_STAGE;
                const uint32_t np = min((uint32_t)PAGES_PER_STAGE, a.npages - p0);
                if (it >= (uint32_t)a.nst) bar_wait(&empty[s], ph ^ 1u);
                bar_expect_tx(&full[s], np * PAGE_BYTES);
                // pages are stored pre-swizzled: one contiguous bulk copy per page
                for (uint32_t pp = 0; pp < np; ++pp)
                    bulk_g2s(stage + (size_t)s * STAGE_BYTES + pp * PAGE_BYTES,
                             a.pages + (size_t)(p0 + pp) * DP * PAGE, PAGE_BYTES, &full[s]);
                if (++s == a.nst) {
                    s = 0;
                    ph ^= 1u;
                }
            }
        }
    } else if (warp == MW + 1) {
        // ---------------- MMA issuer ----------------
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            const uint32_t bbase = su32(btile);
            for (uint32_t it = 0; it < mine; ++it) {
                bar_wait(&full[s], ph);
                tc_fence_after();
                for (int pp = 0; pp < PAGES_PER_STAGE; ++pp) {
                    const uint32_t abase = su32(stage + (size_t)s * STAGE_BYTES + pp * PAGE_BYTES);
                    const uint32_t dcol = tmem + (uint32_t)((s * PAGES_PER_STAGE + pp) * 16);
#pragma unroll
                    for (int ks = 0; ks < KSTEPS; ++ks) {
                        // A: MN-major SWIZZLE_128B_BASE32B (the only MN-major layout for
                        // tf32): LBO = next 32-record block, SBO = next 4-dimension atom
                        const uint64_t ad = umma_desc(abase + ks * 1024, BOX_BYTES, 512, 1);
                        const uint64_t bd = umma_desc(bbase + ks * 512, 128, 256, 0);
                        umma_tf32(dcol, ad, bd, IDESC, ks > 0 ? 1u : 0u);
                    }
                }
                umma_commit(&tfull[s]);
                if (++s == a.nst) {
                    s = 0;
                    ph ^= 1u;
                }
            }
        }
    } else {
        // ---------------- consumers ----------------
        // warp w reads TMEM lane quarter w % 4 of every stage with parity w / 4;
        // the two halves of the consumers work on consecutive stages at once
        const int pp = 0;
        const int par = warp >> 2;
        const int quarter = warp & 3;
        const int rloc = quarter * 32 + lane;  // record within the page
        // Fixed thresholds from the sample pre-pass (T0 <= the global K'-th
        // key): lists are append-only, so consumers never synchronise while
        // streaming.  A record that finds its list full is dropped and only
        // its key is remembered (the bound then covers it).
        float thr_r[2 * QB];
#pragma unroll
        for (int L = 0; L < 2 * QB; ++L) thr_r[L] = L < nl ? a.t0[L] : FLT_MAX;
        const unsigned lt_mask = (1u << lane) - 1u;
        float pmax = 0.f;
        int s = par % a.nst;
        uint32_t ph = (uint32_t)(par / a.nst) & 1u;
        for (uint32_t it = par; it < mine; it += 2) {
            const uint32_t page = (r0 + it * G) * PAGES_PER_STAGE + pp;
            const uint32_t rec = page * PAGE + rloc;
            const bool valid = rec < a.n;
            const float r = valid ? __ldg(a.r32 + rec) : 0.f;
            bar_wait(&full[s], ph);
            // P from the pre-swizzled block: row k at k*128 B, 32-B chunk (lane/8) ^ (k%4)
            const unsigned char* box = stage + (size_t)s * STAGE_BYTES + pp * PAGE_BYTES +
                                       quarter * BOX_BYTES;
            float Pp[4] = {0.f, 0.f, 0.f, 0.f};  // four chains, not one serial FFMA chain
#pragma unroll
            for (int k = 0; k < DP; ++k) {
                const float x = *reinterpret_cast<const float*>(
                    box + k * 128 + ((((lane >> 3) ^ (k & 3)) << 5) | ((lane & 7) << 2)));
                const float y = __fmul_rn(x, ss[k]);
                Pp[k & 3] = fmaf(y, y, Pp[k & 3]);
            }
            const float P = (Pp[0] + Pp[1]) + (Pp[2] + Pp[3]);
            bar_wait(&tfull[s], ph);
            tc_fence_after();
            float acc[16];
            tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) +
                          (uint32_t)((s * PAGES_PER_STAGE + pp) * 16),
                      acc);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) bar_arrive(&empty[s]);
            if (valid) pmax = fmaxf(pmax, P);
            const float lg = log2f(fabsf(fmaf(r, a.c1, -a.c0)) + a.rdelta);
            float key[2 * QB];
            uint32_t pm = 0;
#pragma unroll
            for (int q = 0; q < QB; ++q) {
                const float d2 = (P + a.cc[q]) + (acc[q] + acc[8 + q]);
                key[q] = fmaf(-d2, a.alpha, lg);
                key[QB + q] = -d2;
                pm |= (key[q] > thr_r[q] ? 1u : 0u) << q;
                pm |= (key[QB + q] > thr_r[QB + q] ? 1u : 0u) << (QB + q);
            }
            if (!valid || a.probe) pm = 0;
            if (__any_sync(0xffffffffu, pm)) {
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
                            const int slot = base + __popc(bal & lt_mask);
                            if (slot < lcap(L)) {
                                lkey[lbase(L) + slot] = key[L];
                                lidx[lbase(L) + slot] = rec;
                            } else {
                                atomicMax(&a.dropped[L], f2ord(key[L]));
                            }
                        }
                    }
                }
            }
            // this half consumes every other stage: advance the ring by two
            for (int t = 0; t < 2; ++t)
                if (++s == a.nst) {
                    s = 0;
                    ph ^= 1u;
                }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) pmax = fmaxf(pmax, __shfl_xor_sync(0xffffffffu, pmax, o));
        if (lane == 0) atomicMax(a.pmax, __float_as_uint(pmax));
        asm volatile("bar.sync 1, %0;" ::"n"(MW * 32) : "memory");
        // one compaction per list at the end
        for (int L = warp; L < nl; L += MW) {
            const int c = min(cnt[L], lcap(L));
            __syncwarp();  // every lane has read the count before lane 0 rewrites it
            if (c > lk(L)) {
                warp_keep_topk(lkey + lbase(L), lidx + lbase(L), c, lk(L), hist + warp * 256, lane);
                if (lane == 0) cnt[L] = lk(L);
            } else if (lane == 0) {
                cnt[L] = c;
            }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(MW * 32) : "memory");
        for (int L = 0; L < nl; ++L) {
            const size_t row = ((size_t)blockIdx.x * 2 * QB + L) * a.kmax;
            for (int j = tid; j < lk(L); j += MW * 32) {
                const bool have = j < cnt[L];
                a.out_key[row + j] = have ? lkey[lbase(L) + j] : -INFINITY;
                a.out_idx[row + j] = have ? lidx[lbase(L) + j] : 0xFFFFFFFFu - (uint32_t)(row + j);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == MW + 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(TMEM_COLS));
    }
}

// ------------------------------------------------------ sample pre-pass --
// Page maxima of every list's key over a strided page sample (CUDA cores, the
// stream pass's formula).  The K'-th largest of K' or more page maxima is the
// key of K' distinct records, so it is <= the store's K'-th key: a safe start
// threshold for the stream pass.  One block = one sampled page.
template <int DP, int QB>
__global__ void __launch_bounds__(PAGE)
    sample_keys_kernel(const float* __restrict__ pages, const float* __restrict__ r32, uint32_t n,
                       uint32_t npages, uint32_t sample_pages,
                       const float* __restrict__ consts /* s[DP] | c2[DP][QB] | cc[QB] */,
                       float c1, float c0, float rdelta, float alpha, float* __restrict__ pmaxk) {
    __shared__ float sc[DP + DP * QB + QB];
    __shared__ float wmax[4][2 * QB];
    for (int i = threadIdx.x; i < DP + DP * QB + QB; i += PAGE) sc[i] = consts[i];
    __syncthreads();
    const uint32_t page = (uint32_t)((uint64_t)blockIdx.x * npages / sample_pages);
    const uint32_t rec = page * PAGE + threadIdx.x;
    const bool valid = rec < n;
    float P = 0.f, D[QB];
#pragma unroll
    for (int q = 0; q < QB; ++q) D[q] = 0.f;
    if (valid) {
        // all DP loads in flight at once: the pass is latency-bound, not bandwidth-bound
        float x[DP];
#pragma unroll
        for (int k = 0; k < DP; ++k) x[k] = __ldg(pages + page_index(rec, k, DP));
#pragma unroll
        for (int k = 0; k < DP; ++k) {
            const float y = __fmul_rn(x[k], sc[k]);
            P = fmaf(y, y, P);
#pragma unroll
            for (int q = 0; q < QB; ++q) D[q] = fmaf(y, sc[DP + k * QB + q], D[q]);
        }
    }
    const float r = valid ? __ldg(r32 + rec) : 0.f;
    const float lg = log2f(fabsf(fmaf(r, c1, -c0)) + rdelta);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < QB; ++q) {
        const float d2 = (P + sc[DP + DP * QB + q]) + D[q];
        float ks = valid ? fmaf(-d2, alpha, lg) : -INFINITY;
        float kn = valid ? -d2 : -INFINITY;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            ks = fmaxf(ks, __shfl_xor_sync(0xffffffffu, ks, o));
            kn = fmaxf(kn, __shfl_xor_sync(0xffffffffu, kn, o));
        }
        if (lane == 0) {
            wmax[w][q] = ks;
            wmax[w][QB + q] = kn;
        }
    }
    __syncthreads();
    if (threadIdx.x < 2 * QB) {
        const int L = threadIdx.x;
        pmaxk[(size_t)L * sample_pages + blockIdx.x] =
            fmaxf(fmaxf(wmax[0][L], wmax[1][L]), fmaxf(wmax[2][L], wmax[3][L]));
    }
}

// t0[L] <= the K-th largest of list L's S <= 1024 page maxima: one histogram
// over the ordinal range present (2048 bins); the lower edge of the bin where
// the count from the top reaches K is a lower bound of the K-th value.  It is
// then lowered by a relative 1e-4 so formula differences only loosen it.
__global__ void __launch_bounds__(1024)
    sample_kth_kernel(const float* __restrict__ pmaxk, uint32_t S, int QB, int kp, int knn,
                      float* __restrict__ t0) {
    constexpr int NB = 2048;
    __shared__ uint32_t hist[NB];
    __shared__ uint32_t sh_lo, sh_hi, sh_bin;
    const int L = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
    const int K = L < QB ? kp : knn;
    if ((uint32_t)K > S || K == 0 || S > 1024) {
        if (tid == 0) t0[L] = -FLT_MAX;
        return;
    }
    const bool have = (uint32_t)tid < S;
    const uint32_t o = have ? f2ord(pmaxk[(size_t)L * S + tid]) : 0u;
    const bool valid = have && o > 0x007FFFFFu;  // not -inf (empty page)
    uint32_t lo = valid ? o : 0xFFFFFFFFu, hi = valid ? o : 0u;
    for (int b = tid; b < NB; b += blockDim.x) hist[b] = 0;
    if (tid == 0) {
        sh_lo = 0xFFFFFFFFu;
        sh_hi = 0;
        sh_bin = 0xFFFFFFFFu;
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, d));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, d));
    }
    __syncthreads();
    if (lane == 0) {
        atomicMin(&sh_lo, lo);
        atomicMax(&sh_hi, hi);
    }
    __syncthreads();
    const uint32_t blo = sh_lo, span = sh_hi - sh_lo;
    const int sh = span < NB ? 0 : (32 - __clz(span)) - 11;
    if (valid) atomicAdd(&hist[(o - blo) >> sh], 1u);
    __syncthreads();
    if (tid < 32) {
        uint32_t sum = 0;
        for (int j = 0; j < NB / 32; ++j) sum += hist[NB - 1 - (lane * (NB / 32) + j)];
        uint32_t incl = sum;
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += t;
        }
        const uint32_t excl = incl - sum;
        const unsigned own = __ballot_sync(0xffffffffu, excl < (uint32_t)K && (uint32_t)K <= incl);
        if (lane == __ffs(own) - 1) {
            uint32_t c = excl;
            for (int j = 0; j < NB / 32; ++j) {
                const int b = NB - 1 - (lane * (NB / 32) + j);
                c += hist[b];
                if (c >= (uint32_t)K) {
                    sh_bin = (uint32_t)b;
                    break;
                }
            }
        }
    }
    __syncthreads();
    if (tid == 0) {
        if (sh_bin == 0xFFFFFFFFu) {  // fewer than K non-empty sampled pages
            t0[L] = -FLT_MAX;
        } else {
            const float v = ord2f(blo + (sh_bin << sh));
            t0[L] = v - 1e-4f * (fabsf(v) + 1.f);
        }
    }
}

// ------------------------------------------------------------------- host --

namespace {

inline float tf32_trunc(double v) {
    float f = (float)v;
    uint32_t u;
    std::memcpy(&u, &f, 4);
    u &= 0xFFFFE000u;
    std::memcpy(&f, &u, 4);
    return f;
}

template <int DP, int QB>
void mma_fill_and_launch(sair_store_s* s, const MmaPlan& pl, const QueryPrep& p, const double* zgrp,
                         int nqg, float c1, float c0, float rdelta, float alpha, float* ck,
                         uint32_t* ci, unsigned int* pmax, std::vector<double>& cc_out,
                         const GroupIo& io) {
    MmaArgs<DP, QB> a{};
    a.pages = s->pages;
    a.r32 = s->r32;
    a.probe = std::getenv("SAIR_PROBE") ? 1 : 0;
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
    float* hb = io.hstage;  // 2 DP QB + DP + DP QB + QB floats
    for (int q = 0; q < QB; ++q) {
        const double* z = zgrp + (size_t)(q < nqg ? q : 0) * d;
        double cc = 0.0;
        for (int k = 0; k < DP; ++k) {
            float c = 0.f;
            if (k < d) c = (float)((p.mean[k] - s->shift[k]) / p.sd[k] + z[k]);
            cc += (double)c * (double)c;
            const double bk = k < d ? -2.0 * (double)c * (double)a.s[k] : 0.0;
            const float hi = tf32_trunc(bk);
            hb[k * QB + q] = hi;
            hb[(DP + k) * QB + q] = tf32_trunc(bk - (double)hi);
        }
        a.cc[q] = (float)cc;
        cc_out[q] = cc;
    }
    // device constants: B hi/lo | sample consts (s, -2c, cc) | t0[16] | dropped[16]
    const size_t nb = 2 * DP * QB, nsc = DP + DP * QB + QB;
    for (int k = 0; k < DP; ++k) {
        hb[nb + k] = a.s[k];
        for (int q = 0; q < QB; ++q) {
            const double* z = zgrp + (size_t)(q < nqg ? q : 0) * d;
            const float c = k < d ? (float)((p.mean[k] - s->shift[k]) / p.sd[k] + z[k]) : 0.f;
            hb[nb + DP + k * QB + q] = -2.f * c;
        }
    }
    for (int q = 0; q < QB; ++q) hb[nb + DP + DP * QB + q] = a.cc[q];
    float* db = s->b_mmab.as<float>(nb + nsc + 32 + 64);
    float* dsc = db + nb;
    float* dt0 = dsc + nsc;
    unsigned int* ddrop = reinterpret_cast<unsigned int*>(dt0 + 16);
    SAIR_CUDA(cudaMemcpyAsync(db, hb, (nb + nsc) * sizeof(float), cudaMemcpyHostToDevice, s->st));
    SAIR_CUDA(cudaMemsetAsync(ddrop, 0, 16 * sizeof(unsigned int), s->st));
    a.b = db;
    a.t0 = dt0;
    a.dropped = ddrop;
    s->mma_t0 = dt0;
    s->mma_dropped = ddrop;
    // sample pre-pass over spages strided pages (all pages of a small store)
    const uint32_t npg = a.npages;
    const uint32_t kl = (uint32_t)std::max(pl.kp, pl.knn);
    uint32_t spages = std::min<uint32_t>(npg, std::max<uint32_t>(2 * kl, std::min<uint32_t>(1024, npg / 32)));
    float* dkeys = s->b_sample.as<float>((size_t)2 * QB * spages);
    sample_keys_kernel<DP, QB><<<spages, PAGE, 0, s->st>>>(s->pages, s->r32, a.n, npg, spages, dsc,
                                                          c1, c0, rdelta, alpha, dkeys);
    SAIR_LAUNCH("sample_keys_kernel");
    sample_kth_kernel<<<pl.knn ? 2 * QB : QB, 1024, 0, s->st>>>(
        dkeys, spages, QB, pl.kp, pl.knn, dt0);
    SAIR_LAUNCH("sample_kth_kernel");
    SAIR_CUDA(cudaEventRecord(io.e_mid, s->st));
    SAIR_CUDA(cudaFuncSetAttribute(stream_mma_kernel<DP, QB>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
    stream_mma_kernel<DP, QB><<<pl.grid, MMA_THREADS, pl.smem, s->st>>>(a);
    SAIR_LAUNCH("stream_mma_kernel");
}

template <int DP>
MmaFillFn mma_pick_qb(int qb) {
    switch (qb) {
        case 1: return mma_fill_and_launch<DP, 1>;
        case 2: return mma_fill_and_launch<DP, 2>;
        case 4: return mma_fill_and_launch<DP, 4>;
        default: return mma_fill_and_launch<DP, 8>;
    }
}

}  // namespace

MmaFillFn pick_mma_fill(int dp, int qb) {
    switch (dp) {
        case 8: return mma_pick_qb<8>(qb);
        case 16: return mma_pick_qb<16>(qb);
        case 32: return mma_pick_qb<32>(qb);
        case 64: return mma_pick_qb<64>(qb);
        default: return nullptr;
    }
}

bool make_mma_plan(const sair_store_s* s, size_t nq, size_t m, double lambda, bool nn,
                   MmaPlan* pl) {
    if (s->dp < 8 || s->dp > 64) return false;
    pl->dp = s->dp;
    pl->qb = nq >= 8 ? 8 : (nq >= 4 ? 4 : (nq >= 2 ? 2 : 1));
    pl->kp = 32;
    const size_t want_pool = lambda != 0.0 ? 4 * m : 2 * m;
    while ((size_t)pl->kp < want_pool && pl->kp < 512) pl->kp <<= 1;
    pl->knn = nn ? 16 : 0;
    pl->kmax = std::max(pl->kp, pl->knn);
    // append-only lists above the sample threshold (overflow is tracked, not lost)
    pl->cap_sel = std::max(4 * pl->kp, 512);
    pl->cap_nn = nn ? std::max(4 * pl->knn, 256) : 0;
    const size_t stage = (size_t)PAGES_PER_STAGE * 4 * 32 * pl->dp * 4;  // 32 KB at dp = 64
    const size_t fixed = 1024 /* alignment slack */ + (size_t)(pl->dp / 8) * 512 + pl->dp * 4 +
                         24 * 8 + 16 + 2 * 16 * 4 + MW * 256 * 4 +
                         (size_t)pl->qb * pl->cap_sel * 8 + (nn ? (size_t)pl->qb * pl->cap_nn * 8 : 0);
    const size_t limit = 227 * 1024;
    // deep ring of one-page stages: up to 160 KB in flight (<= 8 stages: TMEM columns)
    pl->nst = (int)std::min<size_t>(8, std::max<size_t>(2, 192 * 1024 / stage));
    while (pl->nst > 2 && fixed + pl->nst * stage > limit) --pl->nst;
    if (fixed + pl->nst * stage > limit) return false;
    if (pl->nst * PAGES_PER_STAGE * 16 > TMEM_COLS) return false;
    pl->smem = fixed + pl->nst * stage;
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, s->device);
    const size_t npages = (s->n + PAGE - 1) / PAGE;
    const size_t nrounds = (npages + PAGES_PER_STAGE - 1) / PAGES_PER_STAGE;
    pl->grid = (int)std::max<size_t>(1, std::min<size_t>(nrounds, (size_t)nsm));
    return true;
}

}  // namespace sair
