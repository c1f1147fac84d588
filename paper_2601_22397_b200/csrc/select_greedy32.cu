// select_greedy32.cu -- select() with lambda_div != 0 over a large store: the
// greedy's steps filtered in fp32, every pick decided in fp64.
//
// experience.cpp:151-205.  On a store of i.i.d. 64-d contexts the diversity
// penalty makes the greedy's later picks come from anywhere in the score
// order (1M records, lambda 0.1: picks 8-32 rank 50k-400k by score), so no
// candidate pool of the best scores can certify them: every step needs an
// arg-max over the whole store.  The fp64 greedy (select_greedy.cu) does that
// in the reference's rounding order for every (query, record) pair -- a
// 64-term fp64 distance per pair per step, ~150 ms per 128 queries at 1M.
//
// Here a step keeps only an fp32 gain per (query, record):
//   step 0   gain = sim32(z_i, z_q) * |r_i - loo_i|        (= score, :163-167)
//   step t   gain -= lambda * sim32(z_i, z_pick(t-1))      (:283-284, :270)
// with sim32 from the fp32 norm expansion (two FFMA2 per two dimensions) and
// ex2, and a per-warp (best, index, second best).  The pick kernel then takes,
// per query, every record whose fp32 gain lies within 2 eps(t) of the fp32
// maximum -- eps(t) a rigorous bound of |gain32 - gain64| over all records
// (error analysis in eps_coeffs below) -- and recomputes their gains exactly:
// score64 and the penalty as the reference sums it (fp64, pick order), then
// the reference's arg-max (gain desc, round asc, index asc).  The true pick is
// always a candidate, so the result is the fp64 greedy's, bit for bit.  A
// query whose candidate set overflows (never seen) goes to the fp64 greedy.
#include <atomic>
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "select_common.cuh"
#include "umma.cuh"

namespace sair {

namespace {

constexpr int FT = 256;     // records per CTA of the step kernel (one per thread)
constexpr int CMAX = 32;    // candidates verified per query and step

struct G32Args {
    const float* z32;      // [DP][n] fp32 standardized rows (dimension-major, zero padded)
    const float* p32;      // [n] |z32_i|^2
    const float* a32;      // [n] |r_i - loo_i| (fp32)
    const double* x64;     // [n][d] stored rows and msd = mean | sd | 1 / sd [3d]: a record's
    const double* msd;     // exact standardized row is computed where needed (zexact)
    const double* r64;
    const int32_t* rnd;
    const double* loo;     // [n] local LOO means or null (global)
    const double* zq;      // [G][d] exact standardized queries
    const float* row32;    // [G][DP] step 0: queries; step t: the previous picks (fp32)
    const float* prow;     // [G] their |.|^2
    size_t n, n_loo;
    int d, G, want;
    double total, two_s2, lambda;
    float c_exp;           // -log2(e) / (2 sigma^2)
    float* gain;           // [G][n], or tiled [n / 32][gs][32] (gs != 0: the tensor-core step)
    int gs;                // tiled layout: rows of the step, padded; else 0
    uint32_t* part;        // [G][nw][3]: best gain (bits), its index, second best (bits)
    uint32_t* part_nn;     // [G][nw][3] step 0: the same for sim32 (veto scan)
    int nw;
    uint32_t* cpart;       // tensor-core step: [G][ncta][3] the same per CTA of the step kernel
    int ncta;              // (0: no CTA level)
    float* pick32;         // [G][DP] the step's picks (the next step's rows)
    float* ppick;          // [G]
    int64_t* picks;        // [G][want]
    double* pscore;        // [G][want] exact score of each pick
    int64_t* nn;           // [G]
    double* nn_sim;        // [G]
    double e0, e1, e2;     // eps(t) = e0 + t e1 + t^2 e2
    double eps_nn;         // |sim32 - sim64|
    int* overflow;         // [G]
    unsigned int* ncand;   // diagnostics: candidates verified (sum)
};

__device__ __forceinline__ float ex2f(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// order-preserving int image of a float (signed compare), and back
__device__ __forceinline__ int f2i(float f) {
    const int b = __float_as_int(f);
    return b >= 0 ? b : b ^ 0x7FFFFFFF;
}
__device__ __forceinline__ float i2f(int b) { return __int_as_float(b >= 0 ? b : b ^ 0x7FFFFFFF); }

// warp: (best value, the lowest lane holding it, second best value) -- two
// redux.sync.max and a ballot (the shuffle tree cost ~40 instructions)
__device__ __forceinline__ void warp_top2(float v, int lane, float& b, int& bl, float& s2) {
    const int iv = f2i(v);
    const int ib = __reduce_max_sync(0xffffffffu, iv);
    const unsigned at = __ballot_sync(0xffffffffu, iv == ib);
    bl = __ffs(at) - 1;
    const int i2 = __reduce_max_sync(0xffffffffu, lane == bl ? (int)0x80000000 : iv);
    b = i2f(ib);
    s2 = i2f(i2);
    (void)lane;
}

// One CTA: FT records (one per thread, its fp32 row in registers) x GQ2
// queries (blockIdx.y).  The gains of the next QB queries are loaded before
// the current ones are computed (the loop is latency-bound otherwise).
constexpr int GQ2 = 32;
constexpr int QB = 4;
template <int DP>
__global__ void __launch_bounds__(FT, 2) g32_step_kernel(const G32Args a, int step) {
    __shared__ __align__(16) float rows[GQ2][DP];
    __shared__ float prow[GQ2];
    const size_t i = (size_t)blockIdx.x * FT + threadIdx.x;
    const bool valid = i < a.n;
    const int lane = threadIdx.x & 31;
    const size_t w = (size_t)blockIdx.x * (FT / 32) + (threadIdx.x >> 5);
    const int g0 = blockIdx.y * GQ2, gn = min(GQ2, a.G - g0);
    for (int e = threadIdx.x; e < gn * DP; e += FT) rows[e / DP][e % DP] = a.row32[(size_t)g0 * DP + e];
    for (int e = threadIdx.x; e < gn; e += FT) prow[e] = a.prow[g0 + e];
    float2 zi[DP / 2];  // register pairs: FFMA2 operands without moves
#pragma unroll
    for (int k = 0; k < DP; k += 2)
        zi[k / 2] = valid ? make_float2(a.z32[(size_t)k * a.n + i], a.z32[(size_t)(k + 1) * a.n + i])
                          : make_float2(0.f, 0.f);
    const float pi = valid ? a.p32[i] : 0.f;
    const float ai = step == 0 && valid ? a.a32[i] : 0.f;
    const float lam = (float)a.lambda;
    __syncthreads();
    // gain of (query g0 + q, record i) at gp + q n; each lane keeps the warp's
    // (best, index, second) of query g0 + lane and stores it once at the end
    float* gp = a.gain + (size_t)g0 * a.n + (valid ? i : 0);
    const size_t gstride = a.n;
    float gcur[QB];
#pragma unroll
    for (int h = 0; h < QB; ++h) gcur[h] = step > 0 && valid && h < gn ? gp[h * gstride] : -INFINITY;
    float my_b = -INFINITY, my_s = -INFINITY, nn_b = -INFINITY, nn_s = -INFINITY;
    uint32_t my_i = 0, nn_i = 0;
    const uint32_t wbase = (uint32_t)(i - lane);
    for (int gb = 0; gb < gn; gb += QB) {
        float gnext[QB];
#pragma unroll
        for (int h = 0; h < QB; ++h) {
            const int q = gb + QB + h;
            gnext[h] = step > 0 && valid && q < gn ? gp[(size_t)q * gstride] : -INFINITY;
        }
#pragma unroll
        for (int h = 0; h < QB; ++h) {
            const int gg = gb + h;
            if (gg >= gn) break;
            float2 acc = make_float2(0.f, 0.f), acc2 = make_float2(0.f, 0.f);
#pragma unroll
            for (int k = 0; k < DP; k += 4) {
                const float4 r = *reinterpret_cast<const float4*>(&rows[gg][k]);
                acc = __ffma2_rn(zi[k / 2], make_float2(r.x, r.y), acc);
                acc2 = __ffma2_rn(zi[k / 2 + 1], make_float2(r.z, r.w), acc2);
            }
            const float d2 = (pi + prow[gg]) - 2.f * ((acc.x + acc.y) + (acc2.x + acc2.y));
            const float sim = ex2f(a.c_exp * d2);
            float gv = -INFINITY;
            if (valid) {
                gv = step == 0 ? sim * ai : (gcur[h] != -INFINITY ? gcur[h] - lam * sim : -INFINITY);
                gp[(size_t)gg * gstride] = gv;
            }
            float b, s2;
            int bl;
            warp_top2(gv, lane, b, bl, s2);
            if (lane == gg) {
                my_b = b;
                my_s = s2;
                my_i = wbase + (uint32_t)bl;
            }
            if (step == 0 && a.part_nn) {
                warp_top2(valid ? sim : -INFINITY, lane, b, bl, s2);
                if (lane == gg) {
                    nn_b = b;
                    nn_s = s2;
                    nn_i = wbase + (uint32_t)bl;
                }
            }
        }
#pragma unroll
        for (int h = 0; h < QB; ++h) gcur[h] = gnext[h];
    }
    if (lane < gn) {
        uint32_t* pp = a.part + ((size_t)(g0 + lane) * a.nw + w) * 3;
        pp[0] = __float_as_uint(my_b);
        pp[1] = my_i;
        pp[2] = __float_as_uint(my_s);
        if (step == 0 && a.part_nn) {
            uint32_t* pn = a.part_nn + ((size_t)(g0 + lane) * a.nw + w) * 3;
            pn[0] = __float_as_uint(nn_b);
            pn[1] = nn_i;
            pn[2] = __float_as_uint(nn_s);
        }
    }
}

// ---------------------------------------------------------------------------
// The step on the tensor cores (d in 33..64): the dots <z_i, row_g> of a
// 128-record tile with all (up to) 256 rows of the step as one M = 128, N =
// 256 accumulator, in 3xTF32 -- each fp32 operand split into TF32 hi + lo
// parts (together within 2^-22 of it), D = hi.hi + lo.hi + hi.lo (the lo.lo
// term, <= 2^-22 |z||row|, dropped): 24 tcgen05.mma kind::tf32 per tile
// (K = 8 each) into TMEM.  The epilogue is the CUDA-core step's per-pair work
// without its 32 FFMA2: d2 = (P_i + P_g) - 2 D, ex2, the gain update and the
// warp's (best, index, second) per row.  Its error bound is g32_eps's with the
// dot's term for the MMA (g32_eps_mma).  One CTA per SM, persistent over the
// tiles; the step is bound by the gain state's HBM traffic (8 B per pair).
constexpr int MT_REC = 128;                   // records per tile (MMA M)
constexpr int MT_N = 256;                     // rows per step (MMA N)
constexpr int MT_A_BYTES = 2 * 8 * 16 * 256;  // [hi, lo][8 K-steps][16 groups][2 x 8 x 16 B] = 64 KB
constexpr int MT_B_BYTES = 2 * 8 * 32 * 256;  // [hi, lo][8 K-steps][32 groups][2 x 8 x 16 B] = 128 KB
constexpr int MT_EPI = 16;                    // epilogue warps: four per TMEM lane quarter
constexpr int MT_TS = 32;                     // transpose row (floats; 4-float groups XOR-swizzled)
constexpr int MT_PROD = MT_EPI, MT_MMA = MT_EPI + 1;
constexpr int MT_THREADS = (MT_EPI + 2) * 32;
constexpr size_t MT_SMEM = MT_B_BYTES + MT_A_BYTES + MT_N * 4 + MT_EPI * 16 * MT_TS * 4 + 256;

__device__ __forceinline__ float mt_tf32(float v) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
    return __uint_as_float(r);
}

// float offset of (row r, dimension k, part) in a K-major no-swizzle operand
// image of `rows` rows: per (part, K-step) rows / 8 groups of two 8 x 16 B
// core matrices (the K halves), 256 B per group
__device__ __forceinline__ size_t mt_off(int part, int k, int r, int rows) {
    return ((size_t)(part * 8 + (k >> 3)) * (rows / 8) + (r >> 3)) * 64 + ((k >> 2) & 1) * 32 +
           (r & 7) * 4 + (k & 3);
}

// the step's rows (queries at step 0, then the picks) as the B operand image
__global__ void g32_mma_bimg_kernel(const float* __restrict__ rows, int G, int DP,
                                    float* __restrict__ img) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < MT_N * 64; e += gridDim.x * blockDim.x) {
        const int g = e / 64, k = e % 64;
        const float v = g < G && k < DP ? rows[(size_t)g * DP + k] : 0.f;
        const float hi = mt_tf32(v), lo = mt_tf32(v - hi);
        img[mt_off(0, k, g, MT_N)] = hi;
        img[mt_off(1, k, g, MT_N)] = lo;
    }
}

__global__ void __launch_bounds__(MT_THREADS, 1)
    g32_mma_step_kernel(const G32Args a, const float* __restrict__ aimg,
                        const float* __restrict__ bimg, int step) {
    using namespace umma;
    extern __shared__ __align__(16) unsigned char smem[];  // (no-swizzle operands: 16 B alignment)
    unsigned char* sb = smem;                       // B image
    unsigned char* sa = smem + MT_B_BYTES;          // A stage
    float* sprow = reinterpret_cast<float*>(sa + MT_A_BYTES);
    float* strans = sprow + MT_N;  // [MT_EPI][16][MT_TS] epilogue transposes
    uint64_t* bar = reinterpret_cast<uint64_t*>(strans + MT_EPI * 16 * MT_TS);
    uint64_t *bfull = bar, *afull = bar + 1, *aempty = bar + 2, *tfull = bar + 3, *tempty = bar + 5;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 8);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const size_t ntiles = (a.n + MT_REC - 1) / MT_REC;
    const uint32_t G = gridDim.x, b0 = blockIdx.x;
    const uint32_t mine = b0 < ntiles ? (uint32_t)((ntiles - 1 - b0) / G + 1) : 0u;
    for (int i = tid; i < MT_N; i += blockDim.x) sprow[i] = i < a.G ? a.prow[i] : 0.f;
    if (tid == 0) {
        bar_init(bfull, 1);
        bar_init(afull, 1);
        bar_init(aempty, 1);
        bar_init(tfull, 1);
        bar_init(tfull + 1, 1);
        // (the epilogue warps with rows: four per 64-row column group in use)
        const int ncg = min(4, (a.G + 63) / 64);
        bar_init(tempty, 4 * ncg);
        bar_init(tempty + 1, 4 * ncg);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == MT_MMA) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         su32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == MT_PROD) {
        if (lane == 0) {
            bar_expect_tx(bfull, MT_B_BYTES);
            for (int c = 0; c < 4; ++c)  // (four 32 KB copies)
                bulk_g2s(sb + c * (MT_B_BYTES / 4), reinterpret_cast<const char*>(bimg) + c * (MT_B_BYTES / 4),
                         MT_B_BYTES / 4, bfull);
            for (uint32_t it = 0; it < mine; ++it) {
                if (it > 0) bar_wait(aempty, (it - 1) & 1u);
                bar_expect_tx(afull, MT_A_BYTES);
                const char* src = reinterpret_cast<const char*>(aimg) + (size_t)(b0 + it * G) * MT_A_BYTES;
                bulk_g2s(sa, src, MT_A_BYTES / 2, afull);
                bulk_g2s(sa + MT_A_BYTES / 2, src + MT_A_BYTES / 2, MT_A_BYTES / 2, afull);
            }
        }
    } else if (warp == MT_MMA) {
        if (lane == 0) {
            // D f32, A / B tf32, both K-major, N = 256, M = 128
            constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(MT_N >> 3) << 17) |
                                       ((uint32_t)(MT_REC >> 4) << 24);
            bar_wait(bfull, 0);
            const uint32_t abase = su32(sa), bbase = su32(sb);
            for (uint32_t it = 0; it < mine; ++it) {
                const uint32_t ts = it & 1u;
                bar_wait(afull, it & 1u);
                if (it >= 2) bar_wait(tempty + ts, ((it >> 1) & 1u) ^ 1u);
                tc_fence_after();
                const uint32_t dcol = tmem + ts * MT_N;
#pragma unroll
                for (int ks = 0; ks < 8; ++ks) {
                    const uint64_t ahi = umma_desc(abase + (0 * 8 + ks) * 4096, 128, 256, 0);
                    const uint64_t alo = umma_desc(abase + (1 * 8 + ks) * 4096, 128, 256, 0);
                    const uint64_t bhi = umma_desc(bbase + (0 * 8 + ks) * 8192, 128, 256, 0);
                    const uint64_t blo = umma_desc(bbase + (1 * 8 + ks) * 8192, 128, 256, 0);
                    umma_tf32(dcol, ahi, bhi, IDESC, ks > 0 ? 1u : 0u);
                    umma_tf32(dcol, alo, bhi, IDESC, 1u);
                    umma_tf32(dcol, ahi, blo, IDESC, 1u);
                }
                umma_commit(aempty);
                umma_commit(tfull + ts);
            }
        }
    } else {
        // epilogue: warp w reads TMEM lane quarter w & 3 (records), columns
        // (rows of the step) [64 (w >> 2), + 64) in chunks of 16.  Gains are
        // tiled [n / 32][gs][32]: a row's gains of a warp's 32 records are one
        // 128-byte line, at a constant offset from the warp's base (no
        // address arithmetic per pair); loaded one chunk ahead.
        // The per-row (best, index, second) over the warp's 32 records goes
        // through a shared-memory transpose (4-float groups XOR-swizzled by
        // row: conflict-free stores and 16-byte loads): lanes q and q + 16 scan
        // records 0-15 / 16-31 of row q and merge (no cross-lane reduction per
        // pair).
        const int quarter = warp & 3, cg = warp >> 2;
        const float lam = (float)a.lambda;
        float* tb = strans + warp * (16 * MT_TS);
        const int nch = max(0, min(4, (a.G - cg * 64 + 15) / 16));  // chunks with rows
        const uint32_t total = mine * (uint32_t)nch;
        // this warp's gains of row c0 + j: gw(w)[(c0 + j) * 32]
        auto gw = [&](size_t w) { return a.gain + w * (size_t)a.gs * 32 + lane; };
        auto load = [&](uint32_t k, float (&gl)[16]) {
            const size_t w = (b0 + (size_t)(k / nch) * G) * 4 + quarter;
            const int c0 = cg * 64 + (int)(k % nch) * 16;
            if (w * 32 + lane < a.n && k < total) {
                const float* gp = gw(w) + (size_t)c0 * 32;
#pragma unroll
                for (int j = 0; j < 16; ++j) gl[j] = gp[j * 32];
            } else {
#pragma unroll
                for (int j = 0; j < 16; ++j) gl[j] = -INFINITY;
            }
        };
        // top-2 of 16 rows x 32 records (values v[j], this lane's record):
        // lane q < 16 ends with row q's (best, index, second)
        auto top2_16 = [&](const float (&v)[16], size_t w, float& b, uint32_t& bi, float& s2) {
#pragma unroll
            for (int j = 0; j < 16; ++j) tb[j * MT_TS + (lane ^ ((j & 7) << 2))] = v[j];
            __syncwarp();
            const int q = lane & 15, r0 = (lane >> 4) * 16;
            b = -INFINITY;
            s2 = -INFINITY;
            int br = r0;
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const float4 x4 =
                    *reinterpret_cast<const float4*>(tb + q * MT_TS + ((r0 + 4 * m) ^ ((q & 7) << 2)));
                const float xs[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float x = xs[e];
                    s2 = fmaxf(s2, fminf(x, b));  // the second: max over min(x, best so far)
                    if (x > b) {
                        b = x;
                        br = r0 + 4 * m + e;
                    }
                }
            }
            __syncwarp();
            // merge with lane q + 16 (its records come later: ties keep ours)
            const float ob = __shfl_xor_sync(0xffffffffu, b, 16);
            const float os = __shfl_xor_sync(0xffffffffu, s2, 16);
            const int obr = __shfl_xor_sync(0xffffffffu, br, 16);
            const bool lo_half = lane < 16;
            const float b1 = lo_half ? b : ob, s1 = lo_half ? s2 : os;   // records 0-15
            const float b2 = lo_half ? ob : b, s22 = lo_half ? os : s2;  // records 16-31
            const int br1 = lo_half ? br : obr, br2 = lo_half ? obr : br;
            if (b2 > b1) {
                b = b2;
                br = br2;
                s2 = fmaxf(b1, s22);
            } else {
                b = b1;
                br = br1;
                s2 = fmaxf(b2, s1);
            }
            bi = (uint32_t)(w * 32) + (uint32_t)br;
        };
        auto put = [&](uint32_t* part, int g, size_t w, float b, uint32_t bi, float s2) {
            if (lane < 16 && g < a.G) {
                uint32_t* pp = part + ((size_t)g * a.nw + w) * 3;
                pp[0] = __float_as_uint(b);
                pp[1] = bi;
                pp[2] = __float_as_uint(s2);
            }
        };
        // running (best, index, second) of this warp's rows over its tiles
        // (lane q < 16: row cg 64 + ch 16 + q), combined per CTA at the end
        float rb[4], rs[4];
        uint32_t ri[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            rb[c] = -INFINITY;
            rs[c] = -INFINITY;
            ri[c] = 0;
        }
        float gq[2][16];
        if (step > 0) load(0, gq[0]);
        for (uint32_t k = 0; k < total; ++k) {
            const uint32_t it = k / (uint32_t)nch;
            const int ch = (int)(k % (uint32_t)nch);
            const uint32_t ts = it & 1u;
            const size_t tile = b0 + (size_t)it * G;
            const size_t rec = tile * MT_REC + quarter * 32 + lane;
            const bool valid = rec < a.n;
            const size_t w = tile * 4 + quarter;  // this warp's 32 records
            const int c0 = cg * 64 + ch * 16;
            if (step > 0) load(k + 1, gq[1]);
            if (ch == 0) {
                bar_wait(tfull + ts, (it >> 1) & 1u);
                tc_fence_after();
            }
            const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + ts * MT_N;
            float acc[16];
            tmem_ld16(taddr + (uint32_t)c0, acc);
            if (ch == nch - 1) {  // the tile's accumulator is read: release the TMEM stage
                tc_fence_before();
                __syncwarp();
                if (lane == 0) bar_arrive(tempty + ts);
            }
            const float pi = valid ? a.p32[rec] : 0.f;
            float pr[16];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const float4 t = *reinterpret_cast<const float4*>(sprow + c0 + 4 * m);
                pr[4 * m] = t.x;
                pr[4 * m + 1] = t.y;
                pr[4 * m + 2] = t.z;
                pr[4 * m + 3] = t.w;
            }
            // rows >= G: their gains stay -inf (never stored, never a best)
            const int gl_n = min(16, a.G - c0);
            float gv[16];
            if (step == 0) {
                const float ai = valid ? a.a32[rec] : 0.f;
                float sv[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const float d2 = (pi + pr[j]) - 2.f * acc[j];
                    const float sim = ex2f(a.c_exp * d2);
                    const bool on = valid && j < gl_n;
                    gv[j] = on ? sim * ai : -INFINITY;
                    sv[j] = on ? sim : -INFINITY;
                }
                if (a.part_nn) {
                    float b, s2;
                    uint32_t bi;
                    top2_16(sv, w, b, bi, s2);
                    put(a.part_nn, c0 + lane, w, b, bi, s2);
                }
            } else {
                const float* gl = gq[0];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const float d2 = (pi + pr[j]) - 2.f * acc[j];
                    const float sim = ex2f(a.c_exp * d2);
                    // (taken records and padding rows hold -inf, invalid records load -inf)
                    gv[j] = gl[j] != -INFINITY && j < gl_n ? fmaf(-lam, sim, gl[j]) : -INFINITY;
                }
#pragma unroll
                for (int j = 0; j < 16; ++j) gq[0][j] = gq[1][j];
            }
            if (valid) {
                float* gp = gw(w) + (size_t)c0 * 32;
#pragma unroll
                for (int j = 0; j < 16; ++j) gp[j * 32] = gv[j];
            }
            float b, s2;
            uint32_t bi;
            top2_16(gv, w, b, bi, s2);
            put(a.part, c0 + lane, w, b, bi, s2);
#pragma unroll
            for (int c = 0; c < 4; ++c)
                if (c == ch) {
                    rs[c] = fmaxf(fmaxf(rs[c], s2), fminf(rb[c], b));
                    if (b > rb[c]) {
                        rb[c] = b;
                        ri[c] = bi;
                    }
                }
        }
        // the CTA's table: the four lane-quarter warps of each column group
        // through shared memory (the transpose buffers, idle now)
        asm volatile("bar.sync 1, %0;" ::"n"(MT_EPI * 32) : "memory");
        float* my = strans + warp * (16 * MT_TS);  // [4 chunks][16 rows][3]
        if (lane < 16)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                my[(c * 16 + lane) * 3] = rb[c];
                my[(c * 16 + lane) * 3 + 1] = __uint_as_float(ri[c]);
                my[(c * 16 + lane) * 3 + 2] = rs[c];
            }
        asm volatile("bar.sync 1, %0;" ::"n"(MT_EPI * 32) : "memory");
        if (quarter == 0 && a.cpart)
            for (int e = lane; e < 64; e += 32) {
                const int g = cg * 64 + e;
                if (e / 16 >= nch || g >= a.G) continue;
                float b = -INFINITY, s2 = -INFINITY;
                uint32_t bi = 0;
#pragma unroll
                for (int qq = 0; qq < 4; ++qq) {
                    const float* o = strans + (cg * 4 + qq) * (16 * MT_TS) + e * 3;
                    const float ob = o[0], os = o[2];
                    s2 = fmaxf(fmaxf(s2, os), fminf(b, ob));
                    if (ob > b) {
                        b = ob;
                        bi = __float_as_uint(o[1]);
                    }
                }
                uint32_t* cp = a.cpart + ((size_t)g * a.ncta + blockIdx.x) * 3;
                cp[0] = __float_as_uint(b);
                cp[1] = bi;
                cp[2] = __float_as_uint(s2);
            }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == MT_MMA) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

// exact similarity of record i to an exact row (experience.cpp:30-40 order)
// standardize(), experience.cpp:71-75, in the reference's rounding
__device__ __forceinline__ double zexact(const G32Args& a, size_t i, int k) {
    return ddiv(dsub(a.x64[i * a.d + k], a.msd[k]), a.msd[a.d + k]);
}

__device__ __forceinline__ double sim64_rec(const G32Args& a, size_t i, const double* row) {
    double d2 = 0.0;
    for (int k = 0; k < a.d; ++k) {
        const double t = dsub(zexact(a, i, k), row[k]);
        d2 = dadd(d2, dmul(t, t));
    }
    return sim_from_d2(d2, a.two_s2);
}

// Candidates of a (best, idx, second) table: every record within `thr`.
// Returns the count (CMAX + 1 on overflow).
__device__ int collect(const G32Args& a, const uint32_t* part, const float* vals, int g,
                       double thr, uint32_t* cand, int* s_cnt) {
    if (threadIdx.x == 0) *s_cnt = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < a.nw; t += blockDim.x) {
        const uint32_t* pp = part + ((size_t)g * a.nw + t) * 3;
        const float b = __uint_as_float(pp[0]), s2 = __uint_as_float(pp[2]);
        if ((double)b < thr) continue;
        if ((double)s2 < thr) {  // this warp's best only
            const int c = atomicAdd(s_cnt, 1);
            if (c < CMAX) cand[c] = pp[1];
        } else if (vals) {  // several: every record of the warp that qualifies
            for (int l = 0; l < 32; ++l) {
                const size_t r = (size_t)t * 32 + l;
                if (r < a.n && (double)vals[a.gs ? ((r >> 5) * a.gs + g) * 32 + (r & 31) : (size_t)g * a.n + r] >= thr) {
                    const int c = atomicAdd(s_cnt, 1);
                    if (c < CMAX) cand[c] = (uint32_t)r;
                }
            }
        } else {
            atomicAdd(s_cnt, CMAX + 1);  // (no per-record values kept: overflow)
        }
    }
    __syncthreads();
    return *s_cnt;
}

// the same from the tensor-core step's per-CTA table: a CTA whose second best
// is below thr contributes its best only; otherwise its warps' table entries
// (its tiles t = c + i ncta, four warps each) are examined as collect() does
__device__ int collect_cta(const G32Args& a, int g, double thr, uint32_t* cand, int* s_cnt) {
    if (threadIdx.x == 0) *s_cnt = 0;
    __syncthreads();
    const size_t ntiles = (a.n + 127) / 128;
    for (int c = threadIdx.x; c < a.ncta; c += blockDim.x) {
        const uint32_t* cp = a.cpart + ((size_t)g * a.ncta + c) * 3;
        const float b = __uint_as_float(cp[0]), s2 = __uint_as_float(cp[2]);
        if ((double)b < thr) continue;
        if ((double)s2 < thr) {
            const int k = atomicAdd(s_cnt, 1);
            if (k < CMAX) cand[k] = cp[1];
            continue;
        }
        for (size_t t = (size_t)c; t < ntiles; t += (size_t)a.ncta)
            for (int qq = 0; qq < 4; ++qq) {
                const size_t w = t * 4 + qq;
                const uint32_t* pp = a.part + ((size_t)g * a.nw + w) * 3;
                const float wb = __uint_as_float(pp[0]), ws = __uint_as_float(pp[2]);
                if ((double)wb < thr) continue;
                if ((double)ws < thr) {
                    const int k = atomicAdd(s_cnt, 1);
                    if (k < CMAX) cand[k] = pp[1];
                    continue;
                }
                for (int l = 0; l < 32; ++l) {
                    const size_t r = w * 32 + l;
                    if (r < a.n && (double)a.gain[(w * a.gs + g) * 32 + l] >= thr) {
                        const int k = atomicAdd(s_cnt, 1);
                        if (k < CMAX) cand[k] = (uint32_t)r;
                    }
                }
            }
    }
    __syncthreads();
    return *s_cnt;
}

// per query: the step's pick, decided in fp64 among the fp32 candidates
__global__ void __launch_bounds__(256) g32_pick_kernel(const G32Args a, int step) {
    const int g = blockIdx.x, tid = threadIdx.x;
    extern __shared__ double sims[];  // [CMAX][step + 1]: sim to the query, then to picks 0..step-1
    __shared__ uint32_t cand[CMAX];
    __shared__ int s_cnt;
    __shared__ float s_m;
    __shared__ Best wb[8];
    const double* zq = a.zq + (size_t)g * a.d;
    // the veto scan's nearest record (step 0): the same filter on sim
    if (step == 0 && a.part_nn) {
        float m = -INFINITY;
        for (int t = tid; t < a.nw; t += blockDim.x)
            m = fmaxf(m, __uint_as_float(a.part_nn[((size_t)g * a.nw + t) * 3]));
#pragma unroll
        for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (tid == 0) s_m = -INFINITY;
        __syncthreads();
        if ((tid & 31) == 0) atomicMax(reinterpret_cast<int*>(&s_m), __float_as_int(m));  // m >= 0
        __syncthreads();
        const int nc = collect(a, a.part_nn, nullptr, g, (double)s_m - 2.0 * a.eps_nn, cand, &s_cnt);
        if (nc > CMAX) {
            if (tid == 0) a.overflow[g] = 1;
        } else {
            Best b{0.0, 0, 0, -1};
            if (tid < nc) {
                const size_t r = cand[tid];
                b = Best{sim64_rec(a, r, zq), 0, (int64_t)r, 1};  // first index on ties
            }
            b = warp_best(b);
            if ((tid & 31) == 0) wb[tid >> 5] = b;
            __syncthreads();
            if (tid == 0) {
                Best c = wb[0];
                for (int x = 1; x < 8; ++x)
                    if (better(wb[x], c)) c = wb[x];
                a.nn[g] = c.j < 0 ? -1 : c.i;
                a.nn_sim[g] = c.j < 0 ? -1.0 : c.g;
            }
        }
        __syncthreads();
    }
    // max fp32 gain, then the candidates within 2 eps(step)
    float m = -INFINITY;
    if (a.ncta)
        for (int c = tid; c < a.ncta; c += blockDim.x)
            m = fmaxf(m, __uint_as_float(a.cpart[((size_t)g * a.ncta + c) * 3]));
    else
        for (int t = tid; t < a.nw; t += blockDim.x)
            m = fmaxf(m, __uint_as_float(a.part[((size_t)g * a.nw + t) * 3]));
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    __shared__ float wm[8];
    if ((tid & 31) == 0) wm[tid >> 5] = m;
    __syncthreads();
    if (tid == 0) {
        float x = wm[0];
        for (int k = 1; k < 8; ++k) x = fmaxf(x, wm[k]);
        s_m = x;
    }
    __syncthreads();
    const double eps = a.e0 + step * a.e1 + (double)step * step * a.e2;
    const int nc = a.ncta ? collect_cta(a, g, (double)s_m - 2.0 * eps, cand, &s_cnt)
                          : collect(a, a.part, a.gain, g, (double)s_m - 2.0 * eps, cand, &s_cnt);
    if (nc > CMAX || nc == 0) {
        if (tid == 0) a.overflow[g] = 1;
        return;
    }
    if (tid == 0 && a.ncand) atomicAdd(a.ncand, (unsigned)nc);
    // exact gains: every (candidate, row) similarity in parallel -- row 0 is
    // the query, rows 1..step the picks so far -- then each candidate's
    // score and penalty in the reference's order
    const int nr = step + 1;
    for (int w = tid; w < nc * nr; w += blockDim.x) {
        const int c = w / nr, j = w % nr;
        const size_t r = cand[c];
        double s;
        if (j == 0) {
            s = sim64_rec(a, r, zq);
        } else {
            const size_t p = (size_t)a.picks[(size_t)g * a.want + (j - 1)];
            double d2 = 0.0;
            for (int k = 0; k < a.d; ++k) {
                const double t = dsub(zexact(a, r, k), zexact(a, p, k));
                d2 = dadd(d2, dmul(t, t));
            }
            s = sim_from_d2(d2, a.two_s2);
        }
        sims[c * nr + j] = s;
    }
    __syncthreads();
    Best b{0.0, 0, 0, -1};
    double sc = 0.0;
    if (tid < nc) {
        const size_t r = cand[tid];
        const double rr = a.r64[r];
        const double loo = a.loo ? a.loo[r]
                                 : (a.n_loo <= 1 ? 0.0 : ddiv(dsub(a.total, rr), (double)(a.n_loo - 1)));
        sc = dmul(sims[tid * nr], fabs(dsub(rr, loo)));
        double pen = 0.0;
        for (int j = 1; j < nr; ++j) pen = dadd(pen, sims[tid * nr + j]);  // :283-284, pick order
        b = Best{dsub(sc, dmul(a.lambda, pen)), a.rnd[r], (int64_t)r, tid};
    }
    b = warp_best(b);
    if ((tid & 31) == 0) wb[tid >> 5] = b;
    __syncthreads();
    if (tid == 0) {
        Best c = wb[0];
        for (int x = 1; x < 8; ++x)
            if (better(wb[x], c)) c = wb[x];
        wb[0] = c;
    }
    __syncthreads();
    const Best win = wb[0];
    const size_t p = (size_t)win.i;
    if (tid == win.j) a.pscore[(size_t)g * a.want + step] = sc;
    if (tid == 0) {
        a.picks[(size_t)g * a.want + step] = (int64_t)p;
        a.gain[a.gs ? ((p >> 5) * a.gs + g) * 32 + (p & 31) : (size_t)g * a.n + p] = -INFINITY;  // taken
        a.ppick[g] = a.p32[p];
    }
}

// the next step's rows: the picks' fp32 rows (DP floats, zero padded)
__global__ void g32_stage_kernel(const G32Args a, int step, int DP) {
    const int g = blockIdx.x;
    const size_t p = (size_t)a.picks[(size_t)g * a.want + step];
    for (int k = threadIdx.x; k < DP; k += blockDim.x)
        a.pick32[(size_t)g * DP + k] = a.z32[(size_t)k * a.n + p];
}

// curriculum order (:290-294) and outputs: a warp per query, a lane per pick
// (its exact similarity, then its position by counting)
__global__ void g32_finish_kernel(const G32Args a, int64_t gbase, int m, int64_t* out_idx,
                                  double* out_sim, double* out_score, double* out_rew,
                                  int32_t* out_round) {
    const int g = blockIdx.x, lane = threadIdx.x;
    const int64_t* pk = a.picks + (size_t)g * a.want;
    const double* zq = a.zq + (size_t)g * a.d;
    for (int x = lane; x < a.want; x += 32) {
        const size_t p = (size_t)pk[x];
        const double rv = a.r64[p];
        const int32_t dv = a.rnd[p];
        int pos = 0;
        for (int y = 0; y < a.want; ++y) {
            const size_t u = (size_t)pk[y];
            const double ru = a.r64[u];
            const int32_t du = a.rnd[u];
            pos += ru != rv ? ru < rv : (du < dv || (du == dv && y < x));
        }
        const size_t o = (size_t)g * m + pos;
        out_idx[o] = gbase + (int64_t)p;
        out_sim[o] = sim64_rec(a, p, zq);
        out_score[o] = a.pscore[(size_t)g * a.want + x];
        out_rew[o] = rv;
        out_round[o] = dv;
    }
}

// fp32 rows, their squared norms, |r - loo| (fp32) and the largest norm
// (z32: (x - mean) * (1 / sd) in fp64, rounded to fp32 -- within 2^-24 + 2^-51
// of the exact standardized value, the storage rounding g32_eps allows);
// img: the tensor-core step's 3xTF32 operand image of the same values (four
// dimensions per 16-byte store), or null
__global__ void g32_prep_kernel(const double* __restrict__ x64, const double* __restrict__ msd,
                                const double* __restrict__ r64,
                                const double* __restrict__ loo, size_t n, size_t n_loo,
                                double total, int d, int DP, float* __restrict__ z32,
                                float* __restrict__ p32, float* __restrict__ a32,
                                unsigned int* __restrict__ pmax, float* __restrict__ amax,
                                float* __restrict__ img) {
    const size_t ntot = img ? (n + 127) / 128 * 128 : n;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < ntot;
         i += (size_t)gridDim.x * blockDim.x) {
        const bool valid = i < n;
        float p = 0.f;
        float* t = img ? img + (i / 128) * (MT_A_BYTES / 4) : nullptr;
        const int r = (int)(i % 128);
        for (int k0 = 0; k0 < DP; k0 += 4) {
            float v[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int k = k0 + e;
                v[e] = valid && k < d ? (float)dmul(dsub(x64[i * d + k], msd[k]), msd[2 * d + k]) : 0.f;
                if (valid) {
                    z32[(size_t)k * n + i] = v[e];
                    p = fmaf(v[e], v[e], p);
                }
            }
            if (t) {
                float4 hi, lo;
                hi.x = mt_tf32(v[0]); lo.x = mt_tf32(v[0] - hi.x);
                hi.y = mt_tf32(v[1]); lo.y = mt_tf32(v[1] - hi.y);
                hi.z = mt_tf32(v[2]); lo.z = mt_tf32(v[2] - hi.z);
                hi.w = mt_tf32(v[3]); lo.w = mt_tf32(v[3] - hi.w);
                *reinterpret_cast<float4*>(t + mt_off(0, k0, r, MT_REC)) = hi;
                *reinterpret_cast<float4*>(t + mt_off(1, k0, r, MT_REC)) = lo;
            }
        }
        if (!valid) continue;
        p32[i] = p;
        const double rr = r64[i];
        const double l = loo ? loo[i] : (n_loo <= 1 ? 0.0 : (total - rr) / (double)(n_loo - 1));
        const float av = (float)fabs(rr - l);
        a32[i] = av;
        atomicMax(pmax, __float_as_uint(p));
        atomicMax(reinterpret_cast<unsigned int*>(amax), __float_as_uint(av));
    }
}

template <int DP>
void g32_steps(const G32Args& a, int nctas, cudaStream_t st) {
    for (int step = 0; step < a.want; ++step) {
        G32Args b = a;
        if (step > 0) {
            b.row32 = a.pick32;
            b.prow = a.ppick;
        }
        g32_step_kernel<DP><<<dim3(nctas, (a.G + GQ2 - 1) / GQ2), FT, 0, st>>>(b, step);
        const size_t smem = (size_t)CMAX * (step + 1) * 8;
        if (smem > 48 * 1024)
            SAIR_CUDA(cudaFuncSetAttribute(g32_pick_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem));
        g32_pick_kernel<<<a.G, 256, smem, st>>>(b, step);
        if (step + 1 < a.want) g32_stage_kernel<<<a.G, 64, 0, st>>>(a, step, DP);
    }
    SAIR_LAUNCH("g32 steps");
}

// ev: 2 want events (each step kernel's start, end), or empty
void g32_steps_mma(const G32Args& a, const float* aimg, float* bimg, const float* q32,
                   cudaStream_t st, const std::vector<cudaEvent_t>& ev) {
    // a per-device function attribute (sharded stores put shards on several GPUs)
    static std::atomic<uint64_t> attr_set{0};
    int dev = 0;
    SAIR_CUDA(cudaGetDevice(&dev));
    const uint64_t bit = 1ull << (dev & 63);
    if (!(attr_set.load() & bit)) {
        SAIR_CUDA(cudaFuncSetAttribute(g32_mma_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)MT_SMEM));
        attr_set.fetch_or(bit);
    }
    const size_t ntiles = (a.n + MT_REC - 1) / MT_REC;
    const int grid = (int)std::min<size_t>(ntiles, 148);
    for (int step = 0; step < a.want; ++step) {
        G32Args b = a;
        if (step > 0) {
            b.row32 = a.pick32;
            b.prow = a.ppick;
        }
        g32_mma_bimg_kernel<<<64, 256, 0, st>>>(b.row32, a.G, 64, bimg);
        if (!ev.empty()) SAIR_CUDA(cudaEventRecord(ev[2 * step], st));
        g32_mma_step_kernel<<<grid, MT_THREADS, MT_SMEM, st>>>(b, aimg, bimg, step);
        if (!ev.empty()) SAIR_CUDA(cudaEventRecord(ev[2 * step + 1], st));
        const size_t smem = (size_t)CMAX * (step + 1) * 8;
        if (smem > 48 * 1024)
            SAIR_CUDA(cudaFuncSetAttribute(g32_pick_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem));
        g32_pick_kernel<<<a.G, 256, smem, st>>>(b, step);
        if (step + 1 < a.want) g32_stage_kernel<<<a.G, 64, 0, st>>>(a, step, 64);
    }
    (void)q32;
    SAIR_LAUNCH("g32 steps (tensor cores)");
}

}  // namespace

// The filter's error bound: with Pm >= every squared
// norm of a record / query row (fp32, rounded up), the fp32 norm expansion
// d2 = (P_i + P_r) - 2 <z_i, z_r> differs from the exact distance by at most
// D = (4 DP + 32) 2^-24 Pm (storage rounding of z, the dot's DP fused terms,
// the norms' sums, the final sums); sim = exp(-d2 / 2 sigma^2) <= 1 moves by
// at most D / (2 sigma^2), plus the argument's rounding and ex2.approx
// (relative 2^-21): e_sim.  score32 = sim32 a32 (a = |r - loo| rounded once):
// e_sim A + 2^-22 A.  Each penalty step subtracts lambda sim32 with two
// roundings: |lambda| (e_sim + 2^-23) + 2^-23 (A + |lambda| t).
// The tensor-core step (mma): the dot in 3xTF32 -- operand splits within
// 2^-22 (x2) and the dropped lo.lo term (2^-22), a chain of 3 DP products
// accumulated in fp32 ((3 DP + 32) 2^-24, plus 2^-20 for the accumulator's
// internal order, as the wide pass's bound) -- doubled in d2: D = (8 DP +
// 160) 2^-24 Pm with the norms' and final sums.
void g32_eps(int DP, double pm, double amax, double two_s2, double lambda, double* e0,
             double* e1, double* e2, double* e_sim, bool mma = false) {
    const double D = (mma ? 8.0 * DP + 160.0 : 4.0 * DP + 32.0) * std::ldexp(1.0, -24) * pm;
    const double argmax = 4.0 * pm / two_s2 * 1.4426950408889634 + 1.0;
    const double es = D / two_s2 + std::ldexp(1.0, -22) * argmax + std::ldexp(1.0, -21);
    const double la = std::fabs(lambda);
    *e_sim = es * 1.01 + 1e-12;
    *e0 = (es * amax + std::ldexp(1.0, -22) * amax) * 1.01 + 1e-12;
    *e1 = (la * (es + std::ldexp(1.0, -23)) + std::ldexp(1.0, -23) * amax) * 1.01;
    *e2 = std::ldexp(1.0, -23) * la * 1.01;
}

bool greedy32_select(sair_store_s* s, const QueryPrep& p, const std::vector<size_t>& qidx,
                     size_t m, double lambda, const double* loo, bool want_nn, int64_t* out_idx,
                     double* out_sim, double* out_score, size_t* out_count, int64_t* out_nn,
                     double* out_nn_sim, double* out_reward, int32_t* out_round,
                     std::vector<size_t>* fallback) {
    const size_t nq = qidx.size();
    const size_t n = s->n;
    const int d = s->d;
    if (nq == 0) return true;
    if (d > 64 || m > 256 || n >= 0xFFFFFFFFull) return false;
    const int DP = d <= 16 ? 16 : (d <= 32 ? 32 : 64);
    const int want = (int)std::min(m, n);
    // queries per batch: 4 B of gain per (query, record) within ~2 GB
    const size_t G = std::max<size_t>(1, std::min<size_t>({nq, 256, ((size_t)2 << 30) / (4 * n)}));
    const int nctas = (int)((n + FT - 1) / FT);
    const int nw = nctas * (FT / 32);
    const size_t ob = G * m * (8 * 4 + 4) + G * 16 + 256;
    size_t off = 0;
    auto sz = [&](size_t b) { const size_t o = off; off += (b + 255) & ~(size_t)255; return o; };
    const size_t o_msd = sz((3 * (size_t)d + G * d) * 8), o_z32 = sz(n * DP * 4),
                 o_p32 = sz(n * 4), o_a32 = sz(n * 4), o_mx = sz(64), o_gain = sz(((G + 15) & ~(size_t)15) * ((n + 127) & ~(size_t)127) * 4),
                 o_part = sz(G * nw * 12), o_pnn = sz(want_nn ? G * nw * 12 : 0),
                 o_q32 = sz(G * DP * 4 + G * 4), o_pick = sz(G * DP * 4 + G * 4),
                 o_picks = sz(G * std::max(want, 1) * 8), o_psc = sz(G * std::max(want, 1) * 8),
                 o_nn = sz(G * 16), o_of = sz(G * 4 + 64), o_out = sz(ob);
    // the tensor-core step (d in 33..64): the records' 3xTF32 operand image
    const bool mma = DP == 64 && !(std::getenv("SAIR_G32_MMA") && std::atoi(std::getenv("SAIR_G32_MMA")) == 0);
    const size_t ntiles = (n + MT_REC - 1) / MT_REC;
    const size_t o_aimg = sz(mma ? ntiles * MT_A_BYTES : 0), o_bimg = sz(mma ? MT_B_BYTES : 0),
                 o_cpart = sz(mma ? G * 148 * 12 : 0);
    char* base = static_cast<char*>(s->b_greedy.get(off + 256));
    double* msd = reinterpret_cast<double*>(base + o_msd);
    double* zq = msd + 3 * (size_t)d;
    float* z32 = reinterpret_cast<float*>(base + o_z32);
    float* p32 = reinterpret_cast<float*>(base + o_p32);
    float* a32 = reinterpret_cast<float*>(base + o_a32);
    unsigned int* mx = reinterpret_cast<unsigned int*>(base + o_mx);
    G32Args a{};
    a.z32 = z32;
    a.p32 = p32;
    a.a32 = a32;
    a.x64 = s->x64;
    a.msd = msd;
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
    a.c_exp = (float)(-1.4426950408889634 / p.two_s2);
    a.gain = reinterpret_cast<float*>(base + o_gain);
    a.part = reinterpret_cast<uint32_t*>(base + o_part);
    a.part_nn = want_nn ? reinterpret_cast<uint32_t*>(base + o_pnn) : nullptr;
    a.nw = nw;
    float* q32 = reinterpret_cast<float*>(base + o_q32);
    a.pick32 = reinterpret_cast<float*>(base + o_pick);
    a.ppick = a.pick32 + G * DP;
    a.picks = reinterpret_cast<int64_t*>(base + o_picks);
    a.pscore = reinterpret_cast<double*>(base + o_psc);
    a.nn = reinterpret_cast<int64_t*>(base + o_nn);
    a.nn_sim = reinterpret_cast<double*>(a.nn + G);
    a.overflow = reinterpret_cast<int*>(base + o_of);
    a.ncand = reinterpret_cast<unsigned int*>(a.overflow + G);
    char* dout = base + o_out;
    char* hout = static_cast<char*>(s->h_out.get(ob + G * 4 + 64));
    // per-call preparation: exact rows, fp32 rows and norms, |r - loo|
    double* hin = s->h_consts.as<double>(3 * (size_t)d + G * d);
    std::copy(p.mean.begin(), p.mean.end(), hin);
    std::copy(p.sd.begin(), p.sd.end(), hin + d);
    for (int k = 0; k < d; ++k) hin[2 * d + k] = 1.0 / p.sd[k];
    SAIR_CUDA(cudaMemcpyAsync(msd, hin, 3 * (size_t)d * 8, cudaMemcpyHostToDevice, s->st));
    SAIR_CUDA(cudaMemsetAsync(mx, 0, 64, s->st));
    float* aimg = mma ? reinterpret_cast<float*>(base + o_aimg) : nullptr;
    float* bimg = mma ? reinterpret_cast<float*>(base + o_bimg) : nullptr;
    g32_prep_kernel<<<(int)std::min<size_t>((n + 255) / 256, 148 * 8), 256, 0, s->st>>>(
        s->x64, msd, s->r64, loo, n, eff_n(s), eff_stats(s).total, d, DP, z32, p32, a32, mx,
        reinterpret_cast<float*>(mx + 1), aimg);
    SAIR_LAUNCH("g32_prep_kernel");
    if (mma) {
        a.nw = (int)(ntiles * 4);
        a.gs = (int)((G + 15) & ~(size_t)15);  // tiled gains (padded rows)
        a.ncta = (int)std::min<size_t>(ntiles, 148);  // the step kernel's grid
        a.cpart = reinterpret_cast<uint32_t*>(base + o_cpart);
    }
    unsigned int hmx[2];
    SAIR_CUDA(cudaMemcpyAsync(hmx, mx, 8, cudaMemcpyDeviceToHost, s->st));
    SAIR_CUDA(cudaStreamSynchronize(s->st));
    float pmr, amr;
    std::memcpy(&pmr, &hmx[0], 4);
    std::memcpy(&amr, &hmx[1], 4);
    std::vector<float> hq(G * DP + G);
    int64_t* o_idx = reinterpret_cast<int64_t*>(dout);
    double* o_sim = reinterpret_cast<double*>(o_idx + G * m);
    double* o_score = o_sim + G * m;
    double* o_rew = o_score + G * m;
    int32_t* o_round = reinterpret_cast<int32_t*>(o_rew + G * m);
    s->last.greedy32_candidates = 0;
    s->last.greedy32_step_ms = 0.f;
    s->last.greedy32_steps = 0;
    for (size_t b0 = 0; b0 < nq; b0 += G) {
        const int g_n = (int)std::min(G, nq - b0);
        a.G = g_n;
        double pq = 0.0;
        for (int g = 0; g < g_n; ++g) {
            const double* zz = p.z.data() + qidx[b0 + g] * d;
            std::copy(zz, zz + d, hin + 3 * d + (size_t)g * d);
            float pr = 0.f;
            for (int k = 0; k < DP; ++k) {
                const float v = k < d ? (float)zz[k] : 0.f;
                hq[(size_t)g * DP + k] = v;
                pr = std::fma(v, v, pr);
            }
            hq[G * DP + g] = pr;
            pq = std::max(pq, (double)pr);
        }
        double e_sim;
        // Pm: the largest squared norm, fp32 sums rounded up by a relative 2^-16
        g32_eps(DP, std::max((double)pmr, pq) * (1.0 + std::ldexp(1.0, -16)), (double)amr * 1.0001,
                p.two_s2, lambda, &a.e0, &a.e1, &a.e2, &e_sim, mma);
        a.eps_nn = e_sim;
        SAIR_CUDA(cudaMemcpyAsync(zq, hin + 3 * d, (size_t)g_n * d * 8, cudaMemcpyHostToDevice, s->st));
        SAIR_CUDA(cudaMemcpyAsync(q32, hq.data(), (G * DP + G) * 4, cudaMemcpyHostToDevice, s->st));
        SAIR_CUDA(cudaMemsetAsync(a.overflow, 0, G * 4 + 64, s->st));
        a.row32 = q32;
        a.prow = q32 + G * DP;
        if (mma) {
            while (s->g32ev.size() < 2 * (size_t)want) {
                cudaEvent_t e;
                SAIR_CUDA(cudaEventCreate(&e));
                s->g32ev.push_back(e);
            }
            g32_steps_mma(a, aimg, bimg, q32, s->st, s->g32ev);
        }
        else switch (DP) {
            case 16: g32_steps<16>(a, nctas, s->st); break;
            case 32: g32_steps<32>(a, nctas, s->st); break;
            default: g32_steps<64>(a, nctas, s->st); break;
        }
        g32_finish_kernel<<<g_n, 32, 0, s->st>>>(a, s->gbase, (int)m, o_idx, o_sim, o_score, o_rew,
                                                 o_round);
        SAIR_LAUNCH("g32_finish_kernel");
        SAIR_CUDA(cudaMemcpyAsync(hout, dout, ob, cudaMemcpyDeviceToHost, s->st));
        SAIR_CUDA(cudaMemcpyAsync(hout + ob, a.overflow, G * 4 + 8, cudaMemcpyDeviceToHost, s->st));
        std::vector<int64_t> hnn(G);
        std::vector<double> hnns(G);
        if (want_nn) {
            SAIR_CUDA(cudaMemcpyAsync(hnn.data(), a.nn, G * 8, cudaMemcpyDeviceToHost, s->st));
            SAIR_CUDA(cudaMemcpyAsync(hnns.data(), a.nn_sim, G * 8, cudaMemcpyDeviceToHost, s->st));
        }
        SAIR_CUDA(cudaStreamSynchronize(s->st));
        if (mma)
            for (int st_i = 0; st_i < want; ++st_i) {
                float ms = 0.f;
                cudaEventElapsedTime(&ms, s->g32ev[2 * st_i], s->g32ev[2 * st_i + 1]);
                s->last.greedy32_step_ms += ms;
                s->last.greedy32_steps++;
            }
        const int64_t* hidx = reinterpret_cast<const int64_t*>(hout);
        const double* hsim = reinterpret_cast<const double*>(hidx + G * m);
        const double* hsc = hsim + G * m;
        const double* hrw = hsc + G * m;
        const int32_t* hrd = reinterpret_cast<const int32_t*>(hrw + G * m);
        const int* hof = reinterpret_cast<const int*>(hout + ob);
        unsigned int nc = 0;
        std::memcpy(&nc, hout + ob + G * 4, 4);
        s->last.greedy32_candidates += nc;
        for (int g = 0; g < g_n; ++g) {
            const size_t q = qidx[b0 + g];
            if (hof[g]) {  // candidate overflow: the fp64 greedy decides this query
                fallback->push_back(q);
                continue;
            }
            out_count[q] = (size_t)want;
            std::copy(hidx + g * m, hidx + g * m + want, out_idx + q * m);
            std::copy(hsim + g * m, hsim + g * m + want, out_sim + q * m);
            std::copy(hsc + g * m, hsc + g * m + want, out_score + q * m);
            if (out_reward) std::copy(hrw + g * m, hrw + g * m + want, out_reward + q * m);
            if (out_round) std::copy(hrd + g * m, hrd + g * m + want, out_round + q * m);
            if (out_nn) {
                out_nn[q] = hnn[g] < 0 ? -1 : s->gbase + hnn[g];
                out_nn_sim[q] = hnns[g];
            }
        }
    }
    return true;
}

}  // namespace sair
