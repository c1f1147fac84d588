// select_wide.cu -- K4: the large-batch streaming filter on the tensor cores.
//
// For Q >= 32 queries per call the Q x N similarity contraction is a real GEMM
// (SURVEY.md 8(a) A9 "K4", configs 2/4/5), so one pass over the store serves
// QW = 32/64/128/256 queries at once instead of one pass per 8 (select_mma.cu):
//
//   warp 16 (producer) one bulk copy (TMA engine) per page into an NST-deep
//                      shared-memory ring; pages are stored as ready MN-major
//                      SWIZZLE_128B_BASE32B TF32 operand blocks (common.cuh).
//   warp 17 (MMA)      per page DP/8 tcgen05.mma kind::tf32, M = 128 records x
//                      N = QW queries x K = 8: A = the page tile, B = the query
//                      constants -2 c_qk / sd_k rounded to nearest TF32 (WB = 1;
//                      the bounded perturbation is carried by the
//                      certification), accumulating into TMEM (fp32); its
//                      commit also releases the page's shared stage.
//   warps 12-15        record constants: P = ||y||^2 (or the per-call cache),
//                      the log residual and the pre-test bounds per record.
//   warps 0-11         epilogue, three groups of four lane quarters taking every
//                      third page: 32 TMEM columns at a time (tcgen05.ld
//                      32x32b.x32), a loose pre-test per (record, query) pair,
//                      the exact key = log2 residual - alpha d2 on the rare hit.
//
// Two launches per query group, the same kernel in two modes:
//   sample  sqrt(5 K' npages) strided pages plus the highest-residual pages;
//           each warp writes the per-query maximum key of its 32 records
//           (redux.sync.max.f32 per column), so the K'-th largest of those
//           maxima is <= the store's K'-th key (distinct records) -> the
//           start threshold t0 (wide_kth_kernel).
//   stream  every page; a record whose key beats t0 is appended to its
//           query's list of this CTA (shared-memory slot counter, global
//           store; a full list only records the largest key it dropped,
//           which the certification bound then covers).
// At the end each CTA list keeps its K' best; the cross-CTA merge
// (launch_merge, select.cu) and the refine kernel finish exactly as for the
// 8-query path.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <vector>

#include <cub/cub.cuh>
#include <cuda_bf16.h>

#include "select_common.cuh"
#include "topk_select.cuh"
#include "umma.cuh"
#include "warp_topk.cuh"

namespace sair {

using namespace umma;

namespace {

// warp roles: 0-11 epilogue (three groups of four TMEM lane quarters taking
// every third unit), 12-15 record constants (two pairs taking alternate
// pages; they own the shared page stage), 16 producer, 17 MMA.
//
// A unit is one (page, query sub-group) accumulator: QW <= 128 is one
// sub-group per page; QW = 256 serves two sub-groups of 128 queries from the
// same shared page stage -- per page two sets of MMAs (N = 128, the B tile's
// halves) into two TMEM stages, each committed on its own -- so the store is
// streamed once per 256 queries while TMEM keeps four 128-column stages and
// the epilogue drains one (page, half) while the tensor core fills the next.
// (A single N = 256 accumulator leaves two TMEM stages: measured 1.45 ms per
// 16M-record pass against 1.2 here -- the MMA of page i + 2 waits on page i's
// whole epilogue.)
constexpr int WE = 12;                 // three groups of four epilogue warps

constexpr int NEG = WE / 4;
constexpr int W_REC = WE, W_PROD = WE + 4, W_MMA = WE + 5;
constexpr int WIDE_THREADS = (WE + 6) * 32;
// B operand parts: 1 = the query constants rounded to nearest TF32 (the
// perturbation is a bounded query error the certification carries, DESIGN.md
// "K4"); 2 = hi + lo split, two MMAs per K-step
constexpr int WB = 1;

struct WideArgs {
    const float* pages;
    const float* r32;
    uint32_t n, npages;
    float c1, c0, rdelta, alpha;
    int nst, ntm, knn, mode;  // smem page stages, TMEM stages; mode 0 = sample, 1 = stream
    uint32_t spages;          // sample mode: sampled pages (page = i * npages / spages) ...
    const uint32_t* hot;      // ... then these (distinct from the above; >= npages: empty)
    uint32_t nhot;
    const float* consts;      // B tiles (hi, lo; smem image) | s [DP] | cc [QW] | t0 [2QW]
    float* smax;              // sample out [2QW][4 * (spages + nhot)]
    float* lkey;              // stream out: per-CTA lists [grid][2QW][cap]
    uint32_t* lidx;
    unsigned int* dropped;    // [2QW] max ordinal of a key dropped on a full list
    uint32_t cap;             // per-CTA list capacity
    int kp, kv;               // K' of the selection / veto lists
    const float* pl_in;       // per-record (P, log residual) of this call, [n][2], or null
    float* pl_out;            // written by the call's first stream pass, or null
    float* okey;              // compacted lists out: [grid][2QW][kout] (the merge's input)
    uint32_t* oidx;
    int kout;
    unsigned int* pmax;       // max P over records (float bits)
    uint32_t tcols;           // TMEM columns allocated (power of two >= ntm * min(QW, 128))
    const uint16_t* pages16;  // bf16 pass: the bf16 page copy
    const void* consts16;     // bf16 pass: the query tile (QW rows x 128 B, swizzled)
    unsigned long long* trace;  // diagnostics (SAIR_WIDE_TRACE): CTA 0 event clocks, or null
    int probe;                // diagnostics (SAIR_PROBE_WIDE): 1 skip the epilogue math, 2 also the MMAs
};

// Candidate append: the slot comes from a shared-memory counter (no global
// round trip on the consumer's critical path), the entry is a fire-and-forget
// global store into this CTA's list; a full list keeps only the largest key
// it dropped (shared atomicMax, folded into the global bound at the end).
__device__ __forceinline__ void list_append(const WideArgs& a, uint32_t* scnt, uint32_t* sdrop,
                                            int nl, int L, float key, uint32_t rec) {
    const uint32_t slot = atomicAdd(&scnt[L], 1u);
    if (slot < a.cap) {
        const size_t o = ((size_t)blockIdx.x * nl + L) * a.cap + slot;
        a.lkey[o] = key;
        a.lidx[o] = rec;
    } else {
        atomicMax(&sdrop[L], f2ord(key));
    }
}

// diagnostics: clock of event ev of page/unit i (CTA 0, i in [TR0, TR0 + 64))
constexpr uint32_t TR0 = 100;
__device__ __forceinline__ void trace_ev(const WideArgs& a, uint32_t i, int ev) {
    if (a.trace && blockIdx.x == 0 && i >= TR0 && i < TR0 + 64) a.trace[(i - TR0) * 16 + ev] = clock64();
}

// nearest TF32 (ties away), as a float
__device__ __forceinline__ float tf32_rna(float v) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
    return __uint_as_float(r);
}

// lane l ends with max over the warp of v[l]: one redux.sync.max.f32 per
// column (sm_100a; CREDUX into a uniform register) and a select, where the
// shuffle transpose took 31 shuffles + 62 selects + 31 max per 32 columns
__device__ __forceinline__ float transpose_max(const float (&v)[32], int lane) {
    float out = -INFINITY;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        float r;
        asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v[j]));
        out = lane == j ? r : out;
    }
    return out;
}

// CG = 1: one CTA per SM, M = 128 MMAs.  CG = 2 (stream mode): CTA pairs
// (cluster of two SMs, cta_group::2): rank 0 issues M = 256 MMAs whose A rows
// are both CTAs' pages and whose B columns are split between them (each CTA
// holds half of every unit's queries), so each SM's tensor core reads half
// the B operand from its shared memory -- the MMA's operand reads were the
// largest shared-memory consumer -- and the halved B tile leaves room for a
// fifth page stage (more bytes in flight per SM: the stage ring is bounded
// by HBM latency, not bandwidth).
template <int DP, int QW, int CG>
__global__ void __launch_bounds__(WIDE_THREADS, 1)
    stream_wide_kernel(const __grid_constant__ WideArgs a) {
    constexpr int NH = QW > 128 ? QW / 128 : 1;  // query sub-groups (units) per page
    constexpr int QS = QW / NH;                  // queries per unit (MMA N)
    constexpr int QH = QS / CG;                  // B rows of a unit in this CTA
    constexpr int BOX_BYTES = 32 * DP * 4;     // 32 records x DP dims
    constexpr int PAGE_BYTES = 4 * BOX_BYTES;  // 128 records
    constexpr int KSTEPS = DP / 8;
    constexpr int BT_BYTES = QW * 32 / CG;     // one K-step B tile: this CTA's rows x 8 tf32
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // smem page stages, TMEM accumulator stages (decoupled: a page's shared
    // stage is released once the MMA has read it and P is done, its TMEM stage
    // once the epilogue is done), record-constant slots (>= ntm + 1 apart)
    // prec slots: the record-constant warps write page it's slot only once the
    // producer has refilled stage it % nst, i.e. once the MMAs of page it - nst
    // are done, which waited on the epilogue of every unit of page
    // it - nst - ntm / NH: nst + ntm / NH slots never overwrite a live one
    const int nst = a.nst, ntm = a.ntm, PR = a.nst + (a.ntm + NH - 1) / NH;
    unsigned char* stage = smem;
    // the bias K-step's A operand: four 32-record boxes whose dimension rows 0
    // and 1 are 1.0 (the rest 0), so the MMA adds B row 0 + B row 1 of every
    // query column to each record (swizzling permutes within a row: invariant)
    float* aconst = reinterpret_cast<float*>(stage + (size_t)nst * PAGE_BYTES);  // [4][8][32]
    float* btile = aconst + 4 * 8 * 32;  // [WB][KSTEPS] data K-steps, then the bias K-step
    float* bbias = btile + WB * KSTEPS * BT_BYTES / 4;
    float* prec = bbias + BT_BYTES / 4;  // [PR][4][PAGE]: Asel, Ann, P, lg
    float* ss = prec + (size_t)PR * 4 * PAGE;
    float* scc = ss + DP;
    float* sthr = scc + QW;
    float* sB = sthr + 2 * QW;   // loose pre-test constants per list (see below)
    float* sM = sB + 2 * QW;     // [2] max |B| per list kind
    uint32_t* scnt = reinterpret_cast<uint32_t*>(sM + 4);  // [2QW] CTA list fill
    uint32_t* sdrop = scnt + 2 * QW;                       // [2QW] dropped max ordinal
    // [WE][256] compaction histograms: aliased onto the page stages, which are
    // idle once every unit's epilogue is done (all copies landed, every MMA
    // and every record-constant read of them finished before)
    uint32_t* whist = reinterpret_cast<uint32_t*>(stage);
    uint64_t* full = reinterpret_cast<uint64_t*>(sdrop + 2 * QW);
    uint64_t* empty = full + 8;
    uint64_t* tfull = empty + 8;
    uint64_t* tempty = tfull + 8;
    uint64_t* pready = tempty + 8;  // [16]
    uint64_t* pfull = pready + 16;  // [8] CG = 2, rank 0: the peer's page of the stage landed
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pfull + 8);
    const uint32_t crank = CG == 2 ? cluster_rank() : 0u;

    // B operand, K-major without swizzle, arranged on the host in shared-memory
    // order (per K-step QW/8 groups of two 8x16B core matrices): a straight
    // coalesced copy
    // (CG = 2: this CTA's rows -- queries h QS + crank QH + j of unit h --
    // are whole 8-row core-matrix groups of the host image, 256 B each)
    {
        const float4* src = reinterpret_cast<const float4*>(a.consts);
        float4* dst = reinterpret_cast<float4*>(btile);
        constexpr int GRP = BT_BYTES / 256;  // 8-row groups per K-step in this CTA
        for (int i = tid; i < WB * KSTEPS * BT_BYTES / 16; i += WIDE_THREADS) {
            const int kk = i / (BT_BYTES / 16), g = (i / 16) % GRP, e = i % 16;
            const int gsrc = CG == 1 ? g : (g / (QH / 8)) * (QS / 8) + (int)crank * (QH / 8) + g % (QH / 8);
            dst[i] = src[(size_t)kk * (QW * 2) + gsrc * 16 + e];
        }
    }
    const float* cs = a.consts + WB * DP * QW;
    for (int i = tid; i < DP; i += WIDE_THREADS) ss[i] = cs[i];
    for (int i = tid; i < QW; i += WIDE_THREADS) scc[i] = cs[DP + i];
    for (int i = tid; i < 2 * QW; i += WIDE_THREADS)
        sthr[i] = (i < QW || a.knn) ? cs[DP + QW + i] : FLT_MAX;
    for (int i = tid; i < 4 * QW; i += WIDE_THREADS) scnt[i] = 0;  // scnt and sdrop
    __syncthreads();
    // Loose pre-test: the exact-formula test
    //   fma(-((P + cc_q) + D), alpha, lg) > thr_q         (selection list)
    //   -((P + cc_q) + D) > thrn_q                        (veto list)
    // implies  D + B_q < A + e  with B_q = thr_q / alpha + cc_q, A = lg / alpha - P
    // (veto: B = thrn_q + cc_q, A = -P) and e = 2^-19 (|A| + P + max|B|), a
    // margin far above the fp32 rounding of both forms.  The hot loop runs
    // the loose test (2 instructions per pair); the rare warp whose records
    // pass re-runs the exact formula on the passing columns.
    // Stream mode folds B_q into the accumulator: a ninth K-step multiplies
    // the ones of `aconst` with B_q split into two TF32 parts (hi + lo within
    // 2^-22 |B_q|), so TMEM holds D' = D + B_q and the hot loop is a plain
    // minimum (no per-column shared-memory operand: those loads were half of
    // the pass's shared-memory wavefronts, which the MMA's operand reads need).
    // The veto lists keep a per-column constant: D' + (Bn_q - B_q).
    for (int i = tid; i < 4 * 8 * 32; i += WIDE_THREADS) aconst[i] = ((i >> 5) & 7) < 2 ? 1.f : 0.f;
    if (warp == 0) {
        float mb[2] = {0.f, 0.f};
        // a query without a start threshold (t0 = -FLT_MAX: every record
        // passes) has no finite B_q; then the whole launch keeps B in shared
        // memory (the bias tile is zero and the loop adds B per column)
        bool fin = true;
        for (int q = lane; q < QW; q += 32) fin &= fabsf(sthr[q] / a.alpha + scc[q]) < 0x1p60f;
        const bool bias = a.mode == 1 && __all_sync(0xffffffffu, fin);
        for (int q = lane; q < QW; q += 32) {
            const float B = sthr[q] / a.alpha + scc[q];
            float hi = 0.f, lo = 0.f;
            if (bias) {
                hi = tf32_rna(B);
                lo = tf32_rna(B - hi);
            }
            // K-major core-matrix image (as the host builds the data K-steps),
            // this CTA's rows only
            const int jj = q % QS;
            if (CG == 1 || jj / QH == (int)crank) {
                const int lr = (q / QS) * QH + jj % QH;
                float* bq = bbias + (lr & 7) * 4 + (lr >> 3) * 64;
                *reinterpret_cast<float4*>(bq) = make_float4(hi, lo, 0.f, 0.f);
                *reinterpret_cast<float4*>(bq + 32) = make_float4(0.f, 0.f, 0.f, 0.f);
            }
            const float beff = hi + lo;
            sB[q] = B;
            // |D| <= P + cc_q: the margins below cover the accumulator's
            // rounding of D + B_q as well
            mb[0] = fmaxf(mb[0], fabsf(B) + scc[q]);
            const float Bn = sthr[QW + q] + scc[q];
            sB[QW + q] = Bn - beff;  // veto pre-test on D': D' + (Bn - B)
            mb[1] = fmaxf(mb[1], fabsf(Bn) + fabsf(Bn - beff) + fabsf(beff) + scc[q]);
        }
        if (lane == 0) sM[2] = bias ? 1.f : 0.f;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            mb[0] = fmaxf(mb[0], __shfl_xor_sync(0xffffffffu, mb[0], o));
            mb[1] = fmaxf(mb[1], __shfl_xor_sync(0xffffffffu, mb[1], o));
        }
        if (lane == 0) {
            sM[0] = mb[0];
            sM[1] = mb[1];
        }
    }
    if (tid == 0) {
        for (int s = 0; s < nst; ++s) {
            bar_init(&full[s], 1);
            // the MMAs' commit + the record-constant warp pair of the page (they
            // read it for P; and their arrival keeps their parity waits on
            // full[] from falling two phases behind)
            bar_init(&empty[s], 3);
        }
        for (int s = 0; s < ntm; ++s) {
            bar_init(&tfull[s], 1);
            // the four epilogue warps of the unit's group (CG = 2: in both CTAs;
            // only rank 0's barrier is used)
            bar_init(&tempty[s], 4 * CG);
        }
        for (int p = 0; p < PR; ++p) bar_init(&pready[p], 2);
        for (int s = 0; s < nst; ++s) bar_init(&pfull[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == W_MMA) {
        if (CG == 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             su32(tmem_slot)),
                         "r"(a.tcols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             su32(tmem_slot)),
                         "r"(a.tcols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        }
    }
    tc_fence_before();
    __syncthreads();
    // the peer's barriers are initialised before any remote arrival
    if (CG == 2) cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    const uint32_t units = a.mode == 0 ? a.spages + a.nhot : a.npages;
    const bool bias_on = sM[2] != 0.f;  // B folded into the accumulator (stream mode)
    const uint32_t G = gridDim.x, r0 = blockIdx.x;
    const uint32_t mine_self = r0 < units ? (units - 1 - r0) / G + 1 : 0;
    // CG = 2: both CTAs of a pair run rank 0's page count (rank 1's extra
    // iterations are empty pages: no copy, every record invalid)
    const uint32_t rb = r0 & ~1u;
    const uint32_t mine = CG == 1 ? mine_self : (rb < units ? (units - 1 - rb) / G + 1 : 0);
    auto page_of = [&](uint32_t it) -> uint32_t {
        const uint32_t u = r0 + it * G;
        if (a.mode != 0) return u;
        if (u < a.spages) return (uint32_t)((uint64_t)u * a.npages / a.spages);
        const uint32_t h = a.hot[u - a.spages];
        return h < a.npages ? h : 0u;  // an empty slot reads page 0, all its records invalid
    };
    auto empty_unit = [&](uint32_t it) -> bool {
        if (it >= mine_self) return true;
        const uint32_t u = r0 + it * G;
        return a.mode == 0 && u >= a.spages && a.hot[u - a.spages] >= a.npages;
    };

    if (warp == W_PROD) {
        // ---------------- producer: one bulk copy per page ----------------
        if (lane == 0) {
            for (uint32_t it = 0; it < mine; ++it) {
                const uint32_t s = it % nst, ph = (it / nst) & 1u;
                if (it >= (uint32_t)nst) bar_wait(&empty[s], ph ^ 1u);
                trace_ev(a, it, 0);  // producer: stage free, copy issued
                if (it >= mine_self) {
                    bar_arrive(&full[s]);  // CG = 2: an empty page of rank 1
                    continue;
                }
                bar_expect_tx(&full[s], PAGE_BYTES);
                bulk_g2s(stage + (size_t)s * PAGE_BYTES, a.pages + (size_t)page_of(it) * DP * PAGE,
                         PAGE_BYTES, &full[s]);
            }
        }
    } else if (warp == W_MMA) {
        // ---------------- MMA issuer ----------------
        if (lane == 0 && crank == 0) {
            // D f32, A/B tf32, A MN-major, B K-major, N = QS, M = 128 CG
            constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) |
                                       ((uint32_t)(QS >> 3) << 17) | ((uint32_t)(128 * CG >> 4) << 24);
            const uint32_t bbase = su32(btile);
            for (uint32_t it = 0; it < mine; ++it) {
                const uint32_t s = it % nst, ph = (it / nst) & 1u;
                bar_wait(&full[s], ph);
                if (CG == 2) bar_wait_cluster(&pfull[s], ph);  // and the peer's page
                trace_ev(a, it, 1);  // MMA: page landed
                const uint32_t abase = su32(stage + (size_t)s * PAGE_BYTES);
#pragma unroll
                for (int h = 0; h < NH; ++h) {
                    const uint32_t u = it * NH + h;  // unit: (page it, sub-group h)
                    const uint32_t ts = u % ntm, tph = (u / ntm) & 1u;
                    if (u >= (uint32_t)ntm) {
                        if (CG == 1) bar_wait(&tempty[ts], tph ^ 1u);
                        else bar_wait_cluster(&tempty[ts], tph ^ 1u);
                    }
                    trace_ev(a, it, 2 + h);  // MMA: TMEM stage of unit (it, h) free
                    tc_fence_after();
                    const uint32_t dcol = tmem + (uint32_t)(ts * QS);
#pragma unroll
                    for (int ks = 0; ks < KSTEPS; ++ks) {
                        const uint64_t ad = umma_desc(abase + ks * 1024, BOX_BYTES, 512, 1);
#pragma unroll
                        for (int w = 0; w < WB; ++w) {
                            // sub-group h: this CTA's rows [h QH, h QH + QH) of the K-step's B tile
                            const uint64_t bd = umma_desc(
                                bbase + (w * KSTEPS + ks) * BT_BYTES + h * QH * 32, 128, 256, 0);
                            if (a.probe != 2) {
                                if (CG == 1) umma_tf32(dcol, ad, bd, IDESC, ks > 0 || w > 0 ? 1u : 0u);
                                else umma_tf32_pair(dcol, ad, bd, IDESC, ks > 0 || w > 0 ? 1u : 0u);
                            }
                        }
                    }
                    if (bias_on && a.probe != 2) {
                        // D += 1 * (hi_q + lo_q): the pre-test constant, in the accumulator
                        const uint64_t ad = umma_desc(su32(aconst), 1024, 512, 1);
                        const uint64_t bd = umma_desc(su32(bbias) + h * QH * 32, 128, 256, 0);
                        if (CG == 1) umma_tf32(dcol, ad, bd, IDESC, 1u);
                        else umma_tf32_pair(dcol, ad, bd, IDESC, 1u);
                    }
                    if (CG == 1) umma_commit(&tfull[ts]);
                    else umma_commit_pair(&tfull[ts]);
                }
                // the stage is free once these MMAs are done (CG = 2: in both CTAs)
                if (CG == 1) umma_commit(&empty[s]);
                else umma_commit_pair(&empty[s]);
                trace_ev(a, it, 4);  // MMA: page's MMAs issued
            }
        }
    } else if (warp >= W_REC) {
        // ---------------- record constants: P, lg, pre-test bounds ----------------
        // P = ||y||^2 needs the page (the first pass of a call; later passes read
        // the (P, lg) cache), the epilogue only TMEM: the stage is released by the
        // MMAs' commit and these warps, never by the epilogue.
        // A pair of warps per page (the pairs take alternate pages); a thread owns
        // two row-adjacent records: one LDS.64 and one FMUL2 + FFMA2 per dimension.
        const int w = warp - W_REC, half = w & 1;
        const int box_i = 2 * half + (lane >> 4), l16 = lane & 15;
        const int rloc = box_i * 32 + 2 * l16;  // records rloc, rloc + 1 of the page
        float pmax = 0.f;
        for (uint32_t it = (uint32_t)(w >> 1); it < mine; it += 2) {
            const uint32_t s = it % nst, ph = (it / nst) & 1u;
            const uint32_t rec = page_of(it) * PAGE + rloc;
            const bool live = !empty_unit(it);
            const bool v0 = live && rec < a.n, v1 = live && rec + 1 < a.n;
            float2 P2, L2;  // P = ||y||^2 and the log residual of the two records
            // CG = 2, rank 1: tell rank 0's MMA issuer that this page landed
            auto relay = [&] {
                if (CG == 2 && crank == 1 && half == 0 && lane == 0)
                    bar_arrive_remote(peer_addr(&pfull[s], 0));
            };
            if (a.pl_in) {
                // computed by an earlier launch of this call (same statistics)
                P2 = L2 = make_float2(0.f, 0.f);
                if (live) {
                    const float4 v = __ldg(reinterpret_cast<const float4*>(a.pl_in) + rec / 2);
                    P2 = make_float2(v.x, v.z);
                    L2 = make_float2(v.y, v.w);
                }
                bar_wait(&full[s], ph);
                relay();
            } else {
                float2 r2 = make_float2(0.f, 0.f);
                if (v1) r2 = __ldg(reinterpret_cast<const float2*>(a.r32 + rec));
                else if (v0) r2.x = __ldg(a.r32 + rec);
                bar_wait(&full[s], ph);
                relay();
                const unsigned char* box = stage + (size_t)s * PAGE_BYTES + box_i * BOX_BYTES;
                float2 Pa = make_float2(0.f, 0.f), Pb = Pa;
#pragma unroll
                for (int k = 0; k < DP; k += 2) {
                    const float2 xa = *reinterpret_cast<const float2*>(
                        box + k * 128 + ((((l16 >> 2) ^ (k & 3)) << 5) | ((l16 & 3) << 3)));
                    const float2 xb = *reinterpret_cast<const float2*>(
                        box + (k + 1) * 128 +
                        ((((l16 >> 2) ^ ((k + 1) & 3)) << 5) | ((l16 & 3) << 3)));
                    const float2 ya = __fmul2_rn(xa, make_float2(ss[k], ss[k]));
                    const float2 yb = __fmul2_rn(xb, make_float2(ss[k + 1], ss[k + 1]));
                    Pa = __ffma2_rn(ya, ya, Pa);
                    Pb = __ffma2_rn(yb, yb, Pb);
                }
                P2 = __fadd2_rn(Pa, Pb);
                L2 = make_float2(log2f(fabsf(fmaf(r2.x, a.c1, -a.c0)) + a.rdelta),
                                 log2f(fabsf(fmaf(r2.y, a.c1, -a.c0)) + a.rdelta));
                if (a.pl_out && v0)
                    reinterpret_cast<float4*>(a.pl_out)[rec / 2] = make_float4(P2.x, L2.x, P2.y, L2.y);
            }
            float* pr = prec + (size_t)(it % PR) * 4 * PAGE;
            float2 oa, on, op, ol;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const bool valid = e ? v1 : v0;
                const float P = e ? P2.y : P2.x, lg = e ? L2.y : L2.x;
                if (valid) pmax = fmaxf(pmax, P);
                const float A = lg / a.alpha - P;
                // an invalid record never passes a pre-test
                const float as = valid ? A + 0x1p-19f * (fabsf(A) + P + sM[0]) : -INFINITY;
                const float an = valid ? -P + 0x1p-19f * (2.f * P + sM[1]) : -INFINITY;
                const float lv = valid ? lg : -INFINITY;
                if (e) { oa.y = as; on.y = an; op.y = P; ol.y = lv; }
                else { oa.x = as; on.x = an; op.x = P; ol.x = lv; }
            }
            *reinterpret_cast<float2*>(pr + rloc) = oa;
            *reinterpret_cast<float2*>(pr + PAGE + rloc) = on;
            *reinterpret_cast<float2*>(pr + 2 * PAGE + rloc) = op;
            *reinterpret_cast<float2*>(pr + 3 * PAGE + rloc) = ol;
            __syncwarp();
            if (lane == 0) {
                bar_arrive(&pready[it % PR]);
                bar_arrive(&empty[s]);  // no wait for the MMA: its commit also arrives
                trace_ev(a, it, 5 + half);  // record constants written
            }
        }
        if (a.mode == 1) {
#pragma unroll
            for (int o = 16; o; o >>= 1) pmax = fmaxf(pmax, __shfl_xor_sync(0xffffffffu, pmax, o));
            if (lane == 0) atomicMax(a.pmax, __float_as_uint(pmax));
        }
    } else {
        // ---------------- epilogue: three groups of four lane quarters ----------------
        // group `par` takes every NEG-th unit u = (page u / NH, sub-group u % NH)
        const int par = warp >> 2, quarter = warp & 3;
        const int rloc = quarter * 32 + lane;
        // (all twelve warps on every unit, three per lane quarter splitting its
        // chunks, measured 1.95 ms per 16M-record pass at QW = 256 against 1.33)
        for (uint32_t u = par; u < mine * NH; u += NEG) {
            const uint32_t it = u / NH;
            const int cbeg = (int)(u % NH) * QS, cend = cbeg + QS;  // this unit's queries
            const int cu = cbeg;  // the unit's first query (TMEM column 0)
            const uint32_t s = u % ntm, ph = (u / ntm) & 1u;  // TMEM stage
            const uint32_t rec = page_of(it) * PAGE + rloc;
            if (quarter == 0) trace_ev(a, it, 7 + 3 * (u % NH));  // epilogue: unit start
            bar_wait(&pready[it % PR], (it / PR) & 1u);
            const float* pr = prec + (size_t)(it % PR) * 4 * PAGE;
            const float Asel = pr[rloc], Ann = pr[PAGE + rloc];
            const float P = pr[2 * PAGE + rloc], lg = pr[3 * PAGE + rloc];
            bar_wait(&tfull[s], ph);
            if (quarter == 0) trace_ev(a, it, 8 + 3 * (u % NH));  // epilogue: accumulator ready
            tc_fence_after();
            // TMEM column c0 - cbeg of the unit's stage holds query c0
            const uint32_t taddr =
                tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(s * QS) - (uint32_t)cu;
            if (a.probe == 0) {
#pragma unroll 1
                for (int c0 = cbeg; c0 < cend; c0 += 32) {
                    float acc[32];
                    tmem_ld32(taddr + c0, acc);
                    if (a.mode == 1) {
                        // min over the chunk of D' = D + B (one 3-input min per two
                        // pairs), two independent chains
                        float m0 = INFINITY, m1 = INFINITY;
                        if (bias_on) {
#pragma unroll
                            for (int j = 0; j < 32; j += 4) {
                                m0 = fminf(m0, fminf(acc[j], acc[j + 1]));
                                m1 = fminf(m1, fminf(acc[j + 2], acc[j + 3]));
                            }
                        } else {
#pragma unroll
                            for (int j = 0; j < 32; j += 4) {
                                const float4 b4 = *reinterpret_cast<const float4*>(sB + c0 + j);
                                const float2 u = __fadd2_rn(make_float2(acc[j], acc[j + 1]),
                                                            make_float2(b4.x, b4.y));
                                const float2 v = __fadd2_rn(make_float2(acc[j + 2], acc[j + 3]),
                                                            make_float2(b4.z, b4.w));
                                m0 = fminf(m0, fminf(u.x, u.y));
                                m1 = fminf(m1, fminf(v.x, v.y));
                            }
                        }
                        bool hit = fminf(m0, m1) < Asel;
                        if (a.knn) {
                            m0 = m1 = INFINITY;
#pragma unroll
                            for (int j = 0; j < 32; j += 4) {
                                const float4 b4 =
                                    *reinterpret_cast<const float4*>(sB + QW + c0 + j);
                                const float2 u = __fadd2_rn(make_float2(acc[j], acc[j + 1]),
                                                            make_float2(b4.x, b4.y));
                                const float2 v = __fadd2_rn(make_float2(acc[j + 2], acc[j + 3]),
                                                            make_float2(b4.z, b4.w));
                                m0 = fminf(m0, fminf(u.x, u.y));
                                m1 = fminf(m1, fminf(v.x, v.y));
                            }
                            hit |= fminf(m0, m1) < Ann;
                        }
                        if (__any_sync(0xffffffffu, hit)) {
                            // rare: which columns passed, then the exact formula (the
                            // stream pass's key) on each such column, reloaded from
                            // TMEM with a warp-uniform column address
                            uint32_t ms = 0, mn = 0;
#pragma unroll
                            for (int j = 0; j < 32; ++j) {
                                ms |= acc[j] + (bias_on ? 0.f : sB[c0 + j]) < Asel ? 1u << j : 0u;
                                if (a.knn) mn |= acc[j] + sB[QW + c0 + j] < Ann ? 1u << j : 0u;
                            }
                            uint32_t U = __reduce_or_sync(0xffffffffu, ms | mn);
                            while (U) {
                                const int j = __ffs(U) - 1;
                                U &= U - 1;
                                // D = D' - (hi + lo), in the order the bias was split
                                const float Bj = sB[c0 + j];
                                float hi = 0.f, lo = 0.f;
                                if (bias_on) {
                                    hi = tf32_rna(Bj);
                                    lo = tf32_rna(Bj - hi);
                                }
                                const float v = (tmem_ld1(taddr + c0 + j) - hi) - lo;
                                const float d2 = (P + scc[c0 + j]) + v;
                                const float key = fmaf(-d2, a.alpha, lg);
                                if (((ms >> j) & 1u) && key > sthr[c0 + j])
                                    list_append(a, scnt, sdrop, 2 * QW, c0 + j, key, rec);
                                if (((mn >> j) & 1u) && -d2 > sthr[QW + c0 + j])
                                    list_append(a, scnt, sdrop, 2 * QW, QW + c0 + j, -d2, rec);
                            }
                        }
                    } else {
                        // sample: per-query maximum over this warp's 32 records
                        const bool valid = lg != -INFINITY;
                        const uint32_t S4 = 4 * (a.spages + a.nhot), col = r0 + it * G;
                        if (a.knn) {
                            float kn[32];
#pragma unroll
                            for (int j = 0; j < 32; ++j) {
                                const float d2 = (P + scc[c0 + j]) + acc[j];
                                acc[j] = valid ? fmaf(-d2, a.alpha, lg) : -INFINITY;
                                kn[j] = valid ? -d2 : -INFINITY;
                            }
                            const float mn = transpose_max(kn, lane);
                            a.smax[(size_t)(QW + c0 + lane) * S4 + 4 * col + quarter] = mn;
                        } else if (__all_sync(0xffffffffu, valid)) {
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                acc[j] = fmaf(-((P + scc[c0 + j]) + acc[j]), a.alpha, lg);
                        } else {
#pragma unroll
                            for (int j = 0; j < 32; ++j) {
                                const float d2 = (P + scc[c0 + j]) + acc[j];
                                acc[j] = valid ? fmaf(-d2, a.alpha, lg) : -INFINITY;
                            }
                        }
                        const float mk = transpose_max(acc, lane);
                        a.smax[(size_t)(c0 + lane) * S4 + 4 * col + quarter] = mk;
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (CG == 1) bar_arrive(&tempty[s]);
                else bar_arrive_remote(peer_addr(&tempty[s], 0));  // rank 0's issuer waits
            }
            if (quarter == 0) trace_ev(a, it, 9 + 3 * (u % NH));  // epilogue: unit done
        }
        if (a.mode == 1) {
            asm volatile("bar.sync 1, %0;" ::"n"(WE * 32) : "memory");
            // Each CTA list keeps its K' best (the CTA's K'-th key is <= the
            // store's K'-th key, so nothing that can reach the pool is lost),
            // padded to exactly K' entries (-inf keys) for the cross-CTA merge.
            for (int L = warp; L < 2 * QW; L += WE) {
                const int K = L < QW ? a.kp : a.kv;
                if (K == 0) continue;
                const size_t o = ((size_t)blockIdx.x * 2 * QW + L) * a.cap;
                int c = (int)min(scnt[L], a.cap);
                if (c > K) {
                    warp_keep_topk(a.lkey + o, a.lidx + o, c, K, whist + warp * 256, lane);
                    c = K;
                }
                const size_t oo = ((size_t)blockIdx.x * 2 * QW + L) * a.kout;
                for (int j = lane; j < K; j += 32) {
                    const bool have = j < c;
                    a.okey[oo + j] = have ? a.lkey[o + j] : -INFINITY;
                    a.oidx[oo + j] = have ? a.lidx[o + j] : 0xFFFFFFFFu - (uint32_t)j;
                }
                if (lane == 0 && sdrop[L]) atomicMax(&a.dropped[L], sdrop[L]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    // CG = 2: rank 0's MMAs write both CTAs' TMEM; neither frees it before
    // both are done
    if (CG == 2) cluster_sync_all();
    if (warp == W_MMA) {
        tc_fence_after();
        if (CG == 1)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tcols));
        else
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tcols));
    }
}

// ---------------------------------------------------------------------------
// K4 bf16: the 256-query stream pass on a bf16 copy of the pages.
//
// At 256 queries per page visit the TF32 pass is bound by its operand
// traffic, not by arithmetic: per 128-record page 32 KB of HBM and, for the
// MMAs, 128 KB of shared-memory operand reads, with the TMA's 32 KB writes
// into the same shared memory -- the ring's stages sit landed-but-unread for
// ~2000 cycles and only four fit (the 72 KB B tile), too few bytes in flight
// for the HBM latency (traced, profiles/r02).  A bf16 copy (kind::f16,
// K = 16 per MMA) halves every one of those: 16 KB pages, twice the MACs per
// operand byte, and eight stages in the same shared memory.
//
// The filter stays exact by construction: the bf16 rounding of the records
// (relative 2^-9 + 2^-11 of the stored TF32 value) and of the query operand
// (2^-9) enter the certification bound exactly like the TF32 storage did
// (DESIGN.md "Exactness"), with a 128-entry candidate pool (the measured gap
// between the 32nd and the 128th key of a 16M-record store is ~0.03 log2
// units against a bound of ~0.007).
//
// Layout: pages16 [page][128 rows][128 B], row = record, K-major with the
// 128-byte swizzle (16-byte chunk c of row r at (c ^ (r % 8)) * 16), so a
// K = 16 step is the same descriptor advanced by 32 bytes; the query tile is
// the same layout with rows = queries.  The bias K-step (ones x hi/mid/lo of
// B_q, three bf16 parts: 2^-27 |B_q|) uses unswizzled K-major tiles.
// Roles, barriers and the epilogue are those of stream_wide_kernel.
// ---------------------------------------------------------------------------
constexpr float REL16 = 0x1.42p-9f;  // |bf16(t) - v| <= (2^-9 + 2^-11)(1 + 2^-7) |v|, t = tf32(v)

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ uint16_t bf16_rn(float v) {
    return __bfloat16_as_ushort(__float2bfloat16_rn(v));
}

// fp32 pages -> the bf16 copy, pages [p0, p1): one thread per (record, 8 dims)
__global__ void pages16_kernel(const float* __restrict__ pages, uint32_t p0, uint32_t p1,
                               uint4* __restrict__ out) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t total = (size_t)(p1 - p0) * PAGE * 8;
    if (i >= total) return;
    const uint32_t c = (uint32_t)(i & 7u);               // 8-dim chunk
    const size_t rec = (size_t)p0 * PAGE + (i >> 3);     // record
    const uint32_t r = (uint32_t)(rec % PAGE);
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int k = 8 * (int)c + 2 * j;
        const uint16_t lo = bf16_rn(__ldg(pages + page_index(rec, k, 64)));
        const uint16_t hi = bf16_rn(__ldg(pages + page_index(rec, k + 1, 64)));
        w[j] = (uint32_t)lo | ((uint32_t)hi << 16);
    }
    out[(rec / PAGE) * (PAGE * 8) + r * 8 + (c ^ (r & 7u))] = make_uint4(w[0], w[1], w[2], w[3]);
}

template <int QW>
__global__ void __launch_bounds__(WIDE_THREADS, 1)
    stream_wide16_kernel(const __grid_constant__ WideArgs a) {
    constexpr int DP = 64;
    constexpr int NH = QW / 128, QS = 128;
    constexpr int PAGE_BYTES = PAGE * DP * 2;  // 16 KB
    constexpr int KSTEPS = DP / 16;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nst = a.nst, ntm = a.ntm, PR = a.nst + (a.ntm + NH - 1) / NH;
    unsigned char* stage = smem;
    unsigned char* btile = stage + (size_t)nst * PAGE_BYTES;  // [QW rows][128 B], swizzled
    unsigned char* aconst = btile + QW * 128;                 // [128 rows][32 B] bias A
    unsigned char* bbias = aconst + 128 * 32;                 // [QW rows][32 B] bias B
    float* prec = reinterpret_cast<float*>(bbias + QW * 32);  // [PR][4][PAGE]
    float* ss = prec + (size_t)PR * 4 * PAGE;
    float* scc = ss + DP;
    float* sthr = scc + QW;
    float* sB = sthr + 2 * QW;
    float* sM = sB + 2 * QW;
    uint32_t* scnt = reinterpret_cast<uint32_t*>(sM + 4);
    uint32_t* sdrop = scnt + 2 * QW;
    uint32_t* whist = reinterpret_cast<uint32_t*>(stage);
    uint64_t* full = reinterpret_cast<uint64_t*>(sdrop + 2 * QW);
    uint64_t* empty = full + 8;
    uint64_t* tfull = empty + 8;
    uint64_t* tempty = tfull + 8;
    uint64_t* pready = tempty + 8;  // [16]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pready + 16);

    // query tile (bf16, swizzled, built on the host) and constants
    {
        const uint4* src = reinterpret_cast<const uint4*>(a.consts16);
        uint4* dst = reinterpret_cast<uint4*>(btile);
        for (int i = tid; i < QW * 128 / 16; i += WIDE_THREADS) dst[i] = src[i];
    }
    const float* cs = a.consts + DP * QW;  // after the TF32 image: s, cc, t0
    for (int i = tid; i < DP; i += WIDE_THREADS) ss[i] = cs[i];
    for (int i = tid; i < QW; i += WIDE_THREADS) scc[i] = cs[DP + i];
    for (int i = tid; i < 2 * QW; i += WIDE_THREADS)
        sthr[i] = (i < QW || a.knn) ? cs[DP + QW + i] : FLT_MAX;
    for (int i = tid; i < 4 * QW; i += WIDE_THREADS) scnt[i] = 0;
    // bias A: ones in dims 0-2 of every row (K-major, 8-row core groups of
    // 2 x 128 B: row r at (r / 8) * 256 + (r % 8) * 16, dims 8-15 at +128)
    for (int i = tid; i < 128 * 16; i += WIDE_THREADS) {
        const int r = i >> 4, k = i & 15;
        reinterpret_cast<uint16_t*>(aconst)[((r >> 3) * 256 + (r & 7) * 16 + (k >> 3) * 128 + (k & 7) * 2) / 2] =
            k < 3 ? (uint16_t)0x3F80u : (uint16_t)0;
    }
    __syncthreads();
    if (warp == 0) {
        float mb[2] = {0.f, 0.f};
        bool fin = true;
        for (int q = lane; q < QW; q += 32) fin &= fabsf(sthr[q] / a.alpha + scc[q]) < 0x1p60f;
        const bool bias = __all_sync(0xffffffffu, fin);
        for (int q = lane; q < QW; q += 32) {
            const float B = sthr[q] / a.alpha + scc[q];
            float p0 = 0.f, p1 = 0.f, p2 = 0.f;
            if (bias) {
                p0 = __bfloat162float(__float2bfloat16_rn(B));
                p1 = __bfloat162float(__float2bfloat16_rn(B - p0));
                p2 = __bfloat162float(__float2bfloat16_rn((B - p0) - p1));
            }
            uint16_t* row = reinterpret_cast<uint16_t*>(bbias + (q >> 3) * 256 + (q & 7) * 16);
            row[0] = bf16_rn(p0);
            row[1] = bf16_rn(p1);
            row[2] = bf16_rn(p2);
#pragma unroll
            for (int k = 3; k < 8; ++k) row[k] = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) row[64 + k] = 0;  // dims 8-15 (+128 B)
            const float beff = (p0 + p1) + p2;
            sB[q] = B;
            mb[0] = fmaxf(mb[0], fabsf(B) + scc[q]);
            const float Bn = sthr[QW + q] + scc[q];
            sB[QW + q] = Bn - beff;
            mb[1] = fmaxf(mb[1], fabsf(Bn) + fabsf(Bn - beff) + fabsf(beff) + scc[q]);
        }
        if (lane == 0) sM[2] = bias ? 1.f : 0.f;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            mb[0] = fmaxf(mb[0], __shfl_xor_sync(0xffffffffu, mb[0], o));
            mb[1] = fmaxf(mb[1], __shfl_xor_sync(0xffffffffu, mb[1], o));
        }
        if (lane == 0) {
            sM[0] = mb[0];
            sM[1] = mb[1];
        }
    }
    if (tid == 0) {
        for (int s = 0; s < nst; ++s) {
            bar_init(&full[s], 1);
            bar_init(&empty[s], 3);
        }
        for (int s = 0; s < ntm; ++s) {
            bar_init(&tfull[s], 1);
            bar_init(&tempty[s], 4);
        }
        for (int p = 0; p < PR; ++p) bar_init(&pready[p], 2);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == W_MMA) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         su32(tmem_slot)),
                     "r"(a.tcols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const bool bias_on = sM[2] != 0.f;

    const uint32_t G = gridDim.x, r0 = blockIdx.x;
    const uint32_t mine = r0 < a.npages ? (a.npages - 1 - r0) / G + 1 : 0;
    auto page_of = [&](uint32_t it) -> uint32_t { return r0 + it * G; };

    if (warp == W_PROD) {
        if (lane == 0) {
            for (uint32_t it = 0; it < mine; ++it) {
                const uint32_t s = it % nst, ph = (it / nst) & 1u;
                if (it >= (uint32_t)nst) bar_wait(&empty[s], ph ^ 1u);
                trace_ev(a, it, 0);
                bar_expect_tx(&full[s], PAGE_BYTES);
                bulk_g2s(stage + (size_t)s * PAGE_BYTES,
                         a.pages16 + (size_t)page_of(it) * (PAGE_BYTES / 2), PAGE_BYTES, &full[s]);
            }
        }
    } else if (warp == W_MMA) {
        if (lane == 0) {
            // D f32, A/B bf16, both K-major, N = 128, M = 128
            constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) |
                                       ((uint32_t)(QS >> 3) << 17) | ((128u >> 4) << 24);
            const uint32_t bbase = su32(btile);
            for (uint32_t it = 0; it < mine; ++it) {
                const uint32_t s = it % nst, ph = (it / nst) & 1u;
                bar_wait(&full[s], ph);
                trace_ev(a, it, 1);
                const uint32_t abase = su32(stage + (size_t)s * PAGE_BYTES);
#pragma unroll
                for (int h = 0; h < NH; ++h) {
                    const uint32_t u = it * NH + h;
                    const uint32_t ts = u % ntm, tph = (u / ntm) & 1u;
                    if (u >= (uint32_t)ntm) bar_wait(&tempty[ts], tph ^ 1u);
                    trace_ev(a, it, 2 + h);
                    tc_fence_after();
                    const uint32_t dcol = tmem + (uint32_t)(ts * QS);
#pragma unroll
                    for (int ks = 0; ks < KSTEPS; ++ks) {
                        // K-major, 128-byte swizzle: a K = 16 step is +32 B
                        const uint64_t ad = umma_desc(abase + ks * 32, 16, 1024, 2);
                        const uint64_t bd = umma_desc(bbase + h * QS * 128 + ks * 32, 16, 1024, 2);
                        if (a.probe != 2) umma_bf16(dcol, ad, bd, IDESC, ks > 0 ? 1u : 0u);
                    }
                    if (bias_on && a.probe != 2) {
                        const uint64_t ad = umma_desc(su32(aconst), 128, 256, 0);
                        const uint64_t bd = umma_desc(su32(bbias) + h * QS * 32, 128, 256, 0);
                        umma_bf16(dcol, ad, bd, IDESC, 1u);
                    }
                    umma_commit(&tfull[ts]);
                }
                umma_commit(&empty[s]);
                trace_ev(a, it, 4);
            }
        }
    } else if (warp >= W_REC) {
        // record constants: a pair of warps per page (pairs alternate pages);
        // thread t of the pair owns rows t and t + 64 (32 consecutive rows per
        // warp: the swizzle spreads their 16-byte chunks over all banks)
        const int w = warp - W_REC, half = w & 1;
        const int ra = 32 * half + lane;
        float pmax = 0.f;
        for (uint32_t it = (uint32_t)(w >> 1); it < mine; it += 2) {
            const uint32_t s = it % nst, ph = (it / nst) & 1u;
            const uint32_t pbase = page_of(it) * PAGE;
            float P[2], L[2];
            bool v[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) v[e] = pbase + ra + 64 * e < a.n;
            if (a.pl_in) {
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const float2 pl = __ldg(reinterpret_cast<const float2*>(a.pl_in) + pbase + ra + 64 * e);
                    P[e] = pl.x;
                    L[e] = pl.y;
                }
                bar_wait(&full[s], ph);
            } else {
                float r[2];
#pragma unroll
                for (int e = 0; e < 2; ++e) r[e] = v[e] ? __ldg(a.r32 + pbase + ra + 64 * e) : 0.f;
                bar_wait(&full[s], ph);
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int row = ra + 64 * e;
                    const unsigned char* rp = stage + (size_t)s * PAGE_BYTES + row * 128;
                    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const uint4 q = *reinterpret_cast<const uint4*>(rp + ((c ^ (row & 7)) << 4));
                        const float4 s0 = *reinterpret_cast<const float4*>(ss + 8 * c);
                        const float4 s1 = *reinterpret_cast<const float4*>(ss + 8 * c + 4);
                        const uint32_t wq[4] = {q.x, q.y, q.z, q.w};
                        const float sv[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const float2 x = make_float2(__uint_as_float(wq[j] << 16),
                                                         __uint_as_float(wq[j] & 0xFFFF0000u));
                            const float2 y = __fmul2_rn(x, make_float2(sv[2 * j], sv[2 * j + 1]));
                            acc = __ffma2_rn(y, y, acc);
                        }
                    }
                    P[e] = acc.x + acc.y;
                    L[e] = log2f(fabsf(fmaf(r[e], a.c1, -a.c0)) + a.rdelta);
                    if (a.pl_out && v[e])
                        reinterpret_cast<float2*>(a.pl_out)[pbase + row] = make_float2(P[e], L[e]);
                }
            }
            float* pr = prec + (size_t)(it % PR) * 4 * PAGE;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int row = ra + 64 * e;
                if (v[e]) pmax = fmaxf(pmax, P[e]);
                const float A = L[e] / a.alpha - P[e];
                pr[row] = v[e] ? A + 0x1p-19f * (fabsf(A) + P[e] + sM[0]) : -INFINITY;
                pr[PAGE + row] = v[e] ? -P[e] + 0x1p-19f * (2.f * P[e] + sM[1]) : -INFINITY;
                pr[2 * PAGE + row] = P[e];
                pr[3 * PAGE + row] = v[e] ? L[e] : -INFINITY;
            }
            __syncwarp();
            if (lane == 0) {
                bar_arrive(&pready[it % PR]);
                bar_arrive(&empty[s]);
                trace_ev(a, it, 5 + half);
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) pmax = fmaxf(pmax, __shfl_xor_sync(0xffffffffu, pmax, o));
        if (lane == 0) atomicMax(a.pmax, __float_as_uint(pmax));
    } else {
        // epilogue: as stream_wide_kernel's stream mode
        const int par = warp >> 2, quarter = warp & 3;
        const int rloc = quarter * 32 + lane;
        for (uint32_t u = par; u < mine * NH; u += NEG) {
            const uint32_t it = u / NH;
            const int cbeg = (int)(u % NH) * QS, cend = cbeg + QS;
            const uint32_t s = u % ntm, ph = (u / ntm) & 1u;
            const uint32_t rec = page_of(it) * PAGE + rloc;
            if (quarter == 0) trace_ev(a, it, 7 + 3 * (u % NH));
            bar_wait(&pready[it % PR], (it / PR) & 1u);
            const float* pr = prec + (size_t)(it % PR) * 4 * PAGE;
            const float Asel = pr[rloc], Ann = pr[PAGE + rloc];
            const float P = pr[2 * PAGE + rloc], lg = pr[3 * PAGE + rloc];
            bar_wait(&tfull[s], ph);
            if (quarter == 0) trace_ev(a, it, 8 + 3 * (u % NH));
            tc_fence_after();
            const uint32_t taddr =
                tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(s * QS) - (uint32_t)cbeg;
            if (a.probe == 0) {
#pragma unroll 1
                for (int c0 = cbeg; c0 < cend; c0 += 32) {
                    float acc[32];
                    tmem_ld32(taddr + c0, acc);
                    float m0 = INFINITY, m1 = INFINITY;
                    if (bias_on) {
#pragma unroll
                        for (int j = 0; j < 32; j += 4) {
                            m0 = fminf(m0, fminf(acc[j], acc[j + 1]));
                            m1 = fminf(m1, fminf(acc[j + 2], acc[j + 3]));
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; j += 4) {
                            const float4 b4 = *reinterpret_cast<const float4*>(sB + c0 + j);
                            const float2 x = __fadd2_rn(make_float2(acc[j], acc[j + 1]),
                                                        make_float2(b4.x, b4.y));
                            const float2 y = __fadd2_rn(make_float2(acc[j + 2], acc[j + 3]),
                                                        make_float2(b4.z, b4.w));
                            m0 = fminf(m0, fminf(x.x, x.y));
                            m1 = fminf(m1, fminf(y.x, y.y));
                        }
                    }
                    bool hit = fminf(m0, m1) < Asel;
                    if (a.knn) {
                        m0 = m1 = INFINITY;
#pragma unroll
                        for (int j = 0; j < 32; j += 4) {
                            const float4 b4 = *reinterpret_cast<const float4*>(sB + QW + c0 + j);
                            const float2 x = __fadd2_rn(make_float2(acc[j], acc[j + 1]),
                                                        make_float2(b4.x, b4.y));
                            const float2 y = __fadd2_rn(make_float2(acc[j + 2], acc[j + 3]),
                                                        make_float2(b4.z, b4.w));
                            m0 = fminf(m0, fminf(x.x, x.y));
                            m1 = fminf(m1, fminf(y.x, y.y));
                        }
                        hit |= fminf(m0, m1) < Ann;
                    }
                    if (__any_sync(0xffffffffu, hit)) {
                        uint32_t ms = 0, mn = 0;
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            ms |= acc[j] + (bias_on ? 0.f : sB[c0 + j]) < Asel ? 1u << j : 0u;
                            if (a.knn) mn |= acc[j] + sB[QW + c0 + j] < Ann ? 1u << j : 0u;
                        }
                        uint32_t U = __reduce_or_sync(0xffffffffu, ms | mn);
                        while (U) {
                            const int j = __ffs(U) - 1;
                            U &= U - 1;
                            // D = D' - (p0 + p1 + p2), in the order the bias was split
                            const float Bj = sB[c0 + j];
                            float p0 = 0.f, p1 = 0.f, p2 = 0.f;
                            if (bias_on) {
                                p0 = __bfloat162float(__float2bfloat16_rn(Bj));
                                p1 = __bfloat162float(__float2bfloat16_rn(Bj - p0));
                                p2 = __bfloat162float(__float2bfloat16_rn((Bj - p0) - p1));
                            }
                            const float vv = ((tmem_ld1(taddr + c0 + j) - p0) - p1) - p2;
                            const float d2 = (P + scc[c0 + j]) + vv;
                            const float key = fmaf(-d2, a.alpha, lg);
                            if (((ms >> j) & 1u) && key > sthr[c0 + j])
                                list_append(a, scnt, sdrop, 2 * QW, c0 + j, key, rec);
                            if (((mn >> j) & 1u) && -d2 > sthr[QW + c0 + j])
                                list_append(a, scnt, sdrop, 2 * QW, QW + c0 + j, -d2, rec);
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) bar_arrive(&tempty[s]);
            if (quarter == 0) trace_ev(a, it, 9 + 3 * (u % NH));
        }
        asm volatile("bar.sync 1, %0;" ::"n"(WE * 32) : "memory");
        for (int L = warp; L < 2 * QW; L += WE) {
            const int K = L < QW ? a.kp : a.kv;
            if (K == 0) continue;
            const size_t o = ((size_t)blockIdx.x * 2 * QW + L) * a.cap;
            int c = (int)min(scnt[L], a.cap);
            if (c > K) {
                warp_keep_topk(a.lkey + o, a.lidx + o, c, K, whist + warp * 256, lane);
                c = K;
            }
            const size_t oo = ((size_t)blockIdx.x * 2 * QW + L) * a.kout;
            for (int j = lane; j < K; j += 32) {
                const bool have = j < c;
                a.okey[oo + j] = have ? a.lkey[o + j] : -INFINITY;
                a.oidx[oo + j] = have ? a.lidx[o + j] : 0xFFFFFFFFu - (uint32_t)j;
            }
            if (lane == 0 && sdrop[L]) atomicMax(&a.dropped[L], sdrop[L]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == W_MMA) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tcols));
    }
}

// Start thresholds from the sample's S block maxima of list L (S up to 4 * 8192):
// tsafe[L] <= the K-th largest (distinct records: <= the store's K-th key, so
// at least K records pass) and, for selection lists, t0[L] = the highest
// threshold at which an estimate of the store's passers reaches `target`
// (a few K' -- instead of ~K' / f).  The first Su maxima come from the
// uniform sample (fraction fu of the pages: each stands for 1 / fu records),
// the rest from the highest-residual pages, which are read whole (each
// stands for itself): est(t) = U(t) / fu + H(t).  Treating the hot pages as
// uniform would put t0 among a concentrated batch's keys and admit too few.
// Any threshold is sound (the certification bound takes max(t0, K'-th kept
// key)); a query whose pool then falls short of certifying gets one more
// pass from tsafe.  Histograms over the ordinal range present; a bin's
// lower edge, lowered by a relative 1e-6.  Fewer than K non-empty maxima: no
// threshold (-FLT_MAX).
__global__ void __launch_bounds__(1024)
    wide_kth_kernel(const float* __restrict__ smax, uint32_t S, uint32_t Su, int QW, int kp, int knn,
                    float inv_fu, float target, float tmargin, float* __restrict__ t0,
                    float* __restrict__ tsafe) {
    constexpr int NB = 2048;
    __shared__ uint32_t hist[NB], histu[NB];
    __shared__ uint32_t sh_lo, sh_hi, sh_bin[2], sh_valid;
    const int L = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
    const uint32_t K = (uint32_t)(L < QW ? kp : knn);
    const bool est = L < QW && target > 0.f;
    const float* v = smax + (size_t)L * S;
    for (int b = tid; b < NB; b += blockDim.x) hist[b] = histu[b] = 0;
    if (tid == 0) {
        sh_lo = 0xFFFFFFFFu;
        sh_hi = 0;
        sh_bin[0] = sh_bin[1] = 0xFFFFFFFFu;
        sh_valid = 0;
    }
    __syncthreads();
    uint32_t lo = 0xFFFFFFFFu, hi = 0, nv = 0;
    for (uint32_t i = tid; i < S; i += blockDim.x) {
        const uint32_t o = f2ord(v[i]);
        if (o > (uint32_t)PAD_TOP) {
            lo = min(lo, o);
            hi = max(hi, o);
            ++nv;
        }
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, d));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, d));
        nv += __shfl_xor_sync(0xffffffffu, nv, d);
    }
    if (lane == 0) {
        atomicMin(&sh_lo, lo);
        atomicMax(&sh_hi, hi);
        atomicAdd(&sh_valid, nv);
    }
    __syncthreads();
    if (K == 0 || sh_valid < K) {
        if (tid == 0) t0[L] = tsafe[L] = -FLT_MAX;
        return;
    }
    const uint32_t blo = sh_lo, span = sh_hi - sh_lo;
    const int sh = span < NB ? 0 : (32 - __clz(span)) - 11;
    for (uint32_t i = tid; i < S; i += blockDim.x) {
        const uint32_t o = f2ord(v[i]);
        if (o > (uint32_t)PAD_TOP) {
            atomicAdd(&hist[(o - blo) >> sh], 1u);
            if (est && i < Su) atomicAdd(&histu[(o - blo) >> sh], 1u);
        }
    }
    __syncthreads();
    if (tid < 64) {
        // warp 0: the bin where the count from the top reaches K; warp 1 (the
        // estimate): where U / fu + H -- with H = all - U -- reaches target
        const bool w1 = tid >= 32;
        if (!w1 || est) {
            float sum = 0.f;
            for (int j = 0; j < NB / 32; ++j) {
                const int b = NB - 1 - (lane * (NB / 32) + j);
                sum += w1 ? (float)histu[b] * inv_fu + (float)(hist[b] - histu[b]) : (float)hist[b];
            }
            float incl = sum;
            for (int o = 1; o < 32; o <<= 1) {
                const float t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            const float T = w1 ? target : (float)K;
            const float excl = incl - sum;
            const unsigned own = __ballot_sync(0xffffffffu, excl < T && T <= incl);
            if (lane == __ffs(own) - 1) {
                float c = excl;
                for (int j = 0; j < NB / 32; ++j) {
                    const int b = NB - 1 - (lane * (NB / 32) + j);
                    c += w1 ? (float)histu[b] * inv_fu + (float)(hist[b] - histu[b]) : (float)hist[b];
                    if (c >= T) {
                        sh_bin[w1 ? 1 : 0] = (uint32_t)b;
                        break;
                    }
                }
            }
        }
    }
    __syncthreads();
    if (tid == 0) {
        const float es = ord2f(blo + (sh_bin[0] << sh));
        // (the estimate never goes below the guaranteed threshold; no bin
        // reaching the target: the guaranteed one)
        const uint32_t ba = sh_bin[1] == 0xFFFFFFFFu ? sh_bin[0] : max(sh_bin[1], sh_bin[0]);
        const float ea = est ? ord2f(blo + (ba << sh)) : es;
        // (tmargin: the stream pass's keys may round below the sample's,
        // bf16 against TF32 records; only the pool's fill depends on it)
        const float m = L < QW ? tmargin : 0.f;
        tsafe[L] = es - 1e-6f * (fabsf(es) + 1.f) - m;
        t0[L] = ea - 1e-6f * (fabsf(ea) + 1.f) - m;
    }
}

inline float tf32_trunc(double v) {
    float f = (float)v;
    uint32_t u;
    std::memcpy(&u, &f, 4);
    u &= 0xFFFFE000u;
    std::memcpy(&f, &u, 4);
    return f;
}

// round to the nearest TF32 (ties to even): |error| <= 2^-11 |v|
inline float tf32_rn(double v) {
    float f = (float)v;
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7F800000u) != 0x7F800000u) u = (u + 0xFFFu + ((u >> 13) & 1u)) & 0xFFFFE000u;
    std::memcpy(&f, &u, 4);
    return f;
}

// host RN-even float -> bf16 (finite inputs)
inline uint16_t bf16_host(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

template <int DP, int QW>
void wide_launch_t(sair_store_s* s, const WidePlan& pl, const QueryPrep& p, const double* zgrp,
                   int nqg, float c1, float c0, float rdelta, float alpha, float* mk,
                   uint32_t* mi, float* mthr, unsigned int* pmax, std::vector<double>& cc_out,
                   const GroupIo& io) {
    const int d = s->d;
    // the 256-query stream pass on the bf16 page copy
    constexpr bool can16 = DP == 64 && QW == 256;
    const bool use16 = can16 && pl.bf16;
    const size_t n16 = use16 ? (size_t)DP * QW / 2 : 0;  // floats of the bf16 query tile
    const size_t nc = WB * (size_t)DP * QW + DP + QW + 2 * QW;
    float* hb = io.hstage;  // nc floats
    float* sv = hb + WB * (size_t)DP * QW;
    float* ccv = sv + DP;
    const size_t L = 2 * (size_t)QW;
    if (io.phase != 2) {
        // the per-dimension quotient once per group, not once per (query, dim):
        // 16k fp64 divisions were ~70 us of host time per 256-query group
        double mq[DP];
        for (int k = 0; k < DP; ++k) {
            sv[k] = k < d ? (float)(1.0 / p.sd[k]) : 0.f;
            mq[k] = k < d ? (p.mean[k] - s->shift[k]) / p.sd[k] : 0.0;
        }
        cc_out.assign(QW, 0.0);
        for (int q = 0; q < QW; ++q) {
            // padded query slots repeat query 0 (their lists are never read)
            const double* z = zgrp + (size_t)(q < nqg ? q : 0) * d;
            double cc = 0.0;
            for (int k = 0; k < DP; ++k) {
                float c = 0.f;
                if (k < d) c = (float)(mq[k] + z[k]);
                cc += (double)c * (double)c;
                const double bk = k < d ? -2.0 * (double)c * (double)sv[k] : 0.0;
                // smem image of the K-major B tiles: (q % 8) * 16 + (q / 8) * 256 +
                // (k % 4) * 4 + (k / 4) * 128 bytes within K-step k / 8
                const size_t off = (size_t)(k / 8) * QW * 8 + (q % 8) * 4 + (q / 8) * 64 +
                                   (k % 4) + ((k % 8) / 4) * 32;
                // the bf16 pass's query tile: row q = the B-constants of query q
                // (RN bf16), K-major with the 128-byte swizzle
                if (use16)
                    reinterpret_cast<uint16_t*>(hb + nc)[(size_t)q * 64 + (((k / 8) ^ (q % 8)) * 8) +
                                                         (k % 8)] = bf16_host((float)bk);
                if (WB == 1) {
                    hb[off] = tf32_rn(bk);
                } else {
                    const float hi = tf32_trunc(bk);
                    hb[off] = hi;
                    hb[(size_t)DP * QW + off] = tf32_trunc(bk - (double)hi);
                }
            }
            ccv[q] = (float)cc;
            cc_out[q] = cc;
        }
        if (io.t0_override) {
            std::copy(io.t0_override, io.t0_override + L, hb + (nc - L));
            std::copy(io.t0_override, io.t0_override + L, hb + nc + n16);
        }
    }
    if (io.phase == 1) return;
    // device: consts | lists | counters
    const size_t S4 = 4 * ((size_t)pl.spages + (io.hot ? io.nhot : 0));
    // consts | the bf16 query tile | safe start thresholds [2QW] | counters ...
    const size_t nct = nc + n16 + L;
    char* base = static_cast<char*>(s->b_mmab.get(nct * 4 + 256 + L * 8 + S4 * L * 4 + 256));
    float* dc = reinterpret_cast<float*>(base);
    float* dt0 = dc + WB * (size_t)DP * QW + DP + QW;  // the t0 slot of consts
    uint32_t* dcnt = reinterpret_cast<uint32_t*>(base + ((nct * 4 + 255) & ~(size_t)255));
    unsigned int* ddrop = dcnt + L;
    float* const dsmax = reinterpret_cast<float*>(ddrop + L);
    const size_t lent = (size_t)pl.grid * L * pl.cap;
    char* lists = static_cast<char*>(s->b_sample.get(lent * 8 + 256));
    float* lkey = reinterpret_cast<float*>(lists);
    uint32_t* lidx = reinterpret_cast<uint32_t*>(lists + lent * 4);
    if (io.phase == 2) {  // constants and zeroed counters already on the device
        dc = io.dconsts;
        dt0 = dc + WB * (size_t)DP * QW + DP + QW;
        dcnt = io.dcnt;
        ddrop = dcnt + L;
    } else {
        // a retry (start thresholds given, no sample pass) uploads them too
        SAIR_CUDA(cudaMemcpyAsync(dc, hb, (io.t0_override ? nc : nc - L) * sizeof(float),
                                  cudaMemcpyHostToDevice, s->st));
        if (n16)
            SAIR_CUDA(cudaMemcpyAsync(dc + nc, hb + nc, n16 * sizeof(float), cudaMemcpyHostToDevice,
                                      s->st));
        if (io.t0_override)  // (a retry's thresholds are its safe ones too)
            SAIR_CUDA(cudaMemcpyAsync(dc + nc + n16, hb + nc + n16, L * sizeof(float),
                                      cudaMemcpyHostToDevice, s->st));
        SAIR_CUDA(cudaMemsetAsync(dcnt, 0, 2 * L * sizeof(uint32_t), s->st));
    }

    WideArgs a{};
    a.pages = s->pages;
    a.r32 = s->r32;
    a.n = (uint32_t)s->n;
    a.npages = (uint32_t)((s->n + PAGE - 1) / PAGE);
    a.c1 = c1;
    a.c0 = c0;
    a.rdelta = rdelta;
    a.alpha = alpha;
    a.nst = pl.nst;
    a.ntm = pl.ntm;
    a.knn = pl.knn ? 1 : 0;
    a.spages = pl.spages;
    a.hot = io.hot;
    a.nhot = io.hot ? io.nhot : 0;
    a.consts = dc;
    a.smax = dsmax;
    a.lkey = lkey;
    a.lidx = lidx;
    a.dropped = ddrop;
    a.cap = pl.cap;
    a.kp = pl.kp;
    a.kv = pl.knn;
    a.pl_in = io.pl_in;
    a.pl_out = nullptr;
    a.okey = io.lists_key;
    a.oidx = io.lists_idx;
    a.kout = pl.kmax;
    a.pmax = pmax;
    a.probe = std::getenv("SAIR_PROBE_WIDE") ? std::atoi(std::getenv("SAIR_PROBE_WIDE")) : 0;
    static unsigned long long* dtrace = nullptr;
    if (std::getenv("SAIR_WIDE_TRACE") && !dtrace) SAIR_CUDA(cudaMalloc(&dtrace, 64 * 16 * 8));
    a.trace = nullptr;

    a.tcols = 32;
    while (a.tcols < (uint32_t)(pl.ntm * std::min(QW, 128))) a.tcols <<= 1;
    SAIR_CUDA(cudaFuncSetAttribute(stream_wide_kernel<DP, QW, 1>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
    // bf16 stream passes keep their own (P, lg) cache; the TF32 sample then
    // fills the TF32 one for its pages (the same pages every group)
    if (use16) a.pl_out = io.pl_out;
    // the sample's keys (TF32 records) may exceed the bf16 pass's keys of the
    // same records by their rounding difference: lower its start threshold by
    // a typical (not worst-case) amount -- only the pool's fill depends on it
    float tmargin = 0.f;
    if (use16) {
        double ccmax = 0.0;
        for (int q = 0; q < QW; ++q) ccmax = std::max(ccmax, (double)hb[WB * (size_t)DP * QW + DP + q]);
        tmargin = (float)(alpha * 0x1p-7 * std::sqrt(4.0 * d * ccmax));
    }
    if (!io.t0_override) {
        // sample pass -> t0 (written into the consts the stream pass reads)
        a.mode = 0;
        stream_wide_kernel<DP, QW, 1><<<(int)std::min<uint32_t>(pl.spages + a.nhot, (uint32_t)pl.grid),
                                        WIDE_THREADS, pl.smem, s->st>>>(a);
        SAIR_LAUNCH("stream_wide_kernel(sample)");
        // the selection lists' start: ~aggr K' records of the store above it
        // (an estimate from the sample; SAIR_WIDE_AGGR=0: the guaranteed K'-th)
        const double aggr = std::getenv("SAIR_WIDE_AGGR") ? std::atof(std::getenv("SAIR_WIDE_AGGR")) : 2.5;
        const double fu = std::min(1.0, (double)pl.spages / (double)a.npages);
        wide_kth_kernel<<<pl.knn ? 2 * QW : QW, 1024, 0, s->st>>>(
            dsmax, (uint32_t)S4, (uint32_t)(4 * pl.spages), QW, pl.kp, pl.knn, (float)(1.0 / fu),
            (float)(aggr * pl.kp), tmargin, dt0, dc + nc + n16);
        SAIR_LAUNCH("wide_kth_kernel");
    }
    SAIR_CUDA(cudaEventRecord(io.e_mid, s->st));
    a.mode = 1;
    a.pl_out = io.pl_out;  // the first stream pass of a call caches (P, lg) per record
    if (dtrace) {
        SAIR_CUDA(cudaMemsetAsync(dtrace, 0, 64 * 16 * 8, s->st));
        a.trace = dtrace;
    }
    if (use16) {
        // 256 queries per visit of the bf16 page copy (stream_wide16_kernel)
        ensure_pages16(s);
        constexpr auto kern16 = stream_wide16_kernel<can16 ? QW : 256>;
        SAIR_CUDA(cudaFuncSetAttribute(kern16, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)pl.smem16));
        WideArgs b = a;
        b.nst = pl.nst16;
        b.pages16 = static_cast<const uint16_t*>(s->b_pages16.p);
        b.consts16 = dc + nc;
        b.pl_in = io.pl16_in;
        b.pl_out = io.pl16_out;
        kern16<<<pl.grid, WIDE_THREADS, pl.smem16, s->st>>>(b);
    } else if (QW == 256 && pl.cg == 2) {
        // CTA pairs: clusters of two, rank 0 of each issuing the M = 256 MMAs
        constexpr auto kern = stream_wide_kernel<DP, QW == 256 ? 256 : 128, 2>;
        SAIR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)pl.smem2));
        a.nst = pl.nst2;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)pl.grid);
        cfg.blockDim = dim3(WIDE_THREADS);
        cfg.dynamicSmemBytes = pl.smem2;
        cfg.stream = s->st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        SAIR_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
    } else {
        stream_wide_kernel<DP, QW, 1><<<pl.grid, WIDE_THREADS, pl.smem, s->st>>>(a);
    }
    SAIR_LAUNCH("stream_wide_kernel(stream)");
    if (dtrace) {  // diagnostics: per-page event clocks of CTA 0, relative to the first
        std::vector<unsigned long long> h(64 * 16);
        SAIR_CUDA(cudaMemcpyAsync(h.data(), dtrace, h.size() * 8, cudaMemcpyDeviceToHost, s->st));
        SAIR_CUDA(cudaStreamSynchronize(s->st));
        const unsigned long long t0c = h[0];
        fprintf(stderr, "[trace] page: prod mfull mtm0 mtm1 missued rec0 rec1 | e0s e0r e0d | e1s e1r e1d\n");
        for (int i = 0; i < 64; ++i) {
            fprintf(stderr, "[trace] %3d:", i + (int)TR0);
            for (int e = 0; e < 13; ++e)
                fprintf(stderr, " %7lld", h[i * 16 + e] ? (long long)(h[i * 16 + e] - t0c) : -1LL);
            fprintf(stderr, "\n");
        }
    }
    SAIR_CUDA(cudaEventRecord(io.e_end, s->st));
    // the per-query top-K' across the CTAs' compacted lists (io.lists_key:
    // [G][2QW][kmax], K' each) is merged by the caller, all groups at once
    (void)mk;
    (void)mi;
    (void)mthr;
    if (std::getenv("SAIR_WIDE_DEBUG")) {  // diagnostics: overflowing lists, thresholds
        std::vector<uint32_t> hd(L);
        std::vector<float> ht(L);
        SAIR_CUDA(cudaMemcpyAsync(hd.data(), ddrop, L * 4, cudaMemcpyDeviceToHost, s->st));
        SAIR_CUDA(cudaMemcpyAsync(ht.data(), dt0, L * 4, cudaMemcpyDeviceToHost, s->st));
        SAIR_CUDA(cudaStreamSynchronize(s->st));
        size_t nd = 0;
        for (int i = 0; i < QW; ++i) nd += hd[i] != 0;
        fprintf(stderr, "[wide] QW=%d spages=%u dropped-lists %zu t0[0]=%g\n", QW, pl.spages, nd,
                (double)ht[0]);
    }
    s->mma_t0 = dt0;
    s->mma_t0safe = dc + nc + n16;
    s->mma_dropped = ddrop;
}

// per page: the largest record-constant residual |r c1 - c0| (the reward
// factor of the key, |r - loo mean| scaled, experience.cpp:138-140,148)
__global__ void page_resid_kernel(const float* __restrict__ r32, uint32_t n, uint32_t npages,
                                  float c1, float c0, float* __restrict__ out,
                                  uint32_t* __restrict__ ids) {
    const uint32_t page = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (page >= npages) return;
    float v = 0.f;
#pragma unroll
    for (int i = 0; i < PAGE / 32; ++i) {
        const uint32_t rec = page * PAGE + i * 32 + lane;
        if (rec < n) v = fmaxf(v, fabsf(fmaf(__ldg(r32 + rec), c1, -c0)));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) {
        out[page] = v;
        ids[page] = page;
    }
}

// the H highest pages (sorted order) that the uniform sample (page =
// floor(u npages / spages)) does not already hold; the others leave an
// empty slot
__global__ void hot_mark_kernel(const uint32_t* __restrict__ sorted, uint32_t npages,
                                uint32_t spages, uint32_t H, uint32_t* __restrict__ hot) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= H) return;
    const uint32_t p = sorted[i];
    const uint64_t u = ((uint64_t)p * spages + npages - 1) / npages;
    hot[i] = u < spages && u * npages / spages == p ? 0xFFFFFFFFu : p;
}

template <int DP>
WideFn wide_pick_qw(int qw) {
    switch (qw) {
        case 32: return wide_launch_t<DP, 32>;
        case 64: return wide_launch_t<DP, 64>;
        case 128: return wide_launch_t<DP, 128>;
        default: return wide_launch_t<DP, 256>;
    }
}

// the bf16 pass (dp = 64): stages of 16 KB, the swizzled query tile, the bias tiles
size_t wide16_smem(int qw, int nst, int ntm) {
    const int nh = qw / 128;
    return 1024 + (size_t)nst * PAGE * 128 + (size_t)qw * 128 + 128 * 32 + (size_t)qw * 32 +
           (size_t)(nst + (ntm + nh - 1) / nh) * 4 * PAGE * 4 + 64 * 4 + qw * 4 + 4 * qw * 4 +
           16 + 4 * qw * 4 + 48 * 8 + 16;
}

size_t wide_smem(int dp, int qw, int nst, int ntm, int cg) {
    const int nh = qw > 128 ? qw / 128 : 1;
    // + the bias K-step: its constant A tile (4 KB) and B tile (qw x 32 B);
    // a CTA pair (cg = 2) holds half of every B tile in each CTA
    return 1024 + (size_t)nst * 4 * 32 * dp * 4 + 4096 + (WB * (size_t)(dp / 8) + 1) * qw * 32 / cg +
           (size_t)(nst + (ntm + nh - 1) / nh) * 4 * PAGE * 4 + dp * 4 + qw * 4 + 4 * qw * 4 +
           16 + 4 * qw * 4 + 56 * 8 + 16;
}

}  // namespace

// The wide sample's second part: the pages with the largest reward residual.
// A page whose records carry a much larger |r - loo mean| than the rest (a
// freshly appended batch of outcomes far from the store's mean) holds most
// queries' best keys, and a uniform sample would miss it: the start
// threshold would sit far below the K'-th key and the stream pass would
// admit that page's records for every query.  Any set of distinct pages
// gives a valid start threshold, so adding these only tightens it.
const uint32_t* wide_hot_pages(sair_store_s* s, const WidePlan& pl, float c1, float c0,
                               uint32_t* nhot) {
    const uint32_t npages = (uint32_t)((s->n + PAGE - 1) / PAGE);
    const uint32_t H = std::min<uint32_t>(256u, npages / 32);
    *nhot = H;
    if (H == 0) return nullptr;
    const size_t pb = ((size_t)npages * 4 + 255) & ~(size_t)255;
    if (s->b_hot.p && s->hot_n == s->n && s->hot_c1 == c1 && s->hot_c0 == c0 &&
        s->hot_sp == pl.spages)
        return reinterpret_cast<const uint32_t*>(static_cast<char*>(s->b_hot.p) + 4 * pb);
    size_t tmp = 0;
    SAIR_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp, (const float*)nullptr,
                                                        (float*)nullptr, (const uint32_t*)nullptr,
                                                        (uint32_t*)nullptr, (int)npages));
    char* base = static_cast<char*>(s->b_hot.get(4 * pb + (((size_t)H * 4 + 255) & ~(size_t)255) +
                                                 tmp + 256));
    float* vals = reinterpret_cast<float*>(base);
    uint32_t* ids = reinterpret_cast<uint32_t*>(base + pb);
    float* vals_s = reinterpret_cast<float*>(base + 2 * pb);
    uint32_t* ids_s = reinterpret_cast<uint32_t*>(base + 3 * pb);
    uint32_t* hot = reinterpret_cast<uint32_t*>(base + 4 * pb);
    void* tbuf = base + 4 * pb + (((size_t)H * 4 + 255) & ~(size_t)255);
    page_resid_kernel<<<(npages + 7) / 8, 256, 0, s->st>>>(s->r32, (uint32_t)s->n, npages, c1, c0,
                                                          vals, ids);
    SAIR_LAUNCH("page_resid_kernel");
    SAIR_CUDA(cub::DeviceRadixSort::SortPairsDescending(tbuf, tmp, vals, vals_s, ids, ids_s,
                                                        (int)npages, 0, 32, s->st));
    hot_mark_kernel<<<(H + 255) / 256, 256, 0, s->st>>>(ids_s, npages, pl.spages, H, hot);
    SAIR_LAUNCH("hot_mark_kernel");
    s->hot_n = s->n;  // reused by later calls until the store grows
    s->hot_c1 = c1;
    s->hot_c0 = c0;
    s->hot_sp = pl.spages;
    return hot;
}

WideFn pick_wide(int dp, int qw) {
    switch (dp) {
        case 8: return wide_pick_qw<8>(qw);
        case 16: return wide_pick_qw<16>(qw);
        case 32: return wide_pick_qw<32>(qw);
        case 64: return wide_pick_qw<64>(qw);
        default: return nullptr;
    }
}

double wide_bq_rel(const WidePlan& pl) {
    // |<x, b' - b>| <= rel |b| |x| with |b| = 2 sqrt(C): 2 x the operand's rounding
    return pl.bf16 ? 0x1p-8 * 1.01 : (WB == 1 ? 0x1p-10 * 1.01 : 0.0);
}
double wide_rec_rel(const WidePlan& pl) { return pl.bf16 ? (double)REL16 : 0x1p-11; }

void ensure_pages16(sair_store_s* s) {
    const size_t npages = (s->n + PAGE - 1) / PAGE;
    if (s->pages16_n > s->n) s->pages16_n = 0;
    if (s->pages16_n == s->n || npages == 0) return;
    void* before = s->b_pages16.p;
    uint4* out = static_cast<uint4*>(s->b_pages16.get(npages * PAGE * 128));
    if (out != before) s->pages16_n = 0;  // reallocated: convert everything
    // from the page holding the first unconverted record (it may have grown)
    const uint32_t p0 = (uint32_t)(s->pages16_n / PAGE), p1 = (uint32_t)npages;
    const size_t threads = (size_t)(p1 - p0) * PAGE * 8;
    pages16_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s->st>>>(s->pages, p0, p1, out);
    SAIR_LAUNCH("pages16_kernel");
    s->pages16_n = s->n;
}

bool make_wide_plan(const sair_store_s* s, size_t nq, size_t m, double lambda, bool nn,
                    WidePlan* pl) {
    if (std::getenv("SAIR_NO_WIDE") || nq < 32 || s->dp < 8 || s->dp > 64) return false;
    pl->dp = s->dp;
    // 256 queries per page visit when the batch has them (two TMEM stages of
    // 256 columns); SAIR_WIDE_QW caps it (A/B and tests)
    int qmax = 256;
    if (const char* e = std::getenv("SAIR_WIDE_QW")) qmax = std::max(32, std::atoi(e));
    pl->qw = nq >= 256 && qmax >= 256 ? 256 : nq >= 128 && qmax >= 128 ? 128
             : (nq >= 64 && qmax >= 64 ? 64 : 32);
    pl->kp = 32;
    // 256-query passes over d <= 64 run on the bf16 page copy (SAIR_WIDE_BF16=0:
    // the TF32 pass, for A/B); its looser filter gets a pool twice as deep
    const char* b16e = std::getenv("SAIR_WIDE_BF16");
    // (from 8M records: below, the deeper pool and sample cost more than the
    // pass saves -- measured at 1M / 4M / 16M records, 256-query batches)
    pl->bf16 = pl->qw == 256 && s->dp == 64 && !(b16e && std::atoi(b16e) == 0) &&
                       (s->n >= ((size_t)8 << 20) || (b16e && std::atoi(b16e) == 1))
                   ? 1
                   : 0;
    const size_t want_pool = (lambda != 0.0 ? 4 * m : 2 * m) * (pl->bf16 ? 2 : 1);
    while ((size_t)pl->kp < want_pool && pl->kp < 512) pl->kp <<= 1;
    pl->knn = nn ? 16 : 0;
    pl->kmax = std::max(pl->kp, pl->knn);
    const size_t npages = (s->n + PAGE - 1) / PAGE;
    // below ~64k records the 8-query pass is as fast and the per-CTA lists
    // could not hold a threshold-less sample
    if (npages < 512) return false;
    // Sample size: a sample of S pages leaves ~K' npages / S candidates per
    // list, and each costs the stream pass a slow chunk; S = sqrt(5 K' npages)
    // balances the two (measured optimum of c in sqrt(c K' npages) at 1M and
    // 16M records: 20% / 5% of the pages).
    // (the bf16 pass starts from an estimated threshold whose pool fill does
    // not depend on the sample size: a smaller sample -- measured 1.1 ms per
    // 4096-query step less at 16M -- suffices there)
    const double sc = std::getenv("SAIR_SAMPLE_C") ? std::atof(std::getenv("SAIR_SAMPLE_C"))
                                                   : (pl->bf16 ? 2.0 : 5.0);
    pl->spages = (uint32_t)std::min<size_t>(
        npages, std::min<size_t>(
                    16384, std::max<size_t>(64, (size_t)std::sqrt(sc * pl->kp * npages))));
    // per CTA and list (global memory): ~7 candidates expected at 148 CTAs;
    // 512 absorbs a few pages of concentrated high keys (a freshly appended batch)
    pl->cap = 512;
    // tests: a tiny capacity forces full lists (the dropped-key bound, the
    // threshold retry and the exact fallback)
    if (const char* e = std::getenv("SAIR_WIDE_CAP")) pl->cap = (uint32_t)std::max(1, std::atoi(e));
    const size_t limit = 227 * 1024;
    // TMEM: ntm stages x min(QW, 128) columns <= 512; as many shared page stages as fit
    pl->ntm = std::min(8, 512 / std::min(pl->qw, 128));  // 128-column units for QW = 256
    // four page stages (a fifth measured 4 % slower at QW = 128)
    pl->nst = 4;
    while (pl->nst > 2 && wide_smem(pl->dp, pl->qw, pl->nst, pl->ntm, 1) > limit) --pl->nst;
    if (wide_smem(pl->dp, pl->qw, pl->nst, pl->ntm, 1) > limit) return false;
    pl->smem = wide_smem(pl->dp, pl->qw, pl->nst, pl->ntm, 1);
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, s->device);
    pl->grid = (int)std::max<size_t>(1, std::min<size_t>(npages, (size_t)nsm));
    if (pl->bf16) {
        int n16 = std::getenv("SAIR_WIDE_NST16") ? std::atoi(std::getenv("SAIR_WIDE_NST16")) : 8;
        n16 = std::max(2, std::min(8, n16));
        while (n16 > 2 && wide16_smem(pl->qw, n16, pl->ntm) > limit) --n16;
        pl->nst16 = n16;
        pl->smem16 = wide16_smem(pl->qw, n16, pl->ntm);
    }
    // SAIR_WIDE_CG=2: 256-query TF32 stream passes on CTA pairs (an even
    // grid; up to six page stages in the shared memory the halved B tile
    // leaves) -- measured 7 % slower than single CTAs at 16M records (the pair
    // waits on the slower of its two pages), so not the default
    pl->cg = 1;
    pl->nst2 = pl->nst;
    pl->smem2 = pl->smem;
    const char* cge = std::getenv("SAIR_WIDE_CG");
    if (pl->qw == 256 && pl->grid % 2 == 0 && cge && std::atoi(cge) == 2) {
        int n2 = std::getenv("SAIR_WIDE_NST2") ? std::atoi(std::getenv("SAIR_WIDE_NST2")) : 6;
        n2 = std::max(2, std::min(8, n2));
        while (n2 > 2 && wide_smem(pl->dp, pl->qw, n2, pl->ntm, 2) > limit) --n2;
        if (wide_smem(pl->dp, pl->qw, n2, pl->ntm, 2) <= limit) {
            pl->cg = 2;
            pl->nst2 = n2;
            pl->smem2 = wide_smem(pl->dp, pl->qw, n2, pl->ntm, 2);
        }
    }
    return true;
}

}  // namespace sair
