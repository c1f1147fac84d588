// topk_select.cuh -- block-wide top-K of one candidate list held in
// registers (<= 1024 * ITEMS entries), shared by the CTA-list merge
// (select.cu) and the per-query global lists of the wide pass (select_wide.cu).
#pragma once

#include "common.cuh"

namespace sair {

constexpr unsigned long long PAD_TOP = 0x007FFFFFull;  // f2ord(-inf): padding entries

// Global top-K of list L for lists of at most 1024 * ITEMS entries, one block
// per list, entries held in registers.  The refine kernel is order-agnostic
// (every tie-break ends on the record index), so the K winners are written
// unsorted.  Selection: one histogram over the ordinal range actually present
// (lo..hi of this list's keys, 2048 bins), the boundary bin resolved by rank
// counting on the composites; a radix select on the registers only when the
// boundary bin is very crowded (many equal keys).
// `load(e, key, idx)` fetches entry e < total (false = no entry); the K
// winners go to out_key/out_idx[0..K) and the K-th key (-inf when every valid
// entry is kept) to *out_thr.  Must be called by all 1024 threads of a block.
template <int ITEMS, class Load>
__device__ __forceinline__ void block_topk(Load load, int total, int K, float* __restrict__ out_key,
                                           uint32_t* __restrict__ out_idx,
                                           float* __restrict__ out_thr) {
    constexpr int NB = 2048, BCAP = 1024;
    __shared__ uint32_t hist[NB];
    __shared__ unsigned long long skey[512];
    __shared__ unsigned long long sb[BCAP];
    __shared__ uint32_t sh_valid, sh_lo, sh_hi, sh_bin, sh_above, sh_cnt, sh_nb;
    __shared__ unsigned long long sh_kth;
    const int tid = threadIdx.x, lane = tid & 31;
    unsigned long long v[ITEMS];
    uint32_t nvalid = 0, lo = 0xFFFFFFFFu, hi = 0;
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
        const int e = tid + it * 1024;
        v[it] = 0ull;  // empty
        float key;
        uint32_t idx;
        if (e < total && load(e, key, idx)) {
            const uint32_t o = f2ord(key);
            if (o > (uint32_t)PAD_TOP) {
                v[it] = ((unsigned long long)o << 32) | (unsigned long long)(~idx);
                ++nvalid;
                lo = min(lo, o);
                hi = max(hi, o);
            }
        }
    }
    if (tid == 0) {
        sh_valid = 0;
        sh_lo = 0xFFFFFFFFu;
        sh_hi = 0;
        sh_cnt = 0;
        sh_nb = 0;
        sh_kth = ~0ull;
    }
    for (int b = tid; b < NB; b += blockDim.x) hist[b] = 0;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        nvalid += __shfl_xor_sync(0xffffffffu, nvalid, o);
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    __syncthreads();
    if (lane == 0 && nvalid) {
        atomicAdd(&sh_valid, nvalid);
        atomicMin(&sh_lo, lo);
        atomicMax(&sh_hi, hi);
    }
    __syncthreads();
    const uint32_t V = sh_valid;
    bool take_all = V <= (uint32_t)K;
    bool radix = false;
    if (!take_all) {
        // bin = (ord - lo) >> sh < NB
        const uint32_t span = sh_hi - sh_lo;
        const int sh = span < NB ? 0 : (32 - __clz(span)) - 11;
        const uint32_t blo = sh_lo;
#pragma unroll
        for (int it = 0; it < ITEMS; ++it)
            if (v[it]) atomicAdd(&hist[((uint32_t)(v[it] >> 32) - blo) >> sh], 1u);
        __syncthreads();
        if (tid < 32) {
            // lane l owns bins [NB - 64 (l + 1), NB - 64 l): counts from the top
            uint32_t sum = 0;
            for (int j = 0; j < NB / 32; ++j) sum += hist[NB - 1 - (lane * (NB / 32) + j)];
            uint32_t incl = sum;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            const uint32_t excl = incl - sum;
            const unsigned own = __ballot_sync(0xffffffffu, excl < (uint32_t)K && (uint32_t)K <= incl);
            if (lane == __ffs(own) - 1) {
                uint32_t c = excl;
                for (int j = 0; j < NB / 32; ++j) {
                    const int b = NB - 1 - (lane * (NB / 32) + j);
                    if (c + hist[b] >= (uint32_t)K) {
                        sh_bin = (uint32_t)b;
                        sh_above = c;
                        break;
                    }
                    c += hist[b];
                }
            }
        }
        __syncthreads();
        const uint32_t bstar = sh_bin, above = sh_above;
        radix = hist[bstar] > (uint32_t)BCAP;
        if (!radix) {
            // bins above the boundary are in; the boundary bin goes to sb
#pragma unroll
            for (int it = 0; it < ITEMS; ++it) {
                if (!v[it]) continue;
                const uint32_t b = ((uint32_t)(v[it] >> 32) - blo) >> sh;
                if (b > bstar) skey[atomicAdd(&sh_cnt, 1u)] = v[it];
                else if (b == bstar) sb[atomicAdd(&sh_nb, 1u)] = v[it];
            }
            __syncthreads();
            // the boundary entries of rank < K - above (composites are unique)
            const uint32_t need = (uint32_t)K - above, nb = sh_nb;
            for (uint32_t t = tid; t < nb; t += blockDim.x) {
                const unsigned long long u = sb[t];
                uint32_t rank = 0;
                for (uint32_t j = 0; j < nb; ++j) rank += sb[j] > u;
                if (rank < need) skey[above + rank] = u;
                if (rank == need - 1) sh_kth = u;
            }
            __syncthreads();
        }
    }
    if (radix) {
        // crowded boundary: 8-bit radix select over the composites
        unsigned long long prefix = 0, pmask = 0;
        uint32_t r = (uint32_t)K;
        for (int shift = 56; shift >= 0; shift -= 8) {
            for (int b = tid; b < 256; b += blockDim.x) hist[b] = 0;
            __syncthreads();
#pragma unroll
            for (int it = 0; it < ITEMS; ++it) {
                const unsigned long long u = v[it];
                if (u && (u & pmask) == prefix) atomicAdd(&hist[(uint32_t)(u >> shift) & 255u], 1u);
            }
            __syncthreads();
            if (tid == 0) {
                uint32_t c = 0;
                for (int b = 255; b >= 0; --b) {
                    if (c + hist[b] >= r) {
                        sh_bin = (uint32_t)b;
                        sh_above = r - c;
                        break;
                    }
                    c += hist[b];
                }
            }
            __syncthreads();
            prefix |= (unsigned long long)sh_bin << shift;
            pmask |= 255ull << shift;
            r = sh_above;
            __syncthreads();
        }
        // prefix is now the K-th composite itself
        if (tid == 0) {
            sh_cnt = 0;
            sh_kth = prefix;
        }
        __syncthreads();
#pragma unroll
        for (int it = 0; it < ITEMS; ++it)
            if (v[it] && v[it] >= prefix) skey[atomicAdd(&sh_cnt, 1u)] = v[it];
        __syncthreads();
    }
    if (take_all) {
#pragma unroll
        for (int it = 0; it < ITEMS; ++it)
            if (v[it]) skey[atomicAdd(&sh_cnt, 1u)] = v[it];
        __syncthreads();
    }
    const int have = take_all ? (int)V : K;
    for (int j = tid; j < K; j += blockDim.x) {
        const size_t o = (size_t)j;
        if (j < have) {
            out_key[o] = ord2f((uint32_t)(skey[j] >> 32));
            out_idx[o] = ~(uint32_t)(skey[j] & 0xffffffffu);
        } else {  // unique padding, idx >= n (skipped by refine)
            out_key[o] = -INFINITY;
            out_idx[o] = 0xFFFFFFFFu - (uint32_t)j;
        }
    }
    if (tid == 0) *out_thr = take_all ? -INFINITY : ord2f((uint32_t)(sh_kth >> 32));
}


}  // namespace sair
