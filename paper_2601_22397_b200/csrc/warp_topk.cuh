// warp_topk.cuh -- warp-level radix select over a shared-memory candidate list
// (used by both streaming kernels; one copy per translation unit).
#pragma once

#include "common.cuh"

namespace sair {

// ------------------------------------------------- warp radix-select (smem) --

// One 8-bit digit step of a descending radix select over `cnt` entries: finds
// the bin (from the top) holding rank r.  Returns the bin; r is reduced by the
// count above it; *binc gets the bin's population.
template <class Get>
static __device__ __forceinline__ int warp_digit(Get get, int cnt, uint32_t prefix, uint32_t pmask,
                                          int shift, int& r, uint32_t* hist, int lane,
                                          uint32_t* binc) {
    for (int b = lane; b < 256; b += 32) hist[b] = 0;
    __syncwarp();
    for (int i = lane; i < cnt; i += 32) {
        uint32_t u;
        if (get(i, u) && (u & pmask) == prefix) atomicAdd(&hist[(u >> shift) & 255u], 1u);
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
    const uint32_t excl = incl - sum;
    const unsigned own = __ballot_sync(0xffffffffu, excl < (uint32_t)r && (uint32_t)r <= incl);
    const int owner = __ffs(own) - 1;
    int bin = 0;
    uint32_t above = 0, pop = 0;
    if (lane == owner) {
        uint32_t c = excl;
        for (int j = 0; j < 8; ++j) {
            if (c + loc[j] >= (uint32_t)r) {
                bin = 255 - (lane * 8 + j);
                above = c;
                pop = loc[j];
                break;
            }
            c += loc[j];
        }
    }
    bin = __shfl_sync(0xffffffffu, bin, owner);
    above = __shfl_sync(0xffffffffu, above, owner);
    *binc = __shfl_sync(0xffffffffu, pop, owner);
    r -= (int)above;
    __syncwarp();
    return bin;
}

// Keep the K largest entries of a candidate list by (key desc, idx asc),
// compacted in place to [0, K).  Returns the ordinal of the K-th key.
static __device__ __noinline__ uint32_t warp_keep_topk(float* key, uint32_t* idx, int cnt, int K, uint32_t* hist,
                                   int lane) {
    uint32_t prefix = 0, pmask = 0, binc = 0;
    int r = K;
    auto by_key = [&](int i, uint32_t& u) {
        u = f2ord(key[i]);
        return true;
    };
    for (int shift = 24; shift >= 0; shift -= 8) {
        int bin = warp_digit(by_key, cnt, prefix, pmask, shift, r, hist, lane, &binc);
        prefix |= (uint32_t)bin << shift;
        pmask |= 255u << shift;
    }
    const uint32_t T = prefix;
    uint32_t TI = 0;  // ties at T are kept when ~idx >= TI
    if ((int)binc > r) {
        uint32_t pre = 0, pm = 0;
        auto by_idx = [&](int i, uint32_t& u) {
            u = ~idx[i];
            return f2ord(key[i]) == T;
        };
        for (int shift = 24; shift >= 0; shift -= 8) {
            int bin = warp_digit(by_idx, cnt, pre, pm, shift, r, hist, lane, &binc);
            pre |= (uint32_t)bin << shift;
            pm |= 255u << shift;
        }
        TI = pre;
    }
    int w = 0;  // in-place compaction: writes never pass the read position
    for (int base = 0; base < cnt; base += 32) {
        const int i = base + lane;
        float kk = 0.f;
        uint32_t ii = 0;
        bool keep = false;
        if (i < cnt) {
            kk = key[i];
            ii = idx[i];
            const uint32_t u = f2ord(kk);
            keep = u > T || (u == T && ~ii >= TI);
        }
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        __syncwarp();
        if (keep) {
            const int pos = w + __popc(bal & ((1u << lane) - 1u));
            key[pos] = kk;
            idx[pos] = ii;
        }
        w += __popc(bal);
        __syncwarp();
    }
    return T;
}


}  // namespace sair
