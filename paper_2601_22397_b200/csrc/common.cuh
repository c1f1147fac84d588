// common.cuh -- shared device/host helpers for libsair (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <stdexcept>
#include <string>

#include "sair.h"

namespace sair {

// Records per store page.  A page holds dp x PAGE fp32 values, dimension-major
// ([k][record]), so one page is one contiguous bulk-copy unit and a warp's
// reads of one dimension are 128 contiguous bytes.
constexpr int PAGE = 128;

// ----------------------------------------------------------------- errors --

struct Error : std::runtime_error {
    sair_status code;
    Error(sair_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw Error(SAIR_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define SAIR_CUDA(x) ::sair::cuda_check((x), #x)
#define SAIR_LAUNCH(what) ::sair::cuda_check(cudaGetLastError(), what)

// ------------------------------------------------- exact fp64 device math --
// The reference is compiled for x86-64 without FMA contraction, so every
// product and sum rounds separately.  nvcc contracts a*b+c into DFMA by
// default; these wrappers pin the reference's rounding sequence.
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// similarity(), experience.cpp:30-40 on standardized vectors:
// d2 = sum_k (a_k - b_k)^2 in k order, exp(-d2 / (2 sigma sigma)).
__device__ __forceinline__ double sim_from_d2(double d2, double two_s2) {
    return exp(ddiv(-d2, two_s2));
}

// total order used for float keys: larger key first, then smaller index
__device__ __forceinline__ uint32_t f2ord(float f) {
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

// Float index of (record, dimension) in the page array.  A page is 4 blocks of
// 32 records; a block is dp rows (one per dimension) of 128 bytes, stored
// pre-swizzled: the 32-byte chunk j of row k holds records 8*(j ^ (k % 4)) ..
// +7.  This is exactly the tcgen05 SWIZZLE_128B_BASE32B image of an MN-major
// TF32 operand block, so one contiguous bulk copy of a page lands a ready UMMA
// operand in shared memory (select_mma.cu), and a warp reading one dimension
// of 32 records still touches 32 distinct banks.
#ifdef __CUDACC__
// the fp32 page copy holds TF32-rounded values (round to nearest): the
// tensor-core filter then reads the stored values exactly (select_mma.cu)
__device__ __forceinline__ float to_tf32(double v) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"((float)v));
    return __uint_as_float(r);
}
#endif

__host__ __device__ __forceinline__ size_t page_index(size_t rec, int k, int dp) {
    const size_t page = rec / PAGE;
    const uint32_t slot = (uint32_t)(rec % PAGE), b = slot >> 5, t = slot & 31u;
    return page * (size_t)dp * PAGE + (size_t)b * dp * 32 + (size_t)k * 32 +
           ((((t >> 3) ^ ((uint32_t)k & 3u)) << 3) | (t & 7u));
}

inline int ceil_div(size_t a, size_t b) { return (int)((a + b - 1) / b); }

// smallest supported padded dimension bucket for the streaming kernel
inline int dp_bucket(int d) {
    if (d <= 8) return 8;
    if (d <= 16) return 16;
    if (d <= 32) return 32;
    if (d <= 64) return 64;
    if (d <= 128) return 128;
    return 256;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) SAIR_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

}  // namespace sair
