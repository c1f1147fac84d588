// mma_rate.cu -- tcgen05.mma issue/exec rate from shared memory on this GPU:
// bf16 (K = 16) and tf32 (K = 8) at N = 128 / 256, M = 128, cta_group::1, one
// CTA per SM, ITERS back-to-back MMAs into one TMEM accumulator, then one
// commit; cycles per MMA (SM clock).  The wide pass's per-page MMA budget.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate mma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)(layout & 7u) << 61;
    return d;
}

template <int KIND, int N>  // KIND 0 = bf16, 1 = tf32
__global__ void mma_kernel(int iters, unsigned long long* cyc) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* s = sm + ((1024u - (su32(sm) & 1023u)) & 1023u);
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s)[i] = 0x3F803F80u;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const uint32_t IDESC = KIND == 0
            ? (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24)
            : (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
        const uint32_t a = su32(s), b = su32(s + 16384);
        const unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                const uint64_t ad = desc(a + ks * 32, 16, 1024, 2);
                const uint64_t bd = desc(b + ks * 32, 16, 1024, 2);
                const uint32_t acc = (it | ks) ? 1u : 0u;
                if (KIND == 0)
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                                 "l"(ad), "l"(bd), "r"(IDESC), "r"(acc));
                else
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                                 "l"(ad), "l"(bd), "r"(IDESC), "r"(acc));
            }
        }
        const unsigned long long t1 = clock64();
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
        asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(su32(&bar)) : "memory");
        const unsigned long long t2 = clock64();
        if (blockIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t0; }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int KIND, int N>
void run(const char* name) {
    unsigned long long* d;
    cudaMalloc(&d, 16);
    const int iters = 4096, smem = 65536 + 1024;
    cudaFuncSetAttribute(mma_kernel<KIND, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    mma_kernel<KIND, N><<<148, 128, smem>>>(iters, d);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    mma_kernel<KIND, N><<<148, 128, smem>>>(iters, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    const double n = 4.0 * iters;
    const double flops = 2.0 * 128 * N * (KIND == 0 ? 16 : 8) * n * 148;
    printf("%s N=%d: issue %.1f cyc/mma, complete %.1f cyc/mma, %.1f TFLOP/s (%s)\n", name, N,
           h[0] / n, h[1] / n, flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    run<0, 128>("bf16");
    run<0, 256>("bf16");
    run<1, 128>("tf32");
    run<1, 256>("tf32");
    return 0;
}
