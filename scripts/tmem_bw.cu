// tmem_bw.cu -- TMEM read bandwidth on this GPU (the bound of the wide pass's
// epilogue: every (record, query) accumulator is read once, 4 bytes).
// One CTA per SM, W warps, each warp reads its lane quarter's columns over and
// over with tcgen05.ld.32x32b.x{16,32,64} and folds them into a register.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bw tmem_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int X>
__device__ __forceinline__ float ldsum(uint32_t taddr);

#define LD_BODY(N, REGS, ...)                                                              \
    uint32_t r[N];                                                                          \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x" #N ".b32 " REGS ", [%" #N "];"          \
                 : __VA_ARGS__                                                               \
                 : "r"(taddr));                                                             \
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");                            \
    float s = 0.f;                                                                          \
    _Pragma("unroll") for (int i = 0; i < N; ++i) s = fminf(s, __uint_as_float(r[i]));     \
    return s;

template <>
__device__ __forceinline__ float ldsum<16>(uint32_t taddr) {
    LD_BODY(16, "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}",
            "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
            "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
            "=r"(r[13]), "=r"(r[14]), "=r"(r[15]))
}
template <>
__device__ __forceinline__ float ldsum<32>(uint32_t taddr) {
    LD_BODY(32,
            "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,"
            "%23,%24,%25,%26,%27,%28,%29,%30,%31}",
            "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
            "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
            "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
            "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
            "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
            "=r"(r[31]))
}

template <int X>
__global__ void tmem_read_kernel(int iters, float* out, unsigned long long* cyc) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = slot;
    const int quarter = warp & 3, part = warp >> 2, nparts = blockDim.x / 128;
    float acc = 0.f;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        // this warp's share of the 512 columns of its lane quarter
        for (int c = part * X; c < 512; c += nparts * X)
            acc += ldsum<X>(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)c);
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (acc == 12345.f) out[threadIdx.x] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int X>
void run(int warps, int nsm) {
    float* out;
    unsigned long long* cyc;
    cudaMalloc(&out, 4096);
    cudaMalloc(&cyc, nsm * 8);
    const int iters = 2000;
    tmem_read_kernel<X><<<nsm, warps * 32>>>(10, out, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    tmem_read_kernel<X><<<nsm, warps * 32>>>(iters, out, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    const double bytes = (double)iters * 128 * 512 * 4;  // per SM
    printf("x%-3d warps %2d: %.1f B/cycle/SM (clock64), %.2f TB/s chip (%d SMs, %.3f ms)\n", X,
           warps, bytes / (double)h, bytes * nsm / (ms * 1e-3) / 1e12, nsm, ms);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    for (int w : {4, 8, 12, 16}) {
        run<16>(w, nsm);
        run<32>(w, nsm);
    }
    return 0;
}
