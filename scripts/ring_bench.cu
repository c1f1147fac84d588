// Microbenchmark: how fast can a persistent 1-CTA/SM bulk-copy ring stream HBM
// with trivial consumers?  Sweeps stage size / depth; compares with LDG.128.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory"); }
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(d)), "l"(s), "r"(n), "r"(su32(b)) : "memory"); }

__global__ void ring(const float* src, size_t nchunks, int chunk_bytes, int nst, float* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* full = (uint64_t*)(sm + (size_t)nst * chunk_bytes);
  uint64_t* empty = full + 8;
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { for (int s = 0; s < nst; ++s) { bar_init(&full[s], 1); bar_init(&empty[s], 8); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  size_t mine = blockIdx.x < nchunks ? (nchunks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (warp == 8) {
    if (lane == 0) { int s = 0; uint32_t ph = 0;
      for (size_t it = 0; it < mine; ++it) {
        if (it >= (size_t)nst) bar_wait(&empty[s], ph ^ 1);
        bar_expect(&full[s], chunk_bytes);
        const char* g = (const char*)src + (blockIdx.x + it * gridDim.x) * (size_t)chunk_bytes;
        for (int off = 0; off < chunk_bytes; off += 32768)
          bulk(sm + (size_t)s * chunk_bytes + off, g + off, min(32768, chunk_bytes - off), &full[s]);
        if (++s == nst) { s = 0; ph ^= 1; } } }
    return;
  }
  float acc = 0.f; int s = 0; uint32_t ph = 0;
  for (size_t it = 0; it < mine; ++it) {
    bar_wait(&full[s], ph);
    acc += ((float*)(sm + (size_t)s * chunk_bytes))[threadIdx.x];
    __syncwarp(); if (lane == 0) bar_arrive(&empty[s]);
    if (++s == nst) { s = 0; ph ^= 1; } }
  if (acc == 12345.f) sink[0] = acc;
}

__global__ void ldg(const float4* src, size_t n4, float* sink) {
  float4 a = make_float4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x * 4) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) { size_t j = i + (size_t)u * gridDim.x * blockDim.x; v[u] = j < n4 ? __ldg(src + j) : make_float4(0,0,0,0); }
#pragma unroll
    for (int u = 0; u < 4; ++u) { a.x += v[u].x; a.y += v[u].y; a.z += v[u].z; a.w += v[u].w; }
  }
  if (a.x + a.y + a.z + a.w == 12345.f) sink[0] = a.x;
}

int main() {
  const size_t bytes = 4362076160ull;  // 16M x 260 B, the stream kernel's traffic
  float* src; float* sink;
  cudaMalloc(&src, bytes); cudaMalloc(&sink, 64); cudaMemset(src, 0, bytes);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int cfgs[][2] = {{16384, 4}, {16384, 8}, {32768, 3}, {32768, 5}, {32768, 6}, {65536, 3}, {65536, 2}};
  cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  for (auto& c : cfgs) {
    size_t nch = bytes / c[0];
    size_t smem = (size_t)c[1] * c[0] + 256;
    if (smem > 227 * 1024) continue;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      ring<<<nsm, 288, smem>>>(src, nch, c[0], c[1], sink);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("ring chunk %6d B x %d stages: %.3f ms  %.0f GB/s  (%s)\n", c[0], c[1], ms, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  for (int g : {nsm * 2, nsm * 4, nsm * 8}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0); ldg<<<g, 256>>>((const float4*)src, bytes / 16, sink); cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("ldg.128 grid %d x 256: %.3f ms  %.0f GB/s\n", g, ms, bytes / ms / 1e6);
  }
  return 0;
}
