// Standalone check of the tcgen05 operand layouts used by select_mma.cu:
// one page (128 records x 64 dims, [k][rec]) through TMA SW128 boxes, 8
// K-steps of M=128 N=16 K=8 tf32 MMAs, D read back with tcgen05.ld.
// Tries descriptor variants and prints the max error of each.
#include "../paper_2601_22397_b200/csrc/select_mma.cu"

#include <cstdio>

using namespace sair;

constexpr int DPD = 64;

__global__ void dbg_kernel(const __grid_constant__ CUtensorMap tmap, const float* btile_g,
                           float* out, uint32_t a_lbo, uint32_t a_sbo, uint32_t b_lbo,
                           uint32_t b_sbo, uint32_t idesc, uint32_t alayout, float* raw_out) {
    extern __shared__ __align__(1024) unsigned char raw[];
    unsigned char* sm = raw + ((1024u - (su32(raw) & 1023u)) & 1023u);
    unsigned char* page = sm;                              // 4 boxes x 8 KB
    float* bt = reinterpret_cast<float*>(sm + 32768);      // 8 x 512 B
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 32768 + 4096);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 1024; i += blockDim.x) bt[i] = btile_g[i];
    if (tid == 0) {
        bar_init(&bar[0], 1);
        bar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 4) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(slot)), "r"(32));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    if (tid == 0) {
        bar_expect_tx(&bar[0], 32768);
        for (int b = 0; b < 4; ++b) tma_load_3d(page + b * 8192, &tmap, &bar[0], 32 * b, 0, 0);
    }
    if (warp == 4 && lane == 0) {
        bar_wait(&bar[0], 0);
        tc_fence_after();
        for (int ks = 0; ks < 8; ++ks) {
            uint64_t ad = umma_desc(su32(page) + ks * 1024, a_lbo, a_sbo, alayout);
            uint64_t bd = umma_desc(su32(bt) + ks * 512, b_lbo, b_sbo, 0);
            umma_tf32(tmem, ad, bd, idesc, ks > 0);
        }
        umma_commit(&bar[1]);
    }
    if (warp < 4) {
        bar_wait(&bar[1], 0);
        for (int i = tid; i < 8192 / 4; i += 128) raw_out[i] = reinterpret_cast<float*>(page)[i];
        tc_fence_after();
        float acc[16];
        tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16), acc);
        for (int c = 0; c < 16; ++c) out[(warp * 32 + lane) * 16 + c] = acc[c];
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 4) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32));
    }
}

int main() {
    // x[k][r] small integers (exact in tf32); b[k][n]
    std::vector<float> x(DPD * 128), b(DPD * 16);
    for (int k = 0; k < DPD; ++k)
        for (int r = 0; r < 128; ++r) x[k * 128 + r] = (float)(((r * 7 + k * 3) % 11) - 5);
    for (int k = 0; k < DPD; ++k)
        for (int n = 0; n < 16; ++n) b[k * 16 + n] = (float)(((k * 5 + n * 3) % 7) - 3);
    // B tiles as the kernel lays them out
    std::vector<float> bt(1024, 0.f);
    for (int ks = 0; ks < 8; ++ks)
        for (int n = 0; n < 16; ++n)
            for (int k = 0; k < 8; ++k) {
                int off = ks * 512 + (n % 8) * 16 + (n / 8) * 256 + (k % 4) * 4 + (k / 4) * 128;
                bt[off / 4] = b[(ks * 8 + k) * 16 + n];
            }
    std::vector<double> want(128 * 16, 0.0);
    for (int r = 0; r < 128; ++r)
        for (int n = 0; n < 16; ++n)
            for (int k = 0; k < DPD; ++k) want[r * 16 + n] += (double)x[k * 128 + r] * b[k * 16 + n];
    float *dx, *db, *dout;
    cudaMalloc(&dx, x.size() * 4);
    cudaMalloc(&db, bt.size() * 4);
    cudaMalloc(&dout, 128 * 16 * 4);
    cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(db, bt.data(), bt.size() * 4, cudaMemcpyHostToDevice);
    CUtensorMap m = make_page_map(dx, DPD, 1);
    CUtensorMap m32;
    {
        std::memset(&m32, 0, sizeof(m32));
        const cuuint64_t dims[3] = {128, (cuuint64_t)DPD, 1};
        const cuuint64_t strides[2] = {128 * 4, (cuuint64_t)DPD * 128 * 4};
        const cuuint32_t box[3] = {32, (cuuint32_t)DPD, 1};
        const cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = encoder()(&m32, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, dx, dims, strides, box, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        std::printf("encode atom32: %d\n", (int)r);
    }
    float* draw;
    cudaMalloc(&draw, 8192);
    cudaFuncSetAttribute(dbg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
    struct V { const char* name; uint32_t alb, asb, blb, bsb, idesc, lay; int map32; };
    const uint32_t I = IDESC;
    const uint32_t I_kmajA = IDESC & ~(1u << 15);
    V vs[] = {{"sw128 (16B atoms)", 8192, 1024, 128, 256, I, 2, 0},
              {"sw128_base32b sbo512", 8192, 512, 128, 256, I, 1, 1},
              {"sw128_base32b sbo1024", 8192, 1024, 128, 256, I, 1, 1},
              {"sw128_base32b swapped", 512, 8192, 128, 256, I, 1, 1},
              {"A K-major bit", 8192, 1024, 128, 256, I_kmajA, 2, 0}};
    for (auto& v : vs) {
        cudaMemset(dout, 0, 128 * 16 * 4);
        dbg_kernel<<<1, 160, 48 * 1024>>>(v.map32 ? m32 : m, db, dout, v.alb, v.asb, v.blb, v.bsb,
                                          v.idesc, v.lay, draw);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> got(128 * 16);
        cudaMemcpy(got.data(), dout, got.size() * 4, cudaMemcpyDeviceToHost);
        double err = 0;
        for (int i = 0; i < 128 * 16; ++i) err = std::max(err, std::abs(got[i] - want[i]));
        std::printf("%-22s err=%g  D[0][0]=%g want %g  D[5][3]=%g want %g  (%s)\n", v.name, err,
                    got[0], want[0], got[5 * 16 + 3], want[5 * 16 + 3], cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
        if (v.map32 && v.asb == 512) {
            std::vector<float> rw(2048);
            cudaMemcpy(rw.data(), draw, 8192, cudaMemcpyDeviceToHost);
            // which record t / dim k landed at each smem float of box 0 (x = (r*7+k*3)%11-5)
            for (int row = 0; row < 9; ++row) {
                std::printf("  smem row %d:", row);
                for (int c = 0; c < 32; c += 1) {
                    float v0 = rw[row * 32 + c];
                    int found = -1;
                    for (int t = 0; t < 32 && found < 0; ++t)
                        if ((float)(((t * 7 + row * 3) % 11) - 5) == v0) found = t;
                    std::printf(" %d", found);
                }
                std::printf("\n");
            }
        }
    }
    return 0;
}
