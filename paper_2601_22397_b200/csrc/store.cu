// store.cu -- the device-resident experience store (ExperienceBuffer state).
//
// Host side keeps exactly the reference's bookkeeping in fp64 (gate, running
// sums in append order, reward total, sigma cache state machine;
// experience.cpp:44-62, :171-212).  Device side holds the SoA arrays
// (DESIGN.md "Data layout in HBM"); rows arrive through pinned staging and a
// scatter kernel that also writes the fp32 page layout.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <new>
#include <cstring>

#include "internal.hpp"

namespace sair {

// ---------------------------------------------------------------- kernels --

// Scatter `cnt` staged rows (fp64, record-major) into the store at [n0, n0+cnt).
__global__ void scatter_rows_kernel(const double* __restrict__ sx, const double* __restrict__ sr,
                                    const int32_t* __restrict__ sround, size_t n0, size_t cnt,
                                    int d, int dp, float* __restrict__ pages,
                                    float* __restrict__ r32, double* __restrict__ r64,
                                    int32_t* __restrict__ rnd, double* __restrict__ x64,
                                    const double* __restrict__ shift) {
    // w covers both layouts: the page row holds dp >= min(d, 256) columns
    // (d > 256 never takes the fp32 filter paths), x64 every one of the d
    const int w = d > dp ? d : dp;
    size_t total = cnt * (size_t)w;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
         t += (size_t)gridDim.x * blockDim.x) {
        size_t i = t / w;
        int k = (int)(t % w);
        size_t rec = n0 + i;
        double v = k < d ? sx[i * d + k] : 0.0;
        if (k < dp) pages[page_index(rec, k, dp)] = k < d ? to_tf32(v - shift[k]) : 0.f;
        if (k < d) x64[rec * d + k] = v;
        if (k == 0) {
            r64[rec] = sr[i];
            r32[rec] = (float)sr[i];
            rnd[rec] = sround[i];
        }
    }
}

// splitmix64 counter generator; paper_2601_22397_b200/synth.py is the host twin.
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t synth_key(uint64_t seed, uint64_t stream) {
    return seed * 0x100000001B3ull + stream * 0x9E3779B1ull;
}
__device__ __forceinline__ double synth_value(uint64_t seed, uint64_t rec, int d, int k) {
    uint64_t h = splitmix64((rec * (uint64_t)d + (uint64_t)k) ^ synth_key(seed, 1));
    int64_t s = (int64_t)(h & 0xFFF) + (int64_t)((h >> 12) & 0xFFF) +
                (int64_t)((h >> 24) & 0xFFF) + (int64_t)((h >> 36) & 0xFFF);
    return (double)(s - 8190) * 0x1p-11;
}

// Generate rows [n0, n0+cnt) (global index gbase+n0+i) and accumulate their
// exact statistics: every value is a multiple of 2^-11 (x^2 of 2^-22, reward
// of 2^-20) so the fp64 sums are exact in any order.
__global__ void synth_rows_kernel(uint64_t seed, int clustered, int64_t gbase, size_t n0,
                                  size_t cnt, int d, int dp, float* __restrict__ pages,
                                  float* __restrict__ r32, double* __restrict__ r64,
                                  int32_t* __restrict__ rnd, double* __restrict__ x64,
                                  double* __restrict__ acc /* [2d + 1] sum, sum_sq, total */,
                                  unsigned long long* __restrict__ amax /* [d + 1] */,
                                  const double* __restrict__ shift) {
    extern __shared__ double sh[];  // [2d+1] block partial sums
    __shared__ unsigned long long shmax[257];
    for (int t = threadIdx.x; t < 2 * d + 1; t += blockDim.x) sh[t] = 0.0;
    for (int t = threadIdx.x; t < d + 1; t += blockDim.x) shmax[t] = 0ull;
    __syncthreads();
    size_t total = cnt * (size_t)dp;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
         t += (size_t)gridDim.x * blockDim.x) {
        size_t i = t / dp;
        int k = (int)(t % dp);
        size_t rec = n0 + i;
        uint64_t g = (uint64_t)(gbase + (int64_t)rec);
        double v = 0.0;
        if (k < d) {
            v = synth_value(seed, g, d, k);
            if (clustered) {
                uint64_t cid = splitmix64(g ^ synth_key(seed, 0xC1)) % 64ull;
                v += synth_value(seed ^ 0x5EEDull, cid, d, k) * 2.0;
            }
            x64[rec * d + k] = v;
            atomicAdd(&sh[k], v);
            atomicAdd(&sh[d + k], v * v);
            atomicMax(&shmax[k], (unsigned long long)__double_as_longlong(fabs(v)));
        }
        pages[page_index(rec, k, dp)] =
            k < d ? to_tf32(v - shift[k]) : 0.f;
        if (k == 0) {
            uint64_t h = splitmix64(g ^ synth_key(seed, 2));
            double r = (double)((h & 0xFFFFFull) + 8192ull) * 0x1p-20;
            r64[rec] = r;
            r32[rec] = (float)r;
            rnd[rec] = (int32_t)g;
            atomicAdd(&sh[2 * d], r);
            atomicMax(&shmax[d], (unsigned long long)__double_as_longlong(r));
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < 2 * d + 1; t += blockDim.x) atomicAdd(&acc[t], sh[t]);
    for (int t = threadIdx.x; t < d + 1; t += blockDim.x) atomicMax(&amax[t], shmax[t]);
}

// sigma refresh (experience.cpp:80-114): z-rows of the subsample, then every
// pairwise distance sqrt(sum (z_i - z_j)^2) in the reference's rounding order.
__global__ void sigma_z_kernel(const double* __restrict__ x64, const int64_t* __restrict__ idx,
                               int m, int d, const double* __restrict__ mean,
                               const double* __restrict__ sd, double* __restrict__ z) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < m * d; t += gridDim.x * blockDim.x) {
        int a = t / d, k = t % d;
        z[t] = ddiv(dsub(x64[idx[a] * d + k], mean[k]), sd[k]);
    }
}

__global__ void sigma_pairs_kernel(const double* __restrict__ z, int m, int d,
                                   double* __restrict__ dists) {
    // block i writes the distances (i, j > i) at row_start(i) + (j - i - 1)
    int i = blockIdx.x;
    size_t row = (size_t)i * (2 * (size_t)m - i - 1) / 2;
    for (int j = i + 1 + threadIdx.x; j < m; j += blockDim.x) {
        double d2 = 0.0;
        for (int k = 0; k < d; ++k) {
            double t = dsub(z[(size_t)i * d + k], z[(size_t)j * d + k]);
            d2 = dadd(d2, dmul(t, t));
        }
        dists[row + (j - i - 1)] = sqrt(d2);
    }
}

// ------------------------------------------------------------------- host --

void store_init(sair_store_s* s, double r_min, int device, size_t capacity_hint) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        throw Error(SAIR_ECUDA, "no CUDA device (libsair has no CPU fallback)");
    if (device < 0 || device >= ndev) throw Error(SAIR_EINVAL, "device ordinal out of range");
    s->device = device;
    s->r_min = r_min;
    DeviceGuard g(device);
    SAIR_CUDA(cudaStreamCreateWithFlags(&s->st, cudaStreamNonBlocking));
    SAIR_CUDA(cudaStreamCreateWithFlags(&s->cst, cudaStreamNonBlocking));
    for (auto& e : s->ev) SAIR_CUDA(cudaEventCreate(&e));
    for (int i = 0; i < 2; ++i) {
        SAIR_CUDA(cudaEventCreateWithFlags(&s->ev_copied[i], cudaEventDisableTiming));
        SAIR_CUDA(cudaEventCreateWithFlags(&s->ev_scattered[i], cudaEventDisableTiming));
    }
    s->cap = 0;
    (void)capacity_hint;  // capacity is fixed once the dimension is known
    s->last = sair_select_stats{};
    s->stats.sum.clear();
}

static void free_arrays(sair_store_s* s) {
    cudaFree(s->pages);
    cudaFree(s->r32);
    cudaFree(s->r64);
    cudaFree(s->rnd);
    cudaFree(s->x64);
    s->pages = nullptr;
    s->r32 = nullptr;
    s->r64 = nullptr;
    s->rnd = nullptr;
    s->x64 = nullptr;
}

void store_free(sair_store_s* s) {
    DeviceGuard g(s->device);
    if (s->st) cudaStreamSynchronize(s->st);
    free_arrays(s);
    cudaFree(s->d_shift);
    s->d_shift = nullptr;
    for (auto* b : {&s->b_stage, &s->b_cand, &s->b_merged, &s->b_thr, &s->b_z, &s->b_consts,
                    &s->b_out, &s->b_exact, &s->b_sigma, &s->b_red, &s->b_mmab, &s->b_sample,
                    &s->b_loo, &s->b_greedy, &s->b_grp,
                    &s->b_wlists, &s->b_pl, &s->b_hot, &s->b_pages16, &s->b_pl16})
        b->release();
    s->pages16_n = 0;
    if (s->cst) cudaStreamSynchronize(s->cst);
    for (int i = 0; i < 2; ++i) {
        s->h_app[i].~HBuf();
        new (&s->h_app[i]) HBuf();
        s->b_app[i].release();
        if (s->ev_copied[i]) cudaEventDestroy(s->ev_copied[i]);
        if (s->ev_scattered[i]) cudaEventDestroy(s->ev_scattered[i]);
        s->ev_copied[i] = s->ev_scattered[i] = nullptr;
    }
    if (s->cst) cudaStreamDestroy(s->cst);
    s->cst = nullptr;
    for (auto& e : s->ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : s->gev) cudaEventDestroy(e);
    for (auto& e : s->g32ev) cudaEventDestroy(e);
    s->g32ev.clear();
    for (auto& e : s->cev) cudaEventDestroy(e);
    s->cev.clear();
    s->gev.clear();
    if (s->st) cudaStreamDestroy(s->st);
    s->st = nullptr;
}

// Ensure capacity for `need` records (page multiple); grows geometrically and
// moves the old contents with device-to-device copies.
void store_reserve(sair_store_s* s, size_t need) {
    if (need <= s->cap) return;
    size_t cap = std::max<size_t>({need, s->cap * 2, (size_t)4 * PAGE});
    cap = (cap + PAGE - 1) / PAGE * PAGE;
    float *pages, *r32;
    double *r64, *x64;
    int32_t* rnd;
    SAIR_CUDA(cudaMalloc(&pages, cap * (size_t)s->dp * sizeof(float)));
    SAIR_CUDA(cudaMalloc(&r32, cap * sizeof(float)));
    SAIR_CUDA(cudaMalloc(&r64, cap * sizeof(double)));
    SAIR_CUDA(cudaMalloc(&rnd, cap * sizeof(int32_t)));
    SAIR_CUDA(cudaMalloc(&x64, cap * (size_t)s->d * sizeof(double)));
    // zero the page layout so padding dims / tail slots read as 0
    SAIR_CUDA(cudaMemsetAsync(pages, 0, cap * (size_t)s->dp * sizeof(float), s->st));
    if (s->n) {
        size_t used_pages = (s->n + PAGE - 1) / PAGE;
        SAIR_CUDA(cudaMemcpyAsync(pages, s->pages, used_pages * PAGE * (size_t)s->dp * 4,
                                  cudaMemcpyDeviceToDevice, s->st));
        SAIR_CUDA(cudaMemcpyAsync(r32, s->r32, s->n * 4, cudaMemcpyDeviceToDevice, s->st));
        SAIR_CUDA(cudaMemcpyAsync(r64, s->r64, s->n * 8, cudaMemcpyDeviceToDevice, s->st));
        SAIR_CUDA(cudaMemcpyAsync(rnd, s->rnd, s->n * 4, cudaMemcpyDeviceToDevice, s->st));
        SAIR_CUDA(cudaMemcpyAsync(x64, s->x64, s->n * (size_t)s->d * 8, cudaMemcpyDeviceToDevice,
                                  s->st));
    }
    SAIR_CUDA(cudaStreamSynchronize(s->st));
    free_arrays(s);
    s->pages = pages;
    s->r32 = r32;
    s->r64 = r64;
    s->rnd = rnd;
    s->x64 = x64;
    s->cap = cap;
}

static void fix_dim(sair_store_s* s, int dim, const double* first_row) {
    s->shift.assign(dim, 0.0);
    if (first_row) s->shift.assign(first_row, first_row + dim);
    if (s->d_shift) cudaFree(s->d_shift);
    s->d_shift = nullptr;
    SAIR_CUDA(cudaMalloc(&s->d_shift, dim * sizeof(double)));
    SAIR_CUDA(cudaMemcpy(s->d_shift, s->shift.data(), dim * sizeof(double), cudaMemcpyHostToDevice));
    s->d = dim;
    s->dp = dp_bucket(dim);
    s->stats.sum.assign(dim, 0.0);
    s->stats.sum_sq.assign(dim, 0.0);
    s->stats.xabs.assign(dim, 0.0);
    s->stats.total = 0.0;
    s->stats.rabs = 0.0;
}

size_t store_append(sair_store_s* s, const double* ctx, size_t count, int dim,
                    const double* reward, const int32_t* round, uint8_t* accepted) {
    if (count == 0) return 0;
    if (dim <= 0) throw Error(SAIR_EINVAL, "experience store: context dimension must be > 0");
    DeviceGuard g(s->device);
    size_t done = 0, n_acc = 0;
    const size_t chunk = 1 << 16;
    std::string err;
    while (done < count && err.empty()) {
        size_t take = std::min(chunk, count - done);
        // this chunk's pinned staging: free once its previous copy (two chunks
        // or calls ago) has landed
        const int slot = s->app_slot;
        SAIR_CUDA(cudaEventSynchronize(s->ev_copied[slot]));
        double* hx = s->h_app[slot].as<double>(take * (size_t)dim + 2 * take);
        double* hr = hx + take * (size_t)dim;
        int32_t* hround = reinterpret_cast<int32_t*>(hr + take);
        size_t k = 0;
        for (size_t i = done; i < done + take; ++i) {
            // gate, experience.cpp:45-48
            if (!(reward[i] > s->r_min)) {
                ++s->rejected;
                if (accepted) accepted[i] = 0;
                continue;
            }
            // dimension fixed on first accepted row, experience.cpp:49-54
            if (s->n + k == 0) {
                fix_dim(s, dim, ctx + i * (size_t)dim);
            } else if (dim != s->d) {
                err = "experience store: context dimension changed";
                break;
            }
            const double* x = ctx + i * (size_t)dim;
            auto& st = s->stats;
            for (int j = 0; j < dim; ++j) {  // experience.cpp:55-58
                st.sum[j] += x[j];
                st.sum_sq[j] += x[j] * x[j];
                st.xabs[j] = std::max(st.xabs[j], std::fabs(x[j]));
            }
            st.total += reward[i];  // loo_mean's total, same order (experience.cpp:138-139)
            st.rabs = std::max(st.rabs, std::fabs(reward[i]));
            std::memcpy(hx + k * (size_t)dim, x, (size_t)dim * sizeof(double));
            hr[k] = reward[i];
            hround[k] = round[i];
            if (accepted) accepted[i] = 1;
            ++k;
            ++s->stale;  // experience.cpp:60
        }
        if (k) {
            store_reserve(s, s->n + k);
            size_t xb = k * (size_t)dim * sizeof(double);
            // The copy runs on the store's copy stream (overlapping the compute
            // stream's work: a select in flight, the previous chunk's scatter);
            // the scatter waits for it on the compute stream, so every later
            // pass sees the rows; the device staging of this slot is rewritten
            // only after its previous scatter
            SAIR_CUDA(cudaStreamWaitEvent(s->cst, s->ev_scattered[slot], 0));
            void* before = s->b_app[slot].p;
            char* dst = static_cast<char*>(s->b_app[slot].get(xb + k * 12 + 64));
            if (dst != before) SAIR_CUDA(cudaStreamSynchronize(s->st));  // (reallocated)
            double* dx = reinterpret_cast<double*>(dst);
            double* dr = reinterpret_cast<double*>(dst + xb);
            int32_t* dround = reinterpret_cast<int32_t*>(dst + xb + k * 8);
            SAIR_CUDA(cudaMemcpyAsync(dx, hx, xb, cudaMemcpyHostToDevice, s->cst));
            SAIR_CUDA(cudaMemcpyAsync(dr, hr, k * 8, cudaMemcpyHostToDevice, s->cst));
            SAIR_CUDA(cudaMemcpyAsync(dround, hround, k * 4, cudaMemcpyHostToDevice, s->cst));
            SAIR_CUDA(cudaEventRecord(s->ev_copied[slot], s->cst));
            SAIR_CUDA(cudaStreamWaitEvent(s->st, s->ev_copied[slot], 0));
            size_t work = k * (size_t)std::max(s->dp, s->d);
            int blocks = (int)std::min<size_t>((work + 255) / 256, 148 * 16);
            scatter_rows_kernel<<<blocks, 256, 0, s->st>>>(dx, dr, dround, s->n, k, s->d, s->dp,
                                                           s->pages, s->r32, s->r64, s->rnd,
                                                           s->x64, s->d_shift);
            SAIR_LAUNCH("scatter_rows_kernel");
            SAIR_CUDA(cudaEventRecord(s->ev_scattered[slot], s->st));
            s->app_slot ^= 1;
            s->n += k;
            n_acc += k;
        }
        done += take;
    }
    if (!err.empty()) throw Error(SAIR_EINVAL, err);
    return n_acc;
}

bool store_append_one_commit(sair_store_s* s, const double* x, double reward) {
    // the host half of store_append for the row the device just wrote (or not)
    if (!(reward > s->r_min)) {
        ++s->rejected;
        return false;
    }
    auto& st = s->stats;
    for (int j = 0; j < s->d; ++j) {  // experience.cpp:55-58
        st.sum[j] += x[j];
        st.sum_sq[j] += x[j] * x[j];
        st.xabs[j] = std::max(st.xabs[j], std::fabs(x[j]));
    }
    st.total += reward;
    st.rabs = std::max(st.rabs, std::fabs(reward));
    s->n += 1;
    ++s->stale;  // experience.cpp:60
    return true;
}

void store_append_synthetic(sair_store_s* s, uint64_t seed, size_t count, int dim,
                            int clustered) {
    if (count == 0) return;
    if (dim <= 0 || dim > 256) throw Error(SAIR_EINVAL, "synthetic: dim must be in 1..256");
    if (!(0x1p-7 > s->r_min))
        throw Error(SAIR_EINVAL, "synthetic rewards start at 2^-7: r_min must be below that");
    if (s->n == 0) {
        fix_dim(s, dim, nullptr);
    } else if (dim != s->d) {
        throw Error(SAIR_EINVAL, "experience store: context dimension changed");
    }
    DeviceGuard g(s->device);
    store_reserve(s, s->n + count);
    double* acc = s->b_red.as<double>(2 * dim + 1 + dim + 1);
    auto* amax = reinterpret_cast<unsigned long long*>(acc + 2 * dim + 1);
    SAIR_CUDA(cudaMemsetAsync(acc, 0, (3 * dim + 2) * sizeof(double), s->st));
    size_t work = count * (size_t)s->dp;
    int blocks = (int)std::min<size_t>((work + 255) / 256, 148 * 8);
    synth_rows_kernel<<<blocks, 256, (2 * dim + 1) * sizeof(double), s->st>>>(
        seed, clustered, s->gbase, s->n, count, s->d, s->dp, s->pages, s->r32, s->r64, s->rnd,
        s->x64, acc, amax, s->d_shift);
    SAIR_LAUNCH("synth_rows_kernel");
    std::vector<double> h(3 * dim + 2);
    SAIR_CUDA(cudaMemcpyAsync(h.data(), acc, h.size() * sizeof(double), cudaMemcpyDeviceToHost,
                              s->st));
    SAIR_CUDA(cudaStreamSynchronize(s->st));
    auto& st = s->stats;
    for (int k = 0; k < dim; ++k) {
        st.sum[k] += h[k];  // exact: every partial sum is representable
        st.sum_sq[k] += h[dim + k];
        double mx;
        std::memcpy(&mx, &h[2 * dim + 1 + k], 8);
        st.xabs[k] = std::max(st.xabs[k], mx);
    }
    st.total += h[2 * dim];
    double rmx;
    std::memcpy(&rmx, &h[3 * dim + 1], 8);
    st.rabs = std::max(st.rabs, rmx);
    s->n += count;
    s->stale += count;
}

void store_mean_sd(const sair_store_s* s, double* mean, double* sd) {
    // standardize's per-dimension statistics, experience.cpp:68-74
    const StoreStats& st = eff_stats(s);
    double nn = static_cast<double>(eff_n(s));
    for (int k = 0; k < s->d; ++k) {
        double m = st.sum[k] / nn;
        double var = std::max(0.0, st.sum_sq[k] / nn - m * m);
        double v = std::sqrt(var);
        if (v < 1e-12) v = 1.0;
        mean[k] = m;
        sd[k] = v;
    }
}

void store_standardize(const sair_store_s* s, const double* x, double* z) {
    // experience.cpp:64-78 (callers check emptiness / dimension)
    std::vector<double> mean(s->d), sd(s->d);
    store_mean_sd(s, mean.data(), sd.data());
    for (int k = 0; k < s->d; ++k) z[k] = (x[k] - mean[k]) / sd[k];
}

// median pairwise z-distance of the rows idx of `x64` (device, record-major),
// experience.cpp:92-112: z rows, every pair's distance, the order statistic
// at size/2 (what nth_element places there) via a device radix sort.
static double sigma_of_rows(cudaStream_t st, DBuf& scratch, const double* x64,
                            const std::vector<int64_t>& idx, int d, const double* mean,
                            const double* sd) {
    const int m = (int)idx.size();
    const size_t np = (size_t)m * (m - 1) / 2;
    if (np == 0) return 1.0;
    size_t tmp_bytes = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, (double*)nullptr, (double*)nullptr,
                                   (int)np);
    size_t off_idx = 0, off_msd = off_idx + m * 8, off_z = off_msd + 2 * d * 8,
           off_d = off_z + (size_t)m * d * 8, off_s = off_d + np * 8, off_t = off_s + np * 8;
    char* base = static_cast<char*>(scratch.get(off_t + tmp_bytes + 256));
    auto* didx = reinterpret_cast<int64_t*>(base + off_idx);
    auto* dmsd = reinterpret_cast<double*>(base + off_msd);
    auto* dz = reinterpret_cast<double*>(base + off_z);
    auto* dd = reinterpret_cast<double*>(base + off_d);
    auto* ds = reinterpret_cast<double*>(base + off_s);
    SAIR_CUDA(cudaMemcpyAsync(didx, idx.data(), m * 8, cudaMemcpyHostToDevice, st));
    SAIR_CUDA(cudaMemcpyAsync(dmsd, mean, d * 8, cudaMemcpyHostToDevice, st));
    SAIR_CUDA(cudaMemcpyAsync(dmsd + d, sd, d * 8, cudaMemcpyHostToDevice, st));
    sigma_z_kernel<<<ceil_div((size_t)m * d, 256), 256, 0, st>>>(x64, didx, m, d, dmsd, dmsd + d,
                                                                 dz);
    SAIR_LAUNCH("sigma_z_kernel");
    sigma_pairs_kernel<<<m, 128, 0, st>>>(dz, m, d, dd);
    SAIR_LAUNCH("sigma_pairs_kernel");
    SAIR_CUDA(cub::DeviceRadixSort::SortKeys(base + off_t, tmp_bytes, dd, ds, (int)np, 0, 64, st));
    double mid = 0.0;
    SAIR_CUDA(cudaMemcpyAsync(&mid, ds + np / 2, 8, cudaMemcpyDeviceToHost, st));
    SAIR_CUDA(cudaStreamSynchronize(st));
    return mid > 1e-12 ? mid : 1.0;
}

// the strided subsample of refresh_sigma_cache, experience.cpp:82-91
std::vector<int64_t> sigma_sample(uint64_t n) {
    const size_t capn = 512;
    std::vector<int64_t> idx;
    if (n <= capn) {
        for (size_t k = 0; k < n; ++k) idx.push_back((int64_t)k);
    } else {
        double stride = static_cast<double>(n) / capn;
        for (size_t k = 0; k < capn; ++k) idx.push_back((int64_t)(size_t)(k * stride));
    }
    return idx;
}

static double refresh_sigma(sair_store_s* s) {
    DeviceGuard g(s->device);
    const int d = s->d;
    std::vector<double> mean(d), sd(d);
    store_mean_sd(s, mean.data(), sd.data());
    return sigma_of_rows(s->st, s->b_sigma, s->x64, sigma_sample(s->n), d, mean.data(), sd.data());
}

double sigma_rows(const double* rows, size_t m, int d, const double* mean, const double* sd,
                  int device) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        throw Error(SAIR_ECUDA, "no CUDA device (libsair has no CPU fallback)");
    DeviceGuard g(device);
    cudaStream_t st;
    SAIR_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    DBuf rb, scratch;
    double* dr = static_cast<double*>(rb.get(m * (size_t)d * 8 + 8));
    SAIR_CUDA(cudaMemcpyAsync(dr, rows, m * (size_t)d * 8, cudaMemcpyHostToDevice, st));
    std::vector<int64_t> idx(m);
    for (size_t i = 0; i < m; ++i) idx[i] = (int64_t)i;
    double v = sigma_of_rows(st, scratch, dr, idx, d, mean, sd);
    cudaStreamDestroy(st);
    return v;
}

double store_effective_sigma(sair_store_s* s, double sigma_sim) {
    // experience.cpp:116-121
    if (sigma_sim > 0.0) return sigma_sim;
    if (s->sharded) {  // the buffer's sigma, computed over its global subsample
        if (s->n_global < 2) return 1.0;
        if (!(s->gsigma > 0.0))
            throw Error(SAIR_EINVAL, "sharded store: set the buffer's sigma (sair_store_set_global)");
        return s->gsigma;
    }
    if (s->n < 2) return 1.0;
    if (s->cached_sigma == 0.0 || s->stale >= 50) {
        s->cached_sigma = refresh_sigma(s);
        s->stale = 0;
    }
    return s->cached_sigma;
}

void store_clone(const sair_store_s* s, sair_store_s* o) {
    {  // the source's enqueued appends complete before its arrays are copied
        DeviceGuard g(s->device);
        SAIR_CUDA(cudaStreamSynchronize(s->st));
    }
    store_init(o, s->r_min, s->device, 0);
    o->rejected = s->rejected;
    o->gbase = s->gbase;
    o->stats = s->stats;
    o->sharded = s->sharded;
    o->n_global = s->n_global;
    o->gst = s->gst;
    o->gsigma = s->gsigma;
    o->shift = s->shift;
    if (!s->shift.empty()) {
        DeviceGuard g0(s->device);
        SAIR_CUDA(cudaMalloc(&o->d_shift, s->shift.size() * sizeof(double)));
        SAIR_CUDA(cudaMemcpy(o->d_shift, s->shift.data(), s->shift.size() * sizeof(double),
                             cudaMemcpyHostToDevice));
    }
    o->cached_sigma = s->cached_sigma;
    o->stale = s->stale;
    if (s->n == 0) {
        o->d = s->d;
        o->dp = s->dp;
        return;
    }
    o->d = s->d;
    o->dp = s->dp;
    DeviceGuard g(s->device);
    SAIR_CUDA(cudaStreamSynchronize(s->st));
    store_reserve(o, s->n);
    size_t used_pages = (s->n + PAGE - 1) / PAGE;
    SAIR_CUDA(cudaMemcpyAsync(o->pages, s->pages, used_pages * PAGE * (size_t)s->dp * 4,
                              cudaMemcpyDeviceToDevice, o->st));
    SAIR_CUDA(cudaMemcpyAsync(o->r32, s->r32, s->n * 4, cudaMemcpyDeviceToDevice, o->st));
    SAIR_CUDA(cudaMemcpyAsync(o->r64, s->r64, s->n * 8, cudaMemcpyDeviceToDevice, o->st));
    SAIR_CUDA(cudaMemcpyAsync(o->rnd, s->rnd, s->n * 4, cudaMemcpyDeviceToDevice, o->st));
    SAIR_CUDA(cudaMemcpyAsync(o->x64, s->x64, s->n * (size_t)s->d * 8, cudaMemcpyDeviceToDevice,
                              o->st));
    SAIR_CUDA(cudaStreamSynchronize(o->st));
    o->n = s->n;
}

}  // namespace sair
