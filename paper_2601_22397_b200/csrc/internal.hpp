// internal.hpp -- host-side state behind the sair_* handles.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <functional>
#include <memory>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace sair {

// growth policy of the scratch buffers: sizes that creep up call by call (a
// store growing one record per decision step) must not reallocate every call
inline size_t grow_to(size_t need, size_t have) {
    size_t n = std::max(need, have + have / 2);
    return (n + 65535) & ~(size_t)65535;
}

// Grow-only device scratch buffer.
struct DBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void* get(size_t need) {
        if (need > bytes) {
            if (p) cudaFree(p);
            p = nullptr;
            const size_t nb = grow_to(need, bytes);
            bytes = 0;
            SAIR_CUDA(cudaMalloc(&p, nb));
            bytes = nb;
        }
        return p;
    }
    template <class T>
    T* as(size_t count) { return static_cast<T*>(get(count * sizeof(T) + 16)); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    ~DBuf() { release(); }
};

// Grow-only pinned host staging buffer.
struct HBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void* get(size_t need) {
        if (need > bytes) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            const size_t nb = grow_to(need, bytes);
            bytes = 0;
            SAIR_CUDA(cudaMallocHost(&p, nb));
            bytes = nb;
        }
        return p;
    }
    template <class T>
    T* as(size_t count) { return static_cast<T*>(get(count * sizeof(T) + 16)); }
    ~HBuf() {
        if (p) cudaFreeHost(p);
    }
};

// Large pageable host->device copy through a pinned ring filled by host
// threads (xfer.cpp); below 8 MB a plain cudaMemcpyAsync.  Returns once every
// chunk's DMA is queued on st and the ring has drained.
void copy_h2d_staged(void* dst, const void* src, size_t bytes, cudaStream_t st);

// Host-maintained fp64 statistics (bit-identical to the reference's
// ExperienceBuffer members sum_, sum_sq_, the reward total of loo_mean, and the
// sigma cache; experience.hpp:82-88).
struct GreedySession;  // select_greedy.cu: a distributed greedy in progress

struct StoreStats {
    std::vector<double> sum, sum_sq, xabs;  // per dim; xabs = max |x| (filter bound)
    double total = 0.0;                     // sum of rewards in index order
    double rabs = 0.0;                      // max |reward| (filter bound)
};

}  // namespace sair

// ------------------------------------------------------------------ store --
struct sair_store_s {
    int device = 0;
    cudaStream_t st = nullptr;
    cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};

    double r_min = 0.0;
    uint64_t rejected = 0;
    // lambda > 0: the last filtered attempt certified < 5 % of its queries
    // (the penalty moves the picks far down the score order): later calls go
    // straight to the filtered greedy, re-trying the pool every 16th call
    int lam_pool_fail = 0;
    uint32_t lam_probe = 0;
    int d = 0;   // 0 until the first accepted row fixes it (experience.cpp:49-54)
    int dp = 0;  // padded dimension of the fp32 page layout
    size_t n = 0, cap = 0;
    int64_t gbase = 0;  // global index of local record 0 (shard offset)

    sair::StoreStats stats;
    // shard mode (multi-GPU): this store holds records [gbase, gbase + n) of a
    // buffer of n_global records whose statistics are gst / gsigma
    bool sharded = false;
    uint64_t n_global = 0;
    sair::StoreStats gst;
    double gsigma = 0.0;
    // per-dimension centring of the fp32 page copy: pages hold fp32(x - shift)
    // (shift = the first stored row), keeping the filter's norm expansion well
    // conditioned for uncentred features (memory_mb, cpu_millicores, ...)
    std::vector<double> shift;
    double* d_shift = nullptr;
    double cached_sigma = 0.0;  // experience.hpp:87
    size_t stale = 0;           // experience.hpp:88

    // device SoA
    float* pages = nullptr;  // [cap/PAGE][dp][PAGE] fp32 filter copy
    float* r32 = nullptr;    // [cap] fp32 rewards (filter)
    double* r64 = nullptr;   // [cap] exact rewards
    int32_t* rnd = nullptr;  // [cap] rounds (tie-break)
    double* x64 = nullptr;   // [cap][d] exact contexts (record-major, refine/gather)

    // appends: a copy stream and two pinned / device staging buffers, so a
    // chunk's host->device copy overlaps the previous chunk's scatter and
    // whatever the compute stream runs
    cudaStream_t cst = nullptr;
    cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_scattered[2] = {nullptr, nullptr};
    sair::HBuf h_app[2];
    sair::DBuf b_app[2];
    int app_slot = 0;
    // scratch
    sair::DBuf b_stage, b_cand, b_merged, b_thr, b_z, b_consts, b_out, b_exact, b_sigma, b_red;
    sair::HBuf h_stage, h_out, h_mmab, h_consts;
    sair::DBuf b_mmab;    // tensor-core B operand constants, t0, dropped
    sair::DBuf b_sample;  // sample pre-pass keys
    sair::DBuf b_loo;     // standardized rows + locally weighted LOO means (per call)
    sair::DBuf b_greedy;  // batched exact greedy: rows + per-(query, record) state
    sair::DBuf b_grp;     // per query group of one select call: merged lists, thresholds, ...
    sair::DBuf b_wlists;  // the wide pass's compacted CTA lists of every group of a call
    sair::DBuf b_pl;      // per record (P, log residual) of the current call (wide pass)
    // bf16 filter copy of the pages for the 256-query wide pass (DESIGN.md
    // "K4 bf16"): [page][128 rows][64 dims] K-major, 128-byte swizzled; derived
    // from `pages` on demand, valid for records [0, pages16_n)
    sair::DBuf b_pages16;
    size_t pages16_n = 0;
    sair::DBuf b_pl16;    // (P, log residual) of the bf16 records (the bf16 pass's cache)
    bool defer_sync = false;         // decision step: the small select leaves its copy-out
    std::function<void()> pending;   // pending, and its host unpack here
    sair::DBuf b_hot;     // the wide sample's highest-residual pages ...
    size_t hot_n = 0;     // ... valid while the store holds hot_n records (append-only)
    float hot_c1 = 0.f, hot_c0 = 0.f;  // and the call's reward constants match
    uint32_t hot_sp = 0;  // and the uniform sample's page count
    sair::HBuf h_ra;      // pinned refine argument blocks
    std::shared_ptr<sair::GreedySession> greedy;  // sharded lambda > 0 select in progress
    std::vector<cudaEvent_t> gev;  // per query group: start, end of pre-pass, end of stream
    std::vector<cudaEvent_t> g32ev;  // the greedy's step kernels: start, end per step
    std::vector<cudaEvent_t> cev;    // wide pass: a group's constants landed (copy stream)
    const float* mma_t0 = nullptr;
    const float* mma_t0safe = nullptr;  // wide pass: the sample's guaranteed start thresholds
    const unsigned int* mma_dropped = nullptr;
    sair_select_stats last{};
};

// --------------------------------------------------------------- frontier --
struct sair_frontier_s {
    int device = 0;
    cudaStream_t st = nullptr;
    double l_max = 1.0, c_max = 1.0;
    size_t F = 0, cap = 0;
    double* fl = nullptr;  // [cap] latency asc
    double* fc = nullptr;  // [cap] cost (strictly desc)
    double hv = 0.0;       // hypervolume() of the current points (host copy)
    std::vector<double> hl, hc;  // host mirror for points()
    sair::DBuf b_tmp, b_in, b_out, b_sort;
    sair::HBuf h_io;
    cudaEvent_t ev_tail = nullptr;  // decision step: reward / frontier work done (pareto.cu)
};

// ----------------------------------------------------------- frontier set --
struct sair_frontier_set_s {
    int device = 0;
    cudaStream_t st = nullptr;
    size_t P = 0, cap = 0, maxf = 0;
    double l_max = 1.0, c_max = 1.0;
    double* fl = nullptr;  // [P][cap]
    double* fc = nullptr;
    size_t* fn = nullptr;  // [P]
    double* hv = nullptr;  // [P]
    sair::DBuf b_in;
};

// ------------------------------------------------- multi-GPU (sharded.cpp) --
struct sair_comm_s {
    std::vector<int> dev;
    std::vector<cudaStream_t> st;
    std::vector<void*> nc;  // ncclComm_t per device (NCCL transport), or empty (copies)
};

struct sair_sharded_s {
    sair_comm_s* comm = nullptr;
    std::vector<sair_store_s*> sh;
    std::vector<size_t> lo;   // global index of each shard's first record
    size_t quota = 0, n = 0;
    uint64_t rejected = 0;
    double r_min = 0.0;
    int d = 0;
    // the buffer-level sigma cache (experience.hpp:87-88) and what the
    // shards' global statistics were last set to
    double cached_sigma = 0.0;
    // the buffer's running sums, accumulated in insertion order on the host
    // (experience.cpp:55-58, :138-139): bit-identical to one buffer's, not a
    // shard-order recombination
    sair::StoreStats gst;
    size_t stale = 0, synced_n = (size_t)-1;
    double synced_sigma = -1.0;
    std::vector<sair::DBuf> b_pack;  // per device: own pack | gathered packs | merged
};

namespace sair {

// statistics the reference's formulas see: the whole buffer's (experience.cpp:68-75, :229-231)
inline const StoreStats& eff_stats(const sair_store_s* s) { return s->sharded ? s->gst : s->stats; }
inline uint64_t eff_n(const sair_store_s* s) { return s->sharded ? s->n_global : s->n; }

// store.cu
void store_init(sair_store_s* s, double r_min, int device, size_t capacity_hint);
void store_free(sair_store_s* s);
void store_clone(const sair_store_s* s, sair_store_s* out);
void store_reserve(sair_store_s* s, size_t need);
size_t store_append(sair_store_s* s, const double* ctx, size_t count, int dim,
                    const double* reward, const int32_t* round, uint8_t* accepted);
void store_append_synthetic(sair_store_s* s, uint64_t seed, size_t count, int dim, int clustered);
// decision step (pareto.cu): the host half of store() for the row its tail
// kernel wrote behind the device-side gate -- the same gate, the host sums
bool store_append_one_commit(sair_store_s* s, const double* x, double reward);
void store_standardize(const sair_store_s* s, const double* x, double* z);
double store_effective_sigma(sair_store_s* s, double sigma_sim);
void store_mean_sd(const sair_store_s* s, double* mean, double* sd);
std::vector<int64_t> sigma_sample(uint64_t n);
double sigma_rows(const double* rows, size_t m, int d, const double* mean, const double* sd,
                  int device);

// select.cu
void store_select(sair_store_s* s, const double* q, size_t nq, int dim,
                  const sair_select_config& cfg, int64_t* out_idx, double* out_sim,
                  double* out_score, size_t* out_count, int64_t* out_nn, double* out_nn_sim,
                  double* out_reward = nullptr, int32_t* out_round = nullptr);
void merge_topk(const double* score, const double* sim, const double* reward,
                const int32_t* round, const int64_t* gidx, const size_t* count, size_t nshards,
                size_t nq, size_t m, int device, int64_t* out_idx, double* out_sim,
                double* out_score, size_t* out_count);
void merge_packed(const double* parts, size_t nshards, size_t nq, size_t m, int device,
                  cudaStream_t st, double* out);
double store_surprisal(sair_store_s* s, size_t index, const double* x,
                       const sair_select_config& cfg);

// pareto.cu
enum { Q_DOMINATED = 0, Q_CONTRIB = 1, Q_DISTANCE = 2, Q_REWARD = 3, Q_HV = 4 };
void frontier_init(sair_frontier_s* f, double l_max, double c_max, int device);
void frontier_free(sair_frontier_s* f);
void frontier_clone(const sair_frontier_s* f, sair_frontier_s* o);
bool frontier_insert_one(sair_frontier_s* f, double pl, double pc);
// one decision step: select + veto, reward, frontier update, store, one sync
void decision_step(sair_store_s* s, sair_frontier_s* f, const double* x, int dim,
                   const sair_select_config& cfg, const sair_reward_inputs* in,
                   const int32_t* deltas, size_t S, const sair_reward_config* rcfg, bool update,
                   double pl, double pc, int32_t round, int64_t* o_idx, double* o_sim,
                   double* o_score, size_t* o_count, int64_t* o_nn, double* o_nn_sim,
                   sair_reward_breakdown* o_rw, int* o_inserted, int* o_stored);
size_t frontier_insert_batch(sair_frontier_s* f, const double* pts, size_t T);
double frontier_point_query(sair_frontier_s* f, double pl, double pc, int op, double* aux);
void frontier_score_batch(sair_frontier_s* f, const double* pts, size_t T, double* out,
                          uint8_t* dom);
void frontier_score_batch_device(sair_frontier_s* f, const double* dpts, size_t T, double* dout,
                                 uint8_t* ddom, cudaStream_t st);
void dominance_counts(const double* tuples, size_t T, int K, int device, uint32_t* counts,
                      uint8_t* member, int part = 0, int nparts = 1);
void compute_reward_batch(const sair_reward_inputs* in, const int32_t* deltas, size_t S, size_t T,
                          sair_frontier_s* f, const sair_reward_config* cfg,
                          sair_reward_breakdown* out);
void compute_reward_replay(const sair_reward_inputs* in, const int32_t* deltas, size_t S,
                           size_t T, const uint8_t* update, sair_frontier_s* f,
                           const sair_reward_config* cfg, sair_reward_breakdown* out);
double action_magnitude(const int32_t* deltas, size_t S, int device);
void frontier_set_init(sair_frontier_set_s* s, size_t P, double l_max, double c_max, int device);
void frontier_set_free(sair_frontier_set_s* s);
void frontier_set_step(sair_frontier_set_s* s, const sair_reward_inputs* in, const int32_t* deltas,
                       size_t S, const uint8_t* update, const sair_reward_config* cfg,
                       sair_reward_breakdown* out);
size_t frontier_set_points(sair_frontier_set_s* s, size_t p, double* l, double* c, size_t cap,
                           double* hv);

// sharded.cpp: one buffer / frontier over the GPUs of this process
void comm_create(const int* devices, int n, sair_comm_s* c);
void comm_free(sair_comm_s* c);
void sharded_init(sair_sharded_s* h, sair_comm_s* c, double r_min, size_t capacity);
void sharded_free(sair_sharded_s* h);
size_t sharded_append(sair_sharded_s* h, const double* ctx, size_t count, int dim,
                      const double* reward, const int32_t* round, uint8_t* accepted);
void sharded_append_synthetic(sair_sharded_s* h, uint64_t seed, size_t count, int dim,
                              int clustered);
double sharded_effective_sigma(sair_sharded_s* h, double sigma_sim);
void sharded_select(sair_sharded_s* h, const double* q, size_t nq, int dim,
                    const sair_select_config& cfg, int64_t* out_idx, double* out_sim,
                    double* out_score, size_t* out_count);
size_t frontier_insert_batch_sharded(sair_comm_s* c, sair_frontier_s* f, const double* pts,
                                     size_t T);

// select_greedy.cu: a shard's side of the distributed exact greedy
void greedy_begin(sair_store_s* s, const double* q, size_t nq, int dim,
                  const sair_select_config& cfg, double* out);
void greedy_next(sair_store_s* s, const int64_t* gpick, const double* rows, double* out);

}  // namespace sair
