// select_common.cuh -- pieces shared by the fast (select.cu) and exact
// (select_exact.cu) retrieval paths.
#pragma once

#include <vector>

#include "internal.hpp"

namespace sair {

// Greedy pick key, experience.cpp:177-187: gain desc, then round asc, then the
// first index scanned (index asc).  j < 0 marks "none".
struct Best {
    double g;
    int32_t r;
    int64_t i;
    int j;
};

__device__ __forceinline__ bool better(const Best& a, const Best& b) {
    if (a.j < 0) return false;
    if (b.j < 0) return true;
    if (a.g > b.g) return true;
    if (a.g < b.g) return false;
    if (a.r != b.r) return a.r < b.r;
    return a.i < b.i;
}

__device__ __forceinline__ Best warp_best(Best b) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        Best c;
        c.g = __shfl_xor_sync(0xffffffffu, b.g, o);
        c.r = __shfl_xor_sync(0xffffffffu, b.r, o);
        c.i = __shfl_xor_sync(0xffffffffu, b.i, o);
        c.j = __shfl_xor_sync(0xffffffffu, b.j, o);
        if (better(c, b)) b = c;
    }
    return b;
}

// Host-side per-call constants: the reference's standardize statistics and the
// standardized queries (experience.cpp:68-75), sigma and 2 sigma^2 (:130).
struct QueryPrep {
    std::vector<double> mean, sd, z;  // z: [nq][d]
    double sigma = 1.0, two_s2 = 2.0;
};

inline QueryPrep prep_queries(const sair_store_s* s, const double* q, size_t nq, double sigma) {
    QueryPrep p;
    const int d = s->d;
    p.mean.resize(d);
    p.sd.resize(d);
    store_mean_sd(s, p.mean.data(), p.sd.data());
    p.z.resize(nq * d);
    for (size_t i = 0; i < nq; ++i)
        for (int k = 0; k < d; ++k) p.z[i * d + k] = (q[i * d + k] - p.mean[k]) / p.sd[k];
    p.sigma = sigma;
    p.two_s2 = 2.0 * sigma * sigma;
    return p;
}

// Per query group: pinned staging for the launcher's constants and the
// events it records (end of the threshold pre-pass, end of the stream pass).
struct GroupIo {
    float* hstage;
    cudaEvent_t e_mid, e_end;
    const float* t0_override;  // wide pass: [2 QW] start thresholds (skip the sample pass)
    float* lists_key;          // wide pass: compacted CTA lists out, [grid][2 QW][kmax]
    uint32_t* lists_idx;
    const float* pl_in;        // wide pass: this call's per-record (P, lg) cache, or null
    float* pl_out;             // wide pass: fill the cache in this group's stream pass
    const uint32_t* hot;       // wide sample: extra pages (highest reward residual), or null
    uint32_t nhot;             // slots in `hot` (entries >= npages are empty)
    // wide pass, batched call: 0 = compute + upload + launch; 1 = only compute
    // this group's constants into hstage (and cc); 2 = only launch, the
    // constants already at dconsts (every group's went up in one copy) and
    // the list counters at dcnt [2 * 2 QW] already zeroed
    int phase;
    float* dconsts;
    uint32_t* dcnt;
    const float* pl16_in;  // bf16 wide pass: its own (P, lg) cache (bf16 records)
    float* pl16_out;
};

// select_mma.cu: the tcgen05 streaming kernel (plan + launcher)
struct MmaPlan {
    int dp, qb, kp, knn, kmax, nst, cap_sel, cap_nn, grid;
    size_t smem;
};
using MmaFillFn = void (*)(sair_store_s*, const MmaPlan&, const QueryPrep&, const double*, int,
                           float, float, float, float, float*, uint32_t*, unsigned int*,
                           std::vector<double>&, const GroupIo&);
MmaFillFn pick_mma_fill(int dp, int qb);
bool make_mma_plan(const sair_store_s* s, size_t nq, size_t m, double lambda, bool nn,
                   MmaPlan* pl);

// select_wide.cu: the tcgen05 large-batch streaming filter (QW = 32/64/128
// queries per pass) -> merged per-query top-K' lists for the refine kernel
struct WidePlan {
    int dp, qw, kp, knn, kmax, nst, ntm, grid;
    size_t smem;
    int cg, nst2;  // stream passes: CTAs per MMA group (2 = CTA pairs) and their page stages
    size_t smem2;
    int bf16, nst16;  // 256-query stream passes on the bf16 page copy (select_wide.cu)
    size_t smem16;
    uint32_t cap, spages;
};
using WideFn = void (*)(sair_store_s*, const WidePlan&, const QueryPrep&, const double*, int, float,
                        float, float, float, float*, uint32_t*, float*, unsigned int*,
                        std::vector<double>&, const GroupIo&);
WideFn pick_wide(int dp, int qw);
// the wide sample's highest-residual pages of this call (nhot slots, empty
// ones >= npages), or null
const uint32_t* wide_hot_pages(sair_store_s* s, const WidePlan& pl, float c1, float c0,
                               uint32_t* nhot);
// select_greedy32.cu: lambda != 0 over a large store, fp32-filtered steps
// decided in fp64 (false: not applicable -- d > 64 or m > 256); queries whose
// candidate set overflowed are appended to `fallback` (the fp64 greedy's)
bool greedy32_select(sair_store_s* s, const QueryPrep& p, const std::vector<size_t>& qidx,
                     size_t m, double lambda, const double* loo, bool want_nn, int64_t* out_idx,
                     double* out_sim, double* out_score, size_t* out_count, int64_t* out_nn,
                     double* out_nn_sim, double* out_reward, int32_t* out_round,
                     std::vector<size_t>* fallback);
double wide_bq_rel(const WidePlan& pl);   // relative error bound of the wide pass's query operand
double wide_rec_rel(const WidePlan& pl);  // relative error bound of its stored records
void ensure_pages16(sair_store_s* s);     // the bf16 page copy covers every record
bool make_wide_plan(const sair_store_s* s, size_t nq, size_t m, double lambda, bool nn,
                    WidePlan* pl);

// select_small.cu: exact select() of small stores (<= 64k records), one
// clustered launch for all given queries
constexpr size_t SMALL_DIRECT_N = 4096;  // lambda == 0: below this, skip the filter
bool small_select_fits(const sair_store_s* s, size_t m);
void small_select(sair_store_s* s, const QueryPrep& p, const std::vector<size_t>& qidx, size_t m,
                  double lambda, bool local, bool want_nn, int64_t* out_idx, double* out_sim,
                  double* out_score, size_t* out_count, int64_t* out_nn, double* out_nn_sim,
                  double* out_reward, int32_t* out_round);

// select.cu: global top-K' of every list across per-CTA lists [G][lists][kmax]
void launch_merge(cudaStream_t st, const float* ck, const uint32_t* ci, int G, int lists, int kmax,
                  int qb, int kp, int knn, float* mk, uint32_t* mi, float* mthr, int kout = 0,
                  int ngroups = 1, size_t in_gstride = 0, size_t out_gstride = 0);

// standardize() of every stored row into z [d][n] (select_small.cu)
void zrows_launch(const double* x64, const double* mean, const double* sd, size_t n, int d,
                  double* z, cudaStream_t st);

// select_greedy.cu: exact select() of many queries over a large store, G
// queries per pass, every greedy step enqueued without a host round trip
void greedy_select(sair_store_s* s, const QueryPrep& p, const std::vector<size_t>& qidx, size_t m,
                   double lambda, const double* loo, bool want_nn, int64_t* out_idx,
                   double* out_sim, double* out_score, size_t* out_count, int64_t* out_nn,
                   double* out_nn_sim, double* out_reward, int32_t* out_round);

// select_exact.cu: one query through the full fp64 pass.
void exact_one(sair_store_s* s, const QueryPrep& p, const double* zq_host, size_t m,
               double lambda, bool local, int64_t* o_idx, double* o_sim, double* o_score,
               size_t* o_cnt, int64_t* o_nn, double* o_nn_sim, double* o_rew = nullptr,
               int32_t* o_round = nullptr, const double* loo_pre = nullptr);
// select_small.cu: the locally weighted LOO means of every record (exact,
// once per call) into a scratch buffer owned by the store
const double* local_loo_all(sair_store_s* s, const QueryPrep& p);

}  // namespace sair
