// scalelab_b200/experience.hpp -- ExperienceBuffer on the device (libsair).
//
// Source-compatible with the reference interface (proj/include/scalelab/
// experience.hpp:10-91).  The buffer's numbers live in a device-resident SoA
// store; the host keeps the Experience records themselves (all() returns
// them, as callers such as the policy's prompt builder need the actions).
// ScalingAction and PipelineState come from the reference's own foundation
// headers (scalelab/action.hpp, scalelab/types.hpp).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "sair.h"
#include "scalelab/action.hpp"
#include "scalelab/types.hpp"

namespace scalelab {

// [replicas, cpu_mc, mem_mb, rate_ratio, queue, u_cpu, u_gpu] per stage, then [p99, rps]
std::vector<double> context_features(const PipelineState& state);

// Gaussian kernel on standardized vectors; std::invalid_argument on length
// mismatch or sigma <= 0
double similarity(const std::vector<double>& a, const std::vector<double>& b, double sigma);

struct Experience {
    std::vector<double> context;
    ScalingAction action;
    double reward = 0.0;
    int round = 0;
    std::string source = "llm";
};

struct SelectionConfig {
    std::size_t m = 15;
    double lambda_div = 0.1;
    double sigma_sim = 0.0;
    bool locally_weighted_mean = false;
};

struct SelectedExperience {
    Experience experience;
    double similarity_to_current = 0.0;
    double score = 0.0;
};

class ExperienceBuffer {
public:
    explicit ExperienceBuffer(double r_min = 0.0);
    ExperienceBuffer(const ExperienceBuffer& other);
    ExperienceBuffer(ExperienceBuffer&& other) noexcept;
    ExperienceBuffer& operator=(const ExperienceBuffer& other);
    ExperienceBuffer& operator=(ExperienceBuffer&& other) noexcept;
    ~ExperienceBuffer();

    bool store(Experience e);
    std::size_t size() const { return items_.size(); }
    bool empty() const { return items_.empty(); }
    std::uint64_t rejected() const;
    double r_min() const { return r_min_; }
    const std::vector<Experience>& all() const { return items_; }

    std::vector<double> standardize(const std::vector<double>& x) const;
    double effective_sigma(const SelectionConfig& cfg) const;
    double surprisal(std::size_t index, const std::vector<double>& x_curr,
                     const SelectionConfig& cfg) const;
    std::vector<SelectedExperience> select(const std::vector<double>& x_curr,
                                           const SelectionConfig& cfg) const;

    void persist(const std::string& path) const;
    static ExperienceBuffer load(const std::string& path, double r_min,
                                 std::size_t* corrupt_lines = nullptr);

    // this library: one device pass for a batch of queries (+ the veto scan)
    std::vector<std::vector<SelectedExperience>> select_batch(
        const std::vector<std::vector<double>>& queries, const SelectionConfig& cfg,
        std::vector<std::int64_t>* nearest = nullptr,
        std::vector<double>* nearest_sim = nullptr) const;
    sair_store_t handle() const { return h_; }
    // GPUs select() runs on (SAIR_DEVICES=0,1,...: >= 2 entries shard the
    // buffer over them; 1 otherwise)
    int select_devices() const;

private:
    void open_shards();        // SAIR_DEVICES -> comm_ / sh_
    void close_shards();
    void mirror_append(const double* ctx, std::size_t count, int dim, const double* reward,
                       const std::int32_t* round);
    sair_store_t h_ = nullptr;
    // multi-GPU select: the records also live in a sharded store over the
    // listed GPUs (sair_store_select_sharded); the other members use h_
    sair_comm_t comm_ = nullptr;
    sair_sharded_t sh_ = nullptr;
    double r_min_ = 0.0;
    std::vector<Experience> items_;
};

}  // namespace scalelab
