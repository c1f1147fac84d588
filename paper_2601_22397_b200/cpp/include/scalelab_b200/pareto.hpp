// scalelab_b200/pareto.hpp -- ParetoFrontier on the device (libsair).
//
// Source-compatible with the reference interface (proj/include/scalelab/
// pareto.hpp:6-72): every public name, signature and exception is the
// reference's; the private state is a device handle plus the host mirror that
// points() returns.  Drop-in builds reach this header through
// compat/scalelab/pareto.hpp.
#pragma once

#include <cstddef>
#include <optional>
#include <vector>

#include "sair.h"

// marks the drop-in (its batch extensions exist)
#define SCALELAB_B200_EXT 1

namespace scalelab {

// normalized (latency, cost), smaller is better on both axes
struct ObjectivePoint {
    double latency = 0.0;
    double cost = 0.0;
    friend bool operator==(const ObjectivePoint&, const ObjectivePoint&) = default;
};

// p is at least as good as q everywhere and strictly better somewhere
bool dominates(const ObjectivePoint& p, const ObjectivePoint& q);

class ParetoFrontier {
public:
    ParetoFrontier(double latency_max_ms, double cost_max);
    ParetoFrontier(const ParetoFrontier& other);
    ParetoFrontier(ParetoFrontier&& other) noexcept;
    ParetoFrontier& operator=(const ParetoFrontier& other);
    ParetoFrontier& operator=(ParetoFrontier&& other) noexcept;
    ~ParetoFrontier();

    struct UpdateResult {
        bool inserted = false;
        bool clamped = false;
    };

    UpdateResult update(double latency_ms, double cost);
    ObjectivePoint normalize(double latency_ms, double cost, bool* clamped = nullptr) const;
    bool strictly_dominated(const ObjectivePoint& p) const;
    double hypervolume() const;
    double contribution(const ObjectivePoint& p) const;  // std::logic_error if dominated
    std::optional<double> distance(const ObjectivePoint& p) const;
    double reward(const ObjectivePoint& p) const;
    bool insert_normalized(const ObjectivePoint& p);

    const std::vector<ObjectivePoint>& points() const { return mirror_; }
    bool empty() const { return mirror_.empty(); }
    std::size_t size() const { return mirror_.size(); }
    double latency_max_ms() const { return l_max_; }
    double cost_max() const { return c_max_; }

    // this library: batch forms of the same operations
    std::size_t insert_batch(const std::vector<ObjectivePoint>& pts);
    std::vector<double> reward_batch(const std::vector<ObjectivePoint>& pts) const;
    sair_frontier_t handle() const { return h_; }

private:
    void refresh();
    sair_frontier_t h_ = nullptr;
    double l_max_ = 1.0, c_max_ = 1.0;
    std::vector<ObjectivePoint> mirror_;
};

}  // namespace scalelab
