// scalelab_b200.cpp -- the reference's retrieval / Pareto / reward classes on
// the libsair C ABI (include/sair.h).  Every number comes from the device; the
// host holds only what the reference's callers hold (Experience records for
// all(), the frontier's points for points()) and does the JSONL I/O.
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <string>
#include <utility>

#include "json.hpp"
#include "scalelab_b200/experience.hpp"
#include "scalelab_b200/pareto.hpp"
#include "scalelab_b200/reward.hpp"

namespace scalelab {
namespace {

// status -> the exception type the reference throws for it
void check(sair_status st) {
    if (st == SAIR_OK) return;
    std::string msg = sair_last_error();
    switch (st) {
        case SAIR_EINVAL: throw std::invalid_argument(msg);
        case SAIR_ERANGE: throw std::out_of_range(msg);
        case SAIR_ELOGIC: throw std::logic_error(msg);
        default: throw std::runtime_error("libsair: " + msg);
    }
}

sair_select_config to_c(const SelectionConfig& c) {
    sair_select_config s{};
    s.m = c.m;
    s.lambda_div = c.lambda_div;
    s.sigma_sim = c.sigma_sim;
    s.locally_weighted_mean = c.locally_weighted_mean ? 1 : 0;
    s.mode = SAIR_SELECT_AUTO;
    return s;
}

std::vector<int32_t> deltas_of(const ScalingAction& a) {
    std::vector<int32_t> d;
    d.reserve(a.stages.size() * 4);
    for (const auto& s : a.stages) {
        d.push_back(s.replicas);
        d.push_back(s.cpu_millicores);
        d.push_back(s.memory_mb);
        d.push_back(s.rate_ratio_tenths);
    }
    return d;
}

}  // namespace

// ------------------------------------------------------------- retrieval --

std::vector<double> context_features(const PipelineState& state) {
    // experience.cpp:13-28: host flattening of the query (the query producer)
    std::vector<double> x;
    x.reserve(state.stages.size() * 7 + 2);
    for (const auto& st : state.stages) {
        x.insert(x.end(), {static_cast<double>(st.config.replicas),
                           static_cast<double>(st.config.cpu_millicores),
                           static_cast<double>(st.config.memory_mb), st.config.rate_ratio,
                           st.queue_depth, st.u_cpu, st.u_gpu_quota});
    }
    x.push_back(state.latency_p99_ms);
    x.push_back(state.throughput_rps);
    return x;
}

double similarity(const std::vector<double>& a, const std::vector<double>& b, double sigma) {
    double v = 0.0;
    check(sair_similarity(a.data(), a.size(), b.data(), b.size(), sigma, &v));
    return v;
}

ExperienceBuffer::ExperienceBuffer(double r_min) : r_min_(r_min) {
    check(sair_store_create(r_min, 0, 0, &h_));
    open_shards();
}

ExperienceBuffer::ExperienceBuffer(const ExperienceBuffer& o) : r_min_(o.r_min_), items_(o.items_) {
    check(sair_store_clone(o.h_, &h_));
    open_shards();
    if (sh_) {  // the copy's shards: the same records in the same order
        for (const auto& e : items_) {
            const int32_t rd = e.round;
            mirror_append(e.context.data(), 1, static_cast<int>(e.context.size()), &e.reward, &rd);
        }
    }
}

ExperienceBuffer::ExperienceBuffer(ExperienceBuffer&& o) noexcept
    : h_(std::exchange(o.h_, nullptr)), comm_(std::exchange(o.comm_, nullptr)),
      sh_(std::exchange(o.sh_, nullptr)), r_min_(o.r_min_), items_(std::move(o.items_)) {}

void ExperienceBuffer::open_shards() {
    const char* e = std::getenv("SAIR_DEVICES");
    if (!e || !*e) return;
    std::vector<int> dev;
    for (const char* p = e; *p;) {
        char* end = nullptr;
        const long v = std::strtol(p, &end, 10);
        if (end == p) throw std::invalid_argument("SAIR_DEVICES: a comma-separated device list");
        dev.push_back(static_cast<int>(v));
        p = *end == ',' ? end + 1 : end;
    }
    if (dev.size() < 2) return;
    const char* cap = std::getenv("SAIR_SHARD_CAPACITY");
    check(sair_comm_create(dev.data(), static_cast<int>(dev.size()), &comm_));
    check(sair_sharded_create(comm_, r_min_, cap ? std::strtoull(cap, nullptr, 10) : (1u << 24),
                              &sh_));
}

void ExperienceBuffer::close_shards() {
    sair_sharded_destroy(sh_);
    sair_comm_destroy(comm_);
    sh_ = nullptr;
    comm_ = nullptr;
}

void ExperienceBuffer::mirror_append(const double* ctx, std::size_t count, int dim,
                                     const double* reward, const std::int32_t* round) {
    if (sh_) check(sair_sharded_append(sh_, ctx, count, dim, reward, round, nullptr, nullptr));
}

int ExperienceBuffer::select_devices() const {
    int n = 1;
    if (comm_) sair_comm_info(comm_, &n, nullptr);
    return n;
}

ExperienceBuffer& ExperienceBuffer::operator=(const ExperienceBuffer& o) {
    if (this != &o) {
        ExperienceBuffer tmp(o);
        *this = std::move(tmp);
    }
    return *this;
}

ExperienceBuffer& ExperienceBuffer::operator=(ExperienceBuffer&& o) noexcept {
    if (this != &o) {
        sair_store_destroy(h_);
        close_shards();
        h_ = std::exchange(o.h_, nullptr);
        comm_ = std::exchange(o.comm_, nullptr);
        sh_ = std::exchange(o.sh_, nullptr);
        r_min_ = o.r_min_;
        items_ = std::move(o.items_);
    }
    return *this;
}

ExperienceBuffer::~ExperienceBuffer() {
    sair_store_destroy(h_);
    close_shards();
}

bool ExperienceBuffer::store(Experience e) {
    uint8_t acc = 0;
    const int32_t round = e.round;
    check(sair_store_append(h_, e.context.data(), 1, static_cast<int>(e.context.size()),
                            &e.reward, &round, &acc, nullptr));
    if (acc) {
        mirror_append(e.context.data(), 1, static_cast<int>(e.context.size()), &e.reward, &round);
        items_.push_back(std::move(e));
    }
    return acc != 0;
}

std::uint64_t ExperienceBuffer::rejected() const {
    uint64_t r = 0;
    check(sair_store_rejected(h_, &r));
    return r;
}

std::vector<double> ExperienceBuffer::standardize(const std::vector<double>& x) const {
    std::vector<double> z(x.size());
    check(sair_store_standardize(h_, x.data(), static_cast<int>(x.size()), z.data()));
    return z;
}

double ExperienceBuffer::effective_sigma(const SelectionConfig& cfg) const {
    double s = 0.0;
    check(sair_store_effective_sigma(h_, cfg.sigma_sim, &s));
    return s;
}

double ExperienceBuffer::surprisal(std::size_t index, const std::vector<double>& x_curr,
                                   const SelectionConfig& cfg) const {
    const sair_select_config c = to_c(cfg);
    double v = 0.0;
    check(sair_store_surprisal(h_, index, x_curr.data(), static_cast<int>(x_curr.size()), &c,
                               &v));
    return v;
}

std::vector<std::vector<SelectedExperience>> ExperienceBuffer::select_batch(
    const std::vector<std::vector<double>>& queries, const SelectionConfig& cfg,
    std::vector<std::int64_t>* nearest, std::vector<double>* nearest_sim) const {
    if ((nearest == nullptr) != (nearest_sim == nullptr))
        throw std::invalid_argument("select_batch: nearest and nearest_sim come in pairs");
    const std::size_t nq = queries.size();
    std::vector<std::vector<SelectedExperience>> out(nq);
    if (nq == 0) return out;
    const int d = static_cast<int>(queries[0].size());
    std::vector<double> q;
    q.reserve(nq * d);
    for (const auto& x : queries) {
        if (static_cast<int>(x.size()) != d)
            throw std::invalid_argument("experience store: feature dimension mismatch");
        q.insert(q.end(), x.begin(), x.end());
    }
    const std::size_t m = cfg.m ? cfg.m : 1;
    std::vector<int64_t> idx(nq * m);
    std::vector<double> sim(nq * m), score(nq * m);
    std::vector<size_t> cnt(nq);
    if (nearest) nearest->assign(nq, -1);
    if (nearest_sim) nearest_sim->assign(nq, -1.0);
    const sair_select_config c = to_c(cfg);
    if (sh_) {
        // over the GPUs of SAIR_DEVICES; the veto scan on the primary store
        check(sair_store_select_sharded(sh_, q.data(), nq, d, &c, idx.data(), sim.data(),
                                        score.data(), cnt.data()));
        if (nearest)
            check(sair_store_nearest(h_, q.data(), nq, d, cfg.sigma_sim, nearest->data(),
                                     nearest_sim->data()));
    } else {
        check(sair_store_select(h_, q.data(), nq, d, &c, idx.data(), sim.data(), score.data(),
                                cnt.data(), nearest ? nearest->data() : nullptr,
                                nearest_sim ? nearest_sim->data() : nullptr));
    }
    for (std::size_t i = 0; i < nq; ++i)
        for (std::size_t j = 0; j < cnt[i]; ++j)
            out[i].push_back({items_.at(static_cast<std::size_t>(idx[i * m + j])),
                              sim[i * m + j], score[i * m + j]});
    return out;
}

std::vector<SelectedExperience> ExperienceBuffer::select(const std::vector<double>& x_curr,
                                                         const SelectionConfig& cfg) const {
    if (items_.empty() || cfg.m == 0) return {};  // experience.cpp:154
    return std::move(select_batch({x_curr}, cfg)[0]);
}

// ---- persistence: the reference's JSONL format (experience.cpp:207-271) --

void ExperienceBuffer::persist(const std::string& path) const {
    std::ofstream out(path, std::ios::trunc);
    if (!out) throw std::runtime_error("experience store: cannot write " + path);
    for (const auto& e : items_) {
        nlohmann::json act = nlohmann::json::array();
        for (const auto& s : e.action.stages)
            act.push_back({{"replicas", s.replicas},
                           {"cpu_millicores", s.cpu_millicores},
                           {"memory_mb", s.memory_mb},
                           {"rate_ratio_tenths", s.rate_ratio_tenths}});
        nlohmann::json j{{"round", e.round}, {"source", e.source}, {"reward", e.reward},
                         {"context", e.context}, {"action", act}};
        out << j.dump() << '\n';
    }
}

ExperienceBuffer ExperienceBuffer::load(const std::string& path, double r_min,
                                        std::size_t* corrupt_lines) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("experience store: cannot read " + path);
    ExperienceBuffer buf(r_min);
    std::size_t bad = 0;
    std::string line;
    std::vector<Experience> rows;
    while (std::getline(in, line)) {
        if (line.empty()) continue;
        try {
            nlohmann::json j = nlohmann::json::parse(line);
            Experience e;
            e.round = j.at("round").get<int>();
            e.source = j.at("source").get<std::string>();
            e.reward = j.at("reward").get<double>();
            e.context = j.at("context").get<std::vector<double>>();
            for (const auto& s : j.at("action")) {
                StageDelta d;
                d.replicas = s.at("replicas").get<int>();
                d.cpu_millicores = s.at("cpu_millicores").get<int>();
                d.memory_mb = s.at("memory_mb").get<int>();
                d.rate_ratio_tenths = s.at("rate_ratio_tenths").get<int>();
                e.action.stages.push_back(d);
            }
            rows.push_back(std::move(e));
        } catch (const nlohmann::json::exception&) {
            ++bad;
        }
    }
    // store() of every parsed row in line order as ONE device append: the gate
    // and the dimension rule are applied here first (a change throws, as the
    // reference's store() inside load() does), rejected rows keep their place
    int dim = -1;
    for (const auto& e : rows) {
        if (!(e.reward > r_min)) continue;
        if (dim < 0) dim = static_cast<int>(e.context.size());
        else if (static_cast<int>(e.context.size()) != dim)
            throw std::invalid_argument("experience store: context dimension changed");
    }
    if (!rows.empty() && dim != 0) {
        const int d = dim > 0 ? dim : 1;
        std::vector<double> ctx(rows.size() * static_cast<std::size_t>(d), 0.0), rew(rows.size());
        std::vector<int32_t> rnd(rows.size());
        std::vector<uint8_t> acc(rows.size(), 0);
        for (std::size_t i = 0; i < rows.size(); ++i) {
            rew[i] = rows[i].reward;
            rnd[i] = rows[i].round;
            if (rows[i].reward > r_min)
                std::copy(rows[i].context.begin(), rows[i].context.end(), ctx.begin() + i * d);
        }
        check(sair_store_append(buf.h_, ctx.data(), rows.size(), d, rew.data(), rnd.data(),
                                acc.data(), nullptr));
        buf.mirror_append(ctx.data(), rows.size(), d, rew.data(), rnd.data());
        for (std::size_t i = 0; i < rows.size(); ++i)
            if (acc[i]) buf.items_.push_back(std::move(rows[i]));
    } else {
        for (auto& e : rows) buf.store(std::move(e));  // empty contexts: one at a time
    }
    if (corrupt_lines) *corrupt_lines = bad;
    return buf;
}

// ---------------------------------------------------------------- pareto --

bool dominates(const ObjectivePoint& p, const ObjectivePoint& q) {
    const double t[4] = {q.latency, q.cost, p.latency, p.cost};  // tuple 1 = p
    uint32_t cnt[2] = {0, 0};
    check(sair_dominance_counts(t, 2, 2, 0, cnt, nullptr));
    return cnt[0] > 0;  // p dominates q
}

ParetoFrontier::ParetoFrontier(double latency_max_ms, double cost_max)
    : l_max_(latency_max_ms), c_max_(cost_max) {
    check(sair_frontier_create(latency_max_ms, cost_max, 0, &h_));
}

ParetoFrontier::ParetoFrontier(const ParetoFrontier& o)
    : l_max_(o.l_max_), c_max_(o.c_max_), mirror_(o.mirror_) {
    check(sair_frontier_clone(o.h_, &h_));
}

ParetoFrontier::ParetoFrontier(ParetoFrontier&& o) noexcept
    : h_(std::exchange(o.h_, nullptr)), l_max_(o.l_max_), c_max_(o.c_max_),
      mirror_(std::move(o.mirror_)) {}

ParetoFrontier& ParetoFrontier::operator=(const ParetoFrontier& o) {
    if (this != &o) {
        ParetoFrontier tmp(o);
        *this = std::move(tmp);
    }
    return *this;
}

ParetoFrontier& ParetoFrontier::operator=(ParetoFrontier&& o) noexcept {
    if (this != &o) {
        sair_frontier_destroy(h_);
        h_ = std::exchange(o.h_, nullptr);
        l_max_ = o.l_max_;
        c_max_ = o.c_max_;
        mirror_ = std::move(o.mirror_);
    }
    return *this;
}

ParetoFrontier::~ParetoFrontier() { sair_frontier_destroy(h_); }

void ParetoFrontier::refresh() {
    size_t F = 0;
    check(sair_frontier_size(h_, &F));
    std::vector<double> l(F), c(F);
    check(sair_frontier_points(h_, l.data(), c.data(), F, &F));
    mirror_.resize(F);
    for (size_t i = 0; i < F; ++i) mirror_[i] = {l[i], c[i]};
}

ParetoFrontier::UpdateResult ParetoFrontier::update(double latency_ms, double cost) {
    int ins = 0, cl = 0;
    check(sair_frontier_update(h_, latency_ms, cost, &ins, &cl));
    if (ins) refresh();
    return {ins != 0, cl != 0};
}

ObjectivePoint ParetoFrontier::normalize(double latency_ms, double cost, bool* clamped) const {
    ObjectivePoint p;
    int cl = 0;
    check(sair_frontier_normalize(h_, latency_ms, cost, &p.latency, &p.cost, &cl));
    if (clamped) *clamped = cl != 0;
    return p;
}

bool ParetoFrontier::strictly_dominated(const ObjectivePoint& p) const {
    int v = 0;
    check(sair_frontier_strictly_dominated(h_, p.latency, p.cost, &v));
    return v != 0;
}

double ParetoFrontier::hypervolume() const {
    double v = 0.0;
    check(sair_frontier_hypervolume(h_, &v));
    return v;
}

double ParetoFrontier::contribution(const ObjectivePoint& p) const {
    double v = 0.0;
    check(sair_frontier_contribution(h_, p.latency, p.cost, &v));
    return v;
}

std::optional<double> ParetoFrontier::distance(const ObjectivePoint& p) const {
    double v = 0.0;
    int has = 0;
    check(sair_frontier_distance(h_, p.latency, p.cost, &v, &has));
    if (!has) return std::nullopt;
    return v;
}

double ParetoFrontier::reward(const ObjectivePoint& p) const {
    double v = 0.0;
    check(sair_frontier_reward(h_, p.latency, p.cost, &v));
    return v;
}

bool ParetoFrontier::insert_normalized(const ObjectivePoint& p) {
    int ins = 0;
    check(sair_frontier_insert_normalized(h_, p.latency, p.cost, &ins));
    if (ins) refresh();
    return ins != 0;
}

std::size_t ParetoFrontier::insert_batch(const std::vector<ObjectivePoint>& pts) {
    std::vector<double> flat;
    flat.reserve(pts.size() * 2);
    for (const auto& p : pts) flat.insert(flat.end(), {p.latency, p.cost});
    size_t F = 0;
    check(sair_frontier_insert_batch(h_, flat.data(), pts.size(), &F));
    refresh();
    return F;
}

std::vector<double> ParetoFrontier::reward_batch(const std::vector<ObjectivePoint>& pts) const {
    std::vector<double> flat, out(pts.size());
    flat.reserve(pts.size() * 2);
    for (const auto& p : pts) flat.insert(flat.end(), {p.latency, p.cost});
    check(sair_frontier_score_batch(h_, flat.data(), pts.size(), out.data(), nullptr));
    return out;
}

// ---------------------------------------------------------------- reward --

double action_magnitude(const ScalingAction& action) {
    const auto d = deltas_of(action);
    double v = 0.0;
    check(sair_action_magnitude(d.data(), action.stages.size(), &v));
    return v;
}

RewardBreakdown compute_reward(const RewardInputs& in, const ScalingAction& action,
                               const ParetoFrontier& frontier, const RewardConfig& cfg) {
    const sair_reward_inputs ri{in.l_before_ms, in.l_after_ms, in.c_before, in.c_after};
    const sair_reward_config rc{cfg.t_sla_ms, cfg.l_baseline_ms, cfg.c_budget, cfg.w_latency,
                                cfg.w_cost, cfg.w_proactive, cfg.r_max};
    const auto d = deltas_of(action);
    sair_reward_breakdown out{};
    check(sair_compute_reward(&ri, d.data(), action.stages.size(), frontier.handle(), &rc, &out));
    return {out.latency, out.cost, out.sla, out.proactive, out.pareto, out.total,
            out.clipped != 0};
}

}  // namespace scalelab
