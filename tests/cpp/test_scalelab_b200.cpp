// The reference's unit and acceptance expectations for the hot path, run
// against the C++ drop-in (scalelab_b200 on libsair).  doctest is not in the
// image, so this is a small self-contained runner; every case cites the
// reference test it restates (paths relative to /root/reference/proj).
// Exit status = number of failed checks.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "scalelab_b200/experience.hpp"
#include "scalelab_b200/pareto.hpp"
#include "scalelab_b200/reward.hpp"

using namespace scalelab;

static int g_fail = 0, g_checks = 0;
#define EXPECT(cond)                                                              \
    do {                                                                          \
        ++g_checks;                                                               \
        if (!(cond)) {                                                            \
            ++g_fail;                                                             \
            std::printf("  FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);         \
        }                                                                         \
    } while (0)
#define EXPECT_THROW(stmt, exc)                                                   \
    do {                                                                          \
        bool hit = false;                                                         \
        try {                                                                     \
            stmt;                                                                 \
        } catch (const exc&) {                                                    \
            hit = true;                                                           \
        } catch (...) {                                                           \
        }                                                                         \
        EXPECT(hit);                                                              \
    } while (0)

static bool close_rel(double a, double b, double eps) {
    return std::abs(a - b) <= eps * std::max(1.0, std::abs(b));
}

static Experience exp_of(std::vector<double> ctx, double r, int round) {
    Experience e;
    e.context = std::move(ctx);
    e.reward = r;
    e.round = round;
    e.action = ScalingAction::noop(1);
    return e;
}

static double subset_value(const ExperienceBuffer& b, const std::vector<std::size_t>& s,
                           const std::vector<double>& x, const SelectionConfig& cfg) {
    // the greedy objective of test_experience.cpp:27-38 / acceptance_main.cpp:452-464
    const double sigma = b.effective_sigma(cfg);
    double v = 0.0;
    for (std::size_t i : s) v += b.surprisal(i, x, cfg);
    for (std::size_t a = 0; a < s.size(); ++a)
        for (std::size_t c = a + 1; c < s.size(); ++c)
            v -= cfg.lambda_div * similarity(b.standardize(b.all()[s[a]].context),
                                             b.standardize(b.all()[s[c]].context), sigma);
    return v;
}

// ---------------------------------------------------------- retrieval --

static void experience_tests() {
    // gate, tests/test_experience.cpp:42-56
    {
        ExperienceBuffer b(0.0);
        EXPECT(b.store(exp_of({1, 2}, 0.5, 0)));
        EXPECT(!b.store(exp_of({1, 2}, -0.2, 1)));
        EXPECT(!b.store(exp_of({1, 2}, 0.0, 2)));
        EXPECT(b.size() == 1 && b.rejected() == 2);
        ExperienceBuffer s(0.0);
        for (int i = 0; i < 100; ++i) s.store(exp_of({double(i), 0.0}, i % 10 < 3 ? -1.0 : 1.0, i));
        EXPECT(s.size() == 70 && s.rejected() == 30);
        EXPECT_THROW(s.store(exp_of({1.0}, 1.0, 200)), std::invalid_argument);
    }
    // kernel, :58-71
    {
        std::vector<double> a{0, 0}, c{std::sqrt(2.0), 0};
        EXPECT(similarity(a, a, 1.0) == 1.0);
        EXPECT(close_rel(similarity(a, c, 1.0), std::exp(-1.0), 1e-12));
        EXPECT_THROW(similarity(a, {1.0}, 1.0), std::invalid_argument);
        EXPECT_THROW(similarity(a, a, 0.0), std::invalid_argument);
        std::mt19937_64 g(5);
        std::uniform_real_distribution<double> u(-3, 3);
        for (int t = 0; t < 20; ++t) {
            std::vector<double> x{u(g), u(g), u(g)}, y{u(g), u(g), u(g)};
            EXPECT(similarity(x, y, 1.7) == similarity(y, x, 1.7));
        }
    }
    // surprisal, :73-93
    {
        SelectionConfig cfg;
        cfg.sigma_sim = 1e9;
        ExperienceBuffer b(-10.0);
        for (int i = 0; i < 3; ++i) b.store(exp_of({0.0}, 0.5, i));
        EXPECT(std::abs(b.surprisal(1, {0.0}, cfg)) <= 1e-9);
        ExperienceBuffer b2(-10.0);
        b2.store(exp_of({0.0}, 1.0, 0));
        b2.store(exp_of({0.0}, 0.4, 1));
        b2.store(exp_of({0.0}, 0.6, 2));
        EXPECT(close_rel(b2.surprisal(0, {0.0}, cfg), 0.5, 1e-9));
        ExperienceBuffer lone(-10.0);
        lone.store(exp_of({0.0}, 0.7, 0));
        EXPECT(close_rel(lone.surprisal(0, {0.0}, cfg), 0.7, 1e-9));
        EXPECT_THROW(lone.surprisal(3, {0.0}, cfg), std::out_of_range);
    }
    // leave-one-out vs naive, :95-117
    {
        std::mt19937_64 g(88);
        std::uniform_real_distribution<double> u(0, 1);
        SelectionConfig cfg;
        cfg.sigma_sim = 1.0;
        ExperienceBuffer b(0.0);
        std::vector<double> r;
        for (int i = 0; i < 40; ++i) {
            r.push_back(0.01 + u(g));
            b.store(exp_of({u(g), u(g)}, r.back(), i));
        }
        std::vector<double> x{0.5, 0.5};
        for (std::size_t i = 0; i < r.size(); ++i) {
            double tot = 0.0;
            for (std::size_t j = 0; j < r.size(); ++j)
                if (j != i) tot += r[j];
            double naive = std::abs(r[i] - tot / (r.size() - 1));
            double sim = similarity(b.standardize(b.all()[i].context), b.standardize(x), 1.0);
            EXPECT(close_rel(b.surprisal(i, x, cfg), sim * naive, 1e-9));
        }
    }
    // top-M without diversity, :119-145
    {
        SelectionConfig cfg;
        cfg.m = 3;
        cfg.lambda_div = 0.0;
        cfg.sigma_sim = 2.0;
        ExperienceBuffer b(0.0);
        const double rs[] = {0.9, 0.2, 1.4, 0.4, 0.6};
        for (int i = 0; i < 5; ++i) b.store(exp_of({0.5 * i, 0.1 * i}, rs[i], i));
        std::vector<double> x{0.4, 0.1};
        auto sel = b.select(x, cfg);
        EXPECT(sel.size() == 3);
        std::vector<std::pair<double, int>> sc;
        for (std::size_t i = 0; i < b.size(); ++i) sc.emplace_back(b.surprisal(i, x, cfg), b.all()[i].round);
        std::sort(sc.rbegin(), sc.rend());
        for (const auto& s : sel) {
            int hits = 0;
            for (int k = 0; k < 3; ++k) hits += sc[k].second == s.experience.round;
            EXPECT(hits == 1);
        }
        for (std::size_t i = 1; i < sel.size(); ++i)
            EXPECT(sel[i - 1].experience.reward <= sel[i].experience.reward);
    }
    // acceptance check 8 (acceptance_main.cpp:466-530): same draw sequence --
    // 200 buffers of 8..32 vs 100 random subsets, then 50 exhaustive C(8,3)
    {
        std::mt19937_64 g(90210);
        std::uniform_real_distribution<double> u(0, 1);
        SelectionConfig cfg;
        cfg.m = 3;
        cfg.lambda_div = 0.1;
        cfg.sigma_sim = 0.8;
        const std::vector<double> x{1.5, 1.5};
        auto fill = [&](ExperienceBuffer& b, int n) {
            for (int i = 0; i < n; ++i) {
                Experience e;
                e.context = {u(g) * 3.0, u(g) * 3.0};
                e.reward = 0.05 + u(g);
                e.round = i;
                e.action = ScalingAction::noop(1);
                b.store(std::move(e));
            }
        };
        // the objective from memoised device surprisals / similarities
        struct Memo {
            std::vector<double> sur;
            std::vector<std::vector<double>> sim;
        };
        auto memo = [&](const ExperienceBuffer& b) {
            Memo mm;
            const std::size_t n = b.size();
            const double sigma = b.effective_sigma(cfg);
            std::vector<std::vector<double>> z;
            for (std::size_t i = 0; i < n; ++i) {
                mm.sur.push_back(b.surprisal(i, x, cfg));
                z.push_back(b.standardize(b.all()[i].context));
            }
            mm.sim.assign(n, std::vector<double>(n, 0.0));
            for (std::size_t i = 0; i < n; ++i)
                for (std::size_t j = i + 1; j < n; ++j) mm.sim[i][j] = similarity(z[i], z[j], sigma);
            return mm;
        };
        auto value = [&](const Memo& mm, std::vector<std::size_t> s3) {
            double v = 0.0;
            for (std::size_t i : s3) v += mm.sur[i];
            for (std::size_t a = 0; a < s3.size(); ++a)
                for (std::size_t c = a + 1; c < s3.size(); ++c)
                    v -= cfg.lambda_div * mm.sim[std::min(s3[a], s3[c])][std::max(s3[a], s3[c])];
            return v;
        };
        auto greedy_value = [&](const ExperienceBuffer& b, const Memo& mm) {
            std::vector<std::size_t> chosen;
            for (const auto& sel : b.select(x, cfg))
                for (std::size_t i = 0; i < b.size(); ++i)
                    if (b.all()[i].round == sel.experience.round) chosen.push_back(i);
            return value(mm, chosen);
        };
        int wins = 0;
        for (int trial = 0; trial < 200; ++trial) {
            ExperienceBuffer b(0.0);
            const int n = 8 + static_cast<int>(g() % 25);
            fill(b, n);
            const Memo mm = memo(b);
            const double gv = greedy_value(b, mm);
            double tot = 0.0;
            for (int dd = 0; dd < 100; ++dd) {
                std::vector<std::size_t> pool(n);
                for (int i = 0; i < n; ++i) pool[i] = i;
                for (int k = 0; k < 3; ++k) std::swap(pool[k], pool[k + g() % (n - k)]);
                tot += value(mm, {pool[0], pool[1], pool[2]});
            }
            wins += gv >= tot / 100.0 - 1e-9;
        }
        int exh = 0;
        for (int trial = 0; trial < 50; ++trial) {
            ExperienceBuffer b(0.0);
            fill(b, 8);
            const Memo mm = memo(b);
            const double gv = greedy_value(b, mm);
            double best = -1e300;
            for (std::size_t a = 0; a < 8; ++a)
                for (std::size_t c = a + 1; c < 8; ++c)
                    for (std::size_t e = c + 1; e < 8; ++e) best = std::max(best, value(mm, {a, c, e}));
            exh += gv >= 0.5 * best - 1e-9;
        }
        std::printf("  acceptance 8: beat random mean on %d/200, >= half optimum on %d/50\n", wins, exh);
        EXPECT(wins >= 190);
        EXPECT(exh == 50);
    }
    // small buffers and determinism, :187-201
    {
        SelectionConfig cfg;
        EXPECT(ExperienceBuffer(0.0).select({1, 2}, cfg).empty());
        ExperienceBuffer b(0.0);
        b.store(exp_of({1, 0}, 0.3, 0));
        b.store(exp_of({0, 1}, 0.8, 1));
        auto a1 = b.select({0.5, 0.5}, cfg), a2 = b.select({0.5, 0.5}, cfg);
        EXPECT(a1.size() == 2 && a2.size() == 2);
        for (std::size_t i = 0; i < a1.size() && i < a2.size(); ++i)
            EXPECT(a1[i].experience.round == a2[i].experience.round);
        EXPECT_THROW(b.select({1.0}, cfg), std::invalid_argument);
    }
    // coverage proxy, :203-230
    {
        std::mt19937_64 g(777);
        std::uniform_real_distribution<double> u(0, 1);
        SelectionConfig cfg;
        cfg.m = 15;
        cfg.sigma_sim = 0.5;
        double d32 = 0, d512 = 0;
        for (int t = 0; t < 10; ++t) {
            ExperienceBuffer b(0.0);
            std::vector<double> probe{u(g), u(g)};
            auto nearest = [&](std::size_t lim) {
                while (b.size() < lim) b.store(exp_of({u(g), u(g)}, 0.05 + u(g), (int)b.size()));
                double best = 1e300;
                for (const auto& s : b.select(probe, cfg))
                    best = std::min(best, std::hypot(s.experience.context[0] - probe[0],
                                                     s.experience.context[1] - probe[1]));
                return best;
            };
            d32 += nearest(32);
            d512 += nearest(512);
        }
        EXPECT(d512 < d32);
    }
    // copies are independent (value semantics, experience.hpp:45)
    {
        ExperienceBuffer a(0.0);
        a.store(exp_of({1, 2}, 0.5, 0));
        ExperienceBuffer b = a;
        b.store(exp_of({2, 3}, 0.6, 1));
        EXPECT(a.size() == 1 && b.size() == 2);
        ExperienceBuffer c = std::move(b);
        EXPECT(c.size() == 2 && c.select({1, 2}, SelectionConfig{}).size() == 2);
    }
    // persistence round trip, :232-273
    {
        const char* path = "/tmp/scalelab_b200_roundtrip.jsonl";
        ExperienceBuffer b(0.0);
        std::mt19937_64 g(31);
        std::uniform_real_distribution<double> u(0, 1);
        for (int i = 0; i < 50; ++i) {
            auto e = exp_of({u(g), u(g), u(g)}, 0.01 + u(g), i);
            e.source = i % 4 == 0 ? "probe" : "llm";
            e.action = ScalingAction::noop(2);
            e.action.stages[i % 2].replicas = (i % 3) - 1;
            b.store(std::move(e));
        }
        b.persist(path);
        std::size_t bad = 7;
        auto l = ExperienceBuffer::load(path, 0.0, &bad);
        EXPECT(bad == 0 && l.size() == b.size());
        for (std::size_t i = 0; i < b.size() && i < l.size(); ++i) {
            EXPECT(l.all()[i].context == b.all()[i].context);
            EXPECT(l.all()[i].action == b.all()[i].action);
            EXPECT(l.all()[i].reward == b.all()[i].reward);
        }
        std::remove(path);
    }
}

// ------------------------------------------------------------- pareto --

static std::vector<ObjectivePoint> brute_frontier(const std::vector<ObjectivePoint>& pts) {
    // the quadratic filter of tests/test_pareto.cpp:17-33, restated
    std::vector<ObjectivePoint> out;
    for (std::size_t i = 0; i < pts.size(); ++i) {
        bool keep = true;
        for (std::size_t j = 0; j < pts.size() && keep; ++j) {
            if (j == i) continue;
            const auto& p = pts[j];
            const auto& q = pts[i];
            bool dom = p.latency <= q.latency && p.cost <= q.cost &&
                       (p.latency < q.latency || p.cost < q.cost);
            if (dom || (p == q && j < i)) keep = false;
        }
        if (keep) out.push_back(pts[i]);
    }
    std::sort(out.begin(), out.end(), [](auto& a, auto& b) { return a.latency < b.latency; });
    return out;
}

static void pareto_tests() {
    // dominance, test_pareto.cpp:55-62
    EXPECT(dominates({0.2, 0.3}, {0.3, 0.3}));
    EXPECT(dominates({0.2, 0.3}, {0.2, 0.4}));
    EXPECT(!dominates({0.2, 0.3}, {0.2, 0.3}));
    EXPECT(!dominates({0.1, 0.9}, {0.9, 0.1}));
    // normalize, :64-76
    {
        ParetoFrontier f(1000.0, 10.0);
        bool cl = true;
        auto p = f.normalize(500.0, 5.0, &cl);
        EXPECT(p.latency == 0.5 && p.cost == 0.5 && !cl);
        p = f.normalize(2500.0, 3.0, &cl);
        EXPECT(p.latency == 1.0 && cl);
        EXPECT_THROW(ParetoFrontier(0.0, 1.0), std::invalid_argument);
        EXPECT_THROW(ParetoFrontier(1.0, -2.0), std::invalid_argument);
    }
    // update, HV, contribution, reward: :78-125
    {
        ParetoFrontier f(1000.0, 10.0);
        EXPECT(f.update(600.0, 4.0).inserted && f.update(200.0, 8.0).inserted);
        EXPECT(!f.update(700.0, 5.0).inserted && !f.update(600.0, 4.0).inserted);
        EXPECT(f.size() == 2);
        EXPECT(close_rel(f.hypervolume(), 0.32, 1e-12));
        EXPECT(close_rel(f.contribution({0.4, 0.5}), 0.06, 1e-12));
        EXPECT_THROW(f.contribution({0.7, 0.9}), std::logic_error);
        double d = std::min(std::hypot(0.5, 0.1), std::hypot(0.1, 0.5));
        EXPECT(close_rel(f.reward({0.7, 0.9}), 0.8 / (1.0 + d), 1e-12));
        EXPECT(close_rel(f.reward({0.4, 0.5}), 1.06, 1e-12));
        EXPECT(close_rel(f.reward({0.2, 0.8}), 1.0, 1e-12));
        ParetoFrontier copy = f;  // copied inside contribution in the reference (pareto.cpp:70)
        EXPECT(f.update(100.0, 1.0).inserted);
        EXPECT(f.size() == 1 && f.points()[0] == (ObjectivePoint{0.1, 0.1}));
        EXPECT(copy.size() == 2);
        ParetoFrontier e(1000.0, 10.0);
        EXPECT(!e.distance({0.3, 0.4}).has_value());
        EXPECT(close_rel(e.reward({0.3, 0.4}), 1.0 + 0.7 * 0.6, 1e-12));
    }
    // random grids vs the brute force, :127-147 and acceptance check 3 (:237-280)
    {
        std::mt19937_64 g(20240817);
        std::uniform_real_distribution<double> u(0, 1);
        int bad = 0;
        for (int t = 0; t < 60; ++t) {
            ParetoFrontier f(1.0, 1.0);
            std::vector<ObjectivePoint> ins;
            int n = 1 + static_cast<int>(g() % 40);
            for (int i = 0; i < n; ++i) {
                ObjectivePoint p{std::round(u(g) * 8) / 8, std::round(u(g) * 8) / 8};
                f.update(p.latency, p.cost);
                ins.push_back(p);
            }
            bad += !(f.points() == brute_frontier(ins));
#ifdef SCALELAB_B200_EXT
            ParetoFrontier h(1.0, 1.0);
            h.insert_batch(ins);
            bad += !(h.points() == f.points());
#endif
        }
        EXPECT(bad == 0);
    }
    // separation >= 0.2, acceptance check 1 (:98-131) / test_reward.cpp:117-138
    {
        std::mt19937_64 g(20260823);
        std::uniform_real_distribution<double> u(0, 1);
        int viol = 0;
        for (int t = 0; t < 200; ++t) {
            ParetoFrontier f(1.0, 1.0);
            int n = 1 + static_cast<int>(g() % 6);
            for (int i = 0; i < n; ++i) f.update(u(g), u(g));
            std::vector<ObjectivePoint> probes;
            for (int k = 0; k < 12; ++k) probes.push_back({u(g), u(g)});
#ifdef SCALELAB_B200_EXT
            auto r = f.reward_batch(probes);
#else
            std::vector<double> r;
            for (const auto& p : probes) r.push_back(f.reward(p));
#endif
            double lo = 1e300, hi = -1e300;
            for (int k = 0; k < 12; ++k)
                (f.strictly_dominated(probes[k]) ? hi : lo) =
                    f.strictly_dominated(probes[k]) ? std::max(hi, r[k]) : std::min(lo, r[k]);
            if (lo < 1e300 && hi > -1e300 && lo - hi < 0.2 - 1e-12) ++viol;
        }
        EXPECT(viol == 0);
    }
}

// -------------------------------------------------------------- reward --

static void reward_tests() {
    // magnitude, test_reward.cpp:21-29
    {
        EXPECT(action_magnitude(ScalingAction::noop(3)) == 0.0);
        auto a = ScalingAction::noop(2);
        a.stages[0].replicas = 2;
        a.stages[0].cpu_millicores = -500;
        a.stages[1].rate_ratio_tenths = 1;
        EXPECT(close_rel(action_magnitude(a), 3.55, 1e-12));
    }
    ParetoFrontier f(2000.0, 10.0);
    RewardConfig cfg;
    // SLA, :31-42
    {
        RewardInputs in{400.0, 1000.0, 1.0, 1.0};
        EXPECT(close_rel(compute_reward(in, ScalingAction::noop(1), f, cfg).sla, -3.0, 1e-12));
        in.l_after_ms = 500.0;
        EXPECT(compute_reward(in, ScalingAction::noop(1), f, cfg).sla == 0.0);
    }
    // golden vector, :57-76
    {
        ParetoFrontier g(400.0, 10.0);
        g.update(100.0, 1.2);
        RewardConfig c;
        c.l_baseline_ms = 400.0;
        auto a = ScalingAction::noop(1);
        a.stages[0].replicas = 1;
        auto r = compute_reward({400.0, 300.0, 1.0, 1.2}, a, g, c);
        EXPECT(close_rel(r.latency, 0.175, 1e-9) && close_rel(r.cost, -0.006, 1e-9));
        EXPECT(r.sla == 0.0 && r.proactive == 0.0 && !r.clipped);
        EXPECT(close_rel(r.pareto, 0.8 / 1.5, 1e-9));
    }
    // proactive, :78-89; clip, :91-102; config errors, :104-115
    {
        auto a = ScalingAction::noop(1);
        a.stages[0].replicas = 1;
        EXPECT(close_rel(compute_reward({750.0, 400.0, 1.0, 1.0}, a, f, cfg).proactive, 0.225, 1e-12));
        auto r = compute_reward({40000.0, 100.0, 5.0, 1.0}, a, f, cfg);
        EXPECT(r.total == cfg.r_max && r.clipped);
        auto r2 = compute_reward({100.0, 40000.0, 1.0, 5.0}, ScalingAction::noop(1), f, cfg);
        EXPECT(r2.total == -cfg.r_max && r2.clipped);
        RewardConfig bad;
        bad.t_sla_ms = 0.0;
        EXPECT_THROW(compute_reward({400, 300, 1, 1}, a, f, bad), std::invalid_argument);
        RewardConfig bad2;
        bad2.c_budget = 0.0;
        EXPECT_THROW(compute_reward({400, 300, 1, 1}, a, f, bad2), std::invalid_argument);
    }
    // acceptance check 2 (acceptance_main.cpp:140-233), vectors a and e
    {
        ParetoFrontier h(1000.0, 10.0);
        h.update(300.0, 4.0);
        h.update(700.0, 2.0);
        RewardConfig c;
        c.l_baseline_ms = 400.0;
        auto a = ScalingAction::noop(2);
        a.stages[0].replicas = 1;
        auto r = compute_reward({900.0, 650.0, 2.0, 2.6}, a, h, c);
        EXPECT(close_rel(r.pareto, 1.0 + 0.05 * 0.14, 1e-9));
        EXPECT(close_rel(r.total, 0.4375 - 0.018 - 0.69 + 0.36 + 1.007, 1e-9));
        auto e = ScalingAction::noop(3);
        e.stages[1].replicas = -1;
        auto r5 = compute_reward({150.0, 180.0, 4.0, 3.2}, e, h, c);
        EXPECT(close_rel(r5.pareto, 1.1136, 1e-9));
    }
}

int main() {
    std::printf("scalelab_b200 drop-in: reference expectations\n");
    experience_tests();
    pareto_tests();
    reward_tests();
    std::printf("%d checks, %d failed\n", g_checks, g_fail);
    return g_fail;
}
