// bench_dropin_decision.cpp -- per-call costs of the drop-in's members in the
// reference's decision loop (harness.cpp / policy.cpp usage) over a 10k store:
// select(m = 15, lambda 0.1), the policy's veto loop (standardize +
// similarity per stored record, policy.cpp:140-153), store().  Diagnostic.
#include <chrono>
#include <cstdio>
#include <string>

#include "scalelab_b200/experience.hpp"

using namespace scalelab;
using clk = std::chrono::steady_clock;

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    auto t0 = clk::now();
    ExperienceBuffer buf = ExperienceBuffer::load(argv[1], 0.0);
    auto t1 = clk::now();
    SelectionConfig cfg;
    const auto& items = buf.all();
    std::vector<double> q = items[17].context;
    for (auto& v : q) v *= 1.01;
    auto ms = [](clk::duration d) { return std::chrono::duration<double, std::milli>(d).count(); };
    buf.select(q, cfg);
    auto t2 = clk::now();
    for (int r = 0; r < 20; ++r) buf.select(q, cfg);
    auto t3 = clk::now();
    double acc = 0.0;
    for (int r = 0; r < 5; ++r) {
        std::vector<double> z = buf.standardize(q);
        double sg = buf.effective_sigma(cfg);
        for (const auto& e : buf.all()) acc += similarity(buf.standardize(e.context), z, sg);
    }
    auto t4 = clk::now();
    for (int r = 0; r < 20; ++r) {
        Experience e = items[r];
        e.round += 100000;
        buf.store(e);
    }
    auto t5 = clk::now();
    std::printf("records %zu: load %.1f ms, first select %.2f ms, select %.3f ms, veto loop %.3f ms, store %.3f ms (%g)\n",
                buf.size(), ms(t1 - t0), ms(t2 - t1), ms(t3 - t2) / 20, ms(t4 - t3) / 5, ms(t5 - t4) / 20, acc);
    return 0;
}
