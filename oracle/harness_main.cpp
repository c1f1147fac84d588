// harness_main.cpp -- runs the reference's decision loop (run_experiment,
// harness.cpp:129-346) on one scenario and writes its episode log CSV.
// Built twice by oracle/Makefile from the unmodified reference sources:
//   _ref/harness_ref   with the reference's experience/pareto/reward.cpp
//   _ref/harness_b200  with the drop-in (scalelab_b200 on libsair) instead
// Identical CSVs for equal seeds (the reference's own determinism check,
// tests/test_harness.cpp:142-150) show the drop-in is exact end to end.
#include <cstdio>
#include <cstdlib>
#include <string>

#include "scalelab/harness.hpp"
#include "scalelab/scenario.hpp"

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: %s scenario.json out.csv [controller] [seed] [rounds]\n", argv[0]);
        return 2;
    }
    scalelab::Scenario sc = scalelab::load_scenario(argv[1]);
    if (argc > 3) sc.controller = argv[3];
    if (argc > 4) sc.seed = std::strtoull(argv[4], nullptr, 10);
    if (argc > 5) sc.rounds = std::atoi(argv[5]);
    scalelab::validate_scenario(sc);
    scalelab::RunResult res = scalelab::run_experiment(sc);
    res.log.to_csv(argv[2]);
    std::printf("{\"p99_ms\": %.17g, \"hypervolume\": %.17g, \"rounds\": %d}\n",
                res.summary.p99_ms, res.summary.frontier_hypervolume, sc.rounds);
    return 0;
}
