// Runs the REFERENCE's own online pipeline (policy::run_open_online,
// policy.cpp:114-191, with the CLI's seeds, opencap_main.cpp:79-87) for the
// 20 paper-scale eval apps, with cf::complete provided by the B200 adapter.
// Prints one line per app: index setting_idx pred_saving(hex) candidates.
#include <cstdio>
#include <fstream>
#include <sstream>

#include "opencap/policy.hpp"
#include "opencap/predictor.hpp"
#include "opencap/rng.hpp"

using namespace opencap;

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: online_demo <predictor.json> [dense.csv]\n");
        return 2;
    }
    const uint64_t seed = 42;
    const auto grid = PowerGrid::default_grid();
    const auto train = sim::make_suite(sim::default_training_params(seed), grid);
    const auto profiled = pred::profile_suite(train, grid, derive_seed(seed, "offline.profile"));
    std::ifstream f(argv[1]);
    std::stringstream buf;
    buf << f.rdbuf();
    const auto predictor = pred::predictor_from_json(buf.str());
    const auto eval = sim::make_suite(sim::default_evaluation_params(seed), grid);
    const auto settings = grid.settings();
    for (size_t e = 0; e < eval.size(); ++e) {
        const auto& spec = eval[e];
        const auto cfg = policy::OnlineConfig::defaults(grid);
        const auto oc = policy::run_open_online(spec, profiled.matrix, predictor, cfg,
                                                derive_seed(seed, "open." + spec.app_id));
        size_t idx = 0;
        while (settings[idx] != oc.decision.setting) ++idx;
        std::printf("%zu %zu %a %zu\n", e, idx, oc.decision.pred_saving, oc.decision.candidates_considered);
    }
    return 0;
}
