// Drives the REFERENCE's own API above paper scale with the B200 adapter
// linked in place of cfcomplete.o:
//   joint_demo complete <matrix.csv>            read_matrix_csv_file (core.cpp:250-254)
//        -> cf::complete (default NcfHyper, seed 42) -> policy::select_caps per row
//        (gamma 0.05); prints "row idx saving(hex) loss(hex) candidates" per row
//   joint_demo fit <matrix.csv> <model.json>    cf::fit (default NcfHyper, seed 42)
//        -> NcfModel::to_json into model.json
#include <cstdio>
#include <cstring>
#include <fstream>
#include <vector>

#include "opencap/cfcomplete.hpp"
#include "opencap/core.hpp"
#include "opencap/policy.hpp"

using namespace opencap;

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: joint_demo complete <matrix.csv> | fit <matrix.csv> <model.json>\n");
        return 2;
    }
    try {
        const auto matrix = read_matrix_csv_file(argv[2]);
        const cf::NcfHyper hyper;
        if (!std::strcmp(argv[1], "fit")) {
            const auto model = cf::fit(matrix, hyper, 42);
            std::ofstream(argv[3], std::ios::binary) << model.to_json();
            std::printf("epochs_run %d best_val %a\n", model.meta().epochs_run, model.meta().best_val_mse);
            return 0;
        }
        const auto done = cf::complete(matrix, hyper, 42);
        std::vector<int> cpu, gpu;  // the matrix's PowerGrid (lexicographic settings)
        for (const auto& st : done.settings()) {
            if (cpu.empty() || cpu.back() != st.cpu_cap_w) cpu.push_back(st.cpu_cap_w);
            if (cpu.size() == 1) gpu.push_back(st.gpu_cap_w);
        }
        const policy::SelectionConfig cfg{PowerGrid(cpu, gpu), 0.05};
        for (size_t i = 0; i < done.rows(); ++i) {
            std::vector<double> row(done.cols());
            for (size_t j = 0; j < done.cols(); ++j) row[j] = done.value(i, j);
            const auto d = policy::select_caps(row, cfg);
            size_t idx = 0;
            while (done.settings()[idx] != d.setting) ++idx;
            std::printf("%zu %zu %a %a %zu\n", i, idx, d.pred_saving, d.pred_loss, d.candidates_considered);
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
