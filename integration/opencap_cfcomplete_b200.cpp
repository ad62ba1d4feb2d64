// Reference-side adapter: a drop-in replacement for the reference's
// proj/src/cfcomplete.cpp entry point `opencap::cf::complete`
// (cfcomplete.hpp:63) that runs the fit + imputation on the B200 through the
// C-ABI in include/ocg.h.  Compiled against the reference's own headers and
// linked INSTEAD of cfcomplete.o, every reference caller — run_open_online
// (policy.cpp:181), evaluate_suite (policy.cpp:368), cmd_online
// (opencap_main.cpp:86) — runs unchanged on the GPU.
//
// Semantics: identical to the reference (same exceptions, same bits): the
// matrix is split into its first m-1 rows (the "offline block") and its last
// row (the app being completed), the per-app kernel fits cf::fit on the whole
// matrix with the reference's RNG streams, and imputes the app row.  The FP
// lane follows the reference process's kern::active_lane() so results match
// whichever lane the reference itself would use.  Missing cells of block rows
// are imputed through ocg_ncf_predict on the fitted parameters.
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "ocg.h"
#include "opencap/cfcomplete.hpp"
#include "opencap/kernels.hpp"

namespace opencap::cf {

namespace {

ocg_ctx* context() {
    static ocg_ctx* ctx = [] {
        ocg_ctx* c = nullptr;
        if (ocg_ctx_create(0, &c) != OCG_OK) throw std::runtime_error(std::string("ocg: ") + ocg_last_error());
        return c;
    }();
    return ctx;
}

[[noreturn]] void rethrow(int rc) {
    const std::string msg = ocg_last_error();
    switch (rc) {
        case OCG_E_INVALID: throw std::invalid_argument(msg);
        case OCG_E_RANGE: throw std::out_of_range(msg);
        case OCG_E_COLD:
        case OCG_E_DIVERGE: throw std::runtime_error(msg);
        case OCG_E_LOGIC: throw std::logic_error(msg);
        default: throw std::runtime_error("ocg: " + msg);
    }
}

ocg_ncf_hyper to_c(const NcfHyper& h) {
    ocg_ncf_hyper c{};
    c.app_dim = static_cast<int64_t>(h.app_dim);
    c.setting_dim = static_cast<int64_t>(h.setting_dim);
    if (h.hidden.size() > 8) throw std::invalid_argument("ncf: too many hidden layers");
    for (size_t i = 0; i < h.hidden.size(); ++i) c.hidden[i] = static_cast<int64_t>(h.hidden[i]);
    c.n_hidden = static_cast<int64_t>(h.hidden.size());
    c.lr = h.lr;
    c.max_epochs = h.max_epochs;
    c.patience = h.patience;
    c.val_fraction = h.val_fraction;
    c.batch_size = h.batch_size;
    return c;
}

}  // namespace

PerformanceMatrix complete(const PerformanceMatrix& matrix, const NcfHyper& hyper, std::uint64_t seed) {
    const size_t m = matrix.rows(), n = matrix.cols();
    // cfcomplete.cpp:199-205 — every row needs an observation
    for (size_t i = 0; i < m; ++i) {
        bool any = false;
        for (size_t j = 0; j < n && !any; ++j) any = matrix.observed(i, j);
        if (!any)
            throw std::invalid_argument("complete: app row '" + matrix.app_ids()[i] +
                                        "' has no observed entries (probe it first)");
    }
    if (matrix.observed_count() == m * n) return matrix;  // :206
    std::vector<double> vals(m * n, 0.0);
    std::vector<uint8_t> mask(m * n, 0);
    for (size_t i = 0; i < m; ++i)
        for (size_t j = 0; j < n; ++j)
            if (matrix.observed(i, j)) {
                vals[i * n + j] = matrix.value(i, j);
                mask[i * n + j] = 1;
            }
    const ocg_ncf_hyper h = to_c(hyper);
    const int lane = kern::active_lane() == kern::Lane::avx2 ? OCG_LANE_AVX2 : OCG_LANE_SCALAR;
    const int64_t T = static_cast<int64_t>(m * hyper.app_dim + n * hyper.setting_dim) + [&] {
        int64_t t = 0, in = static_cast<int64_t>(hyper.app_dim + hyper.setting_dim);
        for (auto w : hyper.hidden) {
            t += in * static_cast<int64_t>(w) + static_cast<int64_t>(w);
            in = static_cast<int64_t>(w);
        }
        return t + in + 1;
    }();
    std::vector<double> params(static_cast<size_t>(T));
    ocg_ncf_meta meta{};
    int32_t status = 0;
    const uint64_t s = seed;
    int rc = ocg_online_fit_batch_params(context(), static_cast<int64_t>(m - 1), vals.data(), mask.data(), 1,
                                         vals.data() + (m - 1) * n, mask.data() + (m - 1) * n, &s,
                                         static_cast<int32_t>(n), &h, lane, params.data(), T, &meta, &status);
    if (rc) rethrow(rc);
    if (status) rethrow(status);
    // impute every unobserved cell in row-major order (cfcomplete.cpp:208-211)
    std::vector<int64_t> rows, cols;
    for (size_t i = 0; i < m; ++i)
        for (size_t j = 0; j < n; ++j)
            if (!mask[i * n + j]) {
                rows.push_back(static_cast<int64_t>(i));
                cols.push_back(static_cast<int64_t>(j));
            }
    std::vector<uint8_t> app_seen(m, 0), set_seen(n, 0);
    for (size_t i = 0; i < m; ++i)
        for (size_t j = 0; j < n; ++j)
            if (mask[i * n + j]) app_seen[i] = set_seen[j] = 1;
    std::vector<double> pred(rows.size());
    rc = ocg_ncf_predict(context(), static_cast<int64_t>(m), static_cast<int64_t>(n), &h, params.data(),
                         app_seen.data(), set_seen.data(), rows.data(), cols.data(), static_cast<int64_t>(rows.size()),
                         lane, pred.data());
    if (rc) rethrow(rc);
    PerformanceMatrix out = matrix;
    for (size_t q = 0; q < rows.size(); ++q) out.set(static_cast<size_t>(rows[q]), static_cast<size_t>(cols[q]), pred[q]);
    return out;
}

}  // namespace opencap::cf
