// Reference-side adapter: a drop-in replacement for the reference's whole
// proj/src/cfcomplete.cpp — cf::fit (cfcomplete.hpp:59), cf::complete (:63),
// NcfModel::predict / app_cold / setting_cold (:27-32) and NcfModel::to_json /
// from_json (:44-45) — that runs on the B200 through the C-ABI in
// include/ocg.h.  Compiled against the reference's own headers and linked
// INSTEAD of cfcomplete.o, every reference caller — run_open_online
// (policy.cpp:181), evaluate_suite (policy.cpp:368), cmd_online
// (opencap_main.cpp:86) — runs unchanged on the GPU.
//
// Semantics: identical to the reference (same exceptions, same bits).  The FP
// lane follows the reference process's kern::active_lane() so results match
// whichever lane the reference itself would use.  Solver: OPENCAP_CF_SOLVER =
// ref (default: FP64, bit-identical) | fast (FP32 NCF, same schedule) | als.
//   * cf::complete on a paper-scale matrix (the online phase's D dense rows + 1
//     app row) runs the per-app kernel (one CTA owns the whole fit);
//   * any larger matrix runs the joint-mode fit (ocg_cf_complete): the same
//     cf::fit, every parameter bit-identical, on the whole GPU.
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "ocg.h"
#include "opencap/cfcomplete.hpp"
#include "opencap/kernels.hpp"
#include "opencap/rng.hpp"

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

int lane() { return kern::active_lane() == kern::Lane::avx2 ? OCG_LANE_AVX2 : OCG_LANE_SCALAR; }

int solver() {
    const char* s = std::getenv("OPENCAP_CF_SOLVER");
    if (!s || !std::strcmp(s, "ref")) return OCG_SOLVER_NCF_REF;
    if (!std::strcmp(s, "fast")) return OCG_SOLVER_NCF_FAST;
    if (!std::strcmp(s, "als")) return OCG_SOLVER_ALS;
    throw std::invalid_argument(std::string("OPENCAP_CF_SOLVER: unknown solver ") + s);
}

struct Csr {
    std::vector<int64_t> rp;
    std::vector<int32_t> col;
    std::vector<double> val;
};

Csr to_csr(const PerformanceMatrix& m) {
    Csr c;
    c.rp.assign(m.rows() + 1, 0);
    for (size_t i = 0; i < m.rows(); ++i) {
        for (size_t j = 0; j < m.cols(); ++j)
            if (m.observed(i, j)) {
                c.col.push_back(static_cast<int32_t>(j));
                c.val.push_back(m.value(i, j));
            }
        c.rp[i + 1] = static_cast<int64_t>(c.col.size());
    }
    return c;
}

int64_t param_count(size_t m, size_t n, const NcfHyper& h) {
    int64_t t = 0, in = static_cast<int64_t>(h.app_dim + h.setting_dim);
    for (auto w : h.hidden) {
        t += in * static_cast<int64_t>(w) + static_cast<int64_t>(w);
        in = static_cast<int64_t>(w);
    }
    return static_cast<int64_t>(m * h.app_dim + n * h.setting_dim) + t + in + 1;
}

}  // namespace

// ---- NcfModel (cfcomplete.cpp:47-61) -----------------------------------
bool NcfModel::app_cold(std::size_t i) const { return app_seen_.at(i) == 0; }
bool NcfModel::setting_cold(std::size_t j) const { return setting_seen_.at(j) == 0; }

double NcfModel::predict(std::size_t app_index, std::size_t setting_index) const {
    ocg_ncf_hyper h{};
    h.app_dim = static_cast<int64_t>(app_emb_.dim);
    h.setting_dim = static_cast<int64_t>(setting_emb_.dim);
    const auto& L = mlp_.layers();
    for (size_t l = 0; l + 1 < L.size(); ++l) h.hidden[l] = static_cast<int64_t>(L[l].out_dim);
    h.n_hidden = static_cast<int64_t>(L.size()) - 1;
    std::vector<double> p(app_emb_.values);
    p.insert(p.end(), setting_emb_.values.begin(), setting_emb_.values.end());
    for (const auto& layer : L) {
        p.insert(p.end(), layer.weights.begin(), layer.weights.end());
        p.insert(p.end(), layer.biases.begin(), layer.biases.end());
    }
    const int64_t r = static_cast<int64_t>(app_index), c = static_cast<int64_t>(setting_index);
    double out = 0.0;
    const int rc = ocg_ncf_predict(context(), static_cast<int64_t>(app_emb_.rows), static_cast<int64_t>(setting_emb_.rows),
                                   &h, p.data(), app_seen_.data(), setting_seen_.data(), &r, &c, 1, lane(), &out);
    if (rc) rethrow(rc);
    return out;
}

// ---- cf::fit (cfcomplete.cpp:63-196): joint-mode fit on the GPU ---------
NcfModel fit(const PerformanceMatrix& matrix, const NcfHyper& hyper, std::uint64_t seed) {
    const size_t m = matrix.rows(), n = matrix.cols();
    const Csr c = to_csr(matrix);
    const ocg_ncf_hyper h = to_c(hyper);
    std::vector<double> p(static_cast<size_t>(param_count(m, n, hyper)));
    NcfModel model;
    model.app_seen_.assign(m, 0);
    model.setting_seen_.assign(n, 0);
    ocg_ncf_meta meta{};
    int sv = solver();
    if (sv == OCG_SOLVER_ALS) sv = OCG_SOLVER_NCF_REF;  // cf::fit returns an NcfModel
    const int rc = ocg_cf_fit(context(), static_cast<int64_t>(m), static_cast<int64_t>(n), c.rp.data(), c.col.data(),
                              c.val.data(), &h, seed, sv, lane(), p.data(), model.app_seen_.data(),
                              model.setting_seen_.data(), &meta);
    if (rc) rethrow(rc);
    size_t off = 0;
    model.app_emb_.rows = m;
    model.app_emb_.dim = hyper.app_dim;
    model.app_emb_.values.assign(p.begin(), p.begin() + static_cast<long>(m * hyper.app_dim));
    off += m * hyper.app_dim;
    model.setting_emb_.rows = n;
    model.setting_emb_.dim = hyper.setting_dim;
    model.setting_emb_.values.assign(p.begin() + static_cast<long>(off), p.begin() + static_cast<long>(off + n * hyper.setting_dim));
    off += n * hyper.setting_dim;
    std::vector<std::size_t> dims{hyper.app_dim + hyper.setting_dim};
    std::vector<nn::Activation> acts;
    for (const auto w : hyper.hidden) {
        dims.push_back(w);
        acts.push_back(nn::Activation::selu);
    }
    dims.push_back(1);
    acts.push_back(nn::Activation::identity);
    Rng scratch(0);  // shapes only: every weight is overwritten below
    model.mlp_ = nn::MlpModel(dims, acts, scratch);
    for (auto& layer : model.mlp_.layers()) {
        for (auto& w : layer.weights) w = p[off++];
        for (auto& b : layer.biases) b = p[off++];
    }
    model.meta_.seed = meta.seed;
    model.meta_.epochs_run = meta.epochs_run;
    model.meta_.initial_train_mse = meta.initial_train_mse;
    model.meta_.final_train_mse = meta.final_train_mse;
    model.meta_.best_val_mse = meta.best_val_mse;
    return model;
}

// ---- cf::complete (cfcomplete.cpp:198-213) -------------------------------
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
    const ocg_ncf_hyper h = to_c(hyper);
    const int ln = lane(), sv = solver();
    std::vector<double> completed(m * n);
    int rc = OCG_E_UNSUPPORTED;
    if (sv == OCG_SOLVER_NCF_REF) {
        // paper scale: one CTA owns the fit (the offline block + the app row)
        std::vector<double> vals(m * n, 0.0);
        std::vector<uint8_t> mask(m * n, 0);
        for (size_t i = 0; i < m; ++i)
            for (size_t j = 0; j < n; ++j)
                if (matrix.observed(i, j)) {
                    vals[i * n + j] = matrix.value(i, j);
                    mask[i * n + j] = 1;
                }
        const int64_t T = param_count(m, n, hyper);
        std::vector<double> params(static_cast<size_t>(T));
        ocg_ncf_meta meta{};
        int32_t status = 0;
        const uint64_t s = seed;
        rc = ocg_online_fit_batch_params(context(), static_cast<int64_t>(m - 1), vals.data(), mask.data(), 1,
                                         vals.data() + (m - 1) * n, mask.data() + (m - 1) * n, &s,
                                         static_cast<int32_t>(n), &h, ln, params.data(), T, &meta, &status);
        if (rc == OCG_OK) {
            if (status) rethrow(status);
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
                                 app_seen.data(), set_seen.data(), rows.data(), cols.data(),
                                 static_cast<int64_t>(rows.size()), ln, pred.data());
            if (rc) rethrow(rc);
            PerformanceMatrix out = matrix;
            for (size_t q = 0; q < rows.size(); ++q)
                out.set(static_cast<size_t>(rows[q]), static_cast<size_t>(cols[q]), pred[q]);
            return out;
        }
        if (rc != OCG_E_UNSUPPORTED) rethrow(rc);
    }
    // any scale / solver: the joint-mode fit + fused imputation over the whole matrix
    const Csr c = to_csr(matrix);
    ocg_als_hyper ah{32, 0.05f, 10, seed};
    if (const char* r = std::getenv("OPENCAP_ALS_RANK")) ah.rank = std::atoi(r);
    rc = ocg_cf_complete(context(), static_cast<int64_t>(m), static_cast<int64_t>(n), c.rp.data(), c.col.data(),
                         c.val.data(), &h, &ah, seed, sv, ln, nullptr, 0, nullptr, 0, 0.05, completed.data(), nullptr,
                         nullptr, nullptr, nullptr);
    if (rc) rethrow(rc);
    PerformanceMatrix out = matrix;
    for (size_t i = 0; i < m; ++i)
        for (size_t j = 0; j < n; ++j)
            if (!matrix.observed(i, j)) out.set(i, j, completed[i * n + j]);
    return out;
}

// ---- model file (cfcomplete.cpp:215-265): the reference's own serializer ---
std::string NcfModel::to_json() const {
    ocg_ncf_hyper h{};
    h.app_dim = static_cast<int64_t>(app_emb_.dim);
    h.setting_dim = static_cast<int64_t>(setting_emb_.dim);
    const auto& L = mlp_.layers();
    for (size_t l = 0; l + 1 < L.size(); ++l) h.hidden[l] = static_cast<int64_t>(L[l].out_dim);
    h.n_hidden = static_cast<int64_t>(L.size()) - 1;
    std::vector<double> p(app_emb_.values);
    p.insert(p.end(), setting_emb_.values.begin(), setting_emb_.values.end());
    for (const auto& layer : L) {
        p.insert(p.end(), layer.weights.begin(), layer.weights.end());
        p.insert(p.end(), layer.biases.begin(), layer.biases.end());
    }
    ocg_ncf_meta mt{meta_.seed, meta_.epochs_run, meta_.initial_train_mse, meta_.final_train_mse, meta_.best_val_mse};
    size_t len = 0;
    const int64_t m = static_cast<int64_t>(app_emb_.rows), n = static_cast<int64_t>(setting_emb_.rows);
    int rc = ocg_ncf_model_to_json(&h, m, n, p.data(), app_seen_.data(), setting_seen_.data(), &mt, nullptr, 0, &len);
    if (rc) rethrow(rc);
    std::string out(len, '\0');
    rc = ocg_ncf_model_to_json(&h, m, n, p.data(), app_seen_.data(), setting_seen_.data(), &mt, out.data(), len, &len);
    if (rc) rethrow(rc);
    out.resize(std::strlen(out.c_str()));
    return out;
}

NcfModel NcfModel::from_json(const std::string& text) {
    ocg_ncf_hyper h{};
    int64_t m = 0, n = 0, np = 0;
    int rc = ocg_ncf_model_from_json(text.c_str(), &h, &m, &n, &np, nullptr, nullptr, nullptr, nullptr);
    if (rc) rethrow(rc);
    std::vector<double> p(static_cast<size_t>(np));
    NcfModel model;
    model.app_seen_.assign(static_cast<size_t>(m), 0);
    model.setting_seen_.assign(static_cast<size_t>(n), 0);
    ocg_ncf_meta mt{};
    rc = ocg_ncf_model_from_json(text.c_str(), &h, &m, &n, &np, p.data(), model.app_seen_.data(),
                                 model.setting_seen_.data(), &mt);
    if (rc) rethrow(rc);
    size_t off = 0;
    model.app_emb_.rows = static_cast<size_t>(m);
    model.app_emb_.dim = static_cast<size_t>(h.app_dim);
    model.app_emb_.values.assign(p.begin(), p.begin() + m * h.app_dim);
    off = static_cast<size_t>(m * h.app_dim);
    model.setting_emb_.rows = static_cast<size_t>(n);
    model.setting_emb_.dim = static_cast<size_t>(h.setting_dim);
    model.setting_emb_.values.assign(p.begin() + static_cast<long>(off), p.begin() + static_cast<long>(off + n * h.setting_dim));
    off += static_cast<size_t>(n * h.setting_dim);
    std::vector<std::size_t> dims{static_cast<size_t>(h.app_dim + h.setting_dim)};
    std::vector<nn::Activation> acts;
    for (int64_t l = 0; l < h.n_hidden; ++l) {
        dims.push_back(static_cast<size_t>(h.hidden[l]));
        acts.push_back(nn::Activation::selu);
    }
    dims.push_back(1);
    acts.push_back(nn::Activation::identity);
    Rng scratch(0);
    model.mlp_ = nn::MlpModel(dims, acts, scratch);
    for (auto& layer : model.mlp_.layers()) {
        for (auto& w : layer.weights) w = p[off++];
        for (auto& b : layer.biases) b = p[off++];
    }
    model.meta_.seed = mt.seed;
    model.meta_.epochs_run = mt.epochs_run;
    model.meta_.initial_train_mse = mt.initial_train_mse;
    model.meta_.final_train_mse = mt.final_train_mse;
    model.meta_.best_val_mse = mt.best_val_mse;
    return model;
}

}  // namespace opencap::cf
