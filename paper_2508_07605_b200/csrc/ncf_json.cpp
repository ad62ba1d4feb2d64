// NCF model file: cf::NcfModel::to_json / from_json (cfcomplete.cpp:215-265)
// with the embedded nn::model_to_json / model_from_json (nnkit.cpp:306-365),
// over the flat parameter layout of this library ([app table | setting table |
// W0 b0 W1 b1 ...], the reference's Adam block order, cfcomplete.cpp:107-110).
//
// Host-only C++ (no device work).  The JSON is written with nlohmann::json
// 3.11.3 -- the library the reference itself links -- and dump(2), so the text
// is byte-identical to the reference's for the same model (keys in map order,
// shortest round-trip doubles); tests/test_ncf_json.py checks exactly that
// against models fitted by the reference.
#include <nlohmann/json.hpp>

#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ocg.h"

int ocg_internal_fail(int code, const std::string& msg);

namespace {

// architecture of cf::fit's MLP (cfcomplete.cpp:77-86): app_dim + setting_dim
// -> hidden... (selu) -> 1 (identity)
std::vector<std::size_t> mlp_dims(const ocg_ncf_hyper& h) {
    std::vector<std::size_t> d{static_cast<std::size_t>(h.app_dim + h.setting_dim)};
    for (int64_t i = 0; i < h.n_hidden; ++i) d.push_back(static_cast<std::size_t>(h.hidden[i]));
    d.push_back(1);
    return d;
}

int64_t param_count(const ocg_ncf_hyper& h, int64_t m, int64_t n) {
    int64_t t = m * h.app_dim + n * h.setting_dim;
    const auto d = mlp_dims(h);
    for (std::size_t l = 0; l + 1 < d.size(); ++l) t += static_cast<int64_t>(d[l] * d[l + 1] + d[l + 1]);
    return t;
}

bool hyper_ok(const ocg_ncf_hyper* h) {
    return h && h->app_dim > 0 && h->setting_dim > 0 && h->n_hidden >= 0 && h->n_hidden <= 8;
}

}  // namespace

extern "C" {

int ocg_ncf_model_to_json(const ocg_ncf_hyper* hyper, int64_t m, int64_t n, const double* params,
                          const uint8_t* app_seen, const uint8_t* setting_seen, const ocg_ncf_meta* meta,
                          char* out, size_t cap, size_t* len) {
    if (!hyper_ok(hyper) || m <= 0 || n <= 0 || !params || !app_seen || !setting_seen || !meta || !len)
        return ocg_internal_fail(OCG_E_INVALID, "ncf model to_json: bad arguments");
    try {
        const ocg_ncf_hyper& h = *hyper;
        const auto dims = mlp_dims(h);
        // nn::model_to_json (nnkit.cpp:306-329)
        nlohmann::json doc;
        doc["format_version"] = 1;
        std::vector<std::string> acts;
        for (std::size_t l = 0; l + 1 < dims.size(); ++l) acts.emplace_back(l + 2 < dims.size() ? "selu" : "identity");
        doc["architecture"] = {{"dims", dims}, {"activations", acts}};
        const double* p = params + m * h.app_dim + n * h.setting_dim;
        nlohmann::json jl = nlohmann::json::array();
        for (std::size_t l = 0; l + 1 < dims.size(); ++l) {
            const std::size_t in = dims[l], outd = dims[l + 1];
            nlohmann::json weights = nlohmann::json::array();
            for (std::size_t o = 0; o < outd; ++o) {
                nlohmann::json row = nlohmann::json::array();
                for (std::size_t i = 0; i < in; ++i) row.push_back(p[o * in + i]);
                weights.push_back(std::move(row));
            }
            p += in * outd;
            jl.push_back({{"weights", std::move(weights)}, {"biases", std::vector<double>(p, p + outd)}});
            p += outd;
        }
        doc["layers"] = std::move(jl);
        // NcfModel::to_json (cfcomplete.cpp:215-236): the MLP text is re-parsed there
        doc = nlohmann::json::parse(doc.dump(2));
        const auto table_json = [](const double* v, int64_t rows, int64_t dim) {
            nlohmann::json r = nlohmann::json::array();
            for (int64_t i = 0; i < rows; ++i) r.push_back(std::vector<double>(v + i * dim, v + (i + 1) * dim));
            return nlohmann::json{{"rows", static_cast<std::size_t>(rows)},
                                  {"dim", static_cast<std::size_t>(dim)},
                                  {"values", std::move(r)}};
        };
        doc["embeddings"] = {{"app", table_json(params, m, h.app_dim)},
                             {"setting", table_json(params + m * h.app_dim, n, h.setting_dim)}};
        doc["observed"] = {{"app_seen", std::vector<std::uint8_t>(app_seen, app_seen + m)},
                           {"setting_seen", std::vector<std::uint8_t>(setting_seen, setting_seen + n)}};
        doc["training"] = {{"seed", meta->seed},
                           {"epochs_run", meta->epochs_run},
                           {"initial_train_mse", meta->initial_train_mse},
                           {"final_train_mse", meta->final_train_mse},
                           {"best_val_mse", meta->best_val_mse}};
        const std::string text = doc.dump(2);
        *len = text.size() + 1;
        if (!out) return OCG_OK;
        if (cap < text.size() + 1) return ocg_internal_fail(OCG_E_INVALID, "ncf model to_json: buffer too small");
        std::memcpy(out, text.c_str(), text.size() + 1);
        return OCG_OK;
    } catch (const std::exception& e) {
        return ocg_internal_fail(OCG_E_LOGIC, std::string("ncf model to_json: ") + e.what());
    }
}

int ocg_ncf_model_from_json(const char* text, ocg_ncf_hyper* hyper, int64_t* m, int64_t* n, int64_t* nparams,
                            double* params, uint8_t* app_seen, uint8_t* setting_seen, ocg_ncf_meta* meta) {
    if (!text || !hyper || !m || !n || !nparams)
        return ocg_internal_fail(OCG_E_INVALID, "ncf model from_json: null argument");
    try {
        const auto doc = nlohmann::json::parse(text);
        // nn::model_from_json's checks (nnkit.cpp:331-365)
        if (!doc.contains("format_version") || doc["format_version"].get<int>() != 1)
            return ocg_internal_fail(OCG_E_INVALID, "model file: unsupported format_version");
        const auto dims = doc.at("architecture").at("dims").get<std::vector<std::size_t>>();
        const auto acts = doc.at("architecture").at("activations").get<std::vector<std::string>>();
        if (dims.size() < 2 || acts.size() != dims.size() - 1 || dims.back() != 1 || dims.size() - 2 > 8)
            return ocg_internal_fail(OCG_E_INVALID, "model file: inconsistent architecture");
        for (std::size_t l = 0; l < acts.size(); ++l)
            if (acts[l] != (l + 1 < acts.size() ? "selu" : "identity"))
                return ocg_internal_fail(OCG_E_UNSUPPORTED, "ncf model: activation layout other than cf::fit's");
        const auto& app = doc.at("embeddings").at("app");
        const auto& set = doc.at("embeddings").at("setting");
        const int64_t mm = app.at("rows").get<int64_t>(), nn = set.at("rows").get<int64_t>();
        ocg_ncf_hyper h;
        ocg_ncf_hyper_default(&h);
        h.app_dim = app.at("dim").get<int64_t>();
        h.setting_dim = set.at("dim").get<int64_t>();
        if (static_cast<int64_t>(dims[0]) != h.app_dim + h.setting_dim)
            return ocg_internal_fail(OCG_E_INVALID, "ncf model: embedding dims do not match the MLP input");
        h.n_hidden = static_cast<int64_t>(dims.size()) - 2;
        for (int64_t i = 0; i < h.n_hidden; ++i) h.hidden[i] = static_cast<int64_t>(dims[i + 1]);
        *hyper = h;
        *m = mm;
        *n = nn;
        *nparams = param_count(h, mm, nn);
        if (!params) return OCG_OK;  // shape query
        double* p = params;
        const auto table_from = [&](const nlohmann::json& j, int64_t rows, int64_t dim) {
            const auto& vals = j.at("values");
            if (static_cast<int64_t>(vals.size()) != rows) throw std::runtime_error("ncf model: embedding shape");
            for (const auto& row : vals) {
                const auto v = row.get<std::vector<double>>();
                if (static_cast<int64_t>(v.size()) != dim) throw std::runtime_error("ncf model: embedding shape");
                for (double x : v) *p++ = x;
            }
        };
        table_from(app, mm, h.app_dim);
        table_from(set, nn, h.setting_dim);
        const auto& jl = doc.at("layers");
        if (jl.size() != dims.size() - 1) throw std::runtime_error("model file: layer count");
        for (std::size_t l = 0; l + 1 < dims.size(); ++l) {
            const auto w = jl[l].at("weights").get<std::vector<std::vector<double>>>();
            const auto b = jl[l].at("biases").get<std::vector<double>>();
            if (w.size() != dims[l + 1] || b.size() != dims[l + 1]) throw std::runtime_error("model file: layer shape");
            for (const auto& row : w) {
                if (row.size() != dims[l]) throw std::runtime_error("model file: layer shape");
                for (double x : row) *p++ = x;
            }
            for (double x : b) *p++ = x;
        }
        const auto as = doc.at("observed").at("app_seen").get<std::vector<std::uint8_t>>();
        const auto ss = doc.at("observed").at("setting_seen").get<std::vector<std::uint8_t>>();
        if (static_cast<int64_t>(as.size()) != mm || static_cast<int64_t>(ss.size()) != nn)
            throw std::runtime_error("ncf model: observed mask shape");
        if (app_seen) std::memcpy(app_seen, as.data(), as.size());
        if (setting_seen) std::memcpy(setting_seen, ss.data(), ss.size());
        if (meta) {
            const auto& tr = doc.at("training");
            meta->seed = tr.at("seed").get<std::uint64_t>();
            meta->epochs_run = tr.at("epochs_run").get<int>();
            meta->initial_train_mse = tr.at("initial_train_mse").get<double>();
            meta->final_train_mse = tr.at("final_train_mse").get<double>();
            meta->best_val_mse = tr.at("best_val_mse").get<double>();
        }
        return OCG_OK;
    } catch (const std::exception& e) {
        return ocg_internal_fail(OCG_E_INVALID, std::string("ncf model from_json: ") + e.what());
    }
}

}  // extern "C"
