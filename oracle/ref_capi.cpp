// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI shim over the *unmodified* reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It lets the
// pytest suite, the golden-vector generator (tests/golden/make_golden.py) and
// bench.py's reference arm drive the reference's own public API through
// ctypes.  Every entry point forwards to the reference symbol named in its
// comment; nothing here re-implements reference arithmetic.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "json.hpp"
#include "opencap/cfcomplete.hpp"
#include "opencap/core.hpp"
#include "opencap/kernels.hpp"
#include "opencap/phasedet.hpp"
#include "opencap/policy.hpp"
#include "opencap/predictor.hpp"
#include "opencap/rng.hpp"
#include "opencap/simnode.hpp"

using namespace opencap;

namespace {

thread_local std::string g_err;

// error codes follow include/ocg.h (OCG_E_*) so tests can compare them
int map_exception() {
    try {
        throw;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 4;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const missing_artifact_error& e) {
        g_err = e.what();
        return 2;
    } catch (const config_error& e) {
        g_err = e.what();
        return 1;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        std::string w = e.what();
        if (w.find("cold") != std::string::npos) return 5;
        if (w.find("divergence") != std::string::npos) return 6;
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

PowerGrid make_grid(const int* cpu, size_t ncpu, const int* gpu, size_t ngpu) {
    return PowerGrid(std::vector<int>(cpu, cpu + ncpu), std::vector<int>(gpu, gpu + ngpu));
}

std::vector<std::string> app_ids(size_t m) {
    std::vector<std::string> ids;
    ids.reserve(m);
    for (size_t i = 0; i < m; ++i) ids.push_back("a" + std::to_string(i));
    return ids;
}

PerformanceMatrix make_matrix(size_t m, const PowerGrid& grid, const double* values,
                              const uint8_t* mask) {
    PerformanceMatrix pm(app_ids(m), grid);
    const size_t n = pm.cols();
    for (size_t i = 0; i < m; ++i)
        for (size_t j = 0; j < n; ++j)
            if (mask[i * n + j]) pm.set(i, j, values[i * n + j]);
    return pm;
}

int copy_text(const std::string& s, char* out, size_t cap, size_t* len) {
    if (len) *len = s.size();
    if (out == nullptr || cap <= s.size()) {
        g_err = "buffer too small";
        return 7;
    }
    std::memcpy(out, s.data(), s.size());
    out[s.size()] = 0;
    return 0;
}

}  // namespace

extern "C" {

struct ref_ncf_hyper {
    uint64_t app_dim, setting_dim;
    uint64_t hidden[8];
    uint64_t n_hidden;
    double lr;
    int32_t max_epochs, patience;
    double val_fraction;
    int32_t batch_size;
};

struct ref_ncf_meta {
    uint64_t seed;
    int32_t epochs_run;
    double initial_train_mse, final_train_mse, best_val_mse;
};

const char* ref_last_error() { return g_err.c_str(); }

// kern::force_lane (kernels.hpp:38) — 0 scalar, 1 avx2
int ref_force_lane(int lane) {
    return kern::force_lane(lane == 0 ? kern::Lane::scalar : kern::Lane::avx2) ? 0 : 1;
}
int ref_active_lane() { return kern::active_lane() == kern::Lane::scalar ? 0 : 1; }

// derive_seed (rng.hpp:53)
uint64_t ref_derive_seed(uint64_t root, const char* tag, uint64_t n) { return derive_seed(root, tag, n); }

// Rng::next_u64 / uniform / uniform_int / normal (rng.hpp:19-38)
void ref_rng_u64(uint64_t seed, uint64_t* out, size_t n) {
    Rng r(seed);
    for (size_t i = 0; i < n; ++i) out[i] = r.next_u64();
}
void ref_rng_uniform(uint64_t seed, double lo, double hi, double* out, size_t n) {
    Rng r(seed);
    for (size_t i = 0; i < n; ++i) out[i] = r.uniform(lo, hi);
}
void ref_rng_normal(uint64_t seed, double* out, size_t n) {
    Rng r(seed);
    for (size_t i = 0; i < n; ++i) out[i] = r.normal();
}

// policy::select_caps (policy.cpp:17-64) applied to `rows` rows of length n
int ref_select_caps(const double* rowsv, size_t rows, const int* cpu, size_t ncpu, const int* gpu,
                    size_t ngpu, double gamma, int32_t* idx, double* saving, double* loss,
                    int32_t* ncand) {
    try {
        policy::SelectionConfig cfg{make_grid(cpu, ncpu, gpu, ngpu), gamma};
        const auto settings = cfg.grid.settings();
        const size_t n = settings.size();
        for (size_t r = 0; r < rows; ++r) {
            const auto d = policy::select_caps(std::span<const double>(rowsv + r * n, n), cfg);
            idx[r] = static_cast<int32_t>(std::find(settings.begin(), settings.end(), d.setting) -
                                          settings.begin());
            saving[r] = d.pred_saving;
            loss[r] = d.pred_loss;
            ncand[r] = static_cast<int32_t>(d.candidates_considered);
        }
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// ProbePlan::default_plan (policy.cpp:66-82) -> setting column indices, in plan order
int ref_default_plan(const int* cpu, size_t ncpu, const int* gpu, size_t ngpu, int32_t* out,
                     size_t* count) {
    try {
        const auto grid = make_grid(cpu, ncpu, gpu, ngpu);
        const auto plan = policy::ProbePlan::default_plan(grid);
        const auto settings = grid.settings();
        *count = plan.settings.size();
        for (size_t k = 0; k < plan.settings.size(); ++k)
            out[k] = static_cast<int32_t>(
                std::find(settings.begin(), settings.end(), plan.settings[k]) - settings.begin());
        return 0;
    } catch (...) {
        return map_exception();
    }
}

static cf::NcfHyper to_hyper(const ref_ncf_hyper* h) {
    cf::NcfHyper hy;
    if (h == nullptr) return hy;
    hy.app_dim = h->app_dim;
    hy.setting_dim = h->setting_dim;
    hy.hidden.assign(h->hidden, h->hidden + h->n_hidden);
    hy.lr = h->lr;
    hy.max_epochs = h->max_epochs;
    hy.patience = h->patience;
    hy.val_fraction = h->val_fraction;
    hy.batch_size = h->batch_size;
    return hy;
}

// cf::fit (cfcomplete.cpp:63-196) + NcfModel::to_json (:215-236)
int ref_ncf_fit(size_t m, const int* cpu, size_t ncpu, const int* gpu, size_t ngpu,
                const double* values, const uint8_t* mask, const ref_ncf_hyper* h, uint64_t seed,
                char* json_out, size_t cap, size_t* len, ref_ncf_meta* meta) {
    try {
        const auto pm = make_matrix(m, make_grid(cpu, ncpu, gpu, ngpu), values, mask);
        const auto model = cf::fit(pm, to_hyper(h), seed);
        if (meta) {
            meta->seed = model.meta().seed;
            meta->epochs_run = model.meta().epochs_run;
            meta->initial_train_mse = model.meta().initial_train_mse;
            meta->final_train_mse = model.meta().final_train_mse;
            meta->best_val_mse = model.meta().best_val_mse;
        }
        return copy_text(model.to_json(), json_out, cap, len);
    } catch (...) {
        return map_exception();
    }
}

// cf::complete (cfcomplete.cpp:198-213): completed values, row-major m x n
int ref_ncf_complete(size_t m, const int* cpu, size_t ncpu, const int* gpu, size_t ngpu,
                     const double* values, const uint8_t* mask, const ref_ncf_hyper* h,
                     uint64_t seed, double* out) {
    try {
        const auto pm = make_matrix(m, make_grid(cpu, ncpu, gpu, ngpu), values, mask);
        const auto done = cf::complete(pm, to_hyper(h), seed);
        for (size_t i = 0; i < done.rows(); ++i)
            for (size_t j = 0; j < done.cols(); ++j) out[i * done.cols() + j] = done.value(i, j);
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// NcfModel::from_json (:238-265) + NcfModel::predict (:47-58)
int ref_ncf_predict(const char* json, const int64_t* rows, const int64_t* cols, size_t count,
                    double* out) {
    try {
        const auto model = cf::NcfModel::from_json(json);
        for (size_t k = 0; k < count; ++k)
            out[k] = model.predict(static_cast<size_t>(rows[k]), static_cast<size_t>(cols[k]));
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// pred::predictor_from_json (predictor.cpp:302) + pred::predict_perf (:151-157)
int ref_predict_perf(const char* json, const double* counters, size_t count, double* out) {
    try {
        const auto model = pred::predictor_from_json(json);
        for (size_t k = 0; k < count; ++k) {
            const double* c = counters + 7 * k;
            CounterSample s{c[0], c[1], c[2], c[3], c[4], c[5], c[6]};
            out[k] = pred::predict_perf(model, s);
        }
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// the same over `threads` host threads (contiguous sample ranges); returns the
// wall seconds of the prediction loop (model parse excluded), <0 on error
double ref_predict_perf_mt(const char* json, const double* counters, size_t count, int threads, double* out) {
    try {
        const auto model = pred::predictor_from_json(json);
        std::atomic<int> bad{0};
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (int t = 0; t < threads; ++t)
            pool.emplace_back([&, t] {
                const size_t lo = count * t / threads, hi = count * (t + 1) / threads;
                try {
                    for (size_t k = lo; k < hi; ++k) {
                        const double* c = counters + 7 * k;
                        CounterSample s{c[0], c[1], c[2], c[3], c[4], c[5], c[6]};
                        out[k] = pred::predict_perf(model, s);
                    }
                } catch (...) {
                    bad = 1;
                }
            });
        for (auto& th : pool) th.join();
        const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return bad ? -1.0 : secs;
    } catch (...) {
        map_exception();
        return -1.0;
    }
}

// ---- reference pipeline pieces used as input generators for goldens ------

struct ref_spec {
    int32_t archetype;
    double kappa_c, alpha_c, kappa_g, alpha_g, base_runtime_s, cpu_phase_s, noise_sigma;
    double ips_max, mem_tput_max, sm_clock_max;
};

static ref_spec to_c(const sim::WorkloadSpec& w) {
    return {static_cast<int32_t>(w.archetype), w.kappa_c, w.alpha_c, w.kappa_g, w.alpha_g,
            w.base_runtime_s, w.cpu_phase_s, w.noise_sigma, w.counter_scales.ips_max,
            w.counter_scales.mem_tput_max, w.counter_scales.sm_clock_max};
}

// sim::make_suite (simnode.cpp:192-244); role 0 training, 1 evaluation
int ref_make_suite(int32_t g, int32_t c, int32_t b, int32_t ins, uint64_t seed, double noise,
                   int32_t role, double cpu_phase_fraction, const int* cpu, size_t ncpu,
                   const int* gpu, size_t ngpu, ref_spec* out) {
    try {
        sim::SuiteParams p;
        p.counts = {g, c, b, ins};
        p.seed = seed;
        p.noise_sigma = noise;
        p.role = role == 0 ? sim::SuiteRole::training : sim::SuiteRole::evaluation;
        p.cpu_phase_fraction = cpu_phase_fraction;
        const auto suite = sim::make_suite(p, make_grid(cpu, ncpu, gpu, ngpu));
        for (size_t k = 0; k < suite.size(); ++k) out[k] = to_c(suite[k]);
        return 0;
    } catch (...) {
        return map_exception();
    }
}

static sim::WorkloadSpec from_c(const ref_spec& s) {
    sim::WorkloadSpec w;
    w.app_id = "x";
    w.archetype = static_cast<sim::Archetype>(s.archetype);
    w.kappa_c = s.kappa_c;
    w.alpha_c = s.alpha_c;
    w.kappa_g = s.kappa_g;
    w.alpha_g = s.alpha_g;
    w.base_runtime_s = s.base_runtime_s;
    w.cpu_phase_s = s.cpu_phase_s;
    w.noise_sigma = s.noise_sigma;
    w.counter_scales.ips_max = s.ips_max;
    w.counter_scales.mem_tput_max = s.mem_tput_max;
    w.counter_scales.sm_clock_max = s.sm_clock_max;
    return w;
}

// sim::true_perf (simnode.cpp:43-45)
double ref_true_perf(const ref_spec* s, int cpu_cap, int gpu_cap) {
    return sim::true_perf(from_c(*s), PowerSetting{cpu_cap, gpu_cap});
}

// sim::sample_counters (simnode.cpp:98-110) -> 7 doubles
void ref_sample_counters(const ref_spec* s, int cpu_cap, int gpu_cap, double* out7) {
    const auto c = sim::sample_counters(from_c(*s), PowerSetting{cpu_cap, gpu_cap});
    const double v[7] = {c.cpu_cap_w, c.gpu_cap_w, c.ips, c.mem_tput, c.sm_clock, c.fp_active, c.dram_active};
    std::memcpy(out7, v, sizeof v);
}

// The reference CLI's offline phase (opencap_main.cpp:44-64) with RunConfig
// defaults and the given root seed: dense profile matrix + predictor JSON.
int ref_offline_default(uint64_t seed, double* dense_out, size_t* rows, char* pred_json, size_t cap,
                        size_t* len) {
    try {
        const auto grid = PowerGrid::default_grid();
        const auto suite = sim::make_suite(sim::default_training_params(seed), grid);
        const auto profiled = pred::profile_suite(suite, grid, derive_seed(seed, "offline.profile"));
        pred::PredictorHyper hyper;
        hyper.seed = derive_seed(seed, "offline.predictor");
        const auto model = pred::train_predictor(profiled.dataset, hyper);
        const auto& mtx = profiled.matrix;
        *rows = mtx.rows();
        if (dense_out)
            for (size_t i = 0; i < mtx.rows(); ++i)
                for (size_t j = 0; j < mtx.cols(); ++j) dense_out[i * mtx.cols() + j] = mtx.value(i, j);
        return copy_text(pred::predictor_to_json(model), pred_json, cap, len);
    } catch (...) {
        return map_exception();
    }
}

struct ref_online_out {
    int32_t setting_idx;
    double pred_saving, pred_loss;
    int32_t candidates;
    int32_t transition;
    int32_t n_probes;
    int32_t probe_idx[64];
    double probe_val[64];
    double completed_row[4096];
};

// policy::run_open_online (policy.cpp:114-191) for eval-suite app `eval_index`
// with the CLI's seeds (opencap_main.cpp:79-87) against the offline block.
int ref_online_default(uint64_t seed, int eval_index, const double* dense, size_t dense_rows,
                       const char* pred_json, ref_online_out* out) {
    try {
        const auto grid = PowerGrid::default_grid();
        const auto train = sim::make_suite(sim::default_training_params(seed), grid);
        std::vector<std::string> ids;
        for (const auto& s : train) ids.push_back(s.app_id);
        if (ids.size() != dense_rows) throw std::invalid_argument("dense rows mismatch");
        PerformanceMatrix dm(ids, grid);
        for (size_t i = 0; i < dm.rows(); ++i)
            for (size_t j = 0; j < dm.cols(); ++j) dm.set(i, j, dense[i * dm.cols() + j]);
        const auto predictor = pred::predictor_from_json(pred_json);
        const auto eval = sim::make_suite(sim::default_evaluation_params(seed), grid);
        const auto& spec = eval.at(static_cast<size_t>(eval_index));
        const auto cfg = policy::OnlineConfig::defaults(grid);
        const auto oc = policy::run_open_online(spec, dm, predictor, cfg, derive_seed(seed, "open." + spec.app_id));
        const auto settings = grid.settings();
        out->setting_idx = static_cast<int32_t>(
            std::find(settings.begin(), settings.end(), oc.decision.setting) - settings.begin());
        out->pred_saving = oc.decision.pred_saving;
        out->pred_loss = oc.decision.pred_loss;
        out->candidates = static_cast<int32_t>(oc.decision.candidates_considered);
        out->transition = oc.transition_detected ? 1 : 0;
        out->n_probes = static_cast<int32_t>(oc.probes.size());
        for (size_t k = 0; k < oc.probes.size(); ++k) {
            out->probe_idx[k] = static_cast<int32_t>(
                std::find(settings.begin(), settings.end(), oc.probes[k].first) - settings.begin());
            out->probe_val[k] = oc.probes[k].second;
        }
        for (size_t j = 0; j < oc.completed_row.size(); ++j) out->completed_row[j] = oc.completed_row[j];
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// ---- reference arm of bench.py ------------------------------------------
//
// Per-app online completion (cf::complete on dense block + one probed row,
// then policy::select_caps on the completed row) exactly as run_open_online
// steps 3-4 (policy.cpp:178-189), for `napps` apps given as rows of
// `probe_vals`/`probe_mask` (napps x n).  Apps are split over `threads`
// std::threads (independent apps, evaluate_suite policy.cpp:360).  Returns the
// wall seconds spent.
double ref_online_batch(size_t d_rows, const int* cpu, size_t ncpu, const int* gpu, size_t ngpu,
                        const double* dense, const double* probe_vals, const uint8_t* probe_mask,
                        const uint64_t* seeds, size_t napps, double gamma, const ref_ncf_hyper* h,
                        int threads, int32_t* sel_idx, double* sel_saving) {
    const auto grid = make_grid(cpu, ncpu, gpu, ngpu);
    const size_t n = grid.settings().size();
    const auto hy = to_hyper(h);
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    int nt = std::max(1, threads);
    for (int t = 0; t < nt; ++t) {
        pool.emplace_back([&, t] {
            for (size_t a = static_cast<size_t>(t); a < napps; a += static_cast<size_t>(nt)) {
                try {
                    auto ids = app_ids(d_rows);
                    ids.push_back("new");
                    PerformanceMatrix pm(ids, grid);
                    for (size_t i = 0; i < d_rows; ++i)
                        for (size_t j = 0; j < n; ++j) pm.set(i, j, dense[i * n + j]);
                    for (size_t j = 0; j < n; ++j)
                        if (probe_mask[a * n + j]) pm.set(d_rows, j, probe_vals[a * n + j]);
                    const auto done = cf::complete(pm, hy, seeds[a]);
                    std::vector<double> row(n);
                    for (size_t j = 0; j < n; ++j) row[j] = done.value(d_rows, j);
                    const auto d = policy::select_caps(row, policy::SelectionConfig{grid, gamma});
                    const auto settings = grid.settings();
                    sel_idx[a] = static_cast<int32_t>(
                        std::find(settings.begin(), settings.end(), d.setting) - settings.begin());
                    sel_saving[a] = d.pred_saving;
                } catch (...) {
                    sel_idx[a] = -1;
                }
            }
        });
    }
    for (auto& th : pool) th.join();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// nprob independent joint problems (each m x n, dense values + mask): per
// problem cf::complete (cfcomplete.cpp:198-213) then policy::select_caps on
// every completed row.  Problems are spread over `threads` std::threads.
// Returns wall seconds.
double ref_complete_select_batch(size_t nprob, size_t m, const int* cpu, size_t ncpu, const int* gpu, size_t ngpu,
                                 const double* values, const uint8_t* mask, const ref_ncf_hyper* h,
                                 const uint64_t* seeds, double gamma, int threads, int32_t* sel_idx) {
    const auto grid = make_grid(cpu, ncpu, gpu, ngpu);
    const size_t n = grid.settings().size();
    const auto hy = to_hyper(h);
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    const int nt = std::max(1, threads);
    for (int t = 0; t < nt; ++t) {
        pool.emplace_back([&, t] {
            for (size_t p = static_cast<size_t>(t); p < nprob; p += static_cast<size_t>(nt)) {
                try {
                    const auto pm = make_matrix(m, grid, values + p * m * n, mask + p * m * n);
                    const auto done = cf::complete(pm, hy, seeds[p]);
                    const policy::SelectionConfig cfg{grid, gamma};
                    const auto settings = grid.settings();
                    std::vector<double> row(n);
                    for (size_t i = 0; i < m; ++i) {
                        for (size_t j = 0; j < n; ++j) row[j] = done.value(i, j);
                        const auto d = policy::select_caps(row, cfg);
                        sel_idx[p * m + i] = static_cast<int32_t>(
                            std::find(settings.begin(), settings.end(), d.setting) - settings.begin());
                    }
                } catch (...) {
                    for (size_t i = 0; i < m; ++i) sel_idx[p * m + i] = -1;
                }
            }
        });
    }
    for (auto& th : pool) th.join();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// ---- NCF completion + selection of given rows (fused-kernel parity / reference arm)
//
// Builds the reference's NCF model file (the layout of NcfModel::to_json,
// cfcomplete.cpp:215-233 + nn::model_to_json nnkit.cpp:306-330) for a model
// whose app table holds `nrows` rows (the rows to complete, in order), loads it
// with NcfModel::from_json (:235-265), then per row: every unobserved cell via
// NcfModel::predict (:47-58), observed cells verbatim (:208-211), and
// policy::select_caps (policy.cpp:17-64) on the completed row.  Rows are spread
// over `threads` std::threads.  *seconds = wall time of the predict + select
// loop (model parse excluded).
static std::string ncf_model_json(size_t ka, size_t ks, const size_t* hidden, size_t nh, size_t m, size_t n,
                                  const double* params, const uint8_t* app_seen, const uint8_t* setting_seen) {
    std::vector<size_t> dims{ka + ks};
    std::vector<std::string> acts;
    for (size_t l = 0; l < nh; ++l) {
        dims.push_back(hidden[l]);
        acts.emplace_back("selu");
    }
    dims.push_back(1);
    acts.emplace_back("identity");
    nlohmann::json doc;
    doc["format_version"] = 1;
    doc["architecture"] = {{"dims", dims}, {"activations", acts}};
    const double* p = params + m * ka + n * ks;
    nlohmann::json jl = nlohmann::json::array();
    for (size_t l = 0; l + 1 < dims.size(); ++l) {
        nlohmann::json w = nlohmann::json::array();
        for (size_t o = 0; o < dims[l + 1]; ++o) {
            nlohmann::json row = nlohmann::json::array();
            for (size_t i = 0; i < dims[l]; ++i) row.push_back(p[o * dims[l] + i]);
            w.push_back(std::move(row));
        }
        p += dims[l] * dims[l + 1];
        std::vector<double> b(p, p + dims[l + 1]);
        p += dims[l + 1];
        jl.push_back({{"weights", std::move(w)}, {"biases", b}});
    }
    doc["layers"] = std::move(jl);
    const auto table = [](const double* v, size_t rows, size_t dim) {
        nlohmann::json vals = nlohmann::json::array();
        for (size_t i = 0; i < rows; ++i) vals.push_back(std::vector<double>(v + i * dim, v + (i + 1) * dim));
        return nlohmann::json{{"rows", rows}, {"dim", dim}, {"values", std::move(vals)}};
    };
    doc["embeddings"] = {{"app", table(params, m, ka)}, {"setting", table(params + m * ka, n, ks)}};
    doc["observed"] = {{"app_seen", std::vector<uint8_t>(app_seen, app_seen + m)},
                       {"setting_seen", std::vector<uint8_t>(setting_seen, setting_seen + n)}};
    doc["training"] = {{"seed", 0}, {"epochs_run", 0}, {"initial_train_mse", 0.0}, {"final_train_mse", 0.0},
                       {"best_val_mse", 0.0}};
    return doc.dump(2);
}

int ref_ncf_complete_select_rows(size_t ka, size_t ks, const size_t* hidden, size_t nh, size_t nrows,
                                 const double* params, const uint8_t* app_seen, const uint8_t* setting_seen,
                                 const int* cpu, size_t ncpu, const int* gpu, size_t ngpu, const double* values,
                                 const uint8_t* mask, double gamma, int threads, double* completed, int32_t* idx,
                                 double* saving, double* loss, int32_t* ncand, double* seconds) {
    try {
        const auto grid = make_grid(cpu, ncpu, gpu, ngpu);
        const size_t n = grid.settings().size();
        const auto model = cf::NcfModel::from_json(
            ncf_model_json(ka, ks, hidden, nh, nrows, n, params, app_seen, setting_seen));
        const policy::SelectionConfig cfg{grid, gamma};
        const auto settings = grid.settings();
        std::atomic<int> rc{0};
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        const int nt = std::max(1, threads);
        for (int t = 0; t < nt; ++t) {
            pool.emplace_back([&, t] {
                std::vector<double> row(n);
                for (size_t i = static_cast<size_t>(t); i < nrows; i += static_cast<size_t>(nt)) {
                    try {
                        for (size_t j = 0; j < n; ++j)
                            row[j] = mask[i * n + j] ? values[i * n + j] : model.predict(i, j);
                        if (completed) std::copy(row.begin(), row.end(), completed + i * n);
                        const auto d = policy::select_caps(row, cfg);
                        idx[i] = static_cast<int32_t>(std::find(settings.begin(), settings.end(), d.setting) -
                                                      settings.begin());
                        saving[i] = d.pred_saving;
                        loss[i] = d.pred_loss;
                        ncand[i] = static_cast<int32_t>(d.candidates_considered);
                    } catch (...) {
                        rc = map_exception();
                    }
                }
            });
        }
        for (auto& th : pool) th.join();
        if (seconds) *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return rc.load();
    } catch (...) {
        return map_exception();
    }
}

// Rows of the SURVEY §8d joint matrix generated with the reference's own code:
// specs from sim::make_suite (evaluation role, noise 0.01, m/4 per archetype),
// the sampled-setting set of ProbePlan::default_plan, a Bernoulli(p) draw over
// the other columns from Rng(derive_seed(seed, "synth.row", i)), values
// clamp(sim::true_perf * exp(0.01 N(0,1)), 0.01, 1.25) — the generator the
// product's synth.cpp restates (tests/test_synth.py pins the two together), so
// the bench's reference arm needs no product code.  as_float: values rounded
// through FP32 (as the FP32 CSR carries them).
int ref_joint_rows_dense(int64_t m, const int* cpu, size_t ncpu, const int* gpu, size_t ngpu, double density,
                         int64_t dense_rows, uint64_t seed, const int64_t* rows, int64_t nrows, int as_float,
                         double* values, uint8_t* mask) {
    try {
        const auto grid = make_grid(cpu, ncpu, gpu, ngpu);
        const auto settings = grid.settings();
        const int64_t n = static_cast<int64_t>(settings.size());
        sim::SuiteParams sp;
        const auto q = static_cast<int32_t>(m / 4);
        sp.counts = {q, q, q, static_cast<int32_t>(m - 3 * static_cast<int64_t>(q))};
        sp.seed = seed;
        sp.noise_sigma = 0.01;
        sp.role = sim::SuiteRole::evaluation;
        sp.cpu_phase_fraction = 0.0;
        const auto specs = sim::make_suite(sp, grid);
        const auto plan = policy::ProbePlan::default_plan(grid);
        std::vector<uint8_t> in_plan(static_cast<size_t>(n), 0);
        for (const auto& st : plan.settings)
            in_plan[static_cast<size_t>(std::find(settings.begin(), settings.end(), st) - settings.begin())] = 1;
        double p = 0.0;
        if (m > dense_rows) {
            const double want = density * static_cast<double>(m) * static_cast<double>(n);
            const double fixed = static_cast<double>(dense_rows) * n + static_cast<double>(m - dense_rows) *
                                 static_cast<double>(plan.settings.size());
            p = (want - fixed) / (static_cast<double>(m - dense_rows) * static_cast<double>(n - plan.settings.size()));
            p = std::min(1.0, std::max(0.0, p));
        }
        std::memset(mask, 0, static_cast<size_t>(nrows * n));
        std::memset(values, 0, sizeof(double) * static_cast<size_t>(nrows * n));
        for (int64_t r = 0; r < nrows; ++r) {
            const int64_t i = rows[r];
            if (i < 0 || i >= m) throw std::out_of_range("row out of range");
            Rng rng(derive_seed(seed, "synth.row", static_cast<uint64_t>(i)));
            for (int64_t j = 0; j < n; ++j) {
                bool obs = i < dense_rows || in_plan[static_cast<size_t>(j)];
                if (!obs) obs = rng.uniform() < p;
                if (!obs) continue;
                const double v = std::clamp(sim::true_perf(specs[static_cast<size_t>(i)], settings[static_cast<size_t>(j)]) *
                                                std::exp(0.01 * rng.normal()),
                                            0.01, 1.25);
                values[r * n + j] = as_float ? static_cast<double>(static_cast<float>(v)) : v;
                mask[r * n + j] = 1;
            }
        }
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// read_matrix_csv_file (core.cpp:250-254) then, if out_path, write_matrix_csv
// (core.cpp:208-211): the reference's own loader / writer for format tests
int ref_matrix_csv_roundtrip(const char* in_path, const char* out_path, size_t* m, size_t* n, size_t* nnz) {
    try {
        const auto pm = read_matrix_csv_file(in_path);
        if (m) *m = pm.rows();
        if (n) *n = pm.cols();
        if (nnz) *nnz = pm.observed_count();
        if (out_path) write_matrix_csv(pm, std::string(out_path));
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// pred::load_predictor (predictor.cpp:325-331): 0 or the mapped exception
int ref_load_predictor(const char* path, int* has_stats) {
    try {
        const auto model = pred::load_predictor(path);
        if (has_stats) *has_stats = model.has_stats ? 1 : 0;
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// One minibatch step of cf::fit's loop body (cfcomplete.cpp:155-178) built from
// the reference's own components at a given model size, for the composed CPU
// figure of a fit too large to run (C2/C3): dense zeroing of the
// embedding-gradient tables, 32 x nn::backprop_sample, nn::AdamState::step over
// every parameter block.  Returns the mean seconds per step over `iters` steps
// (parts[0..2]: zeroing, backprop, adam).
double ref_time_fit_step(size_t m, size_t n, size_t k, const size_t* hidden, size_t nh, int iters, double* parts) {
    try {
        Rng rng(1);
        auto app = nn::EmbeddingTable::random(m, k, rng);
        auto set = nn::EmbeddingTable::random(n, k, rng);
        std::vector<std::size_t> dims{2 * k};
        std::vector<nn::Activation> acts;
        for (size_t l = 0; l < nh; ++l) {
            dims.push_back(hidden[l]);
            acts.push_back(nn::Activation::selu);
        }
        dims.push_back(1);
        acts.push_back(nn::Activation::identity);
        nn::MlpModel mlp(dims, acts, rng);
        std::vector<nn::ParamView> params{{app.values.data(), app.values.size()}, {set.values.data(), set.values.size()}};
        for (const auto& b : mlp.param_blocks()) params.push_back(b);
        nn::AdamState adam(params, 1e-3);
        nn::GradBlocks grads;
        std::vector<double> input_grad;
        double tz = 0, tb = 0, ta = 0;
        using clk = std::chrono::steady_clock;
        for (int it = 0; it < iters; ++it) {
            const auto t0 = clk::now();
            grads.assign(params.size(), {});
            grads[0].assign(app.values.size(), 0.0);
            grads[1].assign(set.values.size(), 0.0);
            nn::GradBlocks mlp_grads;
            for (const auto& layer : mlp.layers()) {
                mlp_grads.emplace_back(layer.weights.size(), 0.0);
                mlp_grads.emplace_back(layer.biases.size(), 0.0);
            }
            const auto t1 = clk::now();
            for (int s = 0; s < 32; ++s) {
                const size_t i = rng.next_u64() % m, j = rng.next_u64() % n;
                std::vector<double> x(app.row(i).begin(), app.row(i).end());
                x.insert(x.end(), set.row(j).begin(), set.row(j).end());
                const double y[] = {0.5};
                nn::backprop_sample(mlp, x, y, 1.0 / 32, mlp_grads, input_grad);
                for (size_t c = 0; c < k; ++c) grads[0][i * k + c] += input_grad[c];
                for (size_t c = 0; c < k; ++c) grads[1][j * k + c] += input_grad[k + c];
            }
            for (size_t b = 0; b < mlp_grads.size(); ++b) grads[2 + b] = std::move(mlp_grads[b]);
            const auto t2 = clk::now();
            adam.step(params, grads);
            const auto t3 = clk::now();
            tz += std::chrono::duration<double>(t1 - t0).count();
            tb += std::chrono::duration<double>(t2 - t1).count();
            ta += std::chrono::duration<double>(t3 - t2).count();
        }
        if (parts) {
            parts[0] = tz / iters;
            parts[1] = tb / iters;
            parts[2] = ta / iters;
        }
        return (tz + tb + ta) / iters;
    } catch (...) {
        map_exception();
        return -1.0;
    }
}

// sim::run (simnode.cpp) of a spec at one setting: its GPU-power trace (the stream the
// phase detector watches); returns the sample count (<= cap) and the sampling interval
int ref_run_trace(const ref_spec* spec, int cpu_cap, int gpu_cap, uint64_t seed, double* power, size_t cap,
                  size_t* count, double* dt) {
    try {
        const auto r = sim::run(from_c(*spec), PowerSetting{cpu_cap, gpu_cap}, seed);
        const size_t n = std::min(cap, r.trace.samples.size());
        for (size_t i = 0; i < n; ++i) power[i] = r.trace.samples[i].gpu_power_w;
        *count = r.trace.samples.size();
        *dt = r.trace.dt;
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// phase::detect_offline (phasedet.cpp:58-67) on a GPU-power stream (armed = 0), or the
// reference Detector fed under run_open_online's arming rule (armed = 1, policy.cpp:138-140):
// index of the firing sample or -1
int ref_detect(const double* power, size_t n, double delta_s, double window_s, double p_th, int armed,
               int64_t* fire) {
    try {
        phase::DetectorConfig cfg{delta_s, window_s, p_th};
        if (!armed) {
            sim::PowerTrace tr;
            tr.dt = delta_s;
            for (size_t i = 0; i < n; ++i) tr.samples.push_back({static_cast<double>(i + 1) * delta_s, 0.0, power[i]});
            const auto t = phase::detect_offline(tr, cfg);
            *fire = -1;
            if (t)
                for (size_t i = 0; i < n; ++i)
                    if (tr.samples[i].t_s == *t) {
                        *fire = static_cast<int64_t>(i);
                        break;
                    }
            return 0;
        }
        phase::Detector det(cfg);
        bool on = false;
        *fire = -1;
        for (size_t i = 0; i < n; ++i) {
            if (!on && power[i] < cfg.p_th_w) on = true;
            if (on && det.feed(power[i]) == phase::Decision::transition) {
                *fire = static_cast<int64_t>(i);
                break;
            }
        }
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// policy::evaluate_suite (policy.cpp:355-405) for the CLI's default evaluation suite and the
// given baseline policies (1 no_cap, 2 gpu_cap_only, 3 cpu_cap_only, 4 oracle) on the default
// grid, plus the simulator runs its truth tables come from (the same sim::run calls
// measure_truth makes): base[a][r] and runs[a][j][r] = {runtime_s, avg_power_w, energy_j}.
// rows[a][p] = {cpu, gpu, true_perf, true_loss, energy_j, avg_power_w, efficiency, pred_saving},
// aggs[p] = {mean_efficiency, mean_gain_vs_no_cap, mean_true_loss, mean_true_perf}
int ref_eval_default(uint64_t seed, int reps, double gamma, const int32_t* pols, size_t npol, double* rows,
                     double* aggs, double* base, double* runs, size_t* napps_out) {
    try {
        const auto grid = PowerGrid::default_grid();
        const auto suite = sim::make_suite(sim::default_evaluation_params(seed), grid);
        std::vector<policy::PolicyKind> kinds;
        for (size_t p = 0; p < npol; ++p) kinds.push_back(static_cast<policy::PolicyKind>(pols[p]));
        auto cfg = policy::EvalConfig::defaults(grid);
        cfg.repetitions = reps;
        cfg.online.selection.gamma = gamma;
        PerformanceMatrix dense({"unused"}, grid);
        pred::PredictorModel predictor;
        const auto report = policy::evaluate_suite(suite, kinds, dense, predictor, cfg, seed);
        const auto settings = grid.settings();
        const size_t n = settings.size();
        for (size_t a = 0; a < suite.size(); ++a) {
            const auto app_seed = derive_seed(seed, "eval." + suite[a].app_id);
            for (int r = 0; r < reps; ++r) {
                const auto rep_seed = derive_seed(app_seed, "rep", static_cast<uint64_t>(r));
                const auto b = sim::run(suite[a], grid.baseline(), rep_seed);
                double* bo = base + (a * reps + r) * 3;
                bo[0] = b.runtime_s;
                bo[1] = b.avg_power_w;
                bo[2] = b.energy_j;
                for (size_t j = 0; j < n; ++j) {
                    const auto c = sim::run(suite[a], settings[j], rep_seed);
                    double* o = runs + ((a * n + j) * reps + r) * 3;
                    o[0] = c.runtime_s;
                    o[1] = c.avg_power_w;
                    o[2] = c.energy_j;
                }
            }
        }
        for (size_t q = 0; q < report.rows.size(); ++q) {
            const auto& w = report.rows[q];
            double* o = rows + q * 8;
            o[0] = w.setting.cpu_cap_w;
            o[1] = w.setting.gpu_cap_w;
            o[2] = w.true_perf;
            o[3] = w.true_loss;
            o[4] = w.energy_j;
            o[5] = w.avg_power_w;
            o[6] = w.efficiency;
            o[7] = w.pred_saving;
        }
        for (size_t p = 0; p < report.aggregates.size(); ++p) {
            const auto& g = report.aggregates[p];
            double* o = aggs + p * 4;
            o[0] = g.mean_efficiency;
            o[1] = g.mean_gain_vs_no_cap;
            o[2] = g.mean_true_loss;
            o[3] = g.mean_true_perf;
        }
        *napps_out = suite.size();
        return 0;
    } catch (...) {
        return map_exception();
    }
}

}  // extern "C"




