// Synthetic input generation for benches and tests (host C++).
//
// Inputs are generated on the host exactly as the reference would produce
// them, so the GPU never regenerates (or re-rounds) anything:
//   * workload specs  — sim::make_suite (simnode.cpp:192-244)
//   * ground truth    — sim::true_perf (simnode.cpp:43-45)
//   * offline block   — pred::profile_suite's normalized-performance matrix
//                       (predictor.cpp:45-69 with sim::run's log-normal noise,
//                       simnode.cpp:125-128), RunConfig defaults
//   * online apps     — the eval suite probed on ProbePlan::default_plan with
//                       the same noise form; cf::complete seeds as
//                       run_open_online derives them (policy.cpp:181,
//                       opencap_main.cpp:86)
//   * joint matrices  — SURVEY §8d: first D rows dense, every other row the
//                       default plan + a Bernoulli(p) draw over the remaining
//                       columns from Rng(derive_seed(seed,"synth.row",i)), values
//                       clamp(true_perf*exp(0.01*N(0,1)), 0.01, 1.25).
// The Rng transforms and derive_seed are the reference's (rng.hpp:13-60) on
// std::mt19937_64 and the host libm, so specs are bit-identical to the
// reference's (tests/test_synth.py).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "../../include/ocg.h"
#include "ocg_common.cuh"

namespace {

struct Rng {
    std::mt19937_64 e;
    explicit Rng(uint64_t s) : e(s) {}
    double uniform() { return static_cast<double>(e() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    double normal() {
        double u1 = uniform();
        while (u1 <= 0.0) u1 = uniform();
        const double u2 = uniform();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925287 * u2);
    }
};

uint64_t derive_seed(uint64_t root, const std::string& tag, uint64_t n = 0) {
    return ocg::derive_seed_h(root, ocg::splitmix64(ocg::fnv1a(tag.c_str())), n);
}

const char* kArchName[4] = {"gpu_sensitive", "cpu_sensitive", "both_sensitive", "insensitive"};

struct Band {
    double lo, hi;
};

double draw_band(Rng& rng, Band tr, Band lo, Band hi, bool training) {
    if (training) return rng.uniform(tr.lo, tr.hi);
    const bool high = rng.uniform() < 0.5;
    const Band b = high ? hi : lo;
    return rng.uniform(b.lo, b.hi);
}

// sim::make_suite (simnode.cpp:192-244)
std::vector<ocg_workload_spec> make_suite(const int32_t counts[4], uint64_t seed, bool training, double noise,
                                          double cpu_phase_fraction, double c_lo, double c_hi, double g_lo,
                                          double g_hi, std::vector<std::string>* ids) {
    const Band knee_tr{0.30, 0.80}, knee_ev_lo{0.15, 0.28}, knee_ev_hi{0.82, 0.95};
    const Band alpha_tr{0.70, 1.20}, alpha_ev_lo{0.55, 0.68}, alpha_ev_hi{1.25, 1.45};
    const Band rt_tr{8.0, 12.0}, rt_ev{12.5, 16.0};
    const Band scale_tr{0.95, 1.05}, scale_ev_lo{0.92, 0.95}, scale_ev_hi{1.05, 1.08};
    Rng rng(derive_seed(seed, training ? "suite.training" : "suite.evaluation"));
    std::vector<ocg_workload_spec> suite;
    for (int a = 0; a < 4; ++a) {
        for (int k = 0; k < counts[a]; ++k) {
            ocg_workload_spec w{};
            w.archetype = a;
            const bool cpu_sens = a == 1 || a == 2, gpu_sens = a == 0 || a == 2;
            if (cpu_sens) {
                const double f = draw_band(rng, knee_tr, knee_ev_lo, knee_ev_hi, training);
                w.kappa_c = c_lo + (c_hi - c_lo) * f;
            } else {
                w.kappa_c = rng.uniform(0.4, 0.95) * c_lo;
            }
            w.alpha_c = cpu_sens ? draw_band(rng, alpha_tr, alpha_ev_lo, alpha_ev_hi, training) : rng.uniform(0.5, 1.5);
            if (gpu_sens) {
                const double f = draw_band(rng, knee_tr, knee_ev_lo, knee_ev_hi, training);
                w.kappa_g = g_lo + (g_hi - g_lo) * f;
            } else {
                w.kappa_g = rng.uniform(0.4, 0.95) * g_lo;
            }
            w.alpha_g = gpu_sens ? draw_band(rng, alpha_tr, alpha_ev_lo, alpha_ev_hi, training) : rng.uniform(0.5, 1.5);
            w.base_runtime_s = training ? rng.uniform(rt_tr.lo, rt_tr.hi) : rng.uniform(rt_ev.lo, rt_ev.hi);
            w.cpu_phase_s = rng.uniform() < cpu_phase_fraction ? rng.uniform(6.0, 14.0) : 0.0;
            w.noise_sigma = noise;
            w.ips_max = 2.0e11 * draw_band(rng, scale_tr, scale_ev_lo, scale_ev_hi, training);
            w.mem_tput_max = 2.5e11 * draw_band(rng, scale_tr, scale_ev_lo, scale_ev_hi, training);
            w.sm_clock_max = 1410.0;
            suite.push_back(w);
            if (ids) ids->push_back(std::string(training ? "tr" : "ev") + "_" + kArchName[a] + "_" + std::to_string(k));
        }
    }
    return suite;
}

inline double knee(double cap, double kappa, double alpha) { return cap >= kappa ? 1.0 : std::pow(cap / kappa, alpha); }
inline double true_perf(const ocg_workload_spec& w, int c, int g) {
    return knee(c, w.kappa_c, w.alpha_c) * knee(g, w.kappa_g, w.alpha_g);
}
inline double clampv(double v) { return std::min(std::max(v, 0.01), 1.25); }

struct Grid {
    const int32_t* cpu;
    int32_t ncpu;
    const int32_t* gpu;
    int32_t ngpu;
    int64_t n() const { return static_cast<int64_t>(ncpu) * ngpu; }
};

std::vector<int32_t> default_plan(const Grid& g) {
    const int32_t wc[6] = {g.ncpu - 1, 0, 0, g.ncpu - 1, g.ncpu / 2, g.ncpu / 4};
    const int32_t wg[6] = {g.ngpu - 1, 0, g.ngpu - 1, 0, g.ngpu / 2, g.ngpu / 4};
    std::vector<int32_t> plan;
    for (int k = 0; k < 6; ++k) {
        const int32_t col = wc[k] * g.ngpu + wg[k];
        if (std::find(plan.begin(), plan.end(), col) == plan.end()) plan.push_back(col);
    }
    return plan;
}

std::vector<ocg_workload_spec> joint_specs(int64_t m, uint64_t seed, const Grid& g) {
    const int32_t q = static_cast<int32_t>(m / 4);
    const int32_t counts[4] = {q, q, q, static_cast<int32_t>(m - 3 * static_cast<int64_t>(q))};
    return make_suite(counts, seed, false, 0.01, 0.0, g.cpu[0], g.cpu[g.ncpu - 1], g.gpu[0], g.gpu[g.ngpu - 1],
                      nullptr);
}

double bernoulli_p(int64_t m, int64_t n, double density, int64_t dense_rows, int64_t plan) {
    if (m <= dense_rows) return 0.0;
    const double want = density * static_cast<double>(m) * static_cast<double>(n);
    const double fixed = static_cast<double>(dense_rows) * n + static_cast<double>(m - dense_rows) * plan;
    const double p = (want - fixed) / (static_cast<double>(m - dense_rows) * static_cast<double>(n - plan));
    return std::min(1.0, std::max(0.0, p));
}

// one row of the §8d joint matrix; emit(col, value) in column order
template <typename F>
void gen_row(int64_t i, int64_t dense_rows, const Grid& g, const std::vector<uint8_t>& in_plan, double p,
             const ocg_workload_spec& w, uint64_t seed, F&& emit) {
    Rng rng(derive_seed(seed, "synth.row", static_cast<uint64_t>(i)));
    const int64_t n = g.n();
    for (int64_t j = 0; j < n; ++j) {
        bool obs = i < dense_rows || in_plan[j];
        if (!obs) obs = rng.uniform() < p;
        if (!obs) continue;
        const int c = g.cpu[j / g.ngpu], gg = g.gpu[j % g.ngpu];
        const double v = clampv(true_perf(w, c, gg) * std::exp(0.01 * rng.normal()));
        emit(j, v);
    }
}

template <typename F>
void parallel_rows(int64_t m, int nthreads, F&& body) {
    nthreads = std::max(1, std::min<int>(nthreads, 256));
    std::vector<std::thread> pool;
    for (int t = 0; t < nthreads; ++t)
        pool.emplace_back([&, t] {
            const int64_t lo = m * t / nthreads, hi = m * (t + 1) / nthreads;
            for (int64_t i = lo; i < hi; ++i) body(i);
        });
    for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

int ocg_synth_suite(const int32_t counts[4], uint64_t seed, int role, double noise_sigma, double cpu_phase_fraction,
                    const int32_t* cpu, int32_t ncpu, const int32_t* gpu, int32_t ngpu, ocg_workload_spec* out) {
    if (!cpu || !gpu || ncpu <= 0 || ngpu <= 0) return OCG_E_INVALID;
    const auto s = make_suite(counts, seed, role == 0, noise_sigma, cpu_phase_fraction, cpu[0], cpu[ncpu - 1], gpu[0],
                              gpu[ngpu - 1], nullptr);
    std::copy(s.begin(), s.end(), out);
    return OCG_OK;
}

int ocg_synth_counters(const ocg_workload_spec* specs, int64_t nspecs, const int32_t* cpu, int32_t ncpu,
                       const int32_t* gpu, int32_t ngpu, int cpu_phase, int nthreads, double* out) {
    if (!specs || !cpu || !gpu || !out || ncpu <= 0 || ngpu <= 0 || nspecs < 0) return OCG_E_INVALID;
    const int64_t n = static_cast<int64_t>(ncpu) * ngpu;
    parallel_rows(nspecs, nthreads, [&](int64_t a) {
        const ocg_workload_spec& w = specs[a];
        for (int32_t i = 0; i < ncpu; ++i)
            for (int32_t j = 0; j < ngpu; ++j) {
                const double fc = knee(cpu[i], w.kappa_c, w.alpha_c), fg = knee(gpu[j], w.kappa_g, w.alpha_g);
                double* c = out + (a * n + static_cast<int64_t>(i) * ngpu + j) * 7;
                c[0] = cpu[i];
                c[1] = gpu[j];
                c[2] = w.ips_max * fc;
                c[3] = w.mem_tput_max * std::pow(fc, 0.8);
                if (cpu_phase) {
                    c[4] = 0.3 * w.sm_clock_max;  // idle clock floor
                    c[5] = 0.02;
                    c[6] = 0.05;
                } else {
                    c[4] = w.sm_clock_max * std::sqrt(std::min(1.0, gpu[j] / w.kappa_g));
                    c[5] = fg;
                    c[6] = std::min(1.0, 0.9 * fg + 0.1);
                }
            }
    });
    return OCG_OK;
}

double ocg_true_perf(const ocg_workload_spec* w, int32_t cpu_cap, int32_t gpu_cap) {
    return true_perf(*w, cpu_cap, gpu_cap);
}

// pred::profile_suite matrix for RunConfig defaults (opencap_main.cpp:47-48):
// training suite default_training_params(seed), profile seed derive_seed(seed,"offline.profile")
int ocg_synth_offline_block(uint64_t seed, const int32_t* cpu, int32_t ncpu, const int32_t* gpu, int32_t ngpu,
                            double* out, int64_t* rows) {
    const int32_t counts[4] = {3, 3, 2, 2};  // default_training_params (simnode.cpp:170-178)
    std::vector<std::string> ids;
    const auto suite = make_suite(counts, seed, true, 0.01, 0.0, cpu[0], cpu[ncpu - 1], gpu[0], gpu[ngpu - 1], &ids);
    const uint64_t pseed = derive_seed(seed, "offline.profile");
    const Grid g{cpu, ncpu, gpu, ngpu};
    const int64_t n = g.n();
    const int cb = cpu[ncpu - 1], gb = gpu[ngpu - 1];
    for (size_t a = 0; a < suite.size(); ++a) {
        const auto& w = suite[a];
        const auto nfr = [&](int c, int gg) {  // noise_free_runtime (simnode.cpp:47-49)
            return w.cpu_phase_s / knee(c, w.kappa_c, w.alpha_c) + w.base_runtime_s / true_perf(w, c, gg);
        };
        const double base = nfr(cb, gb);
        for (int64_t j = 0; j < n; ++j) {
            const int c = cpu[j / ngpu], gg = gpu[j % ngpu];
            Rng rng(derive_seed(pseed, "profile." + ids[a], static_cast<uint64_t>(j)));
            const double noise = std::exp(w.noise_sigma * rng.normal());  // sim::run (simnode.cpp:127)
            const double runtime = nfr(c, gg) * noise;
            out[a * n + j] = std::min(base / runtime, 1.25);
        }
    }
    *rows = static_cast<int64_t>(suite.size());
    return OCG_OK;
}

// eval-suite apps probed on the default plan; cf::complete seeds per app
int ocg_synth_online_apps(int64_t napps, uint64_t seed, const int32_t* cpu, int32_t ncpu, const int32_t* gpu,
                          int32_t ngpu, double* probe_vals, uint8_t* probe_mask, uint64_t* seeds) {
    const int32_t q = static_cast<int32_t>(napps / 4);
    const int32_t counts[4] = {q, q, q, static_cast<int32_t>(napps - 3 * static_cast<int64_t>(q))};
    std::vector<std::string> ids;
    const auto suite = make_suite(counts, seed, false, 0.01, 0.0, cpu[0], cpu[ncpu - 1], gpu[0], gpu[ngpu - 1], &ids);
    const Grid g{cpu, ncpu, gpu, ngpu};
    const int64_t n = g.n();
    const auto plan = default_plan(g);
    std::memset(probe_mask, 0, static_cast<size_t>(napps * n));
    std::memset(probe_vals, 0, sizeof(double) * static_cast<size_t>(napps * n));
    for (int64_t a = 0; a < napps; ++a) {
        Rng rng(derive_seed(seed, "synth.probe." + ids[a]));
        for (const int32_t j : plan) {
            const double v = clampv(true_perf(suite[a], cpu[j / ngpu], gpu[j % ngpu]) * std::exp(0.01 * rng.normal()));
            probe_vals[a * n + j] = v;
            probe_mask[a * n + j] = 1;
        }
        seeds[a] = derive_seed(derive_seed(seed, "open." + ids[a]), "online.ncf." + ids[a]);
    }
    return OCG_OK;
}

// rows [row0, row1) of the m-row joint matrix; row_ptr is local (row_ptr[0] = 0)
int ocg_synth_csr_range_count(int64_t m, int64_t row0, int64_t row1, const int32_t* cpu, int32_t ncpu,
                              const int32_t* gpu, int32_t ngpu, double density, int64_t dense_rows, uint64_t seed,
                              int nthreads, int64_t* row_ptr) {
    if (row0 < 0 || row1 > m || row0 > row1) return OCG_E_RANGE;
    const Grid g{cpu, ncpu, gpu, ngpu};
    const auto specs = joint_specs(m, seed, g);
    const auto plan = default_plan(g);
    std::vector<uint8_t> in_plan(static_cast<size_t>(g.n()), 0);
    for (auto j : plan) in_plan[j] = 1;
    const double p = bernoulli_p(m, g.n(), density, dense_rows, static_cast<int64_t>(plan.size()));
    parallel_rows(row1 - row0, nthreads, [&](int64_t r) {
        const int64_t i = row0 + r;
        int64_t c = 0;
        gen_row(i, dense_rows, g, in_plan, p, specs[i], seed, [&](int64_t, double) { ++c; });
        row_ptr[r + 1] = c;
    });
    row_ptr[0] = 0;
    for (int64_t r = 0; r < row1 - row0; ++r) row_ptr[r + 1] += row_ptr[r];
    return OCG_OK;
}

int ocg_synth_csr_range_fill(int64_t m, int64_t row0, int64_t row1, const int32_t* cpu, int32_t ncpu,
                             const int32_t* gpu, int32_t ngpu, double density, int64_t dense_rows, uint64_t seed,
                             int nthreads, const int64_t* row_ptr, int32_t* col, float* val32, double* val64) {
    if (row0 < 0 || row1 > m || row0 > row1) return OCG_E_RANGE;
    const Grid g{cpu, ncpu, gpu, ngpu};
    const auto specs = joint_specs(m, seed, g);
    const auto plan = default_plan(g);
    std::vector<uint8_t> in_plan(static_cast<size_t>(g.n()), 0);
    for (auto j : plan) in_plan[j] = 1;
    const double p = bernoulli_p(m, g.n(), density, dense_rows, static_cast<int64_t>(plan.size()));
    parallel_rows(row1 - row0, nthreads, [&](int64_t r) {
        const int64_t i = row0 + r;
        int64_t q = row_ptr[r];
        gen_row(i, dense_rows, g, in_plan, p, specs[i], seed, [&](int64_t j, double v) {
            col[q] = static_cast<int32_t>(j);
            if (val32) val32[q] = static_cast<float>(v);
            if (val64) val64[q] = v;
            ++q;
        });
    });
    return OCG_OK;
}

int ocg_synth_csr_count(int64_t m, const int32_t* cpu, int32_t ncpu, const int32_t* gpu, int32_t ngpu,
                        double density, int64_t dense_rows, uint64_t seed, int nthreads, int64_t* row_ptr) {
    return ocg_synth_csr_range_count(m, 0, m, cpu, ncpu, gpu, ngpu, density, dense_rows, seed, nthreads, row_ptr);
}

int ocg_synth_csr_fill(int64_t m, const int32_t* cpu, int32_t ncpu, const int32_t* gpu, int32_t ngpu,
                       double density, int64_t dense_rows, uint64_t seed, int nthreads, const int64_t* row_ptr,
                       int32_t* col, float* val32, double* val64) {
    return ocg_synth_csr_range_fill(m, 0, m, cpu, ncpu, gpu, ngpu, density, dense_rows, seed, nthreads, row_ptr, col,
                                    val32, val64);
}

// selected rows of the joint matrix as dense values + mask (nrows x n)
int ocg_synth_rows_dense(int64_t m, const int32_t* cpu, int32_t ncpu, const int32_t* gpu, int32_t ngpu, double density,
                         int64_t dense_rows, uint64_t seed, const int64_t* rows, int64_t nrows, double* values,
                         uint8_t* mask) {
    const Grid g{cpu, ncpu, gpu, ngpu};
    const auto specs = joint_specs(m, seed, g);
    const auto plan = default_plan(g);
    std::vector<uint8_t> in_plan(static_cast<size_t>(g.n()), 0);
    for (auto j : plan) in_plan[j] = 1;
    const double p = bernoulli_p(m, g.n(), density, dense_rows, static_cast<int64_t>(plan.size()));
    const int64_t n = g.n();
    std::memset(mask, 0, static_cast<size_t>(nrows * n));
    std::memset(values, 0, sizeof(double) * static_cast<size_t>(nrows * n));
    for (int64_t r = 0; r < nrows; ++r) {
        const int64_t i = rows[r];
        if (i < 0 || i >= m) return OCG_E_RANGE;
        gen_row(i, dense_rows, g, in_plan, p, specs[i], seed, [&](int64_t j, double v) {
            values[r * n + j] = static_cast<double>(static_cast<float>(v));  // as the FP32 CSR carries it
            mask[r * n + j] = 1;
        });
    }
    return OCG_OK;
}

// ground truth sim::true_perf (simnode.cpp:43-45) of every cell of selected rows of the
// same joint matrix (nrows x n) — held-out quality of a completion (bench quality block)
int ocg_synth_true_rows(int64_t m, const int32_t* cpu, int32_t ncpu, const int32_t* gpu, int32_t ngpu, uint64_t seed,
                        const int64_t* rows, int64_t nrows, double* out) {
    const Grid g{cpu, ncpu, gpu, ngpu};
    const auto specs = joint_specs(m, seed, g);
    const int64_t n = g.n();
    for (int64_t r = 0; r < nrows; ++r) {
        const int64_t i = rows[r];
        if (i < 0 || i >= m) return OCG_E_RANGE;
        for (int64_t j = 0; j < n; ++j) out[r * n + j] = true_perf(specs[i], g.cpu[j / g.ngpu], g.gpu[j % g.ngpu]);
    }
    return OCG_OK;
}

}  // extern "C"
