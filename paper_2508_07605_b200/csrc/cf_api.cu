// The reference's cf:: operator surface over one whole matrix:
//   ocg_cf_fit      <- cf::fit       (cfcomplete.hpp:59, cfcomplete.cpp:63-196)
//   ocg_cf_complete <- cf::complete  (cfcomplete.hpp:63, cfcomplete.cpp:198-213),
//                      optionally fused with policy::select_caps per row
// with a solver switch: NCF_REF (FP64, the reference's operation order: bit-
// identical), NCF_FAST (FP32 NCF on the same schedule), ALS (the new rank-k
// solver, no reference counterpart).  Host code validates exactly what the
// reference's PerformanceMatrix / NcfHyper / PowerGrid would reject and maps
// the exception type to the OCG_* code; all arithmetic runs on the GPU.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/ocg.h"
#include "ncf_joint.h"

int ocg_internal_fail(int code, const std::string& msg);
cudaStream_t ocg_internal_stream(ocg_ctx* ctx);
int ocg_internal_sm_count(ocg_ctx* ctx);

namespace {

int fail(int code, const std::string& msg) { return ocg_internal_fail(code, msg); }

// cf::fit hyper checks (cfcomplete.cpp:64-66) + MlpModel widths (nnkit.cpp:51-53)
int check_ncf_hyper(const ocg_ncf_hyper* h) {
    if (h == nullptr) return fail(OCG_E_INVALID, "ncf: null hyperparameters");
    if (h->app_dim <= 0 || h->setting_dim <= 0 || !(h->lr > 0) || h->max_epochs <= 0 || h->batch_size <= 0 ||
        !(h->val_fraction >= 0) || h->val_fraction >= 1 || h->n_hidden < 0 || h->n_hidden > 8)
        return fail(OCG_E_INVALID, "ncf: bad hyperparameters");
    for (int64_t l = 0; l < h->n_hidden; ++l)
        if (h->hidden[l] <= 0) return fail(OCG_E_INVALID, "zero layer width");
    return OCG_OK;
}

}  // namespace

// CSR as the reference's PerformanceMatrix would accept it cell by cell
// (core.cpp:142-148): column index in range (out_of_range), value finite in
// (0, 1.25] (invalid_argument); plus the CSR invariants (row_ptr[0] = 0,
// non-decreasing; columns strictly ascending within a row: one value per cell).
int ocg_csr_validate(int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val64,
                     const float* val32) {
    if (m <= 0 || n <= 0) return fail(OCG_E_INVALID, "empty matrix");
    if (!row_ptr || !col || (!val64 && !val32)) return fail(OCG_E_INVALID, "csr: null argument");
    if (row_ptr[0] != 0) return fail(OCG_E_INVALID, "csr: row_ptr[0] must be 0");
    for (int64_t i = 0; i < m; ++i) {
        const int64_t b = row_ptr[i], e = row_ptr[i + 1];
        if (e < b) return fail(OCG_E_INVALID, "csr: row_ptr must be non-decreasing");
        for (int64_t q = b; q < e; ++q) {
            const int32_t c = col[q];
            if (c < 0 || c >= n) return fail(OCG_E_RANGE, "matrix index out of range");
            if (q > b && col[q - 1] >= c)
                return fail(OCG_E_INVALID, "csr: columns must be strictly ascending within a row");
            const double v = val64 ? val64[q] : static_cast<double>(val32[q]);
            if (!std::isfinite(v) || v <= 0.0 || v > 1.25)
                return fail(OCG_E_INVALID, "normalized performance outside (0, 1.25]");
        }
    }
    return OCG_OK;
}

extern "C" {

int ocg_cf_fit(ocg_ctx* ctx, int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
               const ocg_ncf_hyper* hyper, uint64_t seed, int solver, int lane, double* params, uint8_t* app_seen,
               uint8_t* setting_seen, ocg_ncf_meta* meta) {
    int rc = check_ncf_hyper(hyper);
    if (rc) return rc;
    if (solver == OCG_SOLVER_ALS)
        return fail(OCG_E_INVALID, "cf_fit: ALS has no NcfModel (use ocg_cf_complete or ocg_als_plan_*)");
    if (solver != OCG_SOLVER_NCF_REF && solver != OCG_SOLVER_NCF_FAST) return fail(OCG_E_INVALID, "cf_fit: unknown solver");
    if (lane != OCG_LANE_SCALAR && lane != OCG_LANE_AVX2) return fail(OCG_E_INVALID, "unknown lane");
    if ((rc = ocg_csr_validate(m, n, row_ptr, col, val, nullptr))) return rc;
    if (row_ptr[m] == 0) return fail(OCG_E_INVALID, "ncf: matrix has no observed entries");
    if (!ctx) return fail(OCG_E_INVALID, "null context");
    std::string err;
    rc = ocg::joint_ncf_fit(ocg_internal_stream(ctx), ocg_internal_sm_count(ctx), m, n, row_ptr, col, val, *hyper,
                            seed, solver == OCG_SOLVER_NCF_FAST ? OCG_NCF_FAST : OCG_NCF_EXACT, lane, params, app_seen,
                            setting_seen, meta, nullptr, err);
    if (rc) return fail(rc, err);
    return OCG_OK;
}

int ocg_cf_fit_stats(ocg_ctx* ctx, int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
                     const ocg_ncf_hyper* hyper, uint64_t seed, int solver, int lane, double* params, uint8_t* app_seen,
                     uint8_t* setting_seen, ocg_ncf_meta* meta, int64_t* steps, double* device_ms) {
    int rc = check_ncf_hyper(hyper);
    if (rc) return rc;
    if (solver != OCG_SOLVER_NCF_REF && solver != OCG_SOLVER_NCF_FAST) return fail(OCG_E_INVALID, "cf_fit: unknown solver");
    if (lane != OCG_LANE_SCALAR && lane != OCG_LANE_AVX2) return fail(OCG_E_INVALID, "unknown lane");
    if ((rc = ocg_csr_validate(m, n, row_ptr, col, val, nullptr))) return rc;
    if (row_ptr[m] == 0) return fail(OCG_E_INVALID, "ncf: matrix has no observed entries");
    if (!ctx) return fail(OCG_E_INVALID, "null context");
    std::string err;
    ocg::JointFitStats st;
    rc = ocg::joint_ncf_fit(ocg_internal_stream(ctx), ocg_internal_sm_count(ctx), m, n, row_ptr, col, val, *hyper,
                            seed, solver == OCG_SOLVER_NCF_FAST ? OCG_NCF_FAST : OCG_NCF_EXACT, lane, params, app_seen,
                            setting_seen, meta, &st, err);
    if (rc) return fail(rc, err);
    if (steps) *steps = st.steps;
    if (device_ms) *device_ms = st.device_ms;
    return OCG_OK;
}

int ocg_cf_complete(ocg_ctx* ctx, int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
                    const ocg_ncf_hyper* hyper, const ocg_als_hyper* als, uint64_t seed, int solver, int lane,
                    const int32_t* cpu_caps, int32_t ncpu, const int32_t* gpu_caps, int32_t ngpu, double gamma,
                    double* completed, int32_t* idx, double* saving, double* loss, int32_t* ncand) {
    if (solver != OCG_SOLVER_NCF_REF && solver != OCG_SOLVER_NCF_FAST && solver != OCG_SOLVER_ALS)
        return fail(OCG_E_INVALID, "cf_complete: unknown solver");
    if (lane != OCG_LANE_SCALAR && lane != OCG_LANE_AVX2) return fail(OCG_E_INVALID, "unknown lane");
    int rc;
    if (solver == OCG_SOLVER_ALS) {
        if (!als) return fail(OCG_E_INVALID, "als: null hyperparameters");
    } else if ((rc = check_ncf_hyper(hyper))) {
        return rc;
    }
    if ((rc = ocg_csr_validate(m, n, row_ptr, col, val, nullptr))) return rc;
    // cf::complete (cfcomplete.cpp:199-205): every row needs an observed entry
    for (int64_t i = 0; i < m; ++i)
        if (row_ptr[i + 1] == row_ptr[i])
            return fail(OCG_E_INVALID, "complete: app row " + std::to_string(i) +
                                           " has no observed entries (probe it first)");
    // selection grid (PowerGrid, core.cpp:38-45); without one, a placeholder
    // grid of the right width carries the completion (decisions not returned)
    std::vector<int32_t> pc, pg;
    const bool want_sel = cpu_caps != nullptr;
    if (want_sel) {
        if (!gpu_caps || ncpu <= 0 || ngpu <= 0) return fail(OCG_E_INVALID, "cap list is empty");
        if (static_cast<int64_t>(ncpu) * ngpu != n) return fail(OCG_E_INVALID, "grid does not match the matrix width");
    } else {
        pc = {1};
        pg.resize(static_cast<size_t>(n));
        for (int64_t j = 0; j < n; ++j) pg[static_cast<size_t>(j)] = static_cast<int32_t>(j + 1);
        cpu_caps = pc.data();
        gpu_caps = pg.data();
        ncpu = 1;
        ngpu = static_cast<int32_t>(n);
        gamma = 0.05;
    }
    if (!ctx) return fail(OCG_E_INVALID, "null context");
    const bool full = row_ptr[m] == m * n;  // fully observed: returned unchanged, no fit (:206)
    cudaStream_t s = ocg_internal_stream(ctx);
    const int64_t chunk = std::max<int64_t>(1, (int64_t(1) << 24) / n);
    if (solver == OCG_SOLVER_ALS) {
        std::vector<float> v32(static_cast<size_t>(row_ptr[m]));
        for (size_t q = 0; q < v32.size(); ++q) v32[q] = static_cast<float>(val[q]);
        ocg_als_plan* P = nullptr;
        if ((rc = ocg_als_plan_create(ctx, m, row_ptr, col, v32.data(), 0, cpu_caps, ncpu, gpu_caps, ngpu, als, gamma, &P)))
            return rc;
        std::unique_ptr<ocg_als_plan, void (*)(ocg_als_plan*)> g(P, ocg_als_plan_destroy);
        if ((rc = ocg_als_plan_run(P, nullptr, nullptr))) return rc;
        if (want_sel && (rc = ocg_als_plan_results(P, idx, saving, loss, ncand, nullptr, nullptr))) return rc;
        if (completed)
            for (int64_t r0 = 0; r0 < m; r0 += chunk)
                if ((rc = ocg_als_plan_completed_rows(P, r0, std::min(chunk, m - r0), completed + r0 * n))) return rc;
        return OCG_OK;
    }
    // NCF: fit (unless fully observed) then the fused imputation + selection
    const int64_t nparams_emb = m * hyper->app_dim + n * hyper->setting_dim;
    int64_t T = hyper->app_dim + hyper->setting_dim, mlp = 0;
    for (int64_t l = 0; l < hyper->n_hidden; ++l) {
        mlp += T * hyper->hidden[l] + hyper->hidden[l];
        T = hyper->hidden[l];
    }
    mlp += T + 1;
    std::vector<double> params(static_cast<size_t>(nparams_emb + mlp), 0.0);
    std::vector<uint8_t> aseen(static_cast<size_t>(m), 1), sseen(static_cast<size_t>(n), 1);
    if (!full) {
        if ((rc = ocg_cf_fit(ctx, m, n, row_ptr, col, val, hyper, seed, solver, lane, params.data(), aseen.data(),
                             sseen.data(), nullptr)))
            return rc;
    }
    ocg_ncf_model* M = nullptr;
    if ((rc = ocg_ncf_model_create(ctx, hyper, m, n, params.data(), aseen.data(), sseen.data(), &M))) return rc;
    std::unique_ptr<ocg_ncf_model, void (*)(ocg_ncf_model*)> gm(M, ocg_ncf_model_destroy);
    ocg_ncf_plan* P = nullptr;
    const int prec = solver == OCG_SOLVER_NCF_REF ? OCG_NCF_EXACT : OCG_NCF_FAST;
    rc = ocg_ncf_plan_create(M, row_ptr, col, val, 0, cpu_caps, ncpu, gpu_caps, ngpu, gamma, prec, lane, &P);
    if (rc == OCG_E_UNSUPPORTED && prec == OCG_NCF_FAST)  // FP32 tensor-core inference needs hidden {32, 16}
        rc = ocg_ncf_plan_create(M, row_ptr, col, val, 0, cpu_caps, ncpu, gpu_caps, ngpu, gamma, OCG_NCF_EXACT, lane, &P);
    if (rc) return rc;
    std::unique_ptr<ocg_ncf_plan, void (*)(ocg_ncf_plan*)> gp(P, ocg_ncf_plan_destroy);
    if ((rc = ocg_ncf_plan_run(P, nullptr, nullptr))) return rc;
    if ((rc = ocg_ncf_plan_results(P, want_sel ? idx : nullptr, want_sel ? saving : nullptr,
                                   want_sel ? loss : nullptr, want_sel ? ncand : nullptr)))
        return rc;
    if (completed) {
        std::vector<int64_t> rows;
        for (int64_t r0 = 0; r0 < m; r0 += chunk) {
            const int64_t cnt = std::min(chunk, m - r0);
            rows.resize(static_cast<size_t>(cnt));
            for (int64_t i = 0; i < cnt; ++i) rows[static_cast<size_t>(i)] = r0 + i;
            if ((rc = ocg_ncf_plan_completed_rows(P, rows.data(), cnt, completed + r0 * n))) return rc;
        }
    }
    (void)s;
    return OCG_OK;
}

}  // extern "C"
