// Host orchestration of the fused NCF completion + selection path (C-ABI in
// include/ocg.h, ocg_ncf_model_* / ocg_ncf_plan_*).  A model is a fitted
// cf::NcfModel resident in HBM; a plan binds it to a sparse matrix (CSR of the
// observed cells) and a PowerGrid and runs cf::complete's imputation fused with
// policy::select_caps for every row (ncf_select.cu).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/ocg.h"
#include "ncf_select.h"

// from capi.cu
int ocg_internal_fail(int code, const std::string& msg);
cudaStream_t ocg_internal_stream(ocg_ctx* ctx);
int ocg_internal_sm_count(ocg_ctx* ctx);

namespace {

#define NCF_CUDA(call)                                                                                    \
    do {                                                                                                  \
        cudaError_t e_ = (call);                                                                          \
        if (e_ != cudaSuccess) return ocg_internal_fail(OCG_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

template <typename T>
struct Buf {
    T* p = nullptr;
    bool own = true;
    ~Buf() {
        if (p && own) cudaFree(p);
    }
    cudaError_t alloc(size_t n) {
        if (p && own) cudaFree(p);
        p = nullptr;
        own = true;
        return n ? cudaMalloc(&p, sizeof(T) * n) : cudaSuccess;
    }
};

constexpr double kLambda = 1.0507009873554805;  // nnkit.hpp:20

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// CSR checks the reference's PerformanceMatrix enforces cell by cell
// (core.cpp:142-148: out_of_range for an index, invalid_argument for a value
// outside (0, 1.25]); plus sorted / unique columns (a matrix holds one value per cell)
__global__ void ncf_validate_kernel(int64_t m, int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                    const double* __restrict__ val, int* err) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    int bits = 0;
    for (int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < m; i += nw) {
        const int64_t b = rp[i], e = rp[i + 1];
        for (int64_t q = b + lane; q < e; q += 32) {
            const int32_t c = col[q];
            const double v = val[q];
            if (c < 0 || c >= n) bits |= 1 << OCG_E_RANGE;
            if (q > b && col[q - 1] >= c) bits |= 1 << OCG_E_INVALID;
            if (!(v > 0.0 && v <= 1.25)) bits |= 1 << OCG_E_INVALID;  // NaN fails too
        }
    }
    if (bits) atomicOr(err, bits);
}

// columns whose setting embedding is cold but which still hold an unobserved cell
__global__ void ncf_cold_cols_kernel(int64_t m, int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                     const uint8_t* __restrict__ setting_seen, int32_t* counts) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= rp[m]) return;
    const int32_t c = col[t];
    if (c >= 0 && c < n && !setting_seen[c]) atomicAdd(counts + c, 1);
}

int first_error(int bits) {
    static const int order[] = {OCG_E_RANGE, OCG_E_INVALID, OCG_E_COLD, OCG_E_UNSUPPORTED};
    for (int c : order)
        if (bits & (1 << c)) return c;
    return OCG_OK;
}

const char* error_text(int code) {
    switch (code) {
        case OCG_E_RANGE: return "matrix index out of range";
        case OCG_E_INVALID: return "complete: an app row has no observed entries, or a matrix value lies outside (0, 1.25] / columns unsorted";
        case OCG_E_COLD: return "ncf: cold app row / setting column (no observed entries at fit time)";
        case OCG_E_UNSUPPORTED: return "ncf fast path: |W0 . x| too large for the split exponential";
        default: return "ok";
    }
}

}  // namespace

struct ocg_ncf_model {
    ocg_ctx* ctx = nullptr;
    ocg_ncf_hyper h{};
    int64_t m = 0, n = 0, nparams = 0;
    int L = 0;
    int dims[5] = {};
    int64_t off_w[4] = {}, off_b[4] = {}, set_off = 0;
    Buf<double> P;
    Buf<uint8_t> app_seen, setting_seen;
    std::vector<double> mlp;          // host copy of the MLP block (W0 b0 W1 b1 ...)
    std::vector<int32_t> cold_cols;   // setting columns with setting_seen == 0
};

struct ocg_ncf_plan {
    ocg_ncf_model* model = nullptr;
    int64_t m = 0, n = 0, nnz = 0;
    int ngpu = 0, precision = 0, lane = 0;
    double gamma = 0.0, e_base = 0.0;
    Buf<int64_t> row_ptr;
    Buf<int32_t> col;
    Buf<double> val;
    int64_t col_cap = 0;
    Buf<int32_t> cpu, gpu, idx, ncand, cold_counts;
    Buf<double> saving, loss;
    Buf<ocg::NcfRowState> rows;
    Buf<int> err;
    // fast path
    Buf<float> A, EA, BE;
    Buf<uint4> w1img;
    Buf<ocg::NcfFastScale> scale;
    CUtensorMap tmap{};
    int e_w = 0;
    float b1[16] = {}, w2[16] = {}, b2 = 0.0f;
    cudaEvent_t ev[4] = {};
    // pipelined serving (ocg_ncf_plan_stage / _results_async): the next CSR copied on a side
    // stream into the spare buffers while the current step runs; swapped in by the next run
    Buf<int64_t> rp_next;
    Buf<int32_t> col_next;
    Buf<double> val_next;
    int64_t next_cap = 0, staged_nnz = 0;
    bool staged = false;
    cudaStream_t copy_stream = nullptr;
    // ev_free[0]: recorded after the last run that read the current buffers, ev_free[1]: the
    // same for the spare ones (swapped with the buffers), so staging into the spare set waits
    // only for the run before last, not for the run in flight
    cudaEvent_t ev_staged = nullptr, ev_free[2] = {nullptr, nullptr}, ev_results = nullptr;
    bool free_rec[2] = {false, false};
    int* h_err = nullptr;  // pinned error bits of the last async results
    ~ocg_ncf_plan() {
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        if (copy_stream) cudaStreamSynchronize(copy_stream);
        if (ev_staged) cudaEventDestroy(ev_staged);
        for (auto e : ev_free)
            if (e) cudaEventDestroy(e);
        if (ev_results) cudaEventDestroy(ev_results);
        if (copy_stream) cudaStreamDestroy(copy_stream);
        if (h_err) cudaFreeHost(h_err);
    }
};

static ocg::NcfSelArgs sel_args(ocg_ncf_plan* P) {
    const ocg_ncf_model* M = P->model;
    ocg::NcfSelArgs a{};
    a.m = P->m;
    a.n = P->n;
    a.ka = static_cast<int>(M->h.app_dim);
    a.ks = static_cast<int>(M->h.setting_dim);
    a.L = M->L;
    for (int l = 0; l <= M->L; ++l) a.dims[l] = M->dims[l];
    for (int l = 0; l < M->L; ++l) {
        a.off_w[l] = M->off_w[l];
        a.off_b[l] = M->off_b[l];
    }
    a.set_off = M->set_off;
    a.P = M->P.p;
    a.app_seen = M->app_seen.p;
    a.setting_seen = M->setting_seen.p;
    a.row_ptr = P->row_ptr.p;
    a.col = P->col.p;
    a.val = P->val.p;
    a.cpu = P->cpu.p;
    a.gpu = P->gpu.p;
    a.ngpu = P->ngpu;
    a.e_base = P->e_base;
    a.gamma = P->gamma;
    a.rows = P->rows.p;
    a.idx = P->idx.p;
    a.saving = P->saving.p;
    a.loss = P->loss.p;
    a.ncand = P->ncand.p;
    a.err = P->err.p;
    return a;
}

static ocg::NcfFastArgs fast_args(ocg_ncf_plan* P, const ocg::NcfSelArgs& a) {
    ocg::NcfFastArgs f{};
    f.s = a;
    f.A = P->A.p;
    f.EA = P->EA.p;
    f.BE = P->BE.p;
    f.w1img = P->w1img.p;
    f.scale = P->scale.p;
    std::memcpy(f.b1, P->b1, sizeof(f.b1));
    std::memcpy(f.w2, P->w2, sizeof(f.w2));
    f.b2 = P->b2;
    f.e_w = P->e_w;
    return f;
}

extern "C" {

int ocg_ncf_model_create(ocg_ctx* ctx, const ocg_ncf_hyper* h, int64_t m, int64_t n, const double* params,
                         const uint8_t* app_seen, const uint8_t* setting_seen, ocg_ncf_model** out) {
    if (!ctx || !h || !params || !app_seen || !setting_seen || !out)
        return ocg_internal_fail(OCG_E_INVALID, "ncf model: null argument");
    *out = nullptr;
    if (h->app_dim <= 0 || h->setting_dim <= 0 || h->n_hidden < 0 || h->n_hidden > 3)
        return ocg_internal_fail(OCG_E_INVALID, "ncf model: bad hyperparameters");
    if (m <= 0 || n <= 0) return ocg_internal_fail(OCG_E_INVALID, "ncf model: empty embedding table");
    if (h->app_dim + h->setting_dim > 64) return ocg_internal_fail(OCG_E_UNSUPPORTED, "ncf model: input wider than 64");
    auto M = std::make_unique<ocg_ncf_model>();
    M->ctx = ctx;
    M->h = *h;
    M->m = m;
    M->n = n;
    M->L = static_cast<int>(h->n_hidden) + 1;
    M->dims[0] = static_cast<int>(h->app_dim + h->setting_dim);
    for (int l = 0; l < h->n_hidden; ++l) {
        if (h->hidden[l] <= 0 || h->hidden[l] > 64) return ocg_internal_fail(OCG_E_UNSUPPORTED, "ncf model: hidden width");
        M->dims[l + 1] = static_cast<int>(h->hidden[l]);
    }
    M->dims[M->L] = 1;
    int64_t off = m * h->app_dim;
    M->set_off = off;
    off += n * h->setting_dim;
    for (int l = 0; l < M->L; ++l) {
        M->off_w[l] = off;
        off += static_cast<int64_t>(M->dims[l]) * M->dims[l + 1];
        M->off_b[l] = off;
        off += M->dims[l + 1];
    }
    M->nparams = off;
    // MlpModel::check_finite (nnkit.cpp:106-113), as NcfModel::from_json / fit end with it
    for (int64_t e = M->off_w[0]; e < off; ++e)
        if (!std::isfinite(params[e])) return ocg_internal_fail(OCG_E_LOGIC, "non-finite weight");
    M->mlp.assign(params + M->off_w[0], params + off);
    for (int64_t j = 0; j < n; ++j)
        if (!setting_seen[j]) M->cold_cols.push_back(static_cast<int32_t>(j));
    cudaStream_t s = ocg_internal_stream(ctx);
    NCF_CUDA(M->P.alloc(static_cast<size_t>(off)));
    NCF_CUDA(M->app_seen.alloc(static_cast<size_t>(m)));
    NCF_CUDA(M->setting_seen.alloc(static_cast<size_t>(n)));
    NCF_CUDA(cudaMemcpyAsync(M->P.p, params, sizeof(double) * off, cudaMemcpyHostToDevice, s));
    NCF_CUDA(cudaMemcpyAsync(M->app_seen.p, app_seen, m, cudaMemcpyHostToDevice, s));
    NCF_CUDA(cudaMemcpyAsync(M->setting_seen.p, setting_seen, n, cudaMemcpyHostToDevice, s));
    NCF_CUDA(cudaStreamSynchronize(s));
    *out = M.release();
    return OCG_OK;
}

int ocg_ncf_model_from_json_text(ocg_ctx* ctx, const char* text, ocg_ncf_model** out) {
    if (!ctx || !text || !out) return ocg_internal_fail(OCG_E_INVALID, "ncf model: null argument");
    ocg_ncf_hyper h{};
    int64_t m = 0, n = 0, np = 0;
    int rc = ocg_ncf_model_from_json(text, &h, &m, &n, &np, nullptr, nullptr, nullptr, nullptr);
    if (rc) return rc;
    std::vector<double> params(static_cast<size_t>(np));
    std::vector<uint8_t> as(static_cast<size_t>(m)), ss(static_cast<size_t>(n));
    rc = ocg_ncf_model_from_json(text, &h, &m, &n, &np, params.data(), as.data(), ss.data(), nullptr);
    if (rc) return rc;
    return ocg_ncf_model_create(ctx, &h, m, n, params.data(), as.data(), ss.data(), out);
}

void ocg_ncf_model_destroy(ocg_ncf_model* model) { delete model; }

static int plan_upload(ocg_ncf_plan* P, const int64_t* row_ptr, const int32_t* col, const double* val) {
    // row_ptr on the host: non-decreasing from 0 (the per-entry checks run on the device)
    if (row_ptr[0] != 0) return ocg_internal_fail(OCG_E_INVALID, "ncf plan: row_ptr[0] != 0");
    for (int64_t i = 0; i < P->m; ++i)
        if (row_ptr[i + 1] < row_ptr[i]) return ocg_internal_fail(OCG_E_INVALID, "ncf plan: row_ptr decreases");
    const int64_t nnz = row_ptr[P->m];
    cudaStream_t s = ocg_internal_stream(P->model->ctx);
    if (nnz > P->col_cap) {
        NCF_CUDA(cudaStreamSynchronize(s));
        P->col_cap = nnz + nnz / 16 + 1024;
        NCF_CUDA(P->col.alloc(static_cast<size_t>(P->col_cap)));
        NCF_CUDA(P->val.alloc(static_cast<size_t>(P->col_cap)));
    }
    P->nnz = nnz;
    NCF_CUDA(cudaMemcpyAsync(P->row_ptr.p, row_ptr, sizeof(int64_t) * (P->m + 1), cudaMemcpyHostToDevice, s));
    if (nnz > 0) {
        NCF_CUDA(cudaMemcpyAsync(P->col.p, col, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, s));
        NCF_CUDA(cudaMemcpyAsync(P->val.p, val, sizeof(double) * nnz, cudaMemcpyHostToDevice, s));
    }
    return OCG_OK;
}

int ocg_ncf_plan_create(ocg_ncf_model* M, const int64_t* row_ptr, const int32_t* col, const double* val, int on_device,
                        const int32_t* cpu, int32_t ncpu, const int32_t* gpu, int32_t ngpu, double gamma, int precision,
                        int lane, ocg_ncf_plan** out) {
    if (!M || !row_ptr || !col || !val || !cpu || !gpu || !out) return ocg_internal_fail(OCG_E_INVALID, "ncf plan: null argument");
    *out = nullptr;
    // PowerGrid (core.cpp:38-45) and SelectionConfig (policy.cpp:19-25) checks
    for (int k = 0; k < ncpu; ++k)
        if (cpu[k] <= 0 || (k > 0 && cpu[k] <= cpu[k - 1]))
            return ocg_internal_fail(OCG_E_INVALID, "cpu caps must be positive and strictly increasing");
    for (int k = 0; k < ngpu; ++k)
        if (gpu[k] <= 0 || (k > 0 && gpu[k] <= gpu[k - 1]))
            return ocg_internal_fail(OCG_E_INVALID, "gpu caps must be positive and strictly increasing");
    if (ncpu <= 0 || ngpu <= 0) return ocg_internal_fail(OCG_E_INVALID, "cap list is empty");
    if (!(gamma > 0.0 && gamma < 1.0)) return ocg_internal_fail(OCG_E_INVALID, "select_caps: gamma must lie in (0, 1)");
    if (static_cast<int64_t>(ncpu) * ngpu != M->n)
        return ocg_internal_fail(OCG_E_INVALID, "ncf plan: the grid does not match the model's setting table");
    if (precision != OCG_NCF_EXACT && precision != OCG_NCF_FAST)
        return ocg_internal_fail(OCG_E_INVALID, "ncf plan: precision must be OCG_NCF_EXACT or OCG_NCF_FAST");
    if (lane != OCG_LANE_SCALAR && lane != OCG_LANE_AVX2) return ocg_internal_fail(OCG_E_INVALID, "ncf plan: bad lane");
    auto P = std::make_unique<ocg_ncf_plan>();
    P->model = M;
    P->m = M->m;
    P->n = M->n;
    P->ngpu = ngpu;
    P->gamma = gamma;
    P->precision = precision;
    P->lane = lane;
    P->e_base = static_cast<double>(cpu[ncpu - 1] + gpu[ngpu - 1]);
    ocg::NcfSelArgs probe{};
    probe.L = M->L;
    for (int l = 0; l <= M->L; ++l) probe.dims[l] = M->dims[l];
    if (precision == OCG_NCF_FAST && !ocg::ncf_fast_shape_ok(probe))
        return ocg_internal_fail(OCG_E_UNSUPPORTED, "ncf fast path: hidden layers must be {32, 16} (the reference default)");
    cudaStream_t s = ocg_internal_stream(M->ctx);
    if (on_device) {
        P->row_ptr.p = const_cast<int64_t*>(row_ptr);
        P->row_ptr.own = false;
        P->col.p = const_cast<int32_t*>(col);
        P->col.own = false;
        P->val.p = const_cast<double*>(val);
        P->val.own = false;
        NCF_CUDA(cudaMemcpy(&P->nnz, row_ptr + P->m, sizeof(int64_t), cudaMemcpyDeviceToHost));
    } else {
        NCF_CUDA(P->row_ptr.alloc(static_cast<size_t>(P->m + 1)));
        int rc = plan_upload(P.get(), row_ptr, col, val);
        if (rc) return rc;
    }
    NCF_CUDA(P->cpu.alloc(static_cast<size_t>(ncpu)));
    NCF_CUDA(P->gpu.alloc(static_cast<size_t>(ngpu)));
    NCF_CUDA(cudaMemcpyAsync(P->cpu.p, cpu, sizeof(int32_t) * ncpu, cudaMemcpyHostToDevice, s));
    NCF_CUDA(cudaMemcpyAsync(P->gpu.p, gpu, sizeof(int32_t) * ngpu, cudaMemcpyHostToDevice, s));
    NCF_CUDA(P->rows.alloc(static_cast<size_t>(P->m)));
    NCF_CUDA(P->idx.alloc(static_cast<size_t>(P->m)));
    NCF_CUDA(P->ncand.alloc(static_cast<size_t>(P->m)));
    NCF_CUDA(P->saving.alloc(static_cast<size_t>(P->m)));
    NCF_CUDA(P->loss.alloc(static_cast<size_t>(P->m)));
    NCF_CUDA(P->err.alloc(1));
    if (!M->cold_cols.empty()) NCF_CUDA(P->cold_counts.alloc(static_cast<size_t>(P->n)));
    for (auto& e : P->ev) NCF_CUDA(cudaEventCreate(&e));
    if (precision == OCG_NCF_FAST) {
        NCF_CUDA(P->A.alloc(static_cast<size_t>(P->m) * 32));
        NCF_CUDA(P->EA.alloc(static_cast<size_t>(P->m) * 32));
        NCF_CUDA(P->BE.alloc(static_cast<size_t>(P->n) * ocg::kNsColFloats));
        NCF_CUDA(P->scale.alloc(1));
        NCF_CUDA(P->w1img.alloc(192));
        // lambda W1 (SELU's lambda folded out of layer 0), power-of-two scaled, FP16 hi/lo,
        // in the UMMA K-major core-matrix layout (ncf_select.cu aoff: slab / group / chunk / row)
        const double* W1 = M->mlp.data() + (M->off_w[1] - M->off_w[0]);
        const double* B1 = M->mlp.data() + (M->off_b[1] - M->off_w[0]);
        const double* W2 = M->mlp.data() + (M->off_w[2] - M->off_w[0]);
        const double* B2 = M->mlp.data() + (M->off_b[2] - M->off_w[0]);
        double mx = 0.0;
        for (int e = 0; e < 16 * 32; ++e) mx = std::max(mx, std::fabs(kLambda * W1[e]));
        int e2 = 0;
        std::frexp(mx > 0.0 ? mx : 1.0, &e2);
        P->e_w = 14 - e2;
        std::vector<uint16_t> img(1536, 0);  // hi | lo | -hi
        for (int p = 0; p < 16; ++p)
            for (int o = 0; o < 32; ++o) {
                const float w = static_cast<float>(std::ldexp(kLambda * W1[p * 32 + o], P->e_w));
                const __half hi = __float2half_rn(w);
                const __half lo = __float2half_rn(w - __half2float(hi));
                const int kk = o & 15, slab = o >> 4;
                const int off = slab * 256 + (p >> 3) * 128 + (kk >> 3) * 64 + (p & 7) * 8 + (kk & 7);  // in halves
                uint16_t hb, lb;
                std::memcpy(&hb, &hi, 2);
                std::memcpy(&lb, &lo, 2);
                img[off] = hb;
                img[512 + off] = lb;
                img[1024 + off] = static_cast<uint16_t>(hb ^ 0x8000u);
            }
        NCF_CUDA(cudaMemcpyAsync(P->w1img.p, img.data(), 3072, cudaMemcpyHostToDevice, s));
        NCF_CUDA(cudaStreamSynchronize(s));
        for (int p = 0; p < 16; ++p) {
            // the dense epilogue works in log2 units (ncf_select.cu): b1 log2(e), lambda W2 ln(2)
            P->b1[p] = static_cast<float>(B1[p] * 1.4426950408889634);
            P->w2[p] = static_cast<float>(kLambda * W2[p] * 0.6931471805599453);
        }
        P->b2 = static_cast<float>(B2[0]);
        auto enc = tensor_map_encoder();
        if (!enc) return ocg_internal_fail(OCG_E_CUDA, "cuTensorMapEncodeTiled unavailable");
        const cuuint64_t dims[2] = {static_cast<cuuint64_t>(ocg::kNsColFloats), static_cast<cuuint64_t>(P->n)};
        const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ocg::kNsColFloats) * 4};
        const cuuint32_t box[2] = {static_cast<cuuint32_t>(ocg::kNsColFloats), static_cast<cuuint32_t>(ocg::kNsTileCols)};
        const cuuint32_t es[2] = {1, 1};
        const CUresult r = enc(&P->tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, P->BE.p, dims, strides, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return ocg_internal_fail(OCG_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
    }
    NCF_CUDA(cudaStreamSynchronize(s));
    *out = P.release();
    return OCG_OK;
}

int ocg_ncf_plan_upload(ocg_ncf_plan* P, const int64_t* row_ptr, const int32_t* col, const double* val) {
    if (!P || !row_ptr || !col || !val) return ocg_internal_fail(OCG_E_INVALID, "ncf plan: null argument");
    if (!P->row_ptr.own) return ocg_internal_fail(OCG_E_INVALID, "ncf plan: plan uses caller device buffers");
    return plan_upload(P, row_ptr, col, val);
}

static int plan_launch(ocg_ncf_plan* P, const int64_t* d_list, int64_t nlist, double* d_completed, float* phase_ms) {
    cudaStream_t s = ocg_internal_stream(P->model->ctx);
    const int sm = ocg_internal_sm_count(P->model->ctx);
    if (P->staged) {  // swap in the CSR staged by ocg_ncf_plan_stage (a device-side wait, no host sync)
        NCF_CUDA(cudaStreamWaitEvent(s, P->ev_staged, 0));
        std::swap(P->row_ptr.p, P->rp_next.p);
        std::swap(P->col.p, P->col_next.p);
        std::swap(P->val.p, P->val_next.p);
        std::swap(P->col_cap, P->next_cap);
        std::swap(P->ev_free[0], P->ev_free[1]);
        std::swap(P->free_rec[0], P->free_rec[1]);
        P->nnz = P->staged_nnz;
        P->staged = false;
    }
    ocg::NcfSelArgs a = sel_args(P);
    NCF_CUDA(cudaEventRecord(P->ev[0], s));
    NCF_CUDA(cudaMemsetAsync(P->err.p, 0, sizeof(int), s));
    if (P->m > 0) ncf_validate_kernel<<<sm * 8, 256, 0, s>>>(P->m, P->n, P->row_ptr.p, P->col.p, P->val.p, P->err.p);
    NCF_CUDA(cudaGetLastError());
    ocg::NcfFastArgs f{};
    if (P->precision == OCG_NCF_FAST) {
        f = fast_args(P, a);
        NCF_CUDA(ocg::ncf_launch_fast_prep(f, s));
    }
    NCF_CUDA(ocg::ncf_launch_base(a, P->lane, s));
    NCF_CUDA(ocg::ncf_launch_rowprep(a, sm, s));
    NCF_CUDA(cudaEventRecord(P->ev[1], s));
    a.row_list = d_list;
    a.nlist = nlist;
    a.completed = d_completed;
    if (d_list) NCF_CUDA(ocg::ncf_launch_list_observed(a, s));  // observed cells of the listed rows
    if (P->precision == OCG_NCF_FAST) {
        f.s = a;
        NCF_CUDA(ocg::ncf_launch_fast(f, &P->tmap, s));
    } else {
        NCF_CUDA(ocg::ncf_launch_exact(a, P->lane, sm, s));
    }
    NCF_CUDA(cudaEventRecord(P->ev[2], s));
    if (P->ev_free[0]) {  // every read of this step's CSR is behind this point: its buffers may be restaged
        NCF_CUDA(cudaEventRecord(P->ev_free[0], s));
        P->free_rec[0] = true;
    }
    if (phase_ms) {
        NCF_CUDA(cudaEventSynchronize(P->ev[2]));
        NCF_CUDA(cudaEventElapsedTime(phase_ms + 0, P->ev[0], P->ev[1]));
        NCF_CUDA(cudaEventElapsedTime(phase_ms + 1, P->ev[1], P->ev[2]));
    }
    return OCG_OK;
}

int ocg_ncf_plan_run(ocg_ncf_plan* P, float* total_ms, float* phase_ms) {
    if (!P) return ocg_internal_fail(OCG_E_INVALID, "null plan");
    float ph[2];
    int rc = plan_launch(P, nullptr, 0, nullptr, (total_ms || phase_ms) ? ph : nullptr);
    if (rc) return rc;
    if (total_ms) *total_ms = ph[0] + ph[1];
    if (phase_ms) {
        phase_ms[0] = ph[0];
        phase_ms[1] = ph[1];
    }
    return OCG_OK;
}

static int plan_error(ocg_ncf_plan* P) {
    cudaStream_t s = ocg_internal_stream(P->model->ctx);
    int bits = 0;
    NCF_CUDA(cudaMemcpyAsync(&bits, P->err.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    NCF_CUDA(cudaStreamSynchronize(s));
    if (!P->model->cold_cols.empty() && !(bits & ((1 << OCG_E_RANGE) | (1 << OCG_E_INVALID)))) {
        // a cold setting column fails predict unless every row observes it (cfcomplete.cpp:53-55)
        NCF_CUDA(cudaMemsetAsync(P->cold_counts.p, 0, sizeof(int32_t) * P->n, s));
        if (P->nnz > 0)
            ncf_cold_cols_kernel<<<static_cast<unsigned>((P->nnz + 255) / 256), 256, 0, s>>>(
                P->m, P->n, P->row_ptr.p, P->col.p, P->model->setting_seen.p, P->cold_counts.p);
        NCF_CUDA(cudaGetLastError());
        std::vector<int32_t> cnt(static_cast<size_t>(P->n));
        NCF_CUDA(cudaMemcpyAsync(cnt.data(), P->cold_counts.p, sizeof(int32_t) * P->n, cudaMemcpyDeviceToHost, s));
        NCF_CUDA(cudaStreamSynchronize(s));
        for (int32_t j : P->model->cold_cols)
            if (cnt[static_cast<size_t>(j)] < P->m) bits |= 1 << OCG_E_COLD;
    }
    const int code = first_error(bits);
    if (code) return ocg_internal_fail(code, error_text(code));
    return OCG_OK;
}

int ocg_ncf_plan_results(ocg_ncf_plan* P, int32_t* idx, double* saving, double* loss, int32_t* ncand) {
    if (!P) return ocg_internal_fail(OCG_E_INVALID, "null plan");
    int rc = plan_error(P);
    if (rc) return rc;
    cudaStream_t s = ocg_internal_stream(P->model->ctx);
    const size_t m = static_cast<size_t>(P->m);
    if (idx) NCF_CUDA(cudaMemcpyAsync(idx, P->idx.p, sizeof(int32_t) * m, cudaMemcpyDeviceToHost, s));
    if (saving) NCF_CUDA(cudaMemcpyAsync(saving, P->saving.p, sizeof(double) * m, cudaMemcpyDeviceToHost, s));
    if (loss) NCF_CUDA(cudaMemcpyAsync(loss, P->loss.p, sizeof(double) * m, cudaMemcpyDeviceToHost, s));
    if (ncand) NCF_CUDA(cudaMemcpyAsync(ncand, P->ncand.p, sizeof(int32_t) * m, cudaMemcpyDeviceToHost, s));
    NCF_CUDA(cudaStreamSynchronize(s));
    return OCG_OK;
}

int ocg_ncf_plan_completed_rows(ocg_ncf_plan* P, const int64_t* rows, int64_t nrows, double* out) {
    if (!P || (nrows > 0 && (!rows || !out))) return ocg_internal_fail(OCG_E_INVALID, "ncf plan: null argument");
    for (int64_t r = 0; r < nrows; ++r)
        if (rows[r] < 0 || rows[r] >= P->m) return ocg_internal_fail(OCG_E_RANGE, "matrix index out of range");
    if (nrows == 0) return OCG_OK;
    cudaStream_t s = ocg_internal_stream(P->model->ctx);
    Buf<int64_t> dl;
    Buf<double> dout;
    NCF_CUDA(dl.alloc(static_cast<size_t>(nrows)));
    NCF_CUDA(dout.alloc(static_cast<size_t>(nrows * P->n)));
    NCF_CUDA(cudaMemcpyAsync(dl.p, rows, sizeof(int64_t) * nrows, cudaMemcpyHostToDevice, s));
    int rc = plan_launch(P, dl.p, nrows, dout.p, nullptr);
    if (rc) return rc;
    rc = plan_error(P);
    if (rc) return rc;
    NCF_CUDA(cudaMemcpyAsync(out, dout.p, sizeof(double) * nrows * P->n, cudaMemcpyDeviceToHost, s));
    NCF_CUDA(cudaStreamSynchronize(s));
    return OCG_OK;
}

int ocg_ncf_plan_stage(ocg_ncf_plan* P, const int64_t* row_ptr, const int32_t* col, const double* val) {
    if (!P || !row_ptr || !col || !val) return ocg_internal_fail(OCG_E_INVALID, "ncf plan: null argument");
    if (!P->row_ptr.own) return ocg_internal_fail(OCG_E_INVALID, "ncf plan: plan uses caller device buffers");
    if (P->staged) return ocg_internal_fail(OCG_E_INVALID, "ncf plan: a staged CSR is pending (run first)");
    if (row_ptr[0] != 0) return ocg_internal_fail(OCG_E_INVALID, "ncf plan: row_ptr[0] != 0");
    for (int64_t i = 0; i < P->m; ++i)
        if (row_ptr[i + 1] < row_ptr[i]) return ocg_internal_fail(OCG_E_INVALID, "ncf plan: row_ptr decreases");
    const int64_t nnz = row_ptr[P->m];
    cudaStream_t s = ocg_internal_stream(P->model->ctx);
    if (!P->copy_stream) {
        NCF_CUDA(cudaStreamCreateWithFlags(&P->copy_stream, cudaStreamNonBlocking));
        NCF_CUDA(cudaEventCreateWithFlags(&P->ev_staged, cudaEventDisableTiming));
        NCF_CUDA(cudaEventCreateWithFlags(&P->ev_free[0], cudaEventDisableTiming));
        NCF_CUDA(cudaEventCreateWithFlags(&P->ev_free[1], cudaEventDisableTiming));
        NCF_CUDA(P->rp_next.alloc(static_cast<size_t>(P->m + 1)));
    }
    if (nnz > P->next_cap) {  // growth (rare): drain, then size the spare buffers
        NCF_CUDA(cudaStreamSynchronize(s));
        NCF_CUDA(cudaStreamSynchronize(P->copy_stream));
        P->next_cap = nnz + nnz / 16 + 1024;
        NCF_CUDA(P->col_next.alloc(static_cast<size_t>(P->next_cap)));
        NCF_CUDA(P->val_next.alloc(static_cast<size_t>(P->next_cap)));
    }
    cudaStream_t c = P->copy_stream;
    if (P->free_rec[1]) NCF_CUDA(cudaStreamWaitEvent(c, P->ev_free[1], 0));  // the spare buffers' last reader is done
    NCF_CUDA(cudaMemcpyAsync(P->rp_next.p, row_ptr, sizeof(int64_t) * (P->m + 1), cudaMemcpyHostToDevice, c));
    if (nnz > 0) {
        NCF_CUDA(cudaMemcpyAsync(P->col_next.p, col, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, c));
        NCF_CUDA(cudaMemcpyAsync(P->val_next.p, val, sizeof(double) * nnz, cudaMemcpyHostToDevice, c));
    }
    NCF_CUDA(cudaEventRecord(P->ev_staged, c));
    P->staged_nnz = nnz;
    P->staged = true;
    return OCG_OK;
}

int ocg_ncf_plan_results_async(ocg_ncf_plan* P, int32_t* idx, double* saving, double* loss, int32_t* ncand) {
    if (!P || !idx || !saving || !loss || !ncand) return ocg_internal_fail(OCG_E_INVALID, "ncf plan: null argument");
    if (!P->model->cold_cols.empty()) {  // the cold-column rule needs a host-side count: synchronous path
        int rc = plan_error(P);
        if (rc) return rc;
    }
    cudaStream_t s = ocg_internal_stream(P->model->ctx);
    if (!P->ev_results) {
        NCF_CUDA(cudaEventCreateWithFlags(&P->ev_results, cudaEventDisableTiming));
        NCF_CUDA(cudaMallocHost(&P->h_err, sizeof(int)));
    }
    const size_t m = static_cast<size_t>(P->m);
    NCF_CUDA(cudaMemcpyAsync(P->h_err, P->err.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    NCF_CUDA(cudaMemcpyAsync(idx, P->idx.p, sizeof(int32_t) * m, cudaMemcpyDeviceToHost, s));
    NCF_CUDA(cudaMemcpyAsync(saving, P->saving.p, sizeof(double) * m, cudaMemcpyDeviceToHost, s));
    NCF_CUDA(cudaMemcpyAsync(loss, P->loss.p, sizeof(double) * m, cudaMemcpyDeviceToHost, s));
    NCF_CUDA(cudaMemcpyAsync(ncand, P->ncand.p, sizeof(int32_t) * m, cudaMemcpyDeviceToHost, s));
    NCF_CUDA(cudaEventRecord(P->ev_results, s));
    return OCG_OK;
}

int ocg_ncf_plan_results_wait(ocg_ncf_plan* P) {
    if (!P) return ocg_internal_fail(OCG_E_INVALID, "null plan");
    if (!P->ev_results) return OCG_OK;
    NCF_CUDA(cudaEventSynchronize(P->ev_results));
    const int code = first_error(*P->h_err);
    if (code) return ocg_internal_fail(code, error_text(code));
    return OCG_OK;
}

void ocg_ncf_plan_destroy(ocg_ncf_plan* plan) { delete plan; }

}  // extern "C"
