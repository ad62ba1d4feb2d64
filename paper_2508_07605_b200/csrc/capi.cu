// C-ABI (include/ocg.h): host-side orchestration in C++ around the sm_100a
// kernels.  Validation and error behaviour mirror the reference call sites
// named in ocg.h; compute always runs on the GPU (no CPU fallback).
#include <cuda_runtime.h>

#include <algorithm>
#include <memory>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ocg.h"
#include "ncf_batch.h"
#include "ncf_infer.h"
#include "ocg_common.cuh"
#include "select.h"
#include "predictor.h"

constexpr size_t kFlushBytes = size_t(256) << 20;  // > 126 MB L2

struct ocg_ctx {
    void* flush = nullptr;
    int flush_val = 1;
    int device = 0;
    int sm_count = 0;
    int cc_major = 0, cc_minor = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = true;
};

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define OCG_CUDA(call)                                                                       \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess) return fail(OCG_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// owning device buffer
template <typename T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() {
        if (p) cudaFree(p);
    }
    cudaError_t alloc(size_t count) {
        n = count;
        if (count == 0) return cudaSuccess;
        return cudaMalloc(&p, sizeof(T) * count);
    }
    cudaError_t upload(const T* h, size_t count, cudaStream_t s) {
        cudaError_t e = alloc(count);
        if (e != cudaSuccess || count == 0) return e;
        return cudaMemcpyAsync(p, h, sizeof(T) * count, cudaMemcpyHostToDevice, s);
    }
    cudaError_t download(T* h, size_t count, cudaStream_t s) const {
        if (h == nullptr || count == 0) return cudaSuccess;
        return cudaMemcpyAsync(h, p, sizeof(T) * count, cudaMemcpyDeviceToHost, s);
    }
};

// PowerGrid ctor checks (core.cpp:38-45): non-empty, positive, strictly increasing
int check_caps(const int32_t* caps, int32_t k, const char* which) {
    if (caps == nullptr || k <= 0) return fail(OCG_E_INVALID, std::string(which) + " cap list is empty");
    for (int32_t i = 0; i < k; ++i) {
        if (caps[i] <= 0) return fail(OCG_E_INVALID, std::string(which) + " caps must be positive watts");
        if (i > 0 && caps[i] <= caps[i - 1])
            return fail(OCG_E_INVALID, std::string(which) + " caps must be strictly increasing");
    }
    return OCG_OK;
}

int check_grid(const int32_t* cpu, int32_t ncpu, const int32_t* gpu, int32_t ngpu) {
    int rc = check_caps(cpu, ncpu, "cpu");
    if (rc) return rc;
    return check_caps(gpu, ngpu, "gpu");
}

// cf::fit hyper checks (cfcomplete.cpp:64-66) + MlpModel widths (nnkit.cpp:51-53)
int check_hyper(const ocg_ncf_hyper* h) {
    if (h == nullptr) return fail(OCG_E_INVALID, "ncf: null hyperparameters");
    if (h->app_dim == 0 || h->setting_dim == 0 || h->lr <= 0 || h->max_epochs <= 0 || h->batch_size <= 0 ||
        h->val_fraction < 0 || h->val_fraction >= 1)
        return fail(OCG_E_INVALID, "ncf: bad hyperparameters");
    if (h->app_dim < 0 || h->setting_dim < 0 || h->n_hidden < 0 || h->n_hidden > 7)
        return fail(OCG_E_INVALID, "ncf: bad hyperparameters");
    for (int64_t l = 0; l < h->n_hidden; ++l)
        if (h->hidden[l] <= 0) return fail(OCG_E_INVALID, "zero layer width");
    return OCG_OK;
}

// MLP layer table shared by the geometry builders
struct MlpShape {
    int L = 0;
    int dims[ocg::kMaxLayers + 1] = {};
};

int mlp_shape(const ocg_ncf_hyper* h, MlpShape& s) {
    if (h->n_hidden + 1 > ocg::kMaxLayers)
        return fail(OCG_E_UNSUPPORTED, "ncf: more than " + std::to_string(ocg::kMaxLayers - 1) + " hidden layers");
    s.L = static_cast<int>(h->n_hidden) + 1;
    s.dims[0] = static_cast<int>(h->app_dim + h->setting_dim);
    for (int l = 0; l < h->n_hidden; ++l) s.dims[l + 1] = static_cast<int>(h->hidden[l]);
    s.dims[s.L] = 1;
    for (int l = 0; l <= s.L; ++l)
        if (s.dims[l] > ocg::kMaxWidth)
            return fail(OCG_E_UNSUPPORTED, "ncf: layer wider than " + std::to_string(ocg::kMaxWidth));
    return OCG_OK;
}

const uint64_t kFitTagMix = ocg::splitmix64(ocg::fnv1a("ncf.fit"));

struct BatchInputs {
    int64_t d_rows;
    const double* block_vals;
    const uint8_t* block_mask;
    int64_t napps;
    const double* probe_vals;
    const uint8_t* probe_mask;
    const uint64_t* seeds;
    int32_t n;
};

// Builds geometry + uploads the shared block; per-app rows validated on host.
int prepare_batch(ocg_ctx* ctx, const BatchInputs& in, const ocg_ncf_hyper* h, ocg::BatchGeom& g,
                  std::vector<double>& bval, std::vector<uint32_t>& brc, std::vector<uint8_t>& bseen,
                  std::vector<int32_t>& status) {
    (void)ctx;
    int rc = check_hyper(h);
    if (rc) return rc;
    MlpShape ms;
    if ((rc = mlp_shape(h, ms))) return rc;
    if (in.napps < 0 || in.d_rows < 0 || in.n <= 0) return fail(OCG_E_INVALID, "bad batch shape");
    if (h->batch_size > ocg::kMaxBatch)
        return fail(OCG_E_UNSUPPORTED, "per-app kernel supports batch_size <= 32");
    const int64_t m = in.d_rows + 1, n = in.n;
    if (m > 4095 || n > 4095) return fail(OCG_E_UNSUPPORTED, "per-app kernel supports <= 4095 rows/cols");
    std::memset(&g, 0, sizeof g);
    g.m = static_cast<int>(m);
    g.n = static_cast<int>(n);
    g.ka = static_cast<int>(h->app_dim);
    g.ks = static_cast<int>(h->setting_dim);
    g.L = ms.L;
    for (int l = 0; l <= ms.L; ++l) g.dims[l] = ms.dims[l];
    int64_t off = m * g.ka;
    g.set_off = static_cast<int>(off);
    off += n * g.ks;
    for (int l = 0; l < g.L; ++l) {
        g.off_w[l] = static_cast<int>(off);
        off += static_cast<int64_t>(g.dims[l]) * g.dims[l + 1];
        g.off_b[l] = static_cast<int>(off);
        off += g.dims[l + 1];
    }
    if (off > ocg::kMaxParams)
        return fail(OCG_E_UNSUPPORTED, "per-app model has " + std::to_string(off) + " parameters (> " +
                                           std::to_string(ocg::kMaxParams) + ")");
    g.T = static_cast<int>(off);
    for (int l = 0; l <= g.L; ++l) g.stride[l] = g.dims[l] | 1;  // odd stride: no bank conflicts
    // shared block cells, row-major (cfcomplete.cpp:68-71)
    bval.clear();
    brc.clear();
    bseen.assign(static_cast<size_t>(n), 0);
    for (int64_t i = 0; i < in.d_rows; ++i) {
        bool any = false;
        for (int64_t j = 0; j < n; ++j) {
            if (!in.block_mask[i * n + j]) continue;
            const double v = in.block_vals[i * n + j];
            if (!std::isfinite(v) || v <= 0.0 || v > 1.25)  // PerformanceMatrix::set (core.cpp:142-148)
                return fail(OCG_E_INVALID, "normalized performance outside (0, 1.25]");
            bval.push_back(v);
            brc.push_back((static_cast<uint32_t>(i) << 16) | static_cast<uint32_t>(j));
            bseen[j] = 1;
            any = true;
        }
        if (!any) return fail(OCG_E_INVALID, "complete: app row has no observed entries (probe it first)");
    }
    g.block_nnz = static_cast<int>(bval.size());
    g.block_full = g.block_nnz == in.d_rows * n ? 1 : 0;
    g.max_cells = static_cast<int>(g.block_nnz + n);
    if (g.max_cells > ocg::kMaxCells) return fail(OCG_E_UNSUPPORTED, "per-app matrix has too many cells");
    g.batch = h->batch_size;
    g.max_epochs = h->max_epochs;
    g.patience = h->patience;
    g.lr = h->lr;
    g.val_fraction = h->val_fraction;
    g.fit_tag_mix = kFitTagMix;
    status.assign(static_cast<size_t>(in.napps), OCG_OK);
    for (int64_t a = 0; a < in.napps; ++a)
        for (int64_t j = 0; j < n; ++j)
            if (in.probe_mask[a * n + j]) {
                const double v = in.probe_vals[a * n + j];
                if (!std::isfinite(v) || v <= 0.0 || v > 1.25) {
                    status[a] = OCG_E_INVALID;
                    break;
                }
            }
    return OCG_OK;
}

}  // namespace

int ocg_internal_fail(int code, const std::string& msg) { return fail(code, msg); }
cudaStream_t ocg_internal_stream(ocg_ctx* ctx) { return ctx->stream; }
int ocg_internal_sm_count(ocg_ctx* ctx) { return ctx->sm_count; }

// Device-resident per-app batch: inputs uploaded once, kernel re-runnable.
struct ocg_online_plan {
    ocg_ctx* ctx = nullptr;
    ocg::BatchGeom g{};
    ocg::BatchIO io{};
    int lane = 0;
    int64_t napps = 0, n = 0;
    int grid = 0;
    std::vector<int32_t> hstatus;
    DBuf<double> d_bval, d_pv, d_comp, d_sav, d_loss, d_params, d_best;
    DBuf<uint32_t> d_brc;
    DBuf<uint8_t> d_bseen, d_pm;
    DBuf<uint64_t> d_seeds;
    DBuf<int32_t> d_cpu, d_gpu, d_idx, d_ncand, d_status;
    DBuf<ocg::OcgMetaDev> d_meta;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    ~ocg_online_plan() {
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
    }
};

namespace {

int plan_create(ocg_ctx* ctx, const BatchInputs& in, const int32_t* cpu, int32_t ncpu, const int32_t* gpu,
                int32_t ngpu, const ocg_ncf_hyper* h, double gamma, int lane, bool want_completed,
                int64_t params_stride, ocg_online_plan** out) {
    *out = nullptr;
    if (!ctx) return fail(OCG_E_INVALID, "null context");
    if (lane != OCG_LANE_SCALAR && lane != OCG_LANE_AVX2) return fail(OCG_E_INVALID, "unknown lane");
    auto* P = new ocg_online_plan;
    std::unique_ptr<ocg_online_plan> guard(P);
    P->ctx = ctx;
    P->lane = lane;
    std::vector<double> bval;
    std::vector<uint32_t> brc;
    std::vector<uint8_t> bseen;
    int rc = prepare_batch(ctx, in, h, P->g, bval, brc, bseen, P->hstatus);
    if (rc) return rc;
    ocg::BatchGeom& g = P->g;
    g.ngpu = ngpu;
    g.e_base = cpu ? static_cast<double>(cpu[ncpu - 1] + gpu[ngpu - 1]) : 0.0;
    g.gamma = gamma;
    const int64_t n = in.n, napps = in.napps;
    P->napps = napps;
    P->n = n;
    cudaStream_t s = ctx->stream;
    OCG_CUDA(P->d_bval.upload(bval.data(), bval.size(), s));
    OCG_CUDA(P->d_brc.upload(brc.data(), brc.size(), s));
    OCG_CUDA(P->d_bseen.upload(bseen.data(), bseen.size(), s));
    OCG_CUDA(P->d_pv.upload(in.probe_vals, static_cast<size_t>(napps * n), s));
    OCG_CUDA(P->d_pm.upload(in.probe_mask, static_cast<size_t>(napps * n), s));
    OCG_CUDA(P->d_seeds.upload(in.seeds, static_cast<size_t>(napps), s));
    ocg::BatchIO& io = P->io;
    io.napps = napps;
    if (cpu) {
        OCG_CUDA(P->d_cpu.upload(cpu, static_cast<size_t>(ncpu), s));
        OCG_CUDA(P->d_gpu.upload(gpu, static_cast<size_t>(ngpu), s));
        OCG_CUDA(P->d_idx.alloc(static_cast<size_t>(napps)));
        OCG_CUDA(P->d_sav.alloc(static_cast<size_t>(napps)));
        OCG_CUDA(P->d_loss.alloc(static_cast<size_t>(napps)));
        OCG_CUDA(P->d_ncand.alloc(static_cast<size_t>(napps)));
        io.cpu_caps = P->d_cpu.p;
        io.gpu_caps = P->d_gpu.p;
        io.sel_idx = P->d_idx.p;
        io.sel_saving = P->d_sav.p;
        io.sel_loss = P->d_loss.p;
        io.sel_ncand = P->d_ncand.p;
    }
    OCG_CUDA(P->d_status.upload(P->hstatus.data(), P->hstatus.size(), s));
    OCG_CUDA(P->d_meta.alloc(static_cast<size_t>(napps)));
    OCG_CUDA(cudaMemsetAsync(P->d_meta.p, 0, sizeof(ocg::OcgMetaDev) * static_cast<size_t>(napps), s));
    io.block_val = P->d_bval.p;
    io.block_rc = P->d_brc.p;
    io.block_col_seen = P->d_bseen.p;
    io.probe_vals = P->d_pv.p;
    io.probe_mask = P->d_pm.p;
    io.seeds = P->d_seeds.p;
    io.status = P->d_status.p;
    io.meta = P->d_meta.p;
    if (want_completed) {
        OCG_CUDA(P->d_comp.alloc(static_cast<size_t>(napps * n)));
        io.completed = P->d_comp.p;
    }
    if (params_stride > 0) {
        OCG_CUDA(P->d_params.alloc(static_cast<size_t>(napps * params_stride)));
        io.params = P->d_params.p;
        io.params_stride = params_stride;
    }
    const size_t smem = ocg::batch_smem_bytes(g);
    if (smem > 227 * 1024) return fail(OCG_E_UNSUPPORTED, "per-app working set exceeds shared memory");
    const int per_sm = ocg::batch_max_active_per_sm(g, lane);
    if (per_sm < 1) return fail(OCG_E_CUDA, "per-app kernel cannot be resident (smem " + std::to_string(smem) + ")");
    P->grid = static_cast<int>(std::min<int64_t>(std::max<int64_t>(napps, 1), static_cast<int64_t>(per_sm) * ctx->sm_count));
    io.best_stride = (g.T + 31) & ~31;
    OCG_CUDA(P->d_best.alloc(static_cast<size_t>(P->grid) * static_cast<size_t>(io.best_stride)));
    io.best = P->d_best.p;
    OCG_CUDA(cudaEventCreate(&P->ev0));
    OCG_CUDA(cudaEventCreate(&P->ev1));
    OCG_CUDA(cudaStreamSynchronize(s));
    *out = guard.release();
    return OCG_OK;
}

int plan_run(ocg_online_plan* P, float* ms) {
    if (!P) return fail(OCG_E_INVALID, "null plan");
    if (P->napps == 0) return OCG_OK;
    cudaStream_t s = P->ctx->stream;
    OCG_CUDA(cudaEventRecord(P->ev0, s));
    OCG_CUDA(ocg::launch_app_batch(P->g, P->io, P->lane, P->grid, s));
    OCG_CUDA(cudaEventRecord(P->ev1, s));
    if (ms) {
        OCG_CUDA(cudaEventSynchronize(P->ev1));
        OCG_CUDA(cudaEventElapsedTime(ms, P->ev0, P->ev1));
    }
    return OCG_OK;
}

int plan_results(ocg_online_plan* P, double* completed, int32_t* idx, double* saving, double* loss, int32_t* ncand,
                 ocg_ncf_meta* meta, int32_t* status_out, double* params) {
    if (!P) return fail(OCG_E_INVALID, "null plan");
    const int64_t napps = P->napps, n = P->n;
    cudaStream_t s = P->ctx->stream;
    std::vector<int32_t> dev_status(static_cast<size_t>(napps));
    OCG_CUDA(P->d_status.download(dev_status.data(), dev_status.size(), s));
    if (completed && P->io.completed) OCG_CUDA(P->d_comp.download(completed, static_cast<size_t>(napps * n), s));
    if (P->io.sel_idx) {
        OCG_CUDA(P->d_idx.download(idx, static_cast<size_t>(napps), s));
        OCG_CUDA(P->d_sav.download(saving, static_cast<size_t>(napps), s));
        OCG_CUDA(P->d_loss.download(loss, static_cast<size_t>(napps), s));
        OCG_CUDA(P->d_ncand.download(ncand, static_cast<size_t>(napps), s));
    }
    if (meta) OCG_CUDA(P->d_meta.download(reinterpret_cast<ocg::OcgMetaDev*>(meta), static_cast<size_t>(napps), s));
    if (params && P->io.params)
        OCG_CUDA(P->d_params.download(params, static_cast<size_t>(napps * P->io.params_stride), s));
    OCG_CUDA(cudaStreamSynchronize(s));
    if (status_out)
        for (int64_t a = 0; a < napps; ++a)
            status_out[a] = P->hstatus[a] != OCG_OK ? P->hstatus[a] : dev_status[a];
    return OCG_OK;
}

int run_batch(ocg_ctx* ctx, const BatchInputs& in, const int32_t* cpu, int32_t ncpu, const int32_t* gpu,
              int32_t ngpu, const ocg_ncf_hyper* h, double gamma, int lane, double* completed, int32_t* idx,
              double* saving, double* loss, int32_t* ncand, ocg_ncf_meta* meta, int32_t* status_out,
              double* params, int64_t params_stride) {
    if (!status_out) return fail(OCG_E_INVALID, "status output is required");
    ocg_online_plan* P = nullptr;
    int rc = plan_create(ctx, in, cpu, ncpu, gpu, ngpu, h, gamma, lane, completed != nullptr,
                         params ? params_stride : 0, &P);
    if (rc) return rc;
    std::unique_ptr<ocg_online_plan> guard(P);
    if ((rc = plan_run(P, nullptr))) return rc;
    return plan_results(P, completed, idx, saving, loss, ncand, meta, status_out, params);
}

}  // namespace

extern "C" {

const char* ocg_last_error(void) { return g_err.c_str(); }
int ocg_version(void) { return 1; }

void ocg_ncf_hyper_default(ocg_ncf_hyper* h) {
    std::memset(h, 0, sizeof *h);
    h->app_dim = 8;
    h->setting_dim = 8;
    h->hidden[0] = 32;
    h->hidden[1] = 16;
    h->n_hidden = 2;
    h->lr = 1e-3;
    h->max_epochs = 2000;
    h->patience = 100;
    h->val_fraction = 0.1;
    h->batch_size = 32;
}

uint64_t ocg_derive_seed(uint64_t root, const char* tag, uint64_t n) {
    return ocg::derive_seed_h(root, ocg::splitmix64(ocg::fnv1a(tag)), n);
}

int ocg_ctx_create(int device, ocg_ctx** out) {
    if (!out) return fail(OCG_E_INVALID, "null output");
    *out = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        return fail(OCG_E_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
    if (device < 0 || device >= count) return fail(OCG_E_INVALID, "device index out of range");
    OCG_CUDA(cudaSetDevice(device));
    auto* c = new ocg_ctx;
    c->device = device;
    cudaDeviceProp prop{};
    cudaGetDeviceProperties(&prop, device);
    c->sm_count = prop.multiProcessorCount;
    c->cc_major = prop.major;
    c->cc_minor = prop.minor;
    if (prop.major != 10) {
        delete c;
        return fail(OCG_E_CUDA, "kernels are built for sm_100a only (found sm_" + std::to_string(prop.major) +
                                    std::to_string(prop.minor) + ")");
    }
    e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete c;
        return fail(OCG_E_CUDA, cudaGetErrorString(e));
    }
    *out = c;
    return OCG_OK;
}

void ocg_ctx_destroy(ocg_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream && ctx->own_stream) cudaStreamDestroy(ctx->stream);
    if (ctx->flush) cudaFree(ctx->flush);
    delete ctx;
}

int ocg_ctx_device_info(ocg_ctx* ctx, int* sm_count, int* cc_major, int* cc_minor) {
    if (!ctx) return fail(OCG_E_INVALID, "null context");
    if (sm_count) *sm_count = ctx->sm_count;
    if (cc_major) *cc_major = ctx->cc_major;
    if (cc_minor) *cc_minor = ctx->cc_minor;
    return OCG_OK;
}

int ocg_default_plan(const int32_t* cpu, int32_t ncpu, const int32_t* gpu, int32_t ngpu, int32_t* cols,
                     int32_t* count) {
    int rc = check_grid(cpu, ncpu, gpu, ngpu);
    if (rc) return rc;
    const int32_t wc[6] = {ncpu - 1, 0, 0, ncpu - 1, ncpu / 2, ncpu / 4};
    const int32_t wg[6] = {ngpu - 1, 0, ngpu - 1, 0, ngpu / 2, ngpu / 4};
    int32_t k = 0;
    for (int w = 0; w < 6; ++w) {
        const int32_t col = wc[w] * ngpu + wg[w];
        if (std::find(cols, cols + k, col) == cols + k) cols[k++] = col;
    }
    *count = k;
    return OCG_OK;
}

int ocg_select_caps_dev(ocg_ctx* ctx, const void* d_rows, int dtype, int64_t nrows, const int32_t* cpu,
                        int32_t ncpu, const int32_t* gpu, int32_t ngpu, double gamma, int32_t* d_idx,
                        double* d_saving, double* d_loss, int32_t* d_ncand) {
    if (!ctx) return fail(OCG_E_INVALID, "null context");
    int rc = check_grid(cpu, ncpu, gpu, ngpu);
    if (rc) return rc;
    if (gamma <= 0.0 || gamma >= 1.0) return fail(OCG_E_INVALID, "select_caps: gamma must lie in (0, 1)");
    if (dtype != 0 && dtype != 1) return fail(OCG_E_INVALID, "dtype must be 0 (f64) or 1 (f32)");
    if (nrows == 0) return OCG_OK;
    cudaStream_t s = ctx->stream;
    DBuf<int32_t> dc, dg;
    DBuf<int> dbad;
    OCG_CUDA(dc.upload(cpu, static_cast<size_t>(ncpu), s));
    OCG_CUDA(dg.upload(gpu, static_cast<size_t>(ngpu), s));
    OCG_CUDA(dbad.alloc(1));
    OCG_CUDA(cudaMemsetAsync(dbad.p, 0, sizeof(int), s));
    const double e_base = static_cast<double>(cpu[ncpu - 1] + gpu[ngpu - 1]);
    OCG_CUDA(ocg::launch_select_rows(d_rows, dtype, nrows, ncpu * ngpu, dc.p, dg.p, ngpu, e_base, gamma, d_idx,
                                     d_saving, d_loss, d_ncand, dbad.p, ctx->sm_count, s));
    int bad = 0;
    OCG_CUDA(cudaMemcpyAsync(&bad, dbad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    OCG_CUDA(cudaStreamSynchronize(s));
    if (bad) return fail(OCG_E_INVALID, "select_caps: performance entries must be positive");
    return OCG_OK;
}

int ocg_select_caps(ocg_ctx* ctx, const double* rows, int64_t nrows, const int32_t* cpu, int32_t ncpu,
                    const int32_t* gpu, int32_t ngpu, double gamma, int32_t* idx, double* saving, double* loss,
                    int32_t* ncand) {
    if (!ctx) return fail(OCG_E_INVALID, "null context");
    int rc = check_grid(cpu, ncpu, gpu, ngpu);
    if (rc) return rc;
    if (gamma <= 0.0 || gamma >= 1.0) return fail(OCG_E_INVALID, "select_caps: gamma must lie in (0, 1)");
    if (nrows == 0) return OCG_OK;
    const size_t n = static_cast<size_t>(ncpu) * ngpu, R = static_cast<size_t>(nrows);
    cudaStream_t s = ctx->stream;
    DBuf<double> dr, ds, dl;
    DBuf<int32_t> di, dn;
    OCG_CUDA(dr.upload(rows, R * n, s));
    OCG_CUDA(ds.alloc(R));
    OCG_CUDA(dl.alloc(R));
    OCG_CUDA(di.alloc(R));
    OCG_CUDA(dn.alloc(R));
    rc = ocg_select_caps_dev(ctx, dr.p, 0, nrows, cpu, ncpu, gpu, ngpu, gamma, di.p, ds.p, dl.p, dn.p);
    if (rc) return rc;
    OCG_CUDA(di.download(idx, R, s));
    OCG_CUDA(ds.download(saving, R, s));
    OCG_CUDA(dl.download(loss, R, s));
    OCG_CUDA(dn.download(ncand, R, s));
    OCG_CUDA(cudaStreamSynchronize(s));
    return OCG_OK;
}

int ocg_online_complete_batch(ocg_ctx* ctx, int64_t d_rows, const double* block_vals, const uint8_t* block_mask,
                              int64_t napps, const double* probe_vals, const uint8_t* probe_mask,
                              const uint64_t* seeds, const int32_t* cpu, int32_t ncpu, const int32_t* gpu,
                              int32_t ngpu, const ocg_ncf_hyper* hyper, double gamma, int lane, double* completed,
                              int32_t* idx, double* saving, double* loss, int32_t* ncand, ocg_ncf_meta* meta,
                              int32_t* status) {
    int rc = check_grid(cpu, ncpu, gpu, ngpu);
    if (rc) return rc;
    if (gamma <= 0.0 || gamma >= 1.0) return fail(OCG_E_INVALID, "select_caps: gamma must lie in (0, 1)");
    std::vector<int32_t> tmp_i;
    std::vector<double> tmp_s, tmp_l;
    std::vector<int32_t> tmp_n;
    if (!idx) { tmp_i.resize(static_cast<size_t>(napps)); idx = tmp_i.data(); }
    if (!saving) { tmp_s.resize(static_cast<size_t>(napps)); saving = tmp_s.data(); }
    if (!loss) { tmp_l.resize(static_cast<size_t>(napps)); loss = tmp_l.data(); }
    if (!ncand) { tmp_n.resize(static_cast<size_t>(napps)); ncand = tmp_n.data(); }
    BatchInputs in{d_rows, block_vals, block_mask, napps, probe_vals, probe_mask, seeds, ncpu * ngpu};
    return run_batch(ctx, in, cpu, ncpu, gpu, ngpu, hyper, gamma, lane, completed, idx, saving, loss, ncand, meta,
                     status, nullptr, 0);
}

int ocg_online_plan_create(ocg_ctx* ctx, int64_t d_rows, const double* block_vals, const uint8_t* block_mask,
                           int64_t napps, const double* probe_vals, const uint8_t* probe_mask, const uint64_t* seeds,
                           const int32_t* cpu, int32_t ncpu, const int32_t* gpu, int32_t ngpu,
                           const ocg_ncf_hyper* hyper, double gamma, int lane, int want_completed,
                           ocg_online_plan** out) {
    if (!out) return fail(OCG_E_INVALID, "null output");
    int rc = check_grid(cpu, ncpu, gpu, ngpu);
    if (rc) return rc;
    if (gamma <= 0.0 || gamma >= 1.0) return fail(OCG_E_INVALID, "select_caps: gamma must lie in (0, 1)");
    BatchInputs in{d_rows, block_vals, block_mask, napps, probe_vals, probe_mask, seeds, ncpu * ngpu};
    return plan_create(ctx, in, cpu, ncpu, gpu, ngpu, hyper, gamma, lane, want_completed != 0, 0, out);
}

int ocg_online_plan_run(ocg_online_plan* plan, float* kernel_ms) { return plan_run(plan, kernel_ms); }

int ocg_online_plan_results(ocg_online_plan* plan, double* completed, int32_t* idx, double* saving, double* loss,
                            int32_t* ncand, ocg_ncf_meta* meta, int32_t* status) {
    return plan_results(plan, completed, idx, saving, loss, ncand, meta, status, nullptr);
}

void ocg_online_plan_destroy(ocg_online_plan* plan) { delete plan; }

int ocg_ctx_flush_l2(ocg_ctx* ctx) {
    if (!ctx) return fail(OCG_E_INVALID, "null context");
    if (!ctx->flush) OCG_CUDA(cudaMalloc(&ctx->flush, kFlushBytes));
    OCG_CUDA(cudaMemsetAsync(ctx->flush, ctx->flush_val++ & 0xff, kFlushBytes, ctx->stream));
    OCG_CUDA(cudaStreamSynchronize(ctx->stream));
    return OCG_OK;
}

int ocg_ctx_set_stream(ocg_ctx* ctx, void* stream) {
    if (!ctx) return fail(OCG_E_INVALID, "null context");
    // work already queued on the current stream must finish before later kernels run on
    // the new one (they may read what it writes): drain it before switching
    if (ctx->stream) OCG_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
    ctx->own_stream = false;
    ctx->stream = static_cast<cudaStream_t>(stream);
    return OCG_OK;
}

int ocg_ctx_synchronize(ocg_ctx* ctx) {
    if (!ctx) return fail(OCG_E_INVALID, "null context");
    OCG_CUDA(cudaStreamSynchronize(ctx->stream));
    return OCG_OK;
}

int ocg_online_fit_batch_params(ocg_ctx* ctx, int64_t d_rows, const double* block_vals, const uint8_t* block_mask,
                                int64_t napps, const double* probe_vals, const uint8_t* probe_mask,
                                const uint64_t* seeds, int32_t n, const ocg_ncf_hyper* hyper, int lane,
                                double* params, int64_t params_stride, ocg_ncf_meta* meta, int32_t* status) {
    BatchInputs in{d_rows, block_vals, block_mask, napps, probe_vals, probe_mask, seeds, n};
    return run_batch(ctx, in, nullptr, 0, nullptr, 1, hyper, 0.05, lane, nullptr, nullptr, nullptr, nullptr,
                     nullptr, meta, status, params, params_stride);
}

int ocg_ncf_predict(ocg_ctx* ctx, int64_t m, int64_t n, const ocg_ncf_hyper* h, const double* params,
                    const uint8_t* app_seen, const uint8_t* setting_seen, const int64_t* rows, const int64_t* cols,
                    int64_t count, int lane, double* out) {
    if (!ctx) return fail(OCG_E_INVALID, "null context");
    if (!h) return fail(OCG_E_INVALID, "null hyper");
    MlpShape ms;
    int rc = mlp_shape(h, ms);
    if (rc) return rc;
    // NcfModel::predict checks, first offending query wins (cfcomplete.cpp:48-55)
    for (int64_t k = 0; k < count; ++k) {
        if (rows[k] < 0 || rows[k] >= m) return fail(OCG_E_RANGE, "ncf: app index out of range");
        if (cols[k] < 0 || cols[k] >= n) return fail(OCG_E_RANGE, "ncf: setting index out of range");
        if (!app_seen[rows[k]])
            return fail(OCG_E_COLD, "ncf: cold app row " + std::to_string(rows[k]) + " (no observed entries at fit time)");
        if (!setting_seen[cols[k]])
            return fail(OCG_E_COLD,
                        "ncf: cold setting column " + std::to_string(cols[k]) + " (no observed entries at fit time)");
    }
    if (count == 0) return OCG_OK;
    ocg::InferGeom g{};
    g.m = m;
    g.n = n;
    g.ka = static_cast<int>(h->app_dim);
    g.ks = static_cast<int>(h->setting_dim);
    g.L = ms.L;
    for (int l = 0; l <= ms.L; ++l) g.dims[l] = ms.dims[l];
    int64_t off = m * g.ka;
    g.set_off = off;
    off += n * g.ks;
    for (int l = 0; l < g.L; ++l) {
        g.off_w[l] = off;
        off += static_cast<int64_t>(g.dims[l]) * g.dims[l + 1];
        g.off_b[l] = off;
        off += g.dims[l + 1];
    }
    cudaStream_t s = ctx->stream;
    DBuf<double> dp, dout;
    DBuf<int64_t> dr, dc;
    OCG_CUDA(dp.upload(params, static_cast<size_t>(off), s));
    OCG_CUDA(dr.upload(rows, static_cast<size_t>(count), s));
    OCG_CUDA(dc.upload(cols, static_cast<size_t>(count), s));
    OCG_CUDA(dout.alloc(static_cast<size_t>(count)));
    OCG_CUDA(ocg::launch_ncf_predict(g, dp.p, dr.p, dc.p, count, dout.p, lane, s));
    OCG_CUDA(dout.download(out, static_cast<size_t>(count), s));
    OCG_CUDA(cudaStreamSynchronize(s));
    return OCG_OK;
}

struct ocg_predictor {
    ocg_ctx* ctx = nullptr;
    ocg::PredGeom g{};
    DBuf<double> params;
    DBuf<int> bad;
};

int ocg_predictor_create(ocg_ctx* ctx, int32_t n_layers, const int64_t* dims, const int32_t* acts,
                         const double* params, const double* mean7, const double* std7, int has_stats,
                         ocg_predictor** out) {
    if (!ctx || !out || !dims || !acts || !params || !mean7 || !std7) return fail(OCG_E_INVALID, "null argument");
    *out = nullptr;
    // predict_perf (predictor.cpp:151-153): stats first
    if (!has_stats) return fail(OCG_E_MISSING, "predictor model lacks feature standardization stats");
    if (n_layers < 1 || n_layers > ocg::kPredMaxLayers) return fail(OCG_E_UNSUPPORTED, "predictor: layer count");
    if (dims[0] != 7) return fail(OCG_E_INVALID, "forward: input dimension mismatch");
    if (dims[n_layers] != 1) return fail(OCG_E_INVALID, "predictor: output dimension must be 1");
    auto p = std::make_unique<ocg_predictor>();
    ocg::PredGeom& g = p->g;
    g.L = n_layers;
    int off = 0;
    for (int l = 0; l <= n_layers; ++l) {
        if (dims[l] <= 0 || dims[l] > ocg::kPredMaxWidth) return fail(OCG_E_UNSUPPORTED, "predictor: layer width");
        g.dims[l] = static_cast<int>(dims[l]);
    }
    for (int l = 0; l < n_layers; ++l) {
        if (acts[l] < 0 || acts[l] > 2) return fail(OCG_E_INVALID, "unknown activation");
        g.acts[l] = acts[l];
        g.off_w[l] = off;
        off += g.dims[l] * g.dims[l + 1];
        g.off_b[l] = off;
        off += g.dims[l + 1];
    }
    g.T = off;
    for (int q = 0; q < 7; ++q) {
        g.mean[q] = mean7[q];
        g.std[q] = std7[q];
    }
    if (ocg::predictor_smem_bytes(g) > 200 * 1024) return fail(OCG_E_UNSUPPORTED, "predictor too large");
    p->ctx = ctx;
    cudaStream_t s = ctx->stream;
    OCG_CUDA(p->params.upload(params, static_cast<size_t>(g.T), s));
    OCG_CUDA(p->bad.alloc(1));
    OCG_CUDA(cudaStreamSynchronize(s));
    *out = p.release();
    return OCG_OK;
}

int ocg_predictor_run(ocg_predictor* pred, const double* counters, int64_t count, int lane, double* out,
                      uint32_t flags) {
    if (!pred) return fail(OCG_E_INVALID, "null predictor");
    if (count < 0) return fail(OCG_E_INVALID, "negative count");
    if (lane != OCG_LANE_SCALAR && lane != OCG_LANE_AVX2) return fail(OCG_E_INVALID, "unknown kernel lane");
    if (count == 0) return OCG_OK;
    if (!counters || !out) return fail(OCG_E_INVALID, "null buffer");
    ocg_ctx* ctx = pred->ctx;
    cudaStream_t s = ctx->stream;
    const bool on_dev = flags & OCG_PRED_DEVICE_PTRS;
    DBuf<double> dc, dout;
    const double* c = counters;
    double* o = out;
    if (!on_dev) {
        OCG_CUDA(dc.upload(counters, static_cast<size_t>(count) * 7, s));
        OCG_CUDA(dout.alloc(static_cast<size_t>(count)));
        c = dc.p;
        o = dout.p;
    }
    OCG_CUDA(cudaMemsetAsync(pred->bad.p, 0, sizeof(int), s));
    OCG_CUDA(ocg::launch_predict_perf(pred->g, pred->params.p, c, count, o, pred->bad.p, lane, ctx->sm_count, s,
                                      !(flags & OCG_PRED_GENERIC)));
    int bad = 0;
    OCG_CUDA(cudaMemcpyAsync(&bad, pred->bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    if (!on_dev) OCG_CUDA(dout.download(out, static_cast<size_t>(count), s));
    OCG_CUDA(cudaStreamSynchronize(s));
    if (bad) return fail(OCG_E_INVALID, "invalid counter sample (non-finite, negative or activity outside [0,1])");
    return OCG_OK;
}

}  // extern "C"

namespace {

// re-probe rule (policy.cpp:168-176): the counters an app's estimates come from
__global__ void ingest_select_kernel(int64_t napps, int nplan, const double* __restrict__ probe,
                                     const double* __restrict__ reprobe, const int32_t* __restrict__ transition,
                                     double* __restrict__ out) {
    const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t per = static_cast<int64_t>(nplan) * 7;
    if (q >= napps * per) return;
    const int64_t a = q / per;
    out[q] = (reprobe && transition && transition[a]) ? reprobe[q] : probe[q];
}

// validate_counters (core.cpp:74-83) per app, then the estimates into the app rows
__global__ void ingest_scatter_kernel(int64_t napps, int nplan, int64_t n, const int32_t* __restrict__ plan_cols,
                                      const double* __restrict__ counters, const double* __restrict__ est,
                                      double* __restrict__ probe_vals, int32_t* __restrict__ bad_app) {
    const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= napps * nplan) return;
    const int64_t a = q / nplan;
    const int p = static_cast<int>(q - a * nplan);
    const double* c = counters + q * 7;
    bool ok = true;
    for (int f = 0; f < 7; ++f) ok = ok && isfinite(c[f]);
    ok = ok && c[2] >= 0 && c[3] >= 0 && c[4] >= 0 && c[5] >= 0 && c[5] <= 1 && c[6] >= 0 && c[6] <= 1;
    if (!ok) atomicExch(bad_app + a, 1);
    probe_vals[a * n + plan_cols[p]] = ok ? est[q] : 1.0;
}

}  // namespace

extern "C" {

int ocg_online_ingest_complete_batch(ocg_ctx* ctx, int64_t d_rows, const double* block_vals,
                                     const uint8_t* block_mask, int64_t napps, const int32_t* plan_cols,
                                     int32_t nplan, ocg_predictor* pred, const double* counters,
                                     const double* reprobe_counters, const int32_t* transition,
                                     const uint64_t* seeds, const int32_t* cpu, int32_t ncpu, const int32_t* gpu,
                                     int32_t ngpu, const ocg_ncf_hyper* h, double gamma, int lane, double* estimates,
                                     double* completed, int32_t* idx, double* saving, double* loss, int32_t* ncand,
                                     ocg_ncf_meta* meta, int32_t* status) {
    if (!ctx || !pred || !status || (napps > 0 && (!counters || !plan_cols || !seeds)))
        return fail(OCG_E_INVALID, "null argument");
    if (lane != OCG_LANE_SCALAR && lane != OCG_LANE_AVX2) return fail(OCG_E_INVALID, "unknown lane");
    if (cpu && check_grid(cpu, ncpu, gpu, ngpu)) return OCG_E_INVALID;
    const int64_t n = static_cast<int64_t>(ncpu) * ngpu;
    if (nplan <= 0 || nplan > n) return fail(OCG_E_INVALID, "probe plan: bad size");
    for (int32_t p = 0; p < nplan; ++p)  // ProbePlan::validate (policy.cpp:84-96): distinct grid settings
        if (plan_cols[p] < 0 || plan_cols[p] >= n) return fail(OCG_E_INVALID, "probe plan: setting outside the grid");
    if (napps == 0) return OCG_OK;
    // the per-app plan, with placeholder estimates at the plan cells (overwritten on the device)
    std::vector<double> pv(static_cast<size_t>(napps * n), 0.0);
    std::vector<uint8_t> pm(static_cast<size_t>(napps * n), 0);
    for (int64_t a = 0; a < napps; ++a)
        for (int32_t p = 0; p < nplan; ++p) {
            pv[static_cast<size_t>(a * n + plan_cols[p])] = 1.0;
            pm[static_cast<size_t>(a * n + plan_cols[p])] = 1;
        }
    const BatchInputs in{d_rows, block_vals, block_mask, napps, pv.data(), pm.data(), seeds, static_cast<int32_t>(n)};
    ocg_online_plan* P = nullptr;
    int rc = plan_create(ctx, in, cpu, ncpu, gpu, ngpu, h, gamma, lane, completed != nullptr, 0, &P);
    if (rc) return rc;
    std::unique_ptr<ocg_online_plan> guard(P);
    cudaStream_t s = ctx->stream;
    const int64_t ns = napps * nplan;
    DBuf<double> dprobe, dre, dsel, dest;
    DBuf<int32_t> dtr, dplan, dbad;
    OCG_CUDA(dprobe.upload(counters, static_cast<size_t>(ns * 7), s));
    if (reprobe_counters && transition) {
        OCG_CUDA(dre.upload(reprobe_counters, static_cast<size_t>(ns * 7), s));
        OCG_CUDA(dtr.upload(transition, static_cast<size_t>(napps), s));
    }
    OCG_CUDA(dsel.alloc(static_cast<size_t>(ns * 7)));
    OCG_CUDA(dest.alloc(static_cast<size_t>(ns)));
    OCG_CUDA(dplan.upload(plan_cols, static_cast<size_t>(nplan), s));
    OCG_CUDA(dbad.alloc(static_cast<size_t>(napps)));
    OCG_CUDA(cudaMemsetAsync(dbad.p, 0, sizeof(int32_t) * napps, s));
    ingest_select_kernel<<<static_cast<unsigned>((ns * 7 + 255) / 256), 256, 0, s>>>(napps, nplan, dprobe.p, dre.p,
                                                                                     dtr.p, dsel.p);
    OCG_CUDA(cudaGetLastError());
    // pred::predict_perf over every sample; invalid samples are flagged per app below, not fatal
    OCG_CUDA(ocg::launch_predict_perf(pred->g, pred->params.p, dsel.p, ns, dest.p, pred->bad.p, lane, ctx->sm_count, s));
    ingest_scatter_kernel<<<static_cast<unsigned>((ns + 255) / 256), 256, 0, s>>>(napps, nplan, n, dplan.p, dsel.p,
                                                                                  dest.p, P->d_pv.p, dbad.p);
    OCG_CUDA(cudaGetLastError());
    std::vector<int32_t> bad(static_cast<size_t>(napps));
    OCG_CUDA(dbad.download(bad.data(), bad.size(), s));
    if (estimates) OCG_CUDA(dest.download(estimates, static_cast<size_t>(ns), s));
    OCG_CUDA(cudaStreamSynchronize(s));
    for (int64_t a = 0; a < napps; ++a)
        if (bad[static_cast<size_t>(a)] && P->hstatus[static_cast<size_t>(a)] == OCG_OK)
            P->hstatus[static_cast<size_t>(a)] = OCG_E_INVALID;  // predict_perf's validate_counters
    if ((rc = plan_run(P, nullptr))) return rc;
    return plan_results(P, completed, idx, saving, loss, ncand, meta, status, nullptr);
}

int ocg_predictor_destroy(ocg_predictor* pred) {
    delete pred;
    return OCG_OK;
}

int ocg_predict_perf_batch(ocg_ctx* ctx, int32_t n_layers, const int64_t* dims, const int32_t* acts,
                           const double* params, const double* mean7, const double* std7, int has_stats,
                           const double* counters, int64_t count, int lane, double* out) {
    ocg_predictor* p = nullptr;
    int rc = ocg_predictor_create(ctx, n_layers, dims, acts, params, mean7, std7, has_stats, &p);
    if (rc != OCG_OK) return rc;
    rc = ocg_predictor_run(p, counters, count, lane, out, 0);
    ocg_predictor_destroy(p);
    return rc;
}

int ocg_debug_exp(ocg_ctx* ctx, const double* x, int64_t n, double* out) {
    if (!ctx) return fail(OCG_E_INVALID, "null context");
    cudaStream_t s = ctx->stream;
    DBuf<double> dx, dy;
    OCG_CUDA(dx.upload(x, static_cast<size_t>(n), s));
    OCG_CUDA(dy.alloc(static_cast<size_t>(n)));
    OCG_CUDA(ocg::launch_exp_probe(dx.p, n, dy.p, s));
    OCG_CUDA(dy.download(out, static_cast<size_t>(n), s));
    OCG_CUDA(cudaStreamSynchronize(s));
    return OCG_OK;
}

double ocg_debug_exp_host(double x) { return ocg::glibc_exp(x); }

int ocg_debug_rng(ocg_ctx* ctx, uint64_t seed, int64_t n, uint64_t* out) {
    if (!ctx) return fail(OCG_E_INVALID, "null context");
    cudaStream_t s = ctx->stream;
    DBuf<uint64_t> d;
    OCG_CUDA(d.alloc(static_cast<size_t>(n)));
    OCG_CUDA(ocg::launch_rng_probe(seed, n, d.p, s));
    OCG_CUDA(d.download(out, static_cast<size_t>(n), s));
    OCG_CUDA(cudaStreamSynchronize(s));
    return OCG_OK;
}

}  // extern "C"
