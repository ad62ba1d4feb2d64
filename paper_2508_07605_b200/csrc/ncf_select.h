// Fused NCF imputation + Algorithm-2 selection over a whole sparse matrix:
// cf::complete's imputation loop (cfcomplete.cpp:208-211, NcfModel::predict
// :47-58) fused with policy::select_caps (policy.cpp:17-64) per row, never
// materialising the m x n completed matrix.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace ocg {

constexpr int kNsH0 = 32, kNsH1 = 16;  // the reference's default hidden layers (cfcomplete.hpp:14)
constexpr int kNsTileCols = 32;        // fast path: columns per TMA-staged tile
constexpr int kNsColFloats = 68;       // per staged column: s_h*B_j (32) | exp(B_j) (32) | c+g | pad

// per-row state produced by the prep pass, consumed by the dense pass
struct NcfRowState {
    double pbase;      // completed baseline value p_{i,n-1}
    double best_s;     // best observed candidate (incl. the baseline cell): saving, perf
    double best_p;
    int32_t best_j;    // -1: none
    int32_t best_sum;  // c+g of the best
    int32_t ocnt;      // valid observed candidates
    float fthr;        // smallest float p with loss(p) <= gamma (exact FP64 test)
    int32_t lov;       // 1: a completed value clamped to 0.01 is valid
    int32_t status;    // OCG_* code of the exception the reference would throw for the row
    int32_t thr_ok;    // 1: thr is verified exact, so loss(p) <= gamma  <=>  p >= thr
    double thr;        // smallest double p with loss(p) <= gamma
};

// device scalars of the fast path (written by the prep kernels)
struct NcfFastScale {
    unsigned maxA, maxB;  // float bits of max |A_i[o]|, max |B_j[o]|
    float s_h;            // power-of-two scale of the layer-0 activations
    float sd;             // 2^-(e_h + e_w) log2(e): accumulator -> z1 log2(e)
    float alpha_s;        // alpha * s_h
    int bad;              // exp(A) * exp(B) would overflow: the fast path refuses (OCG_E_UNSUPPORTED)
};

struct NcfSelArgs {
    int64_t m, n;
    int ka, ks;
    int L;
    int dims[5];
    int64_t off_w[4], off_b[4], set_off;  // flat parameter layout (app | setting | W0 b0 W1 b1 ...)
    const double* P;
    const uint8_t* app_seen;
    const uint8_t* setting_seen;
    const int64_t* row_ptr;
    const int32_t* col;
    const double* val;
    const int32_t* cpu;
    const int32_t* gpu;
    int ngpu;
    double e_base, gamma;
    NcfRowState* rows;
    // outputs
    int32_t* idx;
    double* saving;
    double* loss;
    int32_t* ncand;
    int* err;  // OR of (1 << status) over rows
    // optional: completed values of the rows in row_list (nlist rows x n); null = none
    const int64_t* row_list;
    int64_t nlist;
    double* completed;
};

struct NcfFastArgs {
    NcfSelArgs s;
    float* A;    // m x 32: W0[:, :ka] . u_i + b0 (unscaled)
    float* EA;   // m x 32: exp(A)
    float* BE;   // n x kNsColFloats
    const uint4* w1img;  // 3 KB: (lambda W1 * s_w) as fp16 hi | lo | -hi in the UMMA core-matrix layout
    NcfFastScale* scale;
    float b1[16], w2[16], b2;  // b1 log2(e), lambda W2 ln(2): the epilogue's log2 units
    int e_w;                   // log2 s_w
};

cudaError_t ncf_launch_base(const NcfSelArgs& a, int lane, cudaStream_t s);
cudaError_t ncf_launch_rowprep(const NcfSelArgs& a, int sm_count, cudaStream_t s);
cudaError_t ncf_launch_list_observed(const NcfSelArgs& a, cudaStream_t s);
cudaError_t ncf_launch_exact(const NcfSelArgs& a, int lane, int sm_count, cudaStream_t s);
cudaError_t ncf_launch_fast_prep(const NcfFastArgs& a, cudaStream_t s);
cudaError_t ncf_launch_fast(const NcfFastArgs& a, const CUtensorMap* tmap, cudaStream_t s);
bool ncf_fast_shape_ok(const NcfSelArgs& a);

}  // namespace ocg
