#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace ocg {

constexpr int kPredMaxLayers = 6;
constexpr int kPredMaxWidth = 128;

struct PredGeom {
    int L;
    int dims[kPredMaxLayers + 1];
    int acts[kPredMaxLayers];  // 0 selu, 1 relu, 2 identity (nnkit.hpp:15)
    int off_w[kPredMaxLayers], off_b[kPredMaxLayers];
    int T;
    double mean[7], std[7];
};

size_t predictor_smem_bytes(const PredGeom& g);
bool predictor_is_fixed(const PredGeom& g);
// allow_fixed: the reference architecture (7-64-64-1) runs the thread-per-sample
// kernel, anything else (and allow_fixed=false) the warp-per-sample one
cudaError_t launch_predict_perf(const PredGeom& g, const double* params, const double* counters, int64_t count,
                                double* out, int* bad, int lane, int sm_count, cudaStream_t s, bool allow_fixed = true);

}  // namespace ocg
