#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "ncf_batch.h"

namespace ocg {

struct InferGeom {
    int64_t m, n;
    int ka, ks, L;
    int dims[kMaxLayers + 1];
    int64_t off_w[kMaxLayers], off_b[kMaxLayers];
    int64_t set_off;
};

cudaError_t launch_ncf_predict(const InferGeom& g, const double* P, const int64_t* rows, const int64_t* cols,
                               int64_t count, double* out, int lane, cudaStream_t stream);
cudaError_t launch_exp_probe(const double* x, int64_t n, double* out, cudaStream_t stream);
cudaError_t launch_rng_probe(uint64_t seed, int64_t n, uint64_t* out, cudaStream_t stream);

}  // namespace ocg
