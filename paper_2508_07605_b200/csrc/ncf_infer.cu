// NcfModel::predict (cfcomplete.cpp:47-58) on given parameters: FP64,
// lane-exact forward (nnkit.cpp:74-89) + clamp to [kPredictMin, kPerfMax].
// One thread per query; parameters are read through the read-only path.
// Index/cold validation happens on the host before launch (the reference
// throws on the first offending query, in query order).
#include <cuda_runtime.h>

#include "lane_ops.cuh"
#include "ncf_infer.h"

namespace ocg {

template <int LANE>
__global__ void __launch_bounds__(128) ncf_predict_kernel(InferGeom g, const double* __restrict__ P,
                                                          const int64_t* __restrict__ rows,
                                                          const int64_t* __restrict__ cols, int64_t count,
                                                          double* __restrict__ out) {
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= count) return;
    double a[kMaxWidth], z[kMaxWidth];
    const int64_t i = rows[k], j = cols[k];
    for (int q = 0; q < g.ka; ++q) a[q] = P[i * g.ka + q];
    for (int q = 0; q < g.ks; ++q) a[g.ka + q] = P[g.set_off + j * g.ks + q];
    for (int l = 0; l < g.L; ++l) {
        const int in = g.dims[l], outd = g.dims[l + 1];
        const double* W = P + g.off_w[l];
        const double* b = P + g.off_b[l];
        for (int o = 0; o < outd; ++o) z[o] = dadd(LaneOps<LANE>::dot(W + o * in, a, in), b[o]);
        const bool hidden = l + 1 < g.L;
        for (int o = 0; o < outd; ++o) {
            double v = z[o], gf;
            if (hidden) selu_fwd(z[o], v, gf);
            a[o] = v;
        }
    }
    const double v = a[0];
    out[k] = v < 0.01 ? 0.01 : (1.25 < v ? 1.25 : v);
}

cudaError_t launch_ncf_predict(const InferGeom& g, const double* P, const int64_t* rows, const int64_t* cols,
                               int64_t count, double* out, int lane, cudaStream_t stream) {
    const int threads = 128;
    const int64_t blocks = (count + threads - 1) / threads;
    if (blocks == 0) return cudaSuccess;
    if (lane == 0)
        ncf_predict_kernel<0><<<static_cast<unsigned>(blocks), threads, 0, stream>>>(g, P, rows, cols, count, out);
    else
        ncf_predict_kernel<1><<<static_cast<unsigned>(blocks), threads, 0, stream>>>(g, P, rows, cols, count, out);
    return cudaGetLastError();
}

// ---- debug probes ----------------------------------------------------------
__global__ void exp_probe_kernel(const double* x, int64_t n, double* out) {
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k < n) out[k] = glibc_exp(x[k]);
}

__global__ void rng_probe_kernel(uint64_t seed, int64_t n, uint64_t* out) {
    __shared__ uint64_t mt[313];
    __shared__ int idx;
    MtWarp w{mt, &idx};
    const int lane = threadIdx.x;
    w.seed(seed, lane);
    for (int64_t base = 0; base < n; base += 32) {
        const int cnt = static_cast<int>(n - base < 32 ? n - base : 32);
        const uint64_t v = w.take(cnt, lane);
        if (lane < cnt) out[base + lane] = v;
    }
}

cudaError_t launch_exp_probe(const double* x, int64_t n, double* out, cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    exp_probe_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(x, n, out);
    return cudaGetLastError();
}

cudaError_t launch_rng_probe(uint64_t seed, int64_t n, uint64_t* out, cudaStream_t stream) {
    rng_probe_kernel<<<1, 32, 0, stream>>>(seed, n, out);
    return cudaGetLastError();
}

}  // namespace ocg
