// Probe ingest: pred::predict_perf (predictor.cpp:151-157) batched over many
// counter samples — validate_counters (core.cpp:97-106), standardize
// (predictor.cpp:74-79), MlpModel::forward (nnkit.cpp:74-89: 7 -> 64 -> 64 -> 1,
// SELU hidden, identity out) and clamp to [kPredictMin, kPerfMax].  FP64 in
// the operation order of the chosen reference kernel lane, so every estimate
// is bit-identical to the reference's.
//
// One warp per sample: lane o computes outputs o, o+32, ... of a layer as a
// dot product over the previous layer's activations (broadcast from shared
// memory) and the layer's weights stored transposed in shared memory (lanes
// read consecutive addresses).  The MLP weights are staged once per CTA.
#include <cuda_runtime.h>

#include "lane_ops.cuh"
#include "predictor.h"

namespace ocg {

namespace {

constexpr int kWarps = 8;

// dot over i of w[i*ws] * x[i] in the lane's FP order (see LaneOps::dot)
template <int LANE>
__device__ __forceinline__ double dot_strided(const double* w, int ws, const double* x, int n) {
    if (LANE == 0) {
        double acc = 0.0;
        for (int i = 0; i < n; ++i) acc = dadd(acc, dmul(w[i * ws], x[i]));
        return acc;
    }
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int i = 0;
    for (; i + 4 <= n; i += 4) {
        a0 = dfma(w[i * ws], x[i], a0);
        a1 = dfma(w[(i + 1) * ws], x[i + 1], a1);
        a2 = dfma(w[(i + 2) * ws], x[i + 2], a2);
        a3 = dfma(w[(i + 3) * ws], x[i + 3], a3);
    }
    double tail = 0.0;
    const int r = n - i;
    if (r >= 2) {
        tail = dadd(tail, dmul(w[i * ws], x[i]));
        tail = dadd(tail, dmul(w[(i + 1) * ws], x[i + 1]));
        if (r == 3) tail = dfma(w[(i + 2) * ws], x[i + 2], tail);
    } else if (r == 1) {
        tail = dfma(w[i * ws], x[i], tail);
    }
    return dadd(dadd(dadd(a0, a2), dadd(a1, a3)), tail);
}

}  // namespace

template <int LANE>
__global__ void __launch_bounds__(256) predict_perf_kernel(PredGeom g, const double* __restrict__ params,
                                                           const double* __restrict__ counters, int64_t count,
                                                           double* __restrict__ out, int* __restrict__ bad) {
    extern __shared__ __align__(16) double sm[];
    double* Wt = sm;                                  // transposed weights + biases, layer by layer
    double* act = sm + g.T + (threadIdx.x >> 5) * 2 * kPredMaxWidth;  // per warp: 2 x width
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // stage parameters: W_l (out x in, row-major) -> Wt_l (in x out), biases after
    for (int l = 0; l < g.L; ++l) {
        const int in = g.dims[l], outd = g.dims[l + 1];
        for (int e = threadIdx.x; e < in * outd; e += blockDim.x) {
            const int o = e / in, i = e - o * in;
            Wt[g.off_w[l] + i * outd + o] = params[g.off_w[l] + e];
        }
        for (int e = threadIdx.x; e < outd; e += blockDim.x) Wt[g.off_b[l] + e] = params[g.off_b[l] + e];
    }
    __syncthreads();
    for (int64_t k = static_cast<int64_t>(blockIdx.x) * kWarps + warp; k < count;
         k += static_cast<int64_t>(gridDim.x) * kWarps) {
        const double* c = counters + k * 7;
        // validate_counters (core.cpp:97-106) + standardize (predictor.cpp:74-79)
        if (lane < 7) {
            const double v = c[lane];
            bool ok = isfinite(v);
            if (lane >= 2 && lane <= 4) ok = ok && !(v < 0.0);
            if (lane >= 5) ok = ok && !(v < 0.0 || v > 1.0);
            if (!ok) atomicExch(bad, 1);
            act[lane] = ddiv(dsub(v, g.mean[lane]), g.std[lane]);
        }
        __syncwarp();
        double* cur = act;
        double* nxt = act + kPredMaxWidth;
        for (int l = 0; l < g.L; ++l) {
            const int in = g.dims[l], outd = g.dims[l + 1];
            for (int o = lane; o < outd; o += 32) {
                double z = dadd(dot_strided<LANE>(Wt + g.off_w[l] + o, outd, cur, in), Wt[g.off_b[l] + o]);
                const int a = g.acts[l];
                if (a == 0) {
                    double gf;
                    selu_fwd(z, z, gf);
                } else if (a == 1) {
                    z = z > 0 ? z : 0.0;
                }
                nxt[o] = z;
            }
            __syncwarp();
            double* t = cur;
            cur = nxt;
            nxt = t;
        }
        if (lane == 0) {
            const double v = cur[0];
            out[k] = v < 0.01 ? 0.01 : (1.25 < v ? 1.25 : v);  // std::clamp(kPredictMin, kPerfMax)
        }
        __syncwarp();
    }
}

size_t predictor_smem_bytes(const PredGeom& g) { return sizeof(double) * (g.T + kWarps * 2 * kPredMaxWidth); }

cudaError_t launch_predict_perf(const PredGeom& g, const double* params, const double* counters, int64_t count,
                                double* out, int* bad, int lane, int sm_count, cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    const size_t smem = predictor_smem_bytes(g);
    int64_t blocks = (count + kWarps - 1) / kWarps;
    if (blocks > static_cast<int64_t>(sm_count) * 8) blocks = static_cast<int64_t>(sm_count) * 8;
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        kern<<<static_cast<unsigned>(blocks), 256, smem, s>>>(g, params, counters, count, out, bad);
    };
    if (lane == 0) go(predict_perf_kernel<0>);
    else go(predict_perf_kernel<1>);
    return cudaGetLastError();
}

}  // namespace ocg
