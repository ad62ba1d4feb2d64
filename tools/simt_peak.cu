// Measured SIMT peaks of this GPU (FP64 DFMA and FP32 FFMA throughput), the
// roofline denominators for the FP64 parity kernels and the FP32 ALS Gram —
// MEASURED_PEAKS.json has only HBM and bf16 tensor figures.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o simt_peak tools/simt_peak.cu && ./simt_peak
// Prints one JSON line: {"fp64_tflops": ..., "fp32_tflops": ..., "sm_count": ...}
#include <cstdio>
#include <cuda_runtime.h>

template <typename T, int CHAINS, int ITERS>
__global__ void __launch_bounds__(256) fma_kernel(T* out, T a, T b) {
    T acc[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = static_cast<T>(threadIdx.x + c);
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
    }
    T s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += acc[c];
    if (s == static_cast<T>(-1.2345)) out[threadIdx.x] = s;  // keep live, never taken
}

template <typename T>
double measure(int sms) {
    constexpr int kChains = 8, kIters = 4096;
    T* out;
    cudaMalloc(&out, 1024 * sizeof(T));
    const int blocks = sms * 8;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
        cudaEventRecord(e0);
        fma_kernel<T, kChains, kIters><<<blocks, 256>>>(out, static_cast<T>(0.999999), static_cast<T>(1e-7));
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;
    }
    cudaFree(out);
    const double flops = 2.0 * blocks * 256.0 * kChains * kIters;
    return flops / (best * 1e-3) / 1e12;
}

int main() {
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const double f64 = measure<double>(sms), f32 = measure<float>(sms);
    std::printf("{\"fp64_tflops\": %.2f, \"fp32_tflops\": %.2f, \"sm_count\": %d, "
                "\"how\": \"dependent-FMA chains x8 per thread, %d x 8 CTAs x 256 threads, best of 5 (CUDA events)\"}\n",
                f64, f32, sms, sms);
    return 0;
}
