// Batched online-phase streaming pieces:
//   * phase::Detector (phasedet.cpp:27-52) over many GPU-power streams at once —
//     the sliding-window CPU->GPU transition detector the online phase feeds
//     (policy.cpp:131-147), one warp per stream;
//   * the online phase's re-probe rule (policy.cpp:159-176) and probe ingest
//     wired into the per-app completion live in capi.cu
//     (ocg_online_ingest_complete_batch) next to the per-app plan.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "../../include/ocg.h"

int ocg_internal_fail(int code, const std::string& msg);
cudaStream_t ocg_internal_stream(ocg_ctx* ctx);
int ocg_internal_sm_count(ocg_ctx* ctx);

namespace {

// One warp per stream, 32 samples per step.  The detector fires on the first fed
// sample that completes a window of n fed samples all >= p_th (phasedet.cpp:37-48:
// "no sample in the buffer below threshold").  Feeding starts at the first sample
// (detect_offline, phasedet.cpp:61-67) or, with armed_start, at the first sample
// below the threshold (run_open_online's arming rule, policy.cpp:138-139).  A
// negative fed sample is the reference's invalid_argument (phasedet.cpp:32).
__global__ void phase_detect_kernel(int64_t nstreams, int64_t nsamples, const double* __restrict__ power,
                                    const int64_t* __restrict__ lengths, double p_th, int64_t n, int armed_start,
                                    int64_t* __restrict__ fire, int32_t* __restrict__ status) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t sidx = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; sidx < nstreams;
         sidx += nw) {
        const int64_t len = lengths ? lengths[sidx] : nsamples;
        const double* p = power + sidx * nsamples;
        bool armed = !armed_start;
        int64_t run = 0;  // consecutive fed samples >= p_th ending at the last fed sample
        int64_t hit = -1;
        int st = OCG_OK;
        for (int64_t base = 0; base < len; base += 32) {
            const int64_t i = base + lane;
            const bool valid = i < len;
            const double v = valid ? p[i] : 0.0;
            const unsigned lowm = __ballot_sync(0xffffffffu, valid && v < p_th);
            const unsigned below = lowm & ((2u << lane) - 1u);  // low samples at positions <= lane
            const bool fed = valid && (armed || below != 0u);
            int64_t r = -1;
            if (fed) r = below ? static_cast<int64_t>(lane - (31 - __clz(below))) : run + lane + 1;
            const unsigned firem = __ballot_sync(0xffffffffu, fed && r >= n);
            const unsigned negm = __ballot_sync(0xffffffffu, fed && v < 0.0);
            if (negm && (!firem || __ffs(negm) <= __ffs(firem))) {
                st = OCG_E_INVALID;
                break;
            }
            if (firem) {
                hit = base + __ffs(firem) - 1;
                break;
            }
            const unsigned validm = __ballot_sync(0xffffffffu, valid);
            const int last = 31 - __clz(validm);
            const unsigned lowv = lowm & validm;
            if (lowv) {
                armed = true;
                run = last - (31 - __clz(lowv));
            } else if (armed) {
                run += __popc(validm);
            }
        }
        if (lane == 0) {
            fire[sidx] = hit;
            if (status) status[sidx] = st;
        }
    }
}

}  // namespace

extern "C" {

int ocg_phase_detect_batch(ocg_ctx* ctx, const ocg_detector_config* cfg, int64_t nstreams, int64_t nsamples,
                           const double* power, const int64_t* lengths, int armed_start, int64_t* fire_index,
                           int32_t* status) {
    if (!cfg) return ocg_internal_fail(OCG_E_INVALID, "null detector config");
    // DetectorConfig::validate (phasedet.cpp:12-25)
    if (cfg->delta_s <= 0 || cfg->window_s <= 0 || cfg->p_th_w <= 0)
        return ocg_internal_fail(OCG_E_INVALID, "detector config: fields must be positive");
    const double nd = static_cast<double>(std::llround(cfg->window_s / cfg->delta_s));
    const int64_t n = static_cast<int64_t>(nd);
    if (n == 0 || std::abs(nd * cfg->delta_s - cfg->window_s) > 1e-9)
        return ocg_internal_fail(OCG_E_INVALID, "detector config: window_s must be a multiple of delta_s");
    const double per_sec = 1.0 / cfg->delta_s;
    if (std::abs(per_sec - std::round(per_sec)) > 1e-9 || std::abs(cfg->window_s - std::round(cfg->window_s)) > 1e-9)
        return ocg_internal_fail(OCG_E_INVALID, "detector config: window must split into 1-second intervals");
    if (nstreams < 0 || nsamples < 0) return ocg_internal_fail(OCG_E_INVALID, "negative stream shape");
    if (nstreams == 0) return OCG_OK;
    if (!ctx || !power || !fire_index) return ocg_internal_fail(OCG_E_INVALID, "null argument");
    if (lengths)
        for (int64_t s = 0; s < nstreams; ++s)
            if (lengths[s] < 0 || lengths[s] > nsamples) return ocg_internal_fail(OCG_E_RANGE, "stream length");
    cudaStream_t st = ocg_internal_stream(ctx);
    const size_t pbytes = sizeof(double) * static_cast<size_t>(nstreams * nsamples);
    double* dp = nullptr;
    int64_t *dl = nullptr, *df = nullptr;
    int32_t* ds = nullptr;
    cudaError_t e = cudaMalloc(&dp, pbytes);
    if (e == cudaSuccess) e = cudaMalloc(&df, sizeof(int64_t) * nstreams);
    if (e == cudaSuccess) e = cudaMalloc(&ds, sizeof(int32_t) * nstreams);
    if (e == cudaSuccess && lengths) e = cudaMalloc(&dl, sizeof(int64_t) * nstreams);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dp, power, pbytes, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess && lengths)
        e = cudaMemcpyAsync(dl, lengths, sizeof(int64_t) * nstreams, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) {
        const int64_t blocks = std::min<int64_t>((nstreams + 7) / 8, 16 * ocg_internal_sm_count(ctx));
        phase_detect_kernel<<<static_cast<unsigned>(std::max<int64_t>(blocks, 1)), 256, 0, st>>>(
            nstreams, nsamples, dp, dl, cfg->p_th_w, n, armed_start, df, ds);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(fire_index, df, sizeof(int64_t) * nstreams, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && status)
        e = cudaMemcpyAsync(status, ds, sizeof(int32_t) * nstreams, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(dp);
    cudaFree(dl);
    cudaFree(df);
    cudaFree(ds);
    if (e != cudaSuccess) return ocg_internal_fail(OCG_E_CUDA, std::string("phase detect: ") + cudaGetErrorString(e));
    return OCG_OK;
}

}  // extern "C"
