// K1 — batched policy::select_caps (policy.cpp:17-64) over completed rows in HBM.
//
// One warp per row, a grid-stride loop of warps over rows.  Row values are
// streamed with coalesced loads (each lane walks the row at a 32-element
// stride), FP32 rows are widened to double exactly before the FP64
// arithmetic.  Validation mirrors the reference (:23-25): any non-finite or
// non-positive entry fails the whole call with invalid_argument.
#include <cuda_runtime.h>

#include "ocg_common.cuh"
#include "select_dev.cuh"
#include "select.h"

namespace ocg {

template <typename T>
__global__ void __launch_bounds__(256) select_rows_kernel(const T* __restrict__ rows, int64_t nrows, int n,
                                                          const int32_t* __restrict__ cpu,
                                                          const int32_t* __restrict__ gpu, int ngpu,
                                                          double e_base, double gamma, int32_t* idx,
                                                          double* saving, double* loss, int32_t* ncand,
                                                          int* bad) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t r = warp; r < nrows; r += nwarps) {
        const T* row = rows + r * n;
        bool ok = true;
        for (int j = lane; j < n; j += 32) {
            const double p = static_cast<double>(row[j]);
            ok &= isfinite(p) && p > 0.0;
        }
        if (!__all_sync(0xffffffffu, ok)) {
            if (lane == 0) {
                atomicExch(bad, 1);
                idx[r] = -1;
            }
            continue;
        }
        const SelResult s = select_row_warp(row, n, cpu, gpu, ngpu, e_base, gamma, lane);
        if (lane == 0) {
            idx[r] = s.idx;
            saving[r] = s.saving;
            loss[r] = s.loss;
            ncand[r] = s.ncand;
        }
    }
}

cudaError_t launch_select_rows(const void* rows, int dtype, int64_t nrows, int n, const int32_t* d_cpu,
                               const int32_t* d_gpu, int ngpu, double e_base, double gamma, int32_t* idx,
                               double* saving, double* loss, int32_t* ncand, int* d_bad, int sm_count,
                               cudaStream_t stream) {
    const int threads = 256;
    const int64_t warps_needed = nrows;
    int64_t blocks = (warps_needed * 32 + threads - 1) / threads;
    const int64_t cap = static_cast<int64_t>(sm_count) * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    if (dtype == 0)
        select_rows_kernel<double><<<static_cast<int>(blocks), threads, 0, stream>>>(
            static_cast<const double*>(rows), nrows, n, d_cpu, d_gpu, ngpu, e_base, gamma, idx, saving, loss,
            ncand, d_bad);
    else
        select_rows_kernel<float><<<static_cast<int>(blocks), threads, 0, stream>>>(
            static_cast<const float*>(rows), nrows, n, d_cpu, d_gpu, ngpu, e_base, gamma, idx, saving, loss,
            ncand, d_bad);
    return cudaGetLastError();
}

}  // namespace ocg
