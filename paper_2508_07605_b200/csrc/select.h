#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace ocg {

cudaError_t launch_select_rows(const void* rows, int dtype, int64_t nrows, int n, const int32_t* d_cpu,
                               const int32_t* d_gpu, int ngpu, double e_base, double gamma, int32_t* idx,
                               double* saving, double* loss, int32_t* ncand, int* d_bad, int sm_count,
                               cudaStream_t stream);

}  // namespace ocg
