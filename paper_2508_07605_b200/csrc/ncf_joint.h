// Joint-mode NCF fit: cf::fit (cfcomplete.cpp:63-196) over one whole sparse
// matrix on one GPU (ncf_joint.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/ocg.h"

namespace ocg {

// precision: OCG_NCF_EXACT (FP64, operation order of `lane`: bit-identical to the
// reference) or OCG_NCF_FAST (FP32, same schedule).  Outputs are host buffers:
// params in the flat layout [app m x ka | setting n x ks | W0 b0 W1 b1 ...]
// (the reference's Adam block order), app_seen[m], setting_seen[n], meta.
// Returns an OCG_* code; err receives the message.
struct JointFitStats {
    int64_t steps = 0;        // minibatch steps run
    int64_t replay_tasks = 0; // helper row replays issued
    double device_ms = 0.0;   // CUDA-event time of the fit on the stream
};

int joint_ncf_fit(cudaStream_t stream, int sm_count, int64_t m, int64_t n, const int64_t* row_ptr,
                  const int32_t* col, const double* val, const ocg_ncf_hyper& h, uint64_t seed, int precision,
                  int lane, double* params, uint8_t* app_seen, uint8_t* setting_seen, ocg_ncf_meta* meta,
                  JointFitStats* stats, std::string& err);

// shapes the joint kernel accepts (OCG_OK or OCG_E_UNSUPPORTED with a message)
int joint_ncf_supported(const ocg_ncf_hyper& h, int precision, std::string& err);

}  // namespace ocg
