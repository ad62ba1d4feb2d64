// Host-visible geometry / IO descriptors of the per-app batched NCF kernel.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/ocg.h"

namespace ocg {

constexpr int kMaxLayers = 4;      // MLP layers (hidden + output)
constexpr int kMaxWidth = 64;      // widest MLP layer / input
constexpr int kMaxParams = 2048;   // parameters of one app's model (8 per compute thread)
constexpr int kFixMaxParams = 1536; // same, reference-default architecture kernel (6 per thread)
constexpr int kMaxCells = 16384;   // observed cells of one app's matrix
constexpr int kMaxBatch = 32;      // minibatch size (one sample per lane)

struct BatchGeom {
    int m, n, ka, ks, L;
    int dims[kMaxLayers + 1];
    int off_w[kMaxLayers], off_b[kMaxLayers];
    int set_off, T;
    int stride[kMaxLayers + 1];
    int block_nnz, block_full, max_cells;
    int batch, max_epochs, patience;
    double lr, val_fraction;
    uint64_t fit_tag_mix;  // splitmix64(fnv1a("ncf.fit"))
    int ngpu;
    double e_base, gamma;
};

struct OcgMetaDev {
    uint64_t seed;
    int32_t epochs_run;
    double initial_train_mse, final_train_mse, best_val_mse;
};
static_assert(sizeof(OcgMetaDev) == sizeof(ocg_ncf_meta), "meta layout");

struct BatchIO {
    int64_t napps;
    const double* block_val;
    const uint32_t* block_rc;
    const uint8_t* block_col_seen;
    const double* probe_vals;
    const uint8_t* probe_mask;
    const uint64_t* seeds;
    const int32_t* cpu_caps;
    const int32_t* gpu_caps;
    double* completed;
    int32_t* sel_idx;
    double* sel_saving;
    double* sel_loss;
    int32_t* sel_ncand;
    OcgMetaDev* meta;
    int32_t* status;
    double* params;
    int64_t params_stride;
    double* best;         // per-CTA best-parameter snapshot (gridDim.x x best_stride), device scratch
    int64_t best_stride;
};

size_t batch_smem_bytes(const BatchGeom& g);
bool batch_is_fixed_k8(const BatchGeom& g);
int batch_threads();
int batch_max_active_per_sm(const BatchGeom& g, int lane);
cudaError_t launch_app_batch(const BatchGeom& g, const BatchIO& io, int lane, int grid, cudaStream_t stream);

}  // namespace ocg
