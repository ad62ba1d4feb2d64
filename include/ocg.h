/* ocg.h — C-ABI of the B200-native online CF completion + selection path
 * (OPEN, arXiv 2508.07605, online phase).  Plain pointers and sizes only.
 *
 * Every entry point replaces a reference interface; the citation after each
 * declaration names it (paths under the reference's proj/).  Semantics and
 * error behaviour follow the reference; return codes map its exception types:
 *
 *   OCG_OK           0
 *   OCG_E_INVALID    1  std::invalid_argument / config_error
 *   OCG_E_MISSING    2  missing_artifact_error
 *   OCG_E_LOGIC      3  std::logic_error / other runtime errors
 *   OCG_E_RANGE      4  std::out_of_range
 *   OCG_E_COLD       5  std::runtime_error "cold app row / setting column"
 *   OCG_E_DIVERGE    6  std::runtime_error "ncf: divergence"
 *   OCG_E_CUDA       7  CUDA / NCCL / allocation failure (no reference analogue)
 *   OCG_E_UNSUPPORTED 8 shape outside what the compiled kernels handle
 *
 * All calls are synchronous on the context's stream.  A context is owned by
 * one thread at a time (as cf::fit is single-owner, SPEC.md "Concurrency
 * Model"); models are immutable after fit and may be shared for predict.
 * "host" pointers are ordinary CPU memory; "_dev" entry points take device
 * pointers already resident in HBM (used by bench.py's kernel-only timing).
 * There is no CPU fallback: without a usable CUDA device every compute entry
 * point returns OCG_E_CUDA. */
#ifndef OCG_H
#define OCG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    OCG_OK = 0,
    OCG_E_INVALID = 1,
    OCG_E_MISSING = 2,
    OCG_E_LOGIC = 3,
    OCG_E_RANGE = 4,
    OCG_E_COLD = 5,
    OCG_E_DIVERGE = 6,
    OCG_E_CUDA = 7,
    OCG_E_UNSUPPORTED = 8
};

/* FP-order lane to reproduce: the reference's kern::Lane (kernels.hpp:28). */
enum { OCG_LANE_SCALAR = 0, OCG_LANE_AVX2 = 1 };

typedef struct ocg_ctx ocg_ctx;

/* cf::NcfHyper (cfcomplete.hpp:11-20) */
typedef struct {
    int64_t app_dim, setting_dim;
    int64_t hidden[8];
    int64_t n_hidden;
    double lr;
    int32_t max_epochs, patience;
    double val_fraction;
    int32_t batch_size;
} ocg_ncf_hyper;

/* cf::NcfModel::Meta (cfcomplete.hpp:34-40) */
typedef struct {
    uint64_t seed;
    int32_t epochs_run;
    double initial_train_mse, final_train_mse, best_val_mse;
} ocg_ncf_meta;

const char* ocg_last_error(void);   /* thread-local message of the last failure */
int ocg_version(void);
void ocg_ncf_hyper_default(ocg_ncf_hyper* h);            /* NcfHyper{} defaults */
uint64_t ocg_derive_seed(uint64_t root, const char* tag, uint64_t n); /* rng.hpp:53-60 */

int ocg_ctx_create(int device, ocg_ctx** out);
void ocg_ctx_destroy(ocg_ctx* ctx);
int ocg_ctx_device_info(ocg_ctx* ctx, int* sm_count, int* cc_major, int* cc_minor);
int ocg_ctx_flush_l2(ocg_ctx* ctx);    /* overwrite a 256 MB scratch buffer (> L2) on the stream */
int ocg_ctx_synchronize(ocg_ctx* ctx);
/* run the context's work on an external stream (e.g. torch's current stream,
 * so NCCL collectives issued by torch are ordered with our kernels) */
int ocg_ctx_set_stream(ocg_ctx* ctx, void* stream);

/* ---- K1: Algorithm 2 selection ---------------------------------------
 * policy::select_caps (policy.cpp:17-64; policy.hpp:34) batched over `nrows`
 * completed rows, row-major nrows x (ncpu*ngpu) FP64, columns in
 * PowerGrid::settings() order (core.cpp:59-65).  Outputs per row: column
 * index of the chosen setting, pred_saving, pred_loss, candidates_considered.
 * Bit-exact with the reference (FP64, same operation order). */
int ocg_select_caps(ocg_ctx* ctx, const double* rows, int64_t nrows, const int32_t* cpu_caps,
                    int32_t ncpu, const int32_t* gpu_caps, int32_t ngpu, double gamma,
                    int32_t* idx, double* saving, double* loss, int32_t* ncand);
/* same, device pointers; rows FP64 (dtype 0) or FP32 (dtype 1, widened to
 * double exactly before the FP64 arithmetic) */
int ocg_select_caps_dev(ocg_ctx* ctx, const void* d_rows, int dtype, int64_t nrows,
                        const int32_t* cpu_caps, int32_t ncpu, const int32_t* gpu_caps,
                        int32_t ngpu, double gamma, int32_t* d_idx, double* d_saving,
                        double* d_loss, int32_t* d_ncand);

/* ProbePlan::default_plan (policy.cpp:66-82): the sampled-setting set as
 * column indices in plan order; returns the count through *count (<= 6). */
int ocg_default_plan(const int32_t* cpu_caps, int32_t ncpu, const int32_t* gpu_caps, int32_t ngpu,
                     int32_t* cols, int32_t* count);

/* ---- per-app online completion (reference orchestration semantics) -----
 * run_open_online steps 3-4 (policy.cpp:178-189) for `napps` independent
 * unseen apps: for app a, sparse = dense block (d_rows x n, values + mask)
 * with the app's probe row appended (probe_vals/probe_mask row a), then
 * cf::complete(sparse, hyper, seeds[a]) (cfcomplete.cpp:198-213, i.e. a full
 * cf::fit :63-196 + NcfModel::predict :47-58 of every missing cell), then
 * policy::select_caps on the app's completed row.  One CTA owns one app's
 * whole fit on the device; FP64, operation order of `lane`.
 * Outputs (host, each may be NULL except status): completed row (napps x n),
 * decision (idx/saving/loss/ncand), meta, per-app status (OCG_* code of the
 * exception the reference would have thrown for that app). */
int ocg_online_complete_batch(ocg_ctx* ctx, int64_t d_rows, const double* block_vals,
                              const uint8_t* block_mask, int64_t napps, const double* probe_vals,
                              const uint8_t* probe_mask, const uint64_t* seeds,
                              const int32_t* cpu_caps, int32_t ncpu, const int32_t* gpu_caps,
                              int32_t ngpu, const ocg_ncf_hyper* hyper, double gamma, int lane,
                              double* completed, int32_t* idx, double* saving, double* loss,
                              int32_t* ncand, ocg_ncf_meta* meta, int32_t* status);

/* Device-resident form of ocg_online_complete_batch: inputs are uploaded once
 * by _create; _run re-runs the completion kernel on data already in HBM and,
 * if kernel_ms is non-NULL, waits and returns its CUDA-event duration on the
 * context stream; _results copies the outputs back. */
typedef struct ocg_online_plan ocg_online_plan;
int ocg_online_plan_create(ocg_ctx* ctx, int64_t d_rows, const double* block_vals,
                           const uint8_t* block_mask, int64_t napps, const double* probe_vals,
                           const uint8_t* probe_mask, const uint64_t* seeds, const int32_t* cpu_caps,
                           int32_t ncpu, const int32_t* gpu_caps, int32_t ngpu,
                           const ocg_ncf_hyper* hyper, double gamma, int lane, int want_completed,
                           ocg_online_plan** out);
int ocg_online_plan_run(ocg_online_plan* plan, float* kernel_ms);
int ocg_online_plan_results(ocg_online_plan* plan, double* completed, int32_t* idx, double* saving,
                            double* loss, int32_t* ncand, ocg_ncf_meta* meta, int32_t* status);
void ocg_online_plan_destroy(ocg_online_plan* plan);

/* ---- batched online-phase streams --------------------------
 * phase::DetectorConfig (phasedet.hpp:13-20) */
typedef struct {
    double delta_s, window_s, p_th_w;  /* defaults 0.2 s, 5 s, 60 W */
} ocg_detector_config;

/* phase::Detector (phasedet.cpp:27-52) over nstreams GPU-power streams (row-major
 * nstreams x nsamples host array; stream s uses its first lengths[s] samples, or all
 * with lengths == NULL): fire_index[s] = index of the sample on which the
 * sliding-window CPU->GPU transition detector first fires (every sample of a full
 * window of window_s/delta_s fed samples >= p_th_w), -1 if it never does.
 * armed_start = 0: every sample is fed (detect_offline, phasedet.cpp:61-67);
 * 1: feeding starts at the first sample below the threshold (run_open_online's
 * arming rule, policy.cpp:138-139).  Config errors as DetectorConfig::validate
 * (OCG_E_INVALID); status[s] (may be NULL) = OCG_E_INVALID for a stream that feeds a
 * negative sample before firing (Detector::feed's invalid_argument). */
int ocg_phase_detect_batch(ocg_ctx* ctx, const ocg_detector_config* cfg, int64_t nstreams, int64_t nsamples,
                           const double* power, const int64_t* lengths, int armed_start, int64_t* fire_index,
                           int32_t* status);


/* Fit-only variant returning every app's parameters in the flat layout
 * [app table | setting table | W0 b0 W1 b1 ... ] (the reference's Adam block
 * order, cfcomplete.cpp:107-110) for parameter-level parity tests. */
int ocg_online_fit_batch_params(ocg_ctx* ctx, int64_t d_rows, const double* block_vals,
                                const uint8_t* block_mask, int64_t napps,
                                const double* probe_vals, const uint8_t* probe_mask,
                                const uint64_t* seeds, int32_t n, const ocg_ncf_hyper* hyper,
                                int lane, double* params, int64_t params_stride,
                                ocg_ncf_meta* meta, int32_t* status);

/* NCF inference on given parameters (NcfModel::predict, cfcomplete.cpp:47-58):
 * FP64 lane-exact forward + clamp for (rows[k], cols[k]) pairs. */
int ocg_ncf_predict(ocg_ctx* ctx, int64_t m, int64_t n, const ocg_ncf_hyper* hyper,
                    const double* params, const uint8_t* app_seen, const uint8_t* setting_seen,
                    const int64_t* rows, const int64_t* cols, int64_t count, int lane,
                    double* out);

/* NCF model file (SURVEY §8b ocg_model_to_json / from_json): cf::NcfModel::to_json
 * / from_json (cfcomplete.cpp:215-265, nn::model_to_json nnkit.cpp:306-365) over
 * the flat parameter layout above, byte-identical text (nlohmann::json dump(2),
 * the reference's own serializer).  Host-only.
 * to_json: out == NULL queries *len (bytes including the terminating NUL).
 * from_json: params == NULL queries the shapes (hyper dims, m, n, *nparams);
 * then params[*nparams], app_seen[m], setting_seen[n], meta (each may be NULL). */
int ocg_ncf_model_to_json(const ocg_ncf_hyper* hyper, int64_t m, int64_t n, const double* params,
                          const uint8_t* app_seen, const uint8_t* setting_seen, const ocg_ncf_meta* meta,
                          char* out, size_t cap, size_t* len);
int ocg_ncf_model_from_json(const char* text, ocg_ncf_hyper* hyper, int64_t* m, int64_t* n, int64_t* nparams,
                            double* params, uint8_t* app_seen, uint8_t* setting_seen, ocg_ncf_meta* meta);

/* ---- NCF completion + selection over a whole matrix (SURVEY §8a a9 + a10) -
 * A fitted cf::NcfModel (cfcomplete.hpp:25-55) resident in HBM, and a plan
 * binding it to a sparse matrix: cf::complete's imputation of every unobserved
 * cell (cfcomplete.cpp:208-211, NcfModel::predict :47-58; observed cells kept
 * verbatim) fused with policy::select_caps (policy.cpp:17-64) on every row.
 * The completed m x n matrix is never materialised.
 *   OCG_NCF_EXACT: FP64 in the operation order of `lane`, glibc exp —
 *                  predictions and decisions bit-identical to the reference.
 *   OCG_NCF_FAST:  FP32 + tcgen05 tensor cores (hidden {32, 16} only), |dp|/p
 *                  ~1e-6; decisions identical wherever the margin exceeds it
 *                  (the baseline p_{i,n-1} is always computed exactly).
 * Model: params in the flat layout [app m x ka | setting n x ks | W0 b0 W1 b1 ...]
 * (as ocg_ncf_model_from_json returns), app_seen[m], setting_seen[n].
 * Matrix: CSR row_ptr[m+1] (int64), col[nnz] (int32, ascending per row), val[nnz]
 * (FP64, (0, 1.25]); on_device = 1: device pointers used in place.
 * Errors (from _results / _completed_rows, as the reference would throw for the
 * whole call): OCG_E_RANGE column index out of range; OCG_E_INVALID row without
 * observed entries (cfcomplete.cpp:199-205) or value outside (0, 1.25]
 * (core.cpp:145-147); OCG_E_COLD cold app row / setting column (:50-55);
 * OCG_E_UNSUPPORTED fast path with |W0 . x| >= 80 (use EXACT). */
typedef struct ocg_ncf_model ocg_ncf_model;
typedef struct ocg_ncf_plan ocg_ncf_plan;
enum { OCG_NCF_EXACT = 0, OCG_NCF_FAST = 1 };
int ocg_ncf_model_create(ocg_ctx* ctx, const ocg_ncf_hyper* hyper, int64_t m, int64_t n, const double* params,
                         const uint8_t* app_seen, const uint8_t* setting_seen, ocg_ncf_model** out);
/* NcfModel::from_json (cfcomplete.cpp:235-265) straight into HBM */
int ocg_ncf_model_from_json_text(ocg_ctx* ctx, const char* text, ocg_ncf_model** out);
void ocg_ncf_model_destroy(ocg_ncf_model* model);
int ocg_ncf_plan_create(ocg_ncf_model* model, const int64_t* row_ptr, const int32_t* col, const double* val,
                        int on_device, const int32_t* cpu_caps, int32_t ncpu, const int32_t* gpu_caps, int32_t ngpu,
                        double gamma, int precision, int lane, ocg_ncf_plan** out);
/* a new matrix (same m) for the plan, host CSR copied on the context stream */
int ocg_ncf_plan_upload(ocg_ncf_plan* plan, const int64_t* row_ptr, const int32_t* col, const double* val);
/* one completion + selection of every row; total_ms / phase_ms[2] (prep: validation,
 * A/B precompute, baselines, observed cells; dense pass) as CUDA-event times (NULL = async) */
int ocg_ncf_plan_run(ocg_ncf_plan* plan, float* total_ms, float* phase_ms);
int ocg_ncf_plan_results(ocg_ncf_plan* plan, int32_t* idx, double* saving, double* loss, int32_t* ncand);
/* pipelined serving: _stage copies the next step's host CSR (pinned memory for an async
 * copy) on a side stream into spare buffers while the current step may still run; the next
 * _run swaps it in (a device-side wait).  _results_async queues the decisions' device->host
 * copies behind the run (the following _run may be enqueued at once); _results_wait blocks
 * until they landed and reports the run's error as _results would.  One staged CSR at a time. */
int ocg_ncf_plan_stage(ocg_ncf_plan* plan, const int64_t* row_ptr, const int32_t* col, const double* val);
int ocg_ncf_plan_results_async(ocg_ncf_plan* plan, int32_t* idx, double* saving, double* loss, int32_t* ncand);
int ocg_ncf_plan_results_wait(ocg_ncf_plan* plan);
/* completed values (nrows x n, FP64) of the listed rows (test / inspection hook) */
int ocg_ncf_plan_completed_rows(ocg_ncf_plan* plan, const int64_t* rows, int64_t nrows, double* out);
void ocg_ncf_plan_destroy(ocg_ncf_plan* plan);

/* ---- cf:: over one whole matrix, every solver ---------------
 * Matrix: host CSR row_ptr[m+1] (int64), col[nnz] (int32, strictly ascending per
 * row), val[nnz] (FP64 in (0, 1.25]), columns in PowerGrid::settings() order.
 * Rejections mirror PerformanceMatrix::set (core.cpp:142-148: OCG_E_RANGE for a
 * column index, OCG_E_INVALID for a value) plus the CSR invariants.
 * Solvers:
 *   OCG_SOLVER_NCF_REF  the reference's NCF and schedule in FP64, operation order
 *                       of `lane`: parameters, meta and predictions bit-identical
 *                       to cf::fit / cf::complete
 *   OCG_SOLVER_NCF_FAST the same NCF and schedule in FP32 (FP32 tensor-core
 *                       inference for hidden {32, 16})
 *   OCG_SOLVER_ALS      rank-k ALS (ocg_als_hyper; no reference counterpart) */
enum { OCG_SOLVER_NCF_REF = 0, OCG_SOLVER_NCF_FAST = 1, OCG_SOLVER_ALS = 2 };

/* cf::fit (cfcomplete.hpp:59; cfcomplete.cpp:63-196), joint mode: one model over
 * the whole matrix on the context's GPU.  Outputs (host, each may be NULL):
 * params in the flat layout [app m x ka | setting n x ks | W0 b0 W1 b1 ...],
 * app_seen[m], setting_seen[n], meta.  Errors: OCG_E_INVALID bad hyperparameters
 * / no observed entries (:64-72), OCG_E_DIVERGE non-finite validation loss
 * (:180), OCG_E_LOGIC non-finite final weight (nnkit.cpp:106-113),
 * OCG_E_UNSUPPORTED dims beyond the kernel (embedding > 64, hidden > 64,
 * > 3 hidden layers, batch_size > 32). */
int ocg_cf_fit(ocg_ctx* ctx, int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
               const ocg_ncf_hyper* hyper, uint64_t seed, int solver, int lane, double* params, uint8_t* app_seen,
               uint8_t* setting_seen, ocg_ncf_meta* meta);
/* same, also returning the minibatch steps run and the fit's CUDA-event time */
int ocg_cf_fit_stats(ocg_ctx* ctx, int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
                     const ocg_ncf_hyper* hyper, uint64_t seed, int solver, int lane, double* params, uint8_t* app_seen,
                     uint8_t* setting_seen, ocg_ncf_meta* meta, int64_t* steps, double* device_ms);

/* ALS hyperparameters (OCG_SOLVER_ALS, ocg_als_plan_*) */
typedef struct {
    int32_t rank;   /* 8, 16, 32 or 64 */
    float lambda;   /* weighted-lambda regularisation */
    int32_t sweeps; /* row + column half-sweeps per fit */
    uint64_t seed;  /* V initialisation (ocgo_als_init_value) */
} ocg_als_hyper;

/* cf::complete (cfcomplete.hpp:63; cfcomplete.cpp:198-213): completed m x n
 * matrix (observed cells verbatim, every other cell the model's clamped
 * prediction; fully observed input returned unchanged without a fit), written
 * row-major into `completed` (host, may be NULL).  With cpu_caps != NULL, also
 * policy::select_caps (policy.cpp:17-64) of every completed row into
 * idx/saving/loss/ncand (host, m each) — fused with the imputation, the
 * completed matrix need not be materialised.  `hyper` is used by the NCF
 * solvers, `als` by OCG_SOLVER_ALS.  Errors as ocg_cf_fit, plus OCG_E_INVALID
 * for a row without observed entries (:199-205) and OCG_E_COLD for a cell in a
 * column that had no observation at fit time (:50-55). */
int ocg_cf_complete(ocg_ctx* ctx, int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
                    const ocg_ncf_hyper* hyper, const ocg_als_hyper* als, uint64_t seed, int solver, int lane,
                    const int32_t* cpu_caps, int32_t ncpu, const int32_t* gpu_caps, int32_t ngpu, double gamma,
                    double* completed, int32_t* idx, double* saving, double* loss, int32_t* ncand);

/* ---- ALS completion + selection (joint mode) -------
 * No reference counterpart: the reference's CF is NCF only.  Semantics are
 * defined by the CPU oracle (oracle/ocg_oracle.c, ocgo_als_fit): weighted-
 * lambda ALS P ~ U V^T of rank k over the observed CSR entries, then
 * cf::complete-style imputation (observed verbatim, clamp(u_i.v_j, 0.01,
 * 1.25) elsewhere) fused with policy::select_caps (policy.cpp:17-64) per row.
 * FP32 factors, FP64 selection arithmetic.  Parity vs the reference:
 * unpinned (vs the oracle: within tolerance; selections exact given the
 * completed rows). */

typedef struct ocg_als_plan ocg_als_plan;
/* CSR input: row_ptr[m+1] (int64), col[nnz] (int32, ascending per row),
 * val[nnz] (FP32 normalized performance).  on_device=0: host buffers are
 * copied; on_device=1: device pointers are used in place (must outlive the
 * plan).  Columns follow PowerGrid::settings() of (cpu_caps x gpu_caps). */
int ocg_als_plan_create(ocg_ctx* ctx, int64_t m, const int64_t* row_ptr, const int32_t* col, const float* val,
                        int on_device, const int32_t* cpu_caps, int32_t ncpu, const int32_t* gpu_caps,
                        int32_t ngpu, const ocg_als_hyper* hyper, double gamma, ocg_als_plan** out);
/* new observations for an existing plan (streaming refits, SURVEY §8d C4;
 * end-to-end timing): host CSR with the plan's m (nnz may change: the
 * nnz-dependent device state is rebuilt, the factors are kept), copied
 * asynchronously on the context stream into the plan's own device buffers
 * (pinned host memory makes the copy overlap-capable); the next _run
 * completes it.  OCG_E_INVALID if the plan was created on device pointers. */
int ocg_als_plan_upload(ocg_als_plan* plan, const int64_t* row_ptr, const int32_t* col, const float* val);
/* the same with 16-bit column indices (n <= 65536: every grid of the paper and
 * of C1-C4), widened on the device: 25% fewer bytes over PCIe per refit */
int ocg_als_plan_upload_compact(ocg_als_plan* plan, const int64_t* row_ptr, const uint16_t* col16, const float* val);
/* double-buffered input (pipelined refits): copies the next step's CSR (16-bit
 * columns, pinned host memory) on a side stream into staging buffers while the
 * current step may still run; the next ocg_als_plan_run swaps it in (waits for the
 * copy on the device, not the host).  The host buffers must stay unchanged until
 * that run has completed.  One staged CSR at a time; _upload / _add_observations
 * are refused while one is pending (OCG_E_INVALID). */
int ocg_als_plan_stage_compact(ocg_als_plan* plan, const int64_t* row_ptr, const uint16_t* col16, const float* val);
/* streaming arrivals: merge `count` new observed cells (host
 * arrays sorted by (row, col); cells not observed yet) into the plan's device CSR
 * -- the same matrix as uploading the merged CSR, with only the new cells crossing
 * PCIe.  OCG_E_INVALID for unsorted / out-of-range / already observed cells (the
 * plan is left unchanged).  Synchronises the context stream. */
int ocg_als_plan_add_observations(ocg_als_plan* plan, int64_t count, const int32_t* rows, const int32_t* cols,
                                  const float* vals);
/* warm refits (a flagged deviation from the reference's from-scratch cf::complete):
 * warm_sweeps > 0 makes every later _run after the first start from the previous
 * factors (no V initialisation) and run warm_sweeps sweeps; 0 restores from-scratch. */
int ocg_als_plan_set_warm(ocg_als_plan* plan, int32_t warm_sweeps);
/* one full step on device data: CSC build, fit, fused imputation+selection.
 * total_ms / phase_ms[6] (CSC, row sweeps, column sweeps, select, and at rank
 * 32 the row / column Gram kernels alone): CUDA-event times on the context
 * stream (either may be NULL = asynchronous). */
int ocg_als_plan_run(ocg_als_plan* plan, float* total_ms, float* phase_ms);
/* Phase-level form of _run for the row-sharded multi-GPU driver (each rank
 * holds a row shard of the CSR with all n columns): begin = CSC +
 * V init; per sweep: row_half (local), col_gram (this shard's column Gram
 * records, n x ocg_als_plan_gram_floats/n floats: k*k + k + 1 at rank 8/16,
 * the 612-float packed lower-triangle record at rank 32, into d_gram) ->
 * allreduce(sum) across
 * ranks -> col_solve(d_gram) (replicated, deterministic); finally select.
 * col_half = the single-GPU fused column half-sweep. */
int ocg_als_plan_begin(ocg_als_plan* plan);
int ocg_als_plan_row_half(ocg_als_plan* plan);
int ocg_als_plan_col_half(ocg_als_plan* plan);
int64_t ocg_als_plan_gram_floats(ocg_als_plan* plan);
int ocg_als_plan_col_gram(ocg_als_plan* plan, float* d_gram);
int ocg_als_plan_col_solve(ocg_als_plan* plan, const float* d_gram);
int ocg_als_plan_select(ocg_als_plan* plan);
int ocg_als_plan_results(ocg_als_plan* plan, int32_t* idx, double* saving, double* loss, int32_t* ncand,
                         float* U, float* V);
/* the decisions (not the factors) copied into host buffers asynchronously on the context
 * stream, behind the run that produced them: a following _run may be enqueued at once
 * (pipelined refits); _results_wait blocks until the copies have landed.  Pinned host
 * buffers make the copies truly asynchronous. */
int ocg_als_plan_results_async(ocg_als_plan* plan, int32_t* idx, double* saving, double* loss, int32_t* ncand);
int ocg_als_plan_results_wait(ocg_als_plan* plan);
int ocg_als_plan_completed_rows(ocg_als_plan* plan, int64_t row0, int64_t nrows, double* out);
void ocg_als_plan_destroy(ocg_als_plan* plan);

/* ---- file formats (host only, no GPU needed; SURVEY §8b loaders, §8f-2) ----
 * A host matrix: app ids, one (cpu, gpu) setting per column, observed cells as
 * CSR (row_ptr int64 [m+1], col int32 ascending, val FP64 in (0, 1.25]).
 * read_csv   <- read_matrix_csv_file (core.cpp:213-254): OCG_E_MISSING if the file
 *               is absent, OCG_E_INVALID for config_error (header, labels, ragged
 *               or non-numeric cells) and invalid_argument (empty / duplicate /
 *               delimiter-bearing app ids, duplicate settings, a value outside
 *               (0, 1.25]) — in the reference's check order.
 * write_csv  <- write_matrix_csv (core.cpp:191-205), round-trip-exact values
 *               (format_double, core.cpp:171-175): byte-identical to the reference's.
 * save_bin / load_bin: the same matrix as a binary CSR ("OCGCSR1"; no reference
 *               counterpart — CSV at C2 is tens of GB of text); load_bin validates
 *               like ocg_matrix_create. */
typedef struct ocg_matrix ocg_matrix;
int ocg_matrix_read_csv(const char* path, ocg_matrix** out);
int ocg_matrix_write_csv(const ocg_matrix* mat, const char* path);
int ocg_matrix_create(int64_t m, int64_t n, const char* const* app_ids, const int32_t* cpu, const int32_t* gpu,
                      const int64_t* row_ptr, const int32_t* col, const double* val, ocg_matrix** out);
int ocg_matrix_shape(const ocg_matrix* mat, int64_t* m, int64_t* n, int64_t* nnz);
int ocg_matrix_get(const ocg_matrix* mat, int32_t* cpu, int32_t* gpu, int64_t* row_ptr, int32_t* col, double* val);
const char* ocg_matrix_app_id(const ocg_matrix* mat, int64_t i);
int ocg_matrix_save_bin(const ocg_matrix* mat, const char* path);
int ocg_matrix_load_bin(const char* path, ocg_matrix** out);
void ocg_matrix_destroy(ocg_matrix* mat);


/* ---- synthetic inputs (benches/tests; host only, no GPU needed) --------
 * Restatements of the reference's input generators so benches never need
 * the reference: sim::make_suite (simnode.cpp:192-244), sim::true_perf
 * (simnode.cpp:43-45), pred::profile_suite's matrix (predictor.cpp:45-69), and
 * the SURVEY §8d joint CSR matrices.  role: 0 training, 1 evaluation. */
typedef struct {
    int32_t archetype; /* 0 gpu_sensitive, 1 cpu_sensitive, 2 both_sensitive, 3 insensitive */
    double kappa_c, alpha_c, kappa_g, alpha_g, base_runtime_s, cpu_phase_s, noise_sigma;
    double ips_max, mem_tput_max, sm_clock_max;
} ocg_workload_spec;

int ocg_synth_suite(const int32_t counts[4], uint64_t seed, int role, double noise_sigma,
                    double cpu_phase_fraction, const int32_t* cpu_caps, int32_t ncpu,
                    const int32_t* gpu_caps, int32_t ngpu, ocg_workload_spec* out);
double ocg_true_perf(const ocg_workload_spec* spec, int32_t cpu_cap, int32_t gpu_cap);
/* offline dense block of the CLI's offline phase for root seed `seed` (10 x n) */
int ocg_synth_offline_block(uint64_t seed, const int32_t* cpu_caps, int32_t ncpu, const int32_t* gpu_caps,
                            int32_t ngpu, double* out, int64_t* rows);
/* napps eval-suite apps probed on the default plan + their cf::complete seeds */
int ocg_synth_online_apps(int64_t napps, uint64_t seed, const int32_t* cpu_caps, int32_t ncpu,
                          const int32_t* gpu_caps, int32_t ngpu, double* probe_vals, uint8_t* probe_mask,
                          uint64_t* seeds);
/* sim::sample_counters (simnode.cpp:98-110; cpu_phase != 0: sample_counters_cpu_phase
 * :112-123) of every spec at every grid setting (lexicographic order):
 * nspecs x ncpu*ngpu x 7 doubles in CounterSample field order */
int ocg_synth_counters(const ocg_workload_spec* specs, int64_t nspecs, const int32_t* cpu_caps, int32_t ncpu,
                       const int32_t* gpu_caps, int32_t ngpu, int cpu_phase, int nthreads, double* out);
/* joint m x n matrix (first dense_rows rows dense) as CSR: count, then fill */
int ocg_synth_csr_count(int64_t m, const int32_t* cpu_caps, int32_t ncpu, const int32_t* gpu_caps, int32_t ngpu,
                        double density, int64_t dense_rows, uint64_t seed, int nthreads, int64_t* row_ptr);
int ocg_synth_csr_fill(int64_t m, const int32_t* cpu_caps, int32_t ncpu, const int32_t* gpu_caps, int32_t ngpu,
                       double density, int64_t dense_rows, uint64_t seed, int nthreads, const int64_t* row_ptr,
                       int32_t* col, float* val32, double* val64);

/* rows [row0, row1) of the same matrix (a rank's shard), local row_ptr */
int ocg_synth_csr_range_count(int64_t m, int64_t row0, int64_t row1, const int32_t* cpu_caps, int32_t ncpu,
                              const int32_t* gpu_caps, int32_t ngpu, double density, int64_t dense_rows,
                              uint64_t seed, int nthreads, int64_t* row_ptr);
int ocg_synth_csr_range_fill(int64_t m, int64_t row0, int64_t row1, const int32_t* cpu_caps, int32_t ncpu,
                             const int32_t* gpu_caps, int32_t ngpu, double density, int64_t dense_rows, uint64_t seed,
                             int nthreads, const int64_t* row_ptr, int32_t* col, float* val32, double* val64);
/* sim::true_perf (simnode.cpp:43-45) of every cell of selected rows of the same joint
 * matrix (nrows x n): the ground truth a completion's held-out quality is measured on */
int ocg_synth_true_rows(int64_t m, const int32_t* cpu_caps, int32_t ncpu, const int32_t* gpu_caps, int32_t ngpu,
                        uint64_t seed, const int64_t* rows, int64_t nrows, double* out);
/* selected rows of the same joint matrix as dense values + mask (values as
 * the FP32 CSR carries them, widened) — CPU-baseline samples */
int ocg_synth_rows_dense(int64_t m, const int32_t* cpu_caps, int32_t ncpu, const int32_t* gpu_caps, int32_t ngpu,
                         double density, int64_t dense_rows, uint64_t seed, const int64_t* rows, int64_t nrows,
                         double* values, uint8_t* mask);

/* ---- probe ingest ----------------------------------
 * pred::predict_perf (predictor.cpp:151-157) for `count` counter samples
 * (count x 7 doubles in CounterSample field order, core.hpp:62-70):
 * validate_counters, standardize with (mean7, std7), MLP forward
 * (dims[0..n_layers], acts: 0 selu / 1 relu / 2 identity; params = per layer
 * W (out x in, row-major) then b — the reference's model-file order,
 * nnkit.cpp:306-330), clamp to [0.01, 1.25].  FP64, lane-exact.
 * has_stats = 0 -> OCG_E_MISSING (missing_artifact_error, :152-153). */
int ocg_predict_perf_batch(ocg_ctx* ctx, int32_t n_layers, const int64_t* dims, const int32_t* acts,
                           const double* params, const double* mean7, const double* std7, int has_stats,
                           const double* counters, int64_t count, int lane, double* out);

/* A loaded predictor (pred::PredictorModel, predictor.hpp:60-68) resident on
 * the context's device: create validates + uploads once, run streams counter
 * batches through it.  run flags: OCG_PRED_DEVICE_PTRS -> counters/out are
 * device pointers on the context's device (no host copies); OCG_PRED_GENERIC
 * -> use the any-architecture kernel even for the reference architecture
 * (7-64-64-1 SELU, which otherwise runs the thread-per-sample kernel).
 * run is synchronous (it reports invalid counters, like validate_counters). */
typedef struct ocg_predictor ocg_predictor;
enum { OCG_PRED_DEVICE_PTRS = 1, OCG_PRED_GENERIC = 2 };
int ocg_predictor_create(ocg_ctx* ctx, int32_t n_layers, const int64_t* dims, const int32_t* acts,
                         const double* params, const double* mean7, const double* std7, int has_stats,
                         ocg_predictor** out);
int ocg_predictor_run(ocg_predictor* pred, const double* counters, int64_t count, int lane, double* out,
                      uint32_t flags);
int ocg_predictor_destroy(ocg_predictor* pred);

/* Predictor model file <- pred::load_predictor / predictor_from_json
 * (predictor.cpp:301-331) over nn::model_from_json (nnkit.cpp:332-365), with
 * the same checks: OCG_E_MISSING absent file; OCG_E_LOGIC bad json, format_version,
 * inconsistent architecture, weight / bias / feature_stats shapes, non-finite
 * weight; OCG_E_INVALID unknown activation.
 * parse: two-phase (NULL arrays query n_layers / nparams); acts 0 selu, 1 relu,
 * 2 identity; params per layer W (out x in, row-major) then b.
 * load / from_json: parse, then ocg_predictor_create on the context's device. */
int ocg_predictor_parse(const char* text, int32_t* n_layers, int64_t* dims, int32_t* acts, double* params,
                        int64_t* nparams, double* mean7, double* std7, int* has_stats);
int ocg_predictor_from_json(ocg_ctx* ctx, const char* text, ocg_predictor** out);
int ocg_predictor_load(ocg_ctx* ctx, const char* path, ocg_predictor** out);

/* run_open_online (policy.cpp:114-191) for napps apps from their counter samples:
 * probe ingest wired into the per-app completion on the device.  For app a the
 * estimates are pred::predict_perf (predictor.cpp:151-157) of its nplan counter
 * samples (napps x nplan x 7, CounterSample field order) at the plan's columns
 * plan_cols[nplan] (ProbePlan order) — the re-probe rule (policy.cpp:168-176): when
 * transition != NULL and transition[a] != 0 the pre-transition samples are dropped
 * and reprobe_counters (same shape) are used instead — then cf::complete of the
 * dense block + that row and policy::select_caps, as ocg_online_complete_batch.
 * estimates (napps x nplan, may be NULL) returns the probe estimates; per-app
 * status OCG_E_INVALID for an invalid counter sample (validate_counters). */
int ocg_online_ingest_complete_batch(ocg_ctx* ctx, int64_t d_rows, const double* block_vals,
                                     const uint8_t* block_mask, int64_t napps, const int32_t* plan_cols,
                                     int32_t nplan, ocg_predictor* predictor, const double* counters,
                                     const double* reprobe_counters, const int32_t* transition,
                                     const uint64_t* seeds, const int32_t* cpu_caps, int32_t ncpu,
                                     const int32_t* gpu_caps, int32_t ngpu, const ocg_ncf_hyper* hyper,
                                     double gamma, int lane, double* estimates, double* completed, int32_t* idx,
                                     double* saving, double* loss, int32_t* ncand, ocg_ncf_meta* meta,
                                     int32_t* status);

/* Evaluation harness: policy::evaluate_suite (policy.cpp:373-405) over napps apps on
 * the device, from the simulator's repetition runs (sim::run is the simulator and stays
 * with the caller).  base_runs[a][r] is sim::run(app a, baseline, rep seed r) and
 * runs[a][j][r] the same at grid setting j (PowerGrid::settings order, cpu-major), rep
 * seed r = derive_seed(derive_seed(seed, "eval." + app_id), "rep", r) as measure_truth
 * (policy.cpp:213-256) draws them.  policies[npol] are ocg_policy_kind values; for the
 * open policy open_idx[a] / open_pred_saving[a] are its run_open_online decision
 * (setting index, pred_saving) and may be NULL otherwise.  rows is napps x npol in the
 * reference's report order; aggs (npol, may be NULL) as its PolicyAggregate (by policy
 * kind).  FP64 in the reference's operation order: bit-exact. */
enum { OCG_POLICY_OPEN = 0, OCG_POLICY_NO_CAP = 1, OCG_POLICY_GPU_CAP_ONLY = 2, OCG_POLICY_CPU_CAP_ONLY = 3,
       OCG_POLICY_ORACLE = 4 };
typedef struct {
    double runtime_s, energy_j, avg_power_w; /* sim::RunResult (simnode.hpp:55-61) scalars */
} ocg_run_result;
typedef struct {
    int32_t policy, setting; /* ocg_policy_kind, setting index */
    int32_t cpu_cap_w, gpu_cap_w;
    double gamma, true_perf, true_loss, energy_j, avg_power_w, efficiency, pred_saving; /* EvalRow */
} ocg_eval_row;
typedef struct {
    int32_t policy;
    double mean_efficiency, mean_gain_vs_no_cap, mean_true_loss, mean_true_perf; /* PolicyAggregate */
} ocg_eval_aggregate;
int ocg_eval_suite(ocg_ctx* ctx, int64_t napps, const int32_t* cpu_caps, int32_t ncpu, const int32_t* gpu_caps,
                   int32_t ngpu, int32_t repetitions, const ocg_run_result* base_runs, const ocg_run_result* runs,
                   double gamma, int32_t npolicies, const int32_t* policies, const int32_t* open_idx,
                   const double* open_pred_saving, ocg_eval_row* rows, ocg_eval_aggregate* aggs);

/* debug / parity probes of device building blocks */
int ocg_debug_exp(ocg_ctx* ctx, const double* x, int64_t n, double* out); /* device glibc-exact exp */
double ocg_debug_exp_host(double x);                                       /* same code, host build */
int ocg_debug_rng(ocg_ctx* ctx, uint64_t seed, int64_t n, uint64_t* out);  /* device mt19937_64 */

#ifdef __cplusplus
}
#endif
#endif /* OCG_H */
