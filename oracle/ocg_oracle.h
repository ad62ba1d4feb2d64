/* TEST INFRASTRUCTURE ONLY — the CPU oracle (plain-C restatement of the
 * reference's online CF completion + selection path).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it, and
 * only as the checker.  The product (paper_2508_07605_b200/) never links it.
 *
 * Parity pinning: every function is checked against the reference library
 * itself (oracle/_ref, built from /root/reference by oracle/Makefile) and
 * against golden vectors in tests/golden/ (tests/test_oracle.py).  The ALS
 * solver has NO reference counterpart: its parity is "unpinned". */
#ifndef OCG_ORACLE_H
#define OCG_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* mirrors cf::NcfHyper (cfcomplete.hpp:11-20); same layout as ocg_ncf_hyper */
typedef struct {
    int64_t app_dim, setting_dim;
    int64_t hidden[8];
    int64_t n_hidden;
    double lr;
    int32_t max_epochs, patience;
    double val_fraction;
    int32_t batch_size;
} ocgo_hyper;

/* mirrors NcfModel::Meta (cfcomplete.hpp:34-40) */
typedef struct {
    uint64_t seed;
    int32_t epochs_run;
    double initial_train_mse, final_train_mse, best_val_mse;
} ocgo_meta;

const char* ocgo_last_error(void);

uint64_t ocgo_derive_seed(uint64_t root, const char* tag, uint64_t n);
void ocgo_rng_u64(uint64_t seed, uint64_t* out, size_t n);
void ocgo_rng_uniform(uint64_t seed, double lo, double hi, double* out, size_t n);

int ocgo_select_caps(const double* rows, int64_t nrows, const int32_t* cpu, int32_t ncpu,
                     const int32_t* gpu, int32_t ngpu, double gamma, int32_t* idx, double* saving,
                     double* loss, int32_t* ncand);
int ocgo_default_plan(const int32_t* cpu, int32_t ncpu, const int32_t* gpu, int32_t ngpu,
                      int32_t* out_cols, int32_t* count);

/* reference kernel lane to follow: 0 scalar (default), 1 AVX2/FMA */
void ocgo_set_lane(int lane);
int64_t ocgo_ncf_param_count(int64_t m, int64_t n, const ocgo_hyper* h);
int ocgo_ncf_fit(int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col,
                 const double* val, const ocgo_hyper* h, uint64_t seed, double* params,
                 ocgo_meta* meta, uint8_t* app_seen, uint8_t* setting_seen);
int ocgo_ncf_predict(int64_t m, int64_t n, const ocgo_hyper* h, const double* params,
                     const uint8_t* app_seen, const uint8_t* setting_seen, const int64_t* rows,
                     const int64_t* cols, int64_t count, double* out);

/* ALS (no reference counterpart; semantics defined in ocg_oracle.c) */
double ocgo_als_init_value(uint64_t seed, int64_t j, int32_t f, int32_t k);
int ocgo_als_fit(int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col, const float* val,
                 const int64_t* col_ptr, const int32_t* row_idx, const float* cval, int32_t k, double lambda,
                 int32_t sweeps, uint64_t seed, double* U, double* V);

void ocgo_als_solve_rows(int64_t nrows, const int64_t* ptr, const int32_t* idx, const float* val, const double* Y,
                         double* X, int32_t k, double lambda);
void ocgo_als_col_gram(int64_t ncols, const int64_t* col_ptr, const int32_t* row_idx, const float* cval,
                       const double* U, int32_t k, double* G);
void ocgo_als_solve_from_gram(int64_t ncols, const double* G, double* X, int32_t k, double lambda);

#ifdef __cplusplus
}
#endif
#endif
