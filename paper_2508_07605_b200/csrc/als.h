#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace ocg {

constexpr int kSeg = 1024;  // observations per ALS work segment

// One half-sweep: solve X (items x K) from Y given the item-major sparse matrix
struct AlsHalf {
    int64_t nitems;
    int32_t max_segs;           // host upper bound (grid sizing)
    const int32_t* total_segs;  // device scalar: actual segment count
    const int64_t* ptr;
    const int32_t* idx;
    const float* val;
    const int32_t* seg_item;
    const int64_t* seg_beg;
    const int32_t* nseg;   // per item
    const int32_t* first;   // per item: first segment
    const int32_t* pfirst;  // per item: first partial-Gram slot (items with >1 segment)
    const float* Y;
    float* X;
    float* partial;   // partial-Gram slots x (K*K + K + 1)
    float* gram_out;  // mode 1: nitems x (K*K + K + 1)
    float lambda;
    // rank-32 tensor-core path (als_mma.cu): Y packed as fp16 hi/lo rows
    const uint4* Yh = nullptr;
    const unsigned* ymax = nullptr;  // max |Y| (float bits) the packing scale came from
    const unsigned* vmax = nullptr;  // max |val|
    const uint32_t* valh = nullptr;  // observed values packed (fp16 hi, fp16 lo) of val * 2^ev
    // optional: multi-segment items (MODE 0 reduce visits only these) and a
    // processing order of the segments (column side: sorted by first row)
    const int32_t* multi_list = nullptr;
    const int32_t* multi_count = nullptr;
    const int32_t* seg_order = nullptr;
    int32_t* blk_ctr = nullptr;  // rank 32: work-block counter (zeroed per launch)
    cudaEvent_t ev_gram0 = nullptr, ev_gram1 = nullptr;  // optional: recorded around the Gram kernel
    unsigned* xmax = nullptr;  // mode 0: the K4 leaves max |X| here (zeroed first)
};

cudaError_t launch_als_init(int64_t n, int k, uint64_t seed, float* V, cudaStream_t s);
cudaError_t launch_seg_count(int64_t nitems, const int64_t* ptr, int32_t* nseg, int32_t* nmulti, int force_partials,
                             int32_t* multi_list, int32_t* multi_count, cudaStream_t s);
cudaError_t launch_seg_key(int32_t max_segs, const int32_t* total, const int64_t* seg_beg, const int32_t* idx,
                           int32_t* key, int32_t* id, cudaStream_t s);
cudaError_t launch_seg_fill(int64_t nitems, const int64_t* ptr, const int32_t* nseg, const int32_t* first,
                            int32_t* seg_item, int64_t* seg_beg, int32_t* total, cudaStream_t s);
size_t als_gram_record_floats(int k);
// mode 0: solve in place; mode 1: write reduced Gram records to gram_out
cudaError_t launch_als_half(int k, const AlsHalf& h, int mode, int sm_count, cudaStream_t s);
// rank-32/64 tensor-core half-sweep (Gram records -> reduce -> batched solve) + the packing
cudaError_t launch_als_mma_half(int k, const AlsHalf& h, int mode, int sm_count, cudaStream_t s);
cudaError_t launch_als_solve_records(int k, int64_t nitems, const float* G, float* X, float lambda, int sm_count,
                                     cudaStream_t s);
size_t als_record_floats_mma(int k);
cudaError_t launch_als_pack(int k, int64_t rows, const float* X, unsigned* maxbits, uint4* Xh, int sm_count,
                            cudaStream_t s, bool have_max = false);
cudaError_t launch_als_pack_vals(int64_t n, const float* val, const unsigned* vmax, uint32_t* out, cudaStream_t s);
cudaError_t launch_absmax(int64_t count, const float* x, unsigned* maxbits, int sm_count, cudaStream_t s);
cudaError_t launch_als_solve_from_gram(int k, int64_t nitems, const float* G, float* X, float lambda, int sm_count,
                                       cudaStream_t s);
cudaError_t launch_expand_pairs(int64_t m, const int64_t* ptr, const uint32_t* vbits, uint64_t* pairs, int sm_count,
                                cudaStream_t s);
cudaError_t launch_split_pairs(int64_t nnz, const uint64_t* pairs, int32_t* crow, uint32_t* cval, cudaStream_t s);
cudaError_t launch_col_ptr(int64_t nnz, int64_t n, const int32_t* skeys, int64_t* cptr, cudaStream_t s);
// packed-key CSC (key = col << rb | row, 32 bits): keys from the CSR, then crow + col_ptr
cudaError_t launch_expand_keys(int64_t m, int rb, const int64_t* ptr, const int32_t* col, uint32_t* keys,
                               int sm_count, cudaStream_t s);
cudaError_t launch_split_keys(int64_t nnz, int64_t n, int rb, const uint32_t* skeys, int32_t* crow, int64_t* cptr,
                              cudaStream_t s);

// fused completion + Algorithm-2 selection over all rows (als_select.cu)
struct AlsSelectArgs {
    int64_t m, n;
    int k;
    const float* U;
    const float* V;   // n x K
    const float* Vt;  // K x n (transposed copy)
    const int64_t* row_ptr;
    const int32_t* col;
    const float* val;
    const int32_t* cpu_caps;
    const int32_t* gpu_caps;
    int ngpu;
    double e_base, gamma;
    int32_t* idx;
    double* saving;
    double* loss;
    int32_t* ncand;
    double* completed;  // optional m x n completed rows (tests), else nullptr
};
cudaError_t launch_als_select(const AlsSelectArgs& a, int sm_count, cudaStream_t s);
// rank 32 on the tensor cores (als_select_mma.cu); Vsel: n x 8 uint4 scratch
cudaError_t launch_als_select_mma(const AlsSelectArgs& a, uint4* Vsel, const unsigned* umax, const unsigned* vmax,
                                  int sm_count, cudaStream_t s);
cudaError_t launch_transpose(int64_t n, int k, const float* V, float* Vt, cudaStream_t s);

}  // namespace ocg
