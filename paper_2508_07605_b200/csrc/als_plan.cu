// Host orchestration of the ALS completion + selection path (C-ABI in
// include/ocg.h).  One step = build the CSC mirror of the CSR input on the
// device (stable radix sort by column -> rows stay ascending inside a column,
// so the column Gram reduction order is fixed), V init, `sweeps` x (row
// half-sweep, column half-sweep), then the fused imputation + selection pass.
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/ocg.h"
#include "als.h"
#include "ocg_common.cuh"

// from capi.cu
int ocg_internal_fail(int code, const std::string& msg);
cudaStream_t ocg_internal_stream(ocg_ctx* ctx);
int ocg_internal_sm_count(ocg_ctx* ctx);

namespace {

#define ALS_CUDA(call)                                                                                    \
    do {                                                                                                  \
        cudaError_t e_ = (call);                                                                          \
        if (e_ != cudaSuccess) return ocg_internal_fail(OCG_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

template <typename T>
struct Buf {
    T* p = nullptr;
    bool own = true;
    ~Buf() {
        if (p && own) cudaFree(p);
    }
    // (re)allocation: an owned previous buffer is released first
    cudaError_t alloc(size_t n) {
        if (p && own) cudaFree(p);
        p = nullptr;
        own = true;
        return n ? cudaMalloc(&p, sizeof(T) * n) : cudaSuccess;
    }
};


// ranks on the tensor-core path (als_mma.cu / als_select_mma.cu)
bool mma_rank(int k) { return k == 32 || k == 64; }

// OCG_CSC_PAIRS=1: the 64-bit-payload radix sort even when packed 32-bit keys fit (A/B runs)
bool csc_pairs_forced() {
    const char* e = std::getenv("OCG_CSC_PAIRS");  // read per build (cheap; tests toggle it)
    return e && e[0] == '1';
}

int bits_for(int64_t n) {
    int b = 1;
    while ((int64_t(1) << b) < n + 1) ++b;
    return b;
}

}  // namespace

struct ocg_als_plan {
    ocg_ctx* ctx = nullptr;
    // input validation (run on the device before every fit on a new CSR): error bits
    // (1 << OCG_E_*) and a column-seen bitmap; dirty = the CSR changed since the last check
    Buf<int> err;
    Buf<unsigned> seen;
    bool dirty = true;
    int64_t m = 0, n = 0, nnz = 0;
    int k = 32, sweeps = 10;
    int warm_sweeps = 0;  // > 0: runs keep the previous factors (no V init) and do this many sweeps
    bool fitted = false;  // a run has completed (factors exist)
    float lambda = 0.05f;
    uint64_t seed = 0;
    double gamma = 0.05, e_base = 0.0;
    int ngpu = 1;
    // CSR (owned copies unless created from device pointers)
    Buf<int64_t> row_ptr;
    Buf<int32_t> col;
    Buf<float> val;
    // CSC mirror + scratch
    Buf<int64_t> col_ptr;
    Buf<int32_t> crow, keys_out;
    Buf<uint64_t> pairs_in, pairs_out;  // (row << 32 | value bits) sorted by column
    Buf<float> cval;
    Buf<uint8_t> sort_tmp;
    size_t sort_tmp_bytes = 0;
    // segment tables (index 0: rows over CSR, 1: columns over CSC)
    struct Side {
        Buf<int32_t> nseg, first, nmulti, pfirst, seg_item, total;  // total: [0] segments, [1] multi items, [2] block counter
        Buf<int32_t> multi_list;
        Buf<int32_t> seg_order, seg_key, seg_key_out, seg_id;  // column side: processing order
        Buf<uint8_t> order_tmp;
        size_t order_tmp_bytes = 0;
        Buf<int64_t> seg_beg;
        Buf<float> partial;
        int32_t max_segs = 0;
    } side[2];
    Buf<uint8_t> scan_tmp;
    size_t scan_tmp_bytes = 0;
    // factors + outputs
    Buf<float> U, V, Vt;
    // rank 32: factors packed as fp16 hi/lo rows for the tensor-core Gram + the
    // max |.| each packing scale came from ([0] U, [1] V, [2] observed values)
    Buf<uint4> Uh, Vh;
    Buf<unsigned> maxbits;
    Buf<uint32_t> valh;
    Buf<uint4> Vsel;  // V in the tensor-core selection layout
    // capacities: nnz_cap sizes every nnz-dependent buffer (als_alloc), col_cap the CSR arrays;
    // both grow with headroom, so streaming arrivals rarely reallocate.  col_alt/val_alt/rp_alt:
    // the merge target of ocg_als_plan_add_observations (swapped with col/val/row_ptr)
    // val_cap / val_next_cap: each value buffer's own size (val swaps with val_alt in
    // add_observations and with val_next at a staged run, so it cannot share col_cap)
    int64_t nnz_cap = 0, col_cap = 0, alt_cap = 0, val_cap = 0, val_next_cap = 0;
    Buf<int32_t> col_alt;
    Buf<float> val_alt;
    Buf<int64_t> rp_alt;
    // add_observations scratch (kept: no allocation per arrival batch)
    Buf<int32_t> add_rc, add_inc, add_ex, add_err;
    Buf<float> add_v;
    Buf<uint8_t> add_tmp;
    int64_t add_cap = 0;
    size_t add_tmp_bytes = 0;
    Buf<uint16_t> col16;  // staging of ocg_als_plan_upload_compact / _stage_compact
    // ocg_als_plan_stage_compact: the next step's CSR copied on a side stream into
    // rp_next / col16 / val_next while the current step runs; the next _run swaps it in
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_staged = nullptr, ev_free = nullptr, ev_results = nullptr;
    bool staged = false, free_recorded = false;
    int64_t staged_nnz = 0;
    Buf<int64_t> rp_next;
    Buf<float> val_next;
    int64_t col16_cap = 0;  // CSR values packed for the tensor-core Gram (the CSC copy is gathered into cval)
    Buf<int32_t> cpu, gpu, idx, ncand;
    Buf<double> saving, loss;
    cudaEvent_t ev[10] = {};
    ~ocg_als_plan() {
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        if (copy_stream) cudaStreamSynchronize(copy_stream);
        if (ev_staged) cudaEventDestroy(ev_staged);
        if (ev_free) cudaEventDestroy(ev_free);
        if (ev_results) cudaEventDestroy(ev_results);
        if (copy_stream) cudaStreamDestroy(copy_stream);
    }
};

static int als_build_csc(ocg_als_plan* P) {
    cudaStream_t s = ocg_internal_stream(P->ctx);
    const int sm = ocg_internal_sm_count(P->ctx);
    const int rb = bits_for(P->m - 1), cb = bits_for(P->n - 1);
    const bool key32 = rb + cb <= 32 && !csc_pairs_forced();
    if (key32) {
        // one 32-bit key (col << rb | row) per observation, sorted on its column bits only
        // (stable: rows stay ascending inside a column); the value word is the payload and
        // lands in cval directly
        const uint32_t* vb = mma_rank(P->k) ? P->valh.p : reinterpret_cast<const uint32_t*>(P->val.p);
        uint32_t* kin = reinterpret_cast<uint32_t*>(P->pairs_in.p);
        uint32_t* kout = reinterpret_cast<uint32_t*>(P->pairs_out.p);
        if (P->nnz > 0) {
            ALS_CUDA(ocg::launch_expand_keys(P->m, rb, P->row_ptr.p, P->col.p, kin, sm, s));
            size_t bytes = P->sort_tmp_bytes;
            ALS_CUDA(cub::DeviceRadixSort::SortPairs(P->sort_tmp.p, bytes, kin, kout, vb,
                                                     reinterpret_cast<uint32_t*>(P->cval.p), P->nnz, rb, rb + cb, s));
        }
        ALS_CUDA(ocg::launch_split_keys(P->nnz, P->n, rb, kout, P->crow.p, P->col_ptr.p, s));
    } else if (P->nnz > 0) {
        // (row, value) travel with the column key through the radix sort (stable:
        // rows stay ascending inside a column), so no random gathers afterwards.
        // Rank 32: the value word is the packed (fp16 hi, lo) form.
        const uint32_t* vb = mma_rank(P->k) ? P->valh.p : reinterpret_cast<const uint32_t*>(P->val.p);
        ALS_CUDA(ocg::launch_expand_pairs(P->m, P->row_ptr.p, vb, P->pairs_in.p, sm, s));
        size_t bytes = P->sort_tmp_bytes;
        ALS_CUDA(cub::DeviceRadixSort::SortPairs(P->sort_tmp.p, bytes, P->col.p, P->keys_out.p, P->pairs_in.p,
                                                 P->pairs_out.p, P->nnz, 0, bits_for(P->n), s));
        ALS_CUDA(ocg::launch_split_pairs(P->nnz, P->pairs_out.p, P->crow.p, reinterpret_cast<uint32_t*>(P->cval.p), s));
    }
    if (!key32) ALS_CUDA(ocg::launch_col_ptr(P->nnz, P->n, P->keys_out.p, P->col_ptr.p, s));
    for (int sd = 0; sd < 2; ++sd) {
        auto& S = P->side[sd];
        const int64_t items = sd == 0 ? P->m : P->n;
        const int64_t* ptr = sd == 0 ? P->row_ptr.p : P->col_ptr.p;
        ALS_CUDA(ocg::launch_seg_count(items, ptr, S.nseg.p, S.nmulti.p, 0, S.multi_list.p, S.total.p + 1, s));
        size_t b = P->scan_tmp_bytes;
        ALS_CUDA(cub::DeviceScan::ExclusiveSum(P->scan_tmp.p, b, S.nseg.p, S.first.p, items, s));
        b = P->scan_tmp_bytes;
        ALS_CUDA(cub::DeviceScan::ExclusiveSum(P->scan_tmp.p, b, S.nmulti.p, S.pfirst.p, items, s));
        ALS_CUDA(ocg::launch_seg_fill(items, ptr, S.nseg.p, S.first.p, S.seg_item.p, S.seg_beg.p, S.total.p, s));
        if (S.seg_order.p) {
            ALS_CUDA(ocg::launch_seg_key(S.max_segs, S.total.p, S.seg_beg.p, P->crow.p, S.seg_key.p, S.seg_id.p, s));
            size_t ob = S.order_tmp_bytes;
            ALS_CUDA(cub::DeviceRadixSort::SortPairs(S.order_tmp.p, ob, S.seg_key.p, S.seg_key_out.p, S.seg_id.p,
                                                     S.seg_order.p, S.max_segs, 0, 31, s));
        }
    }
    return OCG_OK;
}

static ocg::AlsHalf als_half(ocg_als_plan* P, int sd) {
    auto& S = P->side[sd];
    ocg::AlsHalf h{};
    h.nitems = sd == 0 ? P->m : P->n;
    h.max_segs = S.max_segs;
    h.total_segs = S.total.p;
    h.ptr = sd == 0 ? P->row_ptr.p : P->col_ptr.p;
    h.idx = sd == 0 ? P->col.p : P->crow.p;
    h.val = sd == 0 ? P->val.p : P->cval.p;
    h.seg_item = S.seg_item.p;
    h.seg_beg = S.seg_beg.p;
    h.nseg = S.nseg.p;
    h.first = S.first.p;
    h.pfirst = S.pfirst.p;
    h.multi_list = S.multi_list.p;
    h.multi_count = S.total.p + 1;
    h.seg_order = S.seg_order.p;
    h.blk_ctr = S.total.p + 2;
    // K4 fused into the row-side Gram kernel (solve batches of single-segment rows
    // in shared memory): measured 5.1 ms/launch vs 2.0 + 1.7 ms split (7 warps/SM
    // for Gram + batches starve both); kept as an ablation switch, off
    h.Y = sd == 0 ? P->V.p : P->U.p;
    h.X = sd == 0 ? P->U.p : P->V.p;
    h.partial = S.partial.p;
    h.gram_out = nullptr;
    h.lambda = P->lambda;
    if (mma_rank(P->k)) {
        h.valh = sd == 0 ? P->valh.p : reinterpret_cast<const uint32_t*>(P->cval.p);
        h.Yh = sd == 0 ? P->Vh.p : P->Uh.p;
        h.ymax = P->maxbits.p + (sd == 0 ? 1 : 0);
        h.vmax = P->maxbits.p + 2;
    }
    return h;
}

// after a half-sweep (or V init): repack the factor the next half gathers
static int als_pack(ocg_als_plan* P, int sd, bool have_max = false) {
    if (!mma_rank(P->k)) return OCG_OK;
    const int64_t rows = sd == 0 ? P->m : P->n;
    ALS_CUDA(ocg::launch_als_pack(P->k, rows, sd == 0 ? P->U.p : P->V.p, P->maxbits.p + (sd == 0 ? 0 : 1),
                                  sd == 0 ? P->Uh.p : P->Vh.p, ocg_internal_sm_count(P->ctx),
                                  ocg_internal_stream(P->ctx), have_max));
    return OCG_OK;
}

// buffers whose size depends on nnz (reallocated when an upload changes it)
static int als_alloc(ocg_als_plan* P) {
    P->nnz_cap = std::max(P->nnz, P->nnz_cap);
    const int64_t cap = P->nnz_cap;
    ALS_CUDA(P->col_ptr.alloc(static_cast<size_t>(P->n + 1)));
    ALS_CUDA(P->crow.alloc(static_cast<size_t>(cap)));
    ALS_CUDA(P->cval.alloc(static_cast<size_t>(cap)));
    ALS_CUDA(P->keys_out.alloc(static_cast<size_t>(cap)));
    ALS_CUDA(P->pairs_in.alloc(static_cast<size_t>(cap)));
    ALS_CUDA(P->pairs_out.alloc(static_cast<size_t>(cap)));
    size_t bytes = 0, b32 = 0;
    ALS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, P->col.p, P->keys_out.p, P->pairs_in.p, P->pairs_out.p,
                                             cap, 0, bits_for(P->n)));
    ALS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b32, reinterpret_cast<uint32_t*>(P->pairs_in.p),
                                             reinterpret_cast<uint32_t*>(P->pairs_out.p),
                                             static_cast<const uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                             cap, 0, 32));
    bytes = std::max(bytes, b32);
    P->sort_tmp_bytes = bytes;
    ALS_CUDA(P->sort_tmp.alloc(bytes));
    for (int sd = 0; sd < 2; ++sd) {
        auto& S = P->side[sd];
        const int64_t items = sd == 0 ? P->m : P->n;
        const int64_t ms = items + cap / ocg::kSeg + 1;
        if (ms >= (int64_t(1) << 31)) return ocg_internal_fail(OCG_E_UNSUPPORTED, "als: too many segments");
        S.max_segs = static_cast<int32_t>(ms);
        ALS_CUDA(S.nseg.alloc(static_cast<size_t>(items)));
        ALS_CUDA(S.first.alloc(static_cast<size_t>(items)));
        ALS_CUDA(S.total.alloc(3));
        ALS_CUDA(S.multi_list.alloc(static_cast<size_t>(items)));
        if (sd == 1 && mma_rank(P->k)) {
            ALS_CUDA(S.seg_order.alloc(static_cast<size_t>(ms)));
            ALS_CUDA(S.seg_key.alloc(static_cast<size_t>(ms)));
            ALS_CUDA(S.seg_key_out.alloc(static_cast<size_t>(ms)));
            ALS_CUDA(S.seg_id.alloc(static_cast<size_t>(ms)));
            size_t ob = 0;
            ALS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, ob, S.seg_key.p, S.seg_key_out.p, S.seg_id.p,
                                                     S.seg_order.p, static_cast<int>(ms), 0, 31));
            S.order_tmp_bytes = ob;
            ALS_CUDA(S.order_tmp.alloc(ob));
        }
        ALS_CUDA(S.seg_item.alloc(static_cast<size_t>(ms)));
        ALS_CUDA(S.seg_beg.alloc(static_cast<size_t>(ms)));
        // partial Grams only for items with >1 segment: sum of their nseg <= 2*nnz/kSeg
        // (the column side may also run in MODE 1 — every segment keeps a slot)
        // (rank 32: every segment writes a record, slot = segment id)
        const int64_t mp = (sd == 1 || mma_rank(P->k)) ? ms : std::min<int64_t>(ms, 2 * (cap / ocg::kSeg) + 2);
        ALS_CUDA(S.nmulti.alloc(static_cast<size_t>(items)));
        ALS_CUDA(S.pfirst.alloc(static_cast<size_t>(items)));
        ALS_CUDA(S.partial.alloc(static_cast<size_t>(mp) * ocg::als_gram_record_floats(P->k)));
        size_t b = 0;
        ALS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b, S.nseg.p, S.first.p, items));
        P->scan_tmp_bytes = std::max(P->scan_tmp_bytes, b);
    }
    ALS_CUDA(P->scan_tmp.alloc(P->scan_tmp_bytes));
    if (mma_rank(P->k)) ALS_CUDA(P->valh.alloc(static_cast<size_t>(cap)));
    return OCG_OK;
}

// buffers that depend on m, n, k only (they survive an upload with a new nnz)
static int als_alloc_fixed(ocg_als_plan* P) {
    ALS_CUDA(P->U.alloc(static_cast<size_t>(P->m * P->k)));
    ALS_CUDA(P->V.alloc(static_cast<size_t>(P->n * P->k)));
    ALS_CUDA(P->Vt.alloc(static_cast<size_t>(P->n * P->k)));
    if (mma_rank(P->k)) {
        ALS_CUDA(P->Uh.alloc(static_cast<size_t>(P->m * (P->k / 4))));  // K/4 x 16 B per packed row
        ALS_CUDA(P->Vh.alloc(static_cast<size_t>(P->n * (P->k / 4))));
        ALS_CUDA(P->maxbits.alloc(3));
        ALS_CUDA(P->Vsel.alloc(static_cast<size_t>(P->n * (P->k / 4))));
    }
    ALS_CUDA(P->idx.alloc(static_cast<size_t>(P->m)));
    ALS_CUDA(P->ncand.alloc(static_cast<size_t>(P->m)));
    ALS_CUDA(P->saving.alloc(static_cast<size_t>(P->m)));
    ALS_CUDA(P->loss.alloc(static_cast<size_t>(P->m)));
    for (auto& e : P->ev)
        if (!e) ALS_CUDA(cudaEventCreate(&e));
    return OCG_OK;
}

// The checks the reference applies to the same matrix (PerformanceMatrix::set,
// core.cpp:142-148: out_of_range for a column index, invalid_argument for a value
// outside (0, 1.25]; cf::complete, cfcomplete.cpp:199-205: invalid_argument for a
// row without observations; NcfModel::predict :53-55: a cold setting column),
// plus sorted unique columns per row.  Bad entries are neutralised in place
// (column 0, value 1) so the fit that follows stays in bounds; the run's results
// then report the error instead of decisions.  One warp per row.
__global__ void als_validate_kernel(int64_t m, int64_t n, const int64_t* __restrict__ rp, int32_t* col, float* val,
                                    unsigned* seen, int* err) {
    extern __shared__ unsigned sseen[];
    const int nw = static_cast<int>((n + 31) / 32);
    for (int w = threadIdx.x; w < nw; w += blockDim.x) sseen[w] = 0u;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    int bits = 0;
    for (int64_t i = gw; i < m; i += nwarps) {
        const int64_t b = rp[i], e = rp[i + 1];
        if (e <= b) bits |= 1 << OCG_E_INVALID;
        int32_t carry = -1;  // last column of the previous chunk
        for (int64_t q0 = b; q0 < e; q0 += 32) {
            const int64_t q = q0 + lane;
            const bool on = q < e;
            const int32_t c = on ? col[q] : 0;
            const float v = on ? val[q] : 1.0f;
            int32_t prev = __shfl_up_sync(0xffffffffu, c, 1);
            if (lane == 0) prev = carry;
            carry = __shfl_sync(0xffffffffu, c, 31);
            if (on) {
                const bool in = c >= 0 && c < n;
                if (!in) {
                    bits |= 1 << OCG_E_RANGE;
                    col[q] = 0;
                } else {
                    atomicOr(sseen + (c >> 5), 1u << (c & 31));
                }
                if (q > b && prev >= c) bits |= 1 << OCG_E_INVALID;
                if (!(v > 0.0f && v <= 1.25f)) {  // NaN fails too
                    bits |= 1 << OCG_E_INVALID;
                    val[q] = 1.0f;
                }
            }
        }
    }
    bits = __reduce_or_sync(0xffffffffu, bits);
    if (lane == 0 && bits) atomicOr(err, bits);
    __syncthreads();
    for (int w = threadIdx.x; w < nw; w += blockDim.x)
        if (sseen[w]) atomicOr(seen + w, sseen[w]);
}

__global__ void als_cold_kernel(int64_t n, const unsigned* seen, int* err) {
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x)
        if (!((seen[j >> 5] >> (j & 31)) & 1u)) {
            atomicOr(err, 1 << OCG_E_COLD);
            return;
        }
}

static int als_validate(ocg_als_plan* P) {
    if (!P->dirty) return OCG_OK;
    cudaStream_t s = ocg_internal_stream(P->ctx);
    const int nw = static_cast<int>((P->n + 31) / 32);
    if (!P->err.p) {
        ALS_CUDA(P->err.alloc(1));
        ALS_CUDA(P->seen.alloc(static_cast<size_t>(nw)));
    }
    ALS_CUDA(cudaMemsetAsync(P->err.p, 0, sizeof(int), s));
    ALS_CUDA(cudaMemsetAsync(P->seen.p, 0, sizeof(unsigned) * nw, s));
    if (P->m > 0) {
        const int grid = static_cast<int>(std::min<int64_t>((P->m + 7) / 8, 4 * ocg_internal_sm_count(P->ctx)));
        als_validate_kernel<<<grid, 256, sizeof(unsigned) * nw, s>>>(P->m, P->n, P->row_ptr.p, P->col.p, P->val.p,
                                                                      P->seen.p, P->err.p);
        ALS_CUDA(cudaGetLastError());
        als_cold_kernel<<<1, 256, 0, s>>>(P->n, P->seen.p, P->err.p);
        ALS_CUDA(cudaGetLastError());
    }
    P->dirty = false;
    return OCG_OK;
}

// error of the last validated CSR (synchronises the stream), reported like the reference would throw
static int als_error(ocg_als_plan* P) {
    if (!P->err.p) return OCG_OK;
    int bits = 0;
    ALS_CUDA(cudaMemcpyAsync(&bits, P->err.p, sizeof(int), cudaMemcpyDeviceToHost, ocg_internal_stream(P->ctx)));
    ALS_CUDA(cudaStreamSynchronize(ocg_internal_stream(P->ctx)));
    if (bits & (1 << OCG_E_RANGE)) return ocg_internal_fail(OCG_E_RANGE, "matrix index out of range");
    if (bits & (1 << OCG_E_INVALID))
        return ocg_internal_fail(OCG_E_INVALID, "als: a row without observed entries, a value outside (0, 1.25] "
                                                "or unsorted / repeated columns");
    if (bits & (1 << OCG_E_COLD))
        return ocg_internal_fail(OCG_E_COLD, "als: cold setting column (no observed entries at fit time)");
    return OCG_OK;
}

// row_ptr invariants, host side (the device check covers columns and values)
static int check_row_ptr(const int64_t* rp, int64_t m) {
    if (rp[0] != 0) return ocg_internal_fail(OCG_E_INVALID, "csr: row_ptr[0] must be 0");
    for (int64_t i = 0; i < m; ++i)
        if (rp[i + 1] < rp[i]) return ocg_internal_fail(OCG_E_INVALID, "csr: row_ptr must be non-decreasing");
    return OCG_OK;
}

static int als_check(int64_t m, int64_t n, const int32_t* cpu, int32_t ncpu, const int32_t* gpu, int32_t ngpu,
                     const ocg_als_hyper* h, double gamma) {
    if (!h) return ocg_internal_fail(OCG_E_INVALID, "als: null hyperparameters");
    if (h->rank != 8 && h->rank != 16 && h->rank != 32 && h->rank != 64)
        return ocg_internal_fail(OCG_E_UNSUPPORTED, "als: rank must be 8, 16, 32 or 64");
    if (h->lambda <= 0.0f || h->sweeps <= 0) return ocg_internal_fail(OCG_E_INVALID, "als: bad hyperparameters");
    if (m <= 0 || n <= 0) return ocg_internal_fail(OCG_E_INVALID, "als: empty matrix");
    if (gamma <= 0.0 || gamma >= 1.0) return ocg_internal_fail(OCG_E_INVALID, "select_caps: gamma must lie in (0, 1)");
    if (static_cast<int64_t>(ncpu) * ngpu != n) return ocg_internal_fail(OCG_E_INVALID, "row length does not cover the grid");
    if (ncpu + ngpu > 512) return ocg_internal_fail(OCG_E_UNSUPPORTED, "grid too large");
    if (!cpu || !gpu) return ocg_internal_fail(OCG_E_INVALID, "cap list is empty");
    for (int32_t k = 0; k < ncpu; ++k)  // PowerGrid (core.cpp:38-45)
        if (cpu[k] <= 0 || (k > 0 && cpu[k] <= cpu[k - 1]))
            return ocg_internal_fail(OCG_E_INVALID, "cpu caps must be positive and strictly increasing");
    for (int32_t k = 0; k < ngpu; ++k)
        if (gpu[k] <= 0 || (k > 0 && gpu[k] <= gpu[k - 1]))
            return ocg_internal_fail(OCG_E_INVALID, "gpu caps must be positive and strictly increasing");
    return OCG_OK;
}

extern "C" {

int ocg_als_plan_create(ocg_ctx* ctx, int64_t m, const int64_t* row_ptr, const int32_t* col, const float* val,
                        int on_device, const int32_t* cpu, int32_t ncpu, const int32_t* gpu, int32_t ngpu,
                        const ocg_als_hyper* h, double gamma, ocg_als_plan** out) {
    if (!ctx || !out) return ocg_internal_fail(OCG_E_INVALID, "null context/output");
    *out = nullptr;
    const int64_t n = static_cast<int64_t>(ncpu) * ngpu;
    int rc = als_check(m, n, cpu, ncpu, gpu, ngpu, h, gamma);
    if (rc) return rc;
    auto P = std::make_unique<ocg_als_plan>();
    P->ctx = ctx;
    P->m = m;
    P->n = n;
    P->k = h->rank;
    P->sweeps = h->sweeps;
    P->lambda = h->lambda;
    P->seed = h->seed;
    P->gamma = gamma;
    P->ngpu = ngpu;
    P->e_base = static_cast<double>(cpu[ncpu - 1] + gpu[ngpu - 1]);
    cudaStream_t s = ocg_internal_stream(ctx);
    if (on_device) {
        ALS_CUDA(cudaMemcpy(&P->nnz, row_ptr + m, sizeof(int64_t), cudaMemcpyDeviceToHost));
        P->row_ptr.p = const_cast<int64_t*>(row_ptr);
        P->row_ptr.own = false;
        P->col.p = const_cast<int32_t*>(col);
        P->col.own = false;
        P->val.p = const_cast<float*>(val);
        P->val.own = false;
    } else {
        if ((rc = check_row_ptr(row_ptr, m))) return rc;
        P->nnz = row_ptr[m];
        P->col_cap = P->nnz;
        P->val_cap = P->nnz;
        ALS_CUDA(P->row_ptr.alloc(static_cast<size_t>(m + 1)));
        ALS_CUDA(P->col.alloc(static_cast<size_t>(P->nnz)));
        ALS_CUDA(P->val.alloc(static_cast<size_t>(P->nnz)));
        ALS_CUDA(cudaMemcpyAsync(P->row_ptr.p, row_ptr, sizeof(int64_t) * (m + 1), cudaMemcpyHostToDevice, s));
        ALS_CUDA(cudaMemcpyAsync(P->col.p, col, sizeof(int32_t) * P->nnz, cudaMemcpyHostToDevice, s));
        ALS_CUDA(cudaMemcpyAsync(P->val.p, val, sizeof(float) * P->nnz, cudaMemcpyHostToDevice, s));
    }
    if (P->nnz >= (int64_t(1) << 31)) return ocg_internal_fail(OCG_E_UNSUPPORTED, "als: nnz >= 2^31");
    if ((rc = als_alloc(P.get()))) return rc;
    if ((rc = als_alloc_fixed(P.get()))) return rc;
    if (mma_rank(P->k)) {
        ALS_CUDA(ocg::launch_absmax(P->nnz, P->val.p, P->maxbits.p + 2, ocg_internal_sm_count(ctx), s));
        ALS_CUDA(ocg::launch_als_pack_vals(P->nnz, P->val.p, P->maxbits.p + 2, P->valh.p, s));
    }
    ALS_CUDA(P->cpu.alloc(static_cast<size_t>(ncpu)));
    ALS_CUDA(P->gpu.alloc(static_cast<size_t>(ngpu)));
    ALS_CUDA(cudaMemcpyAsync(P->cpu.p, cpu, sizeof(int32_t) * ncpu, cudaMemcpyHostToDevice, s));
    ALS_CUDA(cudaMemcpyAsync(P->gpu.p, gpu, sizeof(int32_t) * ngpu, cudaMemcpyHostToDevice, s));
    ALS_CUDA(cudaStreamSynchronize(s));
    *out = P.release();
    return OCG_OK;
}

static int64_t grow_cap(int64_t n) { return n + n / 16 + 4096; }

// P->nnz = nnz; CSR arrays and nnz-dependent state grow (with headroom) only past their capacity
static int als_set_nnz(ocg_als_plan* P, int64_t nnz) {
    cudaStream_t s = ocg_internal_stream(P->ctx);
    if (nnz > P->col_cap) {
        ALS_CUDA(cudaStreamSynchronize(s));
        P->col_cap = grow_cap(nnz);
        ALS_CUDA(P->col.alloc(static_cast<size_t>(P->col_cap)));
    }
    if (nnz > P->val_cap) {
        ALS_CUDA(cudaStreamSynchronize(s));
        P->val_cap = grow_cap(nnz);
        ALS_CUDA(P->val.alloc(static_cast<size_t>(P->val_cap)));
    }
    P->nnz = nnz;
    if (nnz > P->nnz_cap) {
        ALS_CUDA(cudaStreamSynchronize(s));
        P->nnz_cap = grow_cap(nnz);
        return als_alloc(P);
    }
    return OCG_OK;
}

int ocg_als_plan_upload(ocg_als_plan* P, const int64_t* row_ptr, const int32_t* col, const float* val) {
    if (P && P->staged) return ocg_internal_fail(OCG_E_INVALID, "als upload: a staged CSR is pending (run first)");
    if (!P || !row_ptr || !col || !val) return ocg_internal_fail(OCG_E_INVALID, "null plan/buffer");
    if (!P->row_ptr.own) return ocg_internal_fail(OCG_E_INVALID, "als upload: plan uses caller device buffers");
    if (int rc = check_row_ptr(row_ptr, P->m)) return rc;
    const int64_t nnz = row_ptr[P->m];
    if (nnz < 0 || nnz >= (int64_t(1) << 31)) return ocg_internal_fail(OCG_E_INVALID, "als upload: bad nnz");
    cudaStream_t s = ocg_internal_stream(P->ctx);
    {  // new observations: nnz-dependent device state grows when needed (factors survive)
        int rc = als_set_nnz(P, nnz);
        if (rc) return rc;
    }
    P->dirty = true;
    ALS_CUDA(cudaMemcpyAsync(P->row_ptr.p, row_ptr, sizeof(int64_t) * (P->m + 1), cudaMemcpyHostToDevice, s));
    ALS_CUDA(cudaMemcpyAsync(P->col.p, col, sizeof(int32_t) * P->nnz, cudaMemcpyHostToDevice, s));
    ALS_CUDA(cudaMemcpyAsync(P->val.p, val, sizeof(float) * P->nnz, cudaMemcpyHostToDevice, s));
    if (mma_rank(P->k)) {
        ALS_CUDA(ocg::launch_absmax(P->nnz, P->val.p, P->maxbits.p + 2, ocg_internal_sm_count(P->ctx), s));
        ALS_CUDA(ocg::launch_als_pack_vals(P->nnz, P->val.p, P->maxbits.p + 2, P->valh.p, s));
    }
    return OCG_OK;
}

namespace {
__global__ void widen_u16_kernel(int64_t n, const uint16_t* __restrict__ in, int32_t* __restrict__ out) {
    const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q < n) out[q] = in[q];
}
}  // namespace

namespace {

// ---- streaming arrivals: merge new observations into the device CSR
// per-row insertion counts (additions sorted by (row, col))
__global__ void add_count_kernel(int64_t count, const int32_t* __restrict__ arow, int32_t* __restrict__ inc) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < count) atomicAdd(inc + arow[t], 1);
}
// warp per row: the row's old entries shift by the additions before them (earlier rows:
// ex[r]; this row: those with a smaller column), each addition lands after the old
// entries with a smaller column; an addition on an observed cell sets *err
__global__ void add_merge_kernel(int64_t m, const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                 const float* __restrict__ val, const int32_t* __restrict__ inc,
                                 const int32_t* __restrict__ ex, const int32_t* __restrict__ acol,
                                 const float* __restrict__ aval, int64_t* __restrict__ rp2, int32_t* __restrict__ col2,
                                 float* __restrict__ val2, int32_t* __restrict__ err) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < m; r += nw) {
        const int64_t b = rp[r], e = rp[r + 1];
        const int32_t na = inc[r], a0 = ex[r];
        const int64_t b2 = b + a0;
        if (lane == 0) {
            rp2[r] = b2;
            if (r == m - 1) rp2[m] = e + a0 + na;
        }
        for (int64_t q = b + lane; q < e; q += 32) {
            const int32_t c = col[q];
            int32_t sh = 0;
            for (int32_t t = 0; t < na; ++t) sh += acol[a0 + t] < c;
            col2[b2 + (q - b) + sh] = c;
            val2[b2 + (q - b) + sh] = val[q];
        }
        for (int32_t t = lane; t < na; t += 32) {
            const int32_t c = acol[a0 + t];
            int64_t lo = b, hi = e;  // first old entry with col >= c
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (col[mid] < c) lo = mid + 1;
                else hi = mid;
            }
            if (lo < e && col[lo] == c) atomicExch(err, 1);
            col2[b2 + (lo - b) + t] = c;
            val2[b2 + (lo - b) + t] = aval[a0 + t];
        }
    }
}

}  // namespace

namespace ocg {
cudaError_t launch_widen_u16(int64_t n, const uint16_t* in, int32_t* out, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    widen_u16_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(n, in, out);
    return cudaGetLastError();
}
}  // namespace ocg

// side stream + events of the staged (pipelined) upload path, created on first use
static int als_copy_objs(ocg_als_plan* P) {
    if (!P->copy_stream) {
        ALS_CUDA(cudaStreamCreateWithFlags(&P->copy_stream, cudaStreamNonBlocking));
        ALS_CUDA(cudaEventCreateWithFlags(&P->ev_staged, cudaEventDisableTiming));
        ALS_CUDA(cudaEventCreateWithFlags(&P->ev_free, cudaEventDisableTiming));
    }
    return OCG_OK;
}

int ocg_als_plan_upload_compact(ocg_als_plan* P, const int64_t* row_ptr, const uint16_t* col16, const float* val) {
    if (P && P->staged) return ocg_internal_fail(OCG_E_INVALID, "als upload: a staged CSR is pending (run first)");
    if (!P || !row_ptr || !col16 || !val) return ocg_internal_fail(OCG_E_INVALID, "null plan/buffer");
    if (P->n > 65536) return ocg_internal_fail(OCG_E_INVALID, "als upload_compact: more than 65536 settings");
    if (!P->row_ptr.own) return ocg_internal_fail(OCG_E_INVALID, "als upload: plan uses caller device buffers");
    if (int rc = check_row_ptr(row_ptr, P->m)) return rc;
    const int64_t nnz = row_ptr[P->m];
    if (nnz < 0 || nnz >= (int64_t(1) << 31)) return ocg_internal_fail(OCG_E_INVALID, "als upload: bad nnz");
    cudaStream_t s = ocg_internal_stream(P->ctx);
    {  // new observations: nnz-dependent device state grows when needed (factors survive)
        int rc = als_set_nnz(P, nnz);
        if (rc) return rc;
    }
    P->dirty = true;
    if (P->col16_cap < nnz) {
        ALS_CUDA(P->col16.alloc(static_cast<size_t>(nnz)));
        P->col16_cap = nnz;
    }
    ALS_CUDA(cudaMemcpyAsync(P->row_ptr.p, row_ptr, sizeof(int64_t) * (P->m + 1), cudaMemcpyHostToDevice, s));
    ALS_CUDA(cudaMemcpyAsync(P->col16.p, col16, sizeof(uint16_t) * P->nnz, cudaMemcpyHostToDevice, s));
    ALS_CUDA(cudaMemcpyAsync(P->val.p, val, sizeof(float) * P->nnz, cudaMemcpyHostToDevice, s));
    if (P->nnz > 0) {
        widen_u16_kernel<<<static_cast<unsigned>((P->nnz + 255) / 256), 256, 0, s>>>(P->nnz, P->col16.p, P->col.p);
        ALS_CUDA(cudaGetLastError());
    }
    // col16 is read by the widen above: a later _stage_compact must not overwrite it before
    // the widen has run (its side-stream copy waits on ev_free)
    {
        int rc = als_copy_objs(P);
        if (rc) return rc;
    }
    ALS_CUDA(cudaEventRecord(P->ev_free, s));
    P->free_recorded = true;
    if (mma_rank(P->k)) {
        ALS_CUDA(ocg::launch_absmax(P->nnz, P->val.p, P->maxbits.p + 2, ocg_internal_sm_count(P->ctx), s));
        ALS_CUDA(ocg::launch_als_pack_vals(P->nnz, P->val.p, P->maxbits.p + 2, P->valh.p, s));
    }
    return OCG_OK;
}

int ocg_als_plan_stage_compact(ocg_als_plan* P, const int64_t* row_ptr, const uint16_t* col16, const float* val) {
    if (!P || !row_ptr || !col16 || !val) return ocg_internal_fail(OCG_E_INVALID, "null plan/buffer");
    if (P->n > 65536) return ocg_internal_fail(OCG_E_INVALID, "als stage_compact: more than 65536 settings");
    if (!P->row_ptr.own) return ocg_internal_fail(OCG_E_INVALID, "als upload: plan uses caller device buffers");
    if (P->staged) return ocg_internal_fail(OCG_E_INVALID, "als stage_compact: a staged CSR is pending (run first)");
    if (int rc = check_row_ptr(row_ptr, P->m)) return rc;
    const int64_t nnz = row_ptr[P->m];
    if (nnz < 0 || nnz >= (int64_t(1) << 31)) return ocg_internal_fail(OCG_E_INVALID, "als upload: bad nnz");
    cudaStream_t s = ocg_internal_stream(P->ctx);
    {
        int rc = als_copy_objs(P);
        if (rc) return rc;
    }
    if (nnz > P->col_cap || nnz > P->nnz_cap || P->col16_cap < nnz || !P->rp_next.p || nnz > P->val_next_cap) {
        // growth (rare): drain both streams, then size every buffer for nnz
        ALS_CUDA(cudaStreamSynchronize(s));
        ALS_CUDA(cudaStreamSynchronize(P->copy_stream));
        const int64_t keep = P->nnz;
        int rc = als_set_nnz(P, std::max(nnz, keep));
        if (rc) return rc;
        P->nnz = keep;
        if (P->col16_cap < nnz) {
            P->col16_cap = grow_cap(nnz);
            ALS_CUDA(P->col16.alloc(static_cast<size_t>(P->col16_cap)));
        }
        if (!P->rp_next.p) ALS_CUDA(P->rp_next.alloc(static_cast<size_t>(P->m + 1)));
        if (nnz > P->val_next_cap) {
            P->val_next_cap = grow_cap(nnz);
            ALS_CUDA(P->val_next.alloc(static_cast<size_t>(P->val_next_cap)));
        }
    }
    // rp_next / val_next / col16 are free once the step that last used them has passed its
    // swap point (ev_free, recorded on the compute stream)
    if (P->free_recorded) ALS_CUDA(cudaStreamWaitEvent(P->copy_stream, P->ev_free, 0));
    cudaStream_t c = P->copy_stream;
    ALS_CUDA(cudaMemcpyAsync(P->rp_next.p, row_ptr, sizeof(int64_t) * (P->m + 1), cudaMemcpyHostToDevice, c));
    ALS_CUDA(cudaMemcpyAsync(P->col16.p, col16, sizeof(uint16_t) * nnz, cudaMemcpyHostToDevice, c));
    ALS_CUDA(cudaMemcpyAsync(P->val_next.p, val, sizeof(float) * nnz, cudaMemcpyHostToDevice, c));
    ALS_CUDA(cudaEventRecord(P->ev_staged, c));
    P->staged = true;
    P->staged_nnz = nnz;
    return OCG_OK;
}

int ocg_als_plan_add_observations(ocg_als_plan* P, int64_t count, const int32_t* rows, const int32_t* cols,
                                  const float* vals) {
    if (!P || count < 0 || (count > 0 && (!rows || !cols || !vals)))
        return ocg_internal_fail(OCG_E_INVALID, "als add_observations: bad arguments");
    if (!P->row_ptr.own) return ocg_internal_fail(OCG_E_INVALID, "als upload: plan uses caller device buffers");
    if (P->staged) return ocg_internal_fail(OCG_E_INVALID, "als add_observations: a staged CSR is pending (run first)");
    if (count == 0) return OCG_OK;
    for (int64_t t = 0; t < count; ++t) {  // sorted by (row, col), in range
        if (rows[t] < 0 || rows[t] >= P->m || cols[t] < 0 || cols[t] >= P->n)
            return ocg_internal_fail(OCG_E_INVALID, "als add_observations: cell out of range");
        if (t > 0 && (rows[t] < rows[t - 1] || (rows[t] == rows[t - 1] && cols[t] <= cols[t - 1])))
            return ocg_internal_fail(OCG_E_INVALID, "als add_observations: cells not sorted by (row, col) / repeated");
        if (!(vals[t] > 0.0f && vals[t] <= 1.25f))  // PerformanceMatrix::set (core.cpp:144-146)
            return ocg_internal_fail(OCG_E_INVALID, "normalized performance outside (0, 1.25]");
    }
    P->dirty = true;
    const int64_t nnz2 = P->nnz + count;
    if (nnz2 >= (int64_t(1) << 31)) return ocg_internal_fail(OCG_E_INVALID, "als add_observations: bad nnz");
    cudaStream_t s = ocg_internal_stream(P->ctx);
    const int sm = ocg_internal_sm_count(P->ctx);
    if (!P->add_inc.p) {
        ALS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, P->add_tmp_bytes, P->add_inc.p, P->add_ex.p, P->m));
        ALS_CUDA(P->add_tmp.alloc(P->add_tmp_bytes));
        ALS_CUDA(P->add_inc.alloc(static_cast<size_t>(P->m)));
        ALS_CUDA(P->add_ex.alloc(static_cast<size_t>(P->m)));
        ALS_CUDA(P->add_err.alloc(1));
    }
    if (P->add_cap < count) {
        P->add_cap = grow_cap(count);
        ALS_CUDA(P->add_rc.alloc(static_cast<size_t>(2 * P->add_cap)));
        ALS_CUDA(P->add_v.alloc(static_cast<size_t>(P->add_cap)));
    }
    int32_t* arow = P->add_rc.p;
    int32_t* acol = P->add_rc.p + P->add_cap;
    float* aval = P->add_v.p;
    int32_t* inc = P->add_inc.p;
    int32_t* ex = P->add_ex.p;
    int32_t* err = P->add_err.p;
    size_t tb = P->add_tmp_bytes;
    if (!P->rp_alt.p) ALS_CUDA(P->rp_alt.alloc(static_cast<size_t>(P->m + 1)));
    if (P->alt_cap < nnz2) {
        P->alt_cap = grow_cap(nnz2);
        ALS_CUDA(P->col_alt.alloc(static_cast<size_t>(P->alt_cap)));
        ALS_CUDA(P->val_alt.alloc(static_cast<size_t>(P->alt_cap)));
    }
    ALS_CUDA(cudaMemcpyAsync(arow, rows, sizeof(int32_t) * count, cudaMemcpyHostToDevice, s));
    ALS_CUDA(cudaMemcpyAsync(acol, cols, sizeof(int32_t) * count, cudaMemcpyHostToDevice, s));
    ALS_CUDA(cudaMemcpyAsync(aval, vals, sizeof(float) * count, cudaMemcpyHostToDevice, s));
    ALS_CUDA(cudaMemsetAsync(inc, 0, sizeof(int32_t) * P->m, s));
    ALS_CUDA(cudaMemsetAsync(err, 0, sizeof(int32_t), s));
    add_count_kernel<<<static_cast<unsigned>((count + 255) / 256), 256, 0, s>>>(count, arow, inc);
    ALS_CUDA(cudaGetLastError());
    ALS_CUDA(cub::DeviceScan::ExclusiveSum(P->add_tmp.p, tb, inc, ex, P->m, s));
    add_merge_kernel<<<sm * 8, 256, 0, s>>>(P->m, P->row_ptr.p, P->col.p, P->val.p, inc, ex, acol, aval,
                                            P->rp_alt.p, P->col_alt.p, P->val_alt.p, err);
    ALS_CUDA(cudaGetLastError());
    int32_t herr = 0;
    ALS_CUDA(cudaMemcpyAsync(&herr, err, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    ALS_CUDA(cudaStreamSynchronize(s));
    if (herr) return ocg_internal_fail(OCG_E_INVALID, "als add_observations: a cell is already observed");
    std::swap(P->row_ptr.p, P->rp_alt.p);
    std::swap(P->col.p, P->col_alt.p);
    std::swap(P->val.p, P->val_alt.p);
    // col/val move to the alt pair (both sized alt_cap); the old pair becomes the next merge target
    const int64_t old_col_cap = P->col_cap, old_val_cap = P->val_cap;
    P->col_cap = P->val_cap = P->alt_cap;
    P->alt_cap = std::min(old_col_cap, old_val_cap);
    P->nnz = nnz2;
    if (nnz2 > P->nnz_cap) {
        P->nnz_cap = grow_cap(nnz2);
        int rc = als_alloc(P);
        if (rc) return rc;
    }
    if (mma_rank(P->k)) {
        ALS_CUDA(ocg::launch_absmax(P->nnz, P->val.p, P->maxbits.p + 2, sm, s));
        ALS_CUDA(ocg::launch_als_pack_vals(P->nnz, P->val.p, P->maxbits.p + 2, P->valh.p, s));
    }
    return OCG_OK;
}

int ocg_als_plan_set_warm(ocg_als_plan* P, int32_t warm_sweeps) {
    if (!P) return ocg_internal_fail(OCG_E_INVALID, "null plan");
    if (warm_sweeps < 0) return ocg_internal_fail(OCG_E_INVALID, "als: warm_sweeps < 0");
    P->warm_sweeps = warm_sweeps;
    return OCG_OK;
}

static int launch_select(ocg_als_plan* P) {
    cudaStream_t s = ocg_internal_stream(P->ctx);
    if (!mma_rank(P->k)) ALS_CUDA(ocg::launch_transpose(P->n, P->k, P->V.p, P->Vt.p, s));
    ocg::AlsSelectArgs a{};
    a.m = P->m;
    a.n = P->n;
    a.k = P->k;
    a.U = P->U.p;
    a.V = P->V.p;
    a.Vt = P->Vt.p;
    a.row_ptr = P->row_ptr.p;
    a.col = P->col.p;
    a.val = P->val.p;
    a.cpu_caps = P->cpu.p;
    a.gpu_caps = P->gpu.p;
    a.ngpu = P->ngpu;
    a.e_base = P->e_base;
    a.gamma = P->gamma;
    a.idx = P->idx.p;
    a.saving = P->saving.p;
    a.loss = P->loss.p;
    a.ncand = P->ncand.p;
    a.completed = nullptr;
    if (mma_rank(P->k))
        ALS_CUDA(ocg::launch_als_select_mma(a, P->Vsel.p, P->maxbits.p, P->maxbits.p + 1, ocg_internal_sm_count(P->ctx), s));
    else
        ALS_CUDA(ocg::launch_als_select(a, ocg_internal_sm_count(P->ctx), s));
    return OCG_OK;
}

// phase_ms (optional, 6 floats): CSC build, row half-sweeps, column half-sweeps, select,
// and (rank 32) the row / column Gram kernels alone
int ocg_als_plan_run(ocg_als_plan* P, float* total_ms, float* phase_ms) {
    if (!P) return ocg_internal_fail(OCG_E_INVALID, "null plan");
    cudaStream_t s = ocg_internal_stream(P->ctx);
    const int sm = ocg_internal_sm_count(P->ctx);
    ALS_CUDA(cudaEventRecord(P->ev[0], s));
    if (P->staged) {  // swap in the CSR staged by ocg_als_plan_stage_compact
        ALS_CUDA(cudaStreamWaitEvent(s, P->ev_staged, 0));
        std::swap(P->row_ptr.p, P->rp_next.p);
        std::swap(P->val.p, P->val_next.p);
        std::swap(P->val_cap, P->val_next_cap);
        P->nnz = P->staged_nnz;
        P->staged = false;
        ALS_CUDA(ocg::launch_widen_u16(P->nnz, P->col16.p, P->col.p, s));
        if (mma_rank(P->k)) {
            ALS_CUDA(ocg::launch_absmax(P->nnz, P->val.p, P->maxbits.p + 2, sm, s));
            ALS_CUDA(ocg::launch_als_pack_vals(P->nnz, P->val.p, P->maxbits.p + 2, P->valh.p, s));
        }
        ALS_CUDA(cudaEventRecord(P->ev_free, s));
        P->free_recorded = true;
        P->dirty = true;
    }
    int rc = als_validate(P);
    if (rc) return rc;
    if ((rc = als_build_csc(P))) return rc;
    const bool warm = P->warm_sweeps > 0 && P->fitted;
    if (!warm) {
        ALS_CUDA(ocg::launch_als_init(P->n, P->k, P->seed, P->V.p, s));
        if ((rc = als_pack(P, 1))) return rc;
    }
    const int sweeps = warm ? P->warm_sweeps : P->sweeps;
    ALS_CUDA(cudaEventRecord(P->ev[1], s));
    float row_ms = 0.f, col_ms = 0.f, rgram_ms = 0.f, cgram_ms = 0.f;
    for (int it = 0; it < sweeps; ++it) {
        ocg::AlsHalf hr = als_half(P, 0), hc = als_half(P, 1);
        if (phase_ms) {
            hr.ev_gram0 = P->ev[6];
            hr.ev_gram1 = P->ev[7];
            hc.ev_gram0 = P->ev[8];
            hc.ev_gram1 = P->ev[9];
        }
        const bool track = mma_rank(P->k);
        if (mma_rank(P->k)) {
            hr.xmax = P->maxbits.p + 0;  // U's packing scale, produced by the row-side K4
            hc.xmax = P->maxbits.p + 1;  // V's
        }
        ALS_CUDA(cudaEventRecord(P->ev[2], s));
        ALS_CUDA(ocg::launch_als_half(P->k, hr, 0, sm, s));
        if ((rc = als_pack(P, 0, track))) return rc;
        ALS_CUDA(cudaEventRecord(P->ev[3], s));
        ALS_CUDA(ocg::launch_als_half(P->k, hc, 0, sm, s));
        if ((rc = als_pack(P, 1, track))) return rc;
        ALS_CUDA(cudaEventRecord(P->ev[4], s));
        if (phase_ms) {
            float a = 0, b = 0;
            ALS_CUDA(cudaEventSynchronize(P->ev[4]));
            ALS_CUDA(cudaEventElapsedTime(&a, P->ev[2], P->ev[3]));
            ALS_CUDA(cudaEventElapsedTime(&b, P->ev[3], P->ev[4]));
            row_ms += a;
            col_ms += b;
            if (mma_rank(P->k)) {
                ALS_CUDA(cudaEventElapsedTime(&a, P->ev[6], P->ev[7]));
                ALS_CUDA(cudaEventElapsedTime(&b, P->ev[8], P->ev[9]));
                rgram_ms += a;
                cgram_ms += b;
            }
        }
    }
    ALS_CUDA(cudaEventRecord(P->ev[2], s));
    if ((rc = launch_select(P))) return rc;
    ALS_CUDA(cudaEventRecord(P->ev[5], s));
    P->fitted = true;
    if (total_ms || phase_ms) {
        ALS_CUDA(cudaEventSynchronize(P->ev[5]));
        if (total_ms) ALS_CUDA(cudaEventElapsedTime(total_ms, P->ev[0], P->ev[5]));
        if (phase_ms) {
            ALS_CUDA(cudaEventElapsedTime(&phase_ms[0], P->ev[0], P->ev[1]));
            phase_ms[1] = row_ms;
            phase_ms[2] = col_ms;
            ALS_CUDA(cudaEventElapsedTime(&phase_ms[3], P->ev[2], P->ev[5]));
            phase_ms[4] = rgram_ms;  // Gram kernel alone (rank 32; 0 otherwise)
            phase_ms[5] = cgram_ms;
        }
    }
    return OCG_OK;
}

// ---- phase-level entry points for the row-sharded multi-GPU driver --------
// (all asynchronous on the context stream; see ocg_ctx_set_stream)
int ocg_als_plan_begin(ocg_als_plan* P) {
    if (!P) return ocg_internal_fail(OCG_E_INVALID, "null plan");
    int rc = als_validate(P);
    if (rc) return rc;
    rc = als_build_csc(P);
    if (rc) return rc;
    ALS_CUDA(ocg::launch_als_init(P->n, P->k, P->seed, P->V.p, ocg_internal_stream(P->ctx)));
    return als_pack(P, 1);
}

int ocg_als_plan_row_half(ocg_als_plan* P) {
    if (!P) return ocg_internal_fail(OCG_E_INVALID, "null plan");
    ALS_CUDA(ocg::launch_als_half(P->k, als_half(P, 0), 0, ocg_internal_sm_count(P->ctx), ocg_internal_stream(P->ctx)));
    return als_pack(P, 0);
}

int ocg_als_plan_col_half(ocg_als_plan* P) {
    if (!P) return ocg_internal_fail(OCG_E_INVALID, "null plan");
    ALS_CUDA(ocg::launch_als_half(P->k, als_half(P, 1), 0, ocg_internal_sm_count(P->ctx), ocg_internal_stream(P->ctx)));
    return als_pack(P, 1);
}

int64_t ocg_als_plan_gram_floats(ocg_als_plan* P) {
    return P ? P->n * static_cast<int64_t>(ocg::als_gram_record_floats(P->k)) : 0;
}

// this shard's column Gram records (K*K Gram, K rhs, count per column) -> d_gram
int ocg_als_plan_col_gram(ocg_als_plan* P, float* d_gram) {
    if (!P || !d_gram) return ocg_internal_fail(OCG_E_INVALID, "null plan/buffer");
    ocg::AlsHalf h = als_half(P, 1);
    h.gram_out = d_gram;
    ALS_CUDA(ocg::launch_als_half(P->k, h, 1, ocg_internal_sm_count(P->ctx), ocg_internal_stream(P->ctx)));
    return OCG_OK;
}

// V from (allreduced) column Gram records
int ocg_als_plan_col_solve(ocg_als_plan* P, const float* d_gram) {
    if (!P || !d_gram) return ocg_internal_fail(OCG_E_INVALID, "null plan/buffer");
    ALS_CUDA(ocg::launch_als_solve_from_gram(P->k, P->n, d_gram, P->V.p, P->lambda, ocg_internal_sm_count(P->ctx),
                                             ocg_internal_stream(P->ctx)));
    return als_pack(P, 1);
}

int ocg_als_plan_select(ocg_als_plan* P) {
    if (!P) return ocg_internal_fail(OCG_E_INVALID, "null plan");
    return launch_select(P);
}

int ocg_als_plan_results(ocg_als_plan* P, int32_t* idx, double* saving, double* loss, int32_t* ncand, float* U,
                         float* V) {
    if (!P) return ocg_internal_fail(OCG_E_INVALID, "null plan");
    if (idx || saving || loss || ncand)  // decisions of a rejected matrix are not returned (factors stay inspectable)
        if (int rc = als_error(P)) return rc;
    cudaStream_t s = ocg_internal_stream(P->ctx);
    const size_t m = static_cast<size_t>(P->m);
    if (idx) ALS_CUDA(cudaMemcpyAsync(idx, P->idx.p, sizeof(int32_t) * m, cudaMemcpyDeviceToHost, s));
    if (saving) ALS_CUDA(cudaMemcpyAsync(saving, P->saving.p, sizeof(double) * m, cudaMemcpyDeviceToHost, s));
    if (loss) ALS_CUDA(cudaMemcpyAsync(loss, P->loss.p, sizeof(double) * m, cudaMemcpyDeviceToHost, s));
    if (ncand) ALS_CUDA(cudaMemcpyAsync(ncand, P->ncand.p, sizeof(int32_t) * m, cudaMemcpyDeviceToHost, s));
    if (U) ALS_CUDA(cudaMemcpyAsync(U, P->U.p, sizeof(float) * m * P->k, cudaMemcpyDeviceToHost, s));
    if (V) ALS_CUDA(cudaMemcpyAsync(V, P->V.p, sizeof(float) * P->n * P->k, cudaMemcpyDeviceToHost, s));
    ALS_CUDA(cudaStreamSynchronize(s));
    return OCG_OK;
}

int ocg_als_plan_results_async(ocg_als_plan* P, int32_t* idx, double* saving, double* loss, int32_t* ncand) {
    if (!P || !idx || !saving || !loss || !ncand) return ocg_internal_fail(OCG_E_INVALID, "null plan/buffer");
    cudaStream_t s = ocg_internal_stream(P->ctx);
    const size_t m = static_cast<size_t>(P->m);
    if (!P->ev_results) ALS_CUDA(cudaEventCreateWithFlags(&P->ev_results, cudaEventDisableTiming));
    ALS_CUDA(cudaMemcpyAsync(idx, P->idx.p, sizeof(int32_t) * m, cudaMemcpyDeviceToHost, s));
    ALS_CUDA(cudaMemcpyAsync(saving, P->saving.p, sizeof(double) * m, cudaMemcpyDeviceToHost, s));
    ALS_CUDA(cudaMemcpyAsync(loss, P->loss.p, sizeof(double) * m, cudaMemcpyDeviceToHost, s));
    ALS_CUDA(cudaMemcpyAsync(ncand, P->ncand.p, sizeof(int32_t) * m, cudaMemcpyDeviceToHost, s));
    ALS_CUDA(cudaEventRecord(P->ev_results, s));
    return OCG_OK;
}

int ocg_als_plan_results_wait(ocg_als_plan* P) {
    if (!P) return ocg_internal_fail(OCG_E_INVALID, "null plan");
    if (P->ev_results) ALS_CUDA(cudaEventSynchronize(P->ev_results));
    return als_error(P);
}

// completed rows [row0, row0+nrows) as the selection saw them (FP64), for tests
int ocg_als_plan_completed_rows(ocg_als_plan* P, int64_t row0, int64_t nrows, double* out) {
    if (!P) return ocg_internal_fail(OCG_E_INVALID, "null plan");
    if (row0 < 0 || nrows < 0 || row0 + nrows > P->m) return ocg_internal_fail(OCG_E_RANGE, "row range");
    if (int rc = als_error(P)) return rc;
    cudaStream_t s = ocg_internal_stream(P->ctx);
    Buf<double> d;
    Buf<int32_t> di, dn;
    Buf<double> ds, dl;
    ALS_CUDA(d.alloc(static_cast<size_t>(nrows * P->n)));
    ALS_CUDA(di.alloc(static_cast<size_t>(nrows)));
    ALS_CUDA(dn.alloc(static_cast<size_t>(nrows)));
    ALS_CUDA(ds.alloc(static_cast<size_t>(nrows)));
    ALS_CUDA(dl.alloc(static_cast<size_t>(nrows)));
    ocg::AlsSelectArgs a{};
    a.m = nrows;
    a.n = P->n;
    a.k = P->k;
    a.U = P->U.p + row0 * P->k;
    a.V = P->V.p;
    a.Vt = P->Vt.p;
    // the rows' CSR slice: row_ptr offsets stay absolute, so pass shifted pointers
    a.row_ptr = P->row_ptr.p + row0;
    a.col = P->col.p;
    a.val = P->val.p;
    a.cpu_caps = P->cpu.p;
    a.gpu_caps = P->gpu.p;
    a.ngpu = P->ngpu;
    a.e_base = P->e_base;
    a.gamma = P->gamma;
    a.idx = di.p;
    a.saving = ds.p;
    a.loss = dl.p;
    a.ncand = dn.p;
    a.completed = d.p;
    if (mma_rank(P->k))
        ALS_CUDA(ocg::launch_als_select_mma(a, P->Vsel.p, P->maxbits.p, P->maxbits.p + 1, ocg_internal_sm_count(P->ctx), s));
    else
        ALS_CUDA(ocg::launch_als_select(a, ocg_internal_sm_count(P->ctx), s));
    ALS_CUDA(cudaMemcpyAsync(out, d.p, sizeof(double) * nrows * P->n, cudaMemcpyDeviceToHost, s));
    ALS_CUDA(cudaStreamSynchronize(s));
    return OCG_OK;
}

void ocg_als_plan_destroy(ocg_als_plan* P) { delete P; }

}  // extern "C"
