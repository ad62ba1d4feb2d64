// ALS completion kernels (K3 Gram accumulation + K4 batched Cholesky solve).
//
// No reference counterpart (the reference's CF is NCF only): the
// semantics are defined by oracle/ocg_oracle.c (ocgo_als_fit) — weighted-
// lambda ALS, u_i = (sum_j v_j v_j^T + lambda n_i I)^-1 sum_j r_ij v_j.
//
// als_gram_solve_kernel: one ITEM (a row for the row half-sweep, a column for
// the column half-sweep) is owned by WPI warps.  Each warp streams 32
// observations at a time: the (index, value) pairs are read coalesced, the 32
// gathered factor rows (K floats each, 128 B at K=32) are staged in shared
// memory, and every lane accumulates a (K/8) x (K/4) block of the K x K Gram
// in registers (all loads are conflict-free 16-byte LDS within one staged
// row).  The WPI partial Grams are reduced in a fixed order in shared memory
// (deterministic), lambda*n is added to the diagonal, and one warp factors
// the system with a register-resident right-looking Cholesky (lane l owns row
// l) followed by forward/back substitution.  MODE_GRAM instead writes the
// reduced Gram + rhs to global memory (multi-GPU: allreduced over ranks, then
// als_solve_from_gram_kernel).
#include <cuda_runtime.h>

#include "als.h"
#include "ocg_common.cuh"

namespace ocg {

namespace {

template <int K>
struct GramShape {
    static constexpr int RB = K / 8;  // rows per lane block
    static constexpr int CB = K / 4;  // cols per lane block
    static constexpr int GS = K + 1;  // padded Gram row stride (floats)
    static constexpr int TS = K + 4;  // staged-row stride (floats), keeps 16-byte alignment
};

// Cholesky-solve A x = b on one warp; lane l < K owns row l of A (in smem G,
// row stride GS) and b_l.  Returns x_l.  A is overwritten with L.
template <int K>
__device__ __forceinline__ float chol_solve_warp(float* G, float* colb, float b, float diag_add, int lane) {
    constexpr int GS = GramShape<K>::GS;
    float a[K];
#pragma unroll
    for (int m = 0; m < K; ++m) a[m] = lane < K ? G[lane * GS + m] : 0.0f;
    if (lane < K) a[lane] += diag_add;
    // right-looking factorisation, column c per step
#pragma unroll
    for (int c = 0; c < K; ++c) {
        if (lane == c) {
            a[c] = sqrtf(a[c]);
            colb[c] = a[c];
        }
        __syncwarp();
        const float d = colb[c];
        if (lane > c && lane < K) {
            a[c] = a[c] / d;
            colb[lane] = a[c];
        }
        __syncwarp();
        if (lane > c && lane < K) {
#pragma unroll
            for (int m = c + 1; m < K; ++m)
                if (m <= lane) a[m] = fmaf(-a[c], colb[m], a[m]);
        }
        __syncwarp();
    }
    // L y = b
    float y = b;
#pragma unroll
    for (int c = 0; c < K; ++c) {
        if (lane == c) {
            y = y / a[c];
            colb[c] = y;
        }
        __syncwarp();
        const float yc = colb[c];
        if (lane > c && lane < K) y = fmaf(-a[c], yc, y);
        __syncwarp();
    }
    // L^T x = y : needs L[c][l] -> stage L in G
    if (lane < K) {
#pragma unroll
        for (int m = 0; m < K; ++m)
            if (m <= lane) G[lane * GS + m] = a[m];
    }
    __syncwarp();
#pragma unroll
    for (int c = K - 1; c >= 0; --c) {
        if (lane == c) {
            y = y / a[c];
            colb[c] = y;
        }
        __syncwarp();
        const float xc = colb[c];
        if (lane < c) y = fmaf(-G[c * GS + lane], xc, y);
        __syncwarp();
    }
    return y;
}

// Accumulate one warp's share of an item's Gram (register blocks) and rhs.
template <int K>
__device__ __forceinline__ void gram_accumulate(const int32_t* __restrict__ idx, const float* __restrict__ val,
                                                int64_t beg, int64_t end, int64_t step_chunks, int64_t first_chunk,
                                                const float* __restrict__ Y, float* stage, float* rstage,
                                                float (&acc)[GramShape<K>::RB][GramShape<K>::CB], float& bacc,
                                                int lane) {
    constexpr int RB = GramShape<K>::RB, CB = GramShape<K>::CB, TS = GramShape<K>::TS;
    constexpr int PER = 32 / K > 0 ? 32 / K : 1;  // observations loaded per instruction
    const int bi = lane >> 2, bj = lane & 3;
    for (int64_t base = beg + first_chunk * 32; base < end; base += step_chunks * 32) {
        const int cnt = static_cast<int>(end - base < 32 ? end - base : 32);
        int j = 0;
        float r = 0.0f;
        if (lane < cnt) {
            j = __ldg(idx + base + lane);
            r = __ldg(val + base + lane);
        }
        rstage[lane] = r;
        // gather the cnt factor rows into the stage (coalesced K-float rows)
#pragma unroll 8
        for (int o0 = 0; o0 < 32; o0 += PER) {
            const int o = o0 + lane / K;
            const int f = lane % K;
            const int jo = __shfl_sync(0xffffffffu, j, o);
            if (o < cnt) stage[o * TS + f] = __ldg(Y + static_cast<int64_t>(jo) * K + f);
        }
        __syncwarp();
        for (int o = 0; o < cnt; ++o) {
            const float* row = stage + o * TS;
            float x[RB], yv[CB];
#pragma unroll
            for (int q = 0; q < RB; ++q) x[q] = row[bi * RB + q];
#pragma unroll
            for (int q = 0; q < CB; ++q) yv[q] = row[bj * CB + q];
#pragma unroll
            for (int p = 0; p < RB; ++p)
#pragma unroll
                for (int q = 0; q < CB; ++q) acc[p][q] = fmaf(x[p], yv[q], acc[p][q]);
            if (lane < K) bacc = fmaf(rstage[o], row[lane], bacc);
        }
        __syncwarp();
    }
}

}  // namespace

template <int K, int WPI, int MODE>
__global__ void __launch_bounds__(256) als_gram_solve_kernel(int64_t nitems, const int64_t* __restrict__ ptr,
                                                             const int32_t* __restrict__ idx,
                                                             const float* __restrict__ val,
                                                             const float* __restrict__ Y, float* __restrict__ X,
                                                             float* __restrict__ Gout, float lambda) {
    constexpr int RB = GramShape<K>::RB, CB = GramShape<K>::CB, GS = GramShape<K>::GS, TS = GramShape<K>::TS;
    constexpr int WARPS = 8;
    constexpr int ITEMS_PER_CTA = WARPS / WPI;
    static_assert(32 * TS >= K * GS, "Gram aliases the item's first stage buffer");
    __shared__ __align__(16) float stage_all[WARPS][32 * TS];
    __shared__ float rstage_all[WARPS][32];
    __shared__ float rhs_all[ITEMS_PER_CTA][WPI][K];
    __shared__ float colb_all[ITEMS_PER_CTA][K];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int slot = warp / WPI, sub = warp % WPI;
    float* stage = stage_all[warp];
    float* rstage = rstage_all[warp];
    float* G = stage_all[slot * WPI];  // free once the item's sub-0 warp finished accumulating
    float* colb = colb_all[slot];
    const int bi = lane >> 2, bj = lane & 3;
    for (int64_t item0 = static_cast<int64_t>(blockIdx.x) * ITEMS_PER_CTA; item0 < nitems;
         item0 += static_cast<int64_t>(gridDim.x) * ITEMS_PER_CTA) {
        const int64_t item = item0 + slot;
        const bool live = item < nitems;
        const int64_t beg = live ? ptr[item] : 0, end = live ? ptr[item + 1] : 0;
        float acc[RB][CB];
#pragma unroll
        for (int p = 0; p < RB; ++p)
#pragma unroll
            for (int q = 0; q < CB; ++q) acc[p][q] = 0.0f;
        float bacc = 0.0f;
        if (live) gram_accumulate<K>(idx, val, beg, end, WPI, sub, Y, stage, rstage, acc, bacc, lane);
        // deterministic reduction of the WPI partial Grams: sub 0 writes, others add in order
        for (int s = 0; s < WPI; ++s) {
            if (sub == s && live) {
#pragma unroll
                for (int p = 0; p < RB; ++p)
#pragma unroll
                    for (int q = 0; q < CB; ++q) {
                        float* g = G + (bi * RB + p) * GS + bj * CB + q;
                        *g = s == 0 ? acc[p][q] : *g + acc[p][q];
                    }
                if (lane < K) rhs_all[slot][s][lane] = bacc;
            }
            if (WPI > 1) __syncthreads();
            else __syncwarp();
        }
        if (sub == 0 && live) {
            float b = 0.0f;
            if (lane < K)
                for (int s = 0; s < WPI; ++s) b += rhs_all[slot][s][lane];
            const int64_t cnt = end - beg;
            if (MODE == 1) {  // write Gram + rhs for the cross-rank allreduce
                float* out = Gout + item * (K * K + K);
                for (int e = lane; e < K * K; e += 32) out[e] = G[(e / K) * GS + (e % K)];
                if (lane < K) out[K * K + lane] = b;
            } else if (cnt == 0) {
                if (lane < K) X[item * K + lane] = 0.0f;
            } else {
                const float x = chol_solve_warp<K>(G, colb, b, lambda * static_cast<float>(cnt), lane);
                if (lane < K) X[item * K + lane] = x;
            }
        }
        if (WPI > 1) __syncthreads();
        else __syncwarp();
    }
}

// Solve from a (possibly allreduced) Gram + rhs buffer; cnt per item from ptr.
template <int K>
__global__ void __launch_bounds__(256) als_solve_from_gram_kernel(int64_t nitems, const int64_t* __restrict__ counts,
                                                                  const float* __restrict__ Gin, float* __restrict__ X,
                                                                  float lambda) {
    constexpr int GS = GramShape<K>::GS;
    __shared__ float gram_all[8][K * GS];
    __shared__ float colb_all[8][K];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t item = static_cast<int64_t>(blockIdx.x) * 8 + warp; item < nitems;
         item += static_cast<int64_t>(gridDim.x) * 8) {
        const float* in = Gin + item * (K * K + K);
        float* G = gram_all[warp];
        for (int e = lane; e < K * K; e += 32) G[(e / K) * GS + (e % K)] = in[e];
        const float b = lane < K ? in[K * K + lane] : 0.0f;
        __syncwarp();
        const int64_t cnt = counts[item];
        if (cnt == 0) {
            if (lane < K) X[item * K + lane] = 0.0f;
        } else {
            const float x = chol_solve_warp<K>(G, colb_all[warp], b, lambda * static_cast<float>(cnt), lane);
            if (lane < K) X[item * K + lane] = x;
        }
        __syncwarp();
    }
}

// V[j][0] = 1, V[j][f>0] = 0.01*(2u-1) (ocgo_als_init_value)
__global__ void als_init_kernel(int64_t n, int k, uint64_t seed, float* V) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= n * k) return;
    const int64_t j = e / k;
    const int f = static_cast<int>(e - j * k);
    double v = 1.0;
    if (f != 0) {
        const uint64_t h = splitmix64(seed ^ splitmix64(static_cast<uint64_t>(j * k + f)));
        const double u = static_cast<double>(h >> 11) * 0x1.0p-53;
        v = dmul(0.01, dsub(dmul(2.0, u), 1.0));
    }
    V[e] = static_cast<float>(v);
}

// CSR row ids (expand row_ptr), used to build the CSC mirror
__global__ void expand_rows_kernel(int64_t m, const int64_t* __restrict__ ptr, int32_t* __restrict__ rowid) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp; i < m; i += nw)
        for (int64_t q = ptr[i] + lane; q < ptr[i + 1]; q += 32) rowid[q] = static_cast<int32_t>(i);
}

__global__ void gather_csc_kernel(int64_t nnz, const int32_t* __restrict__ perm, const int32_t* __restrict__ rowid,
                                  const float* __restrict__ val, int32_t* __restrict__ crow, float* __restrict__ cval) {
    const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= nnz) return;
    const int32_t p = perm[q];
    crow[q] = rowid[p];
    cval[q] = val[p];
}

// col_ptr from the sorted column keys (first occurrence per column)
__global__ void col_ptr_kernel(int64_t nnz, int64_t n, const int32_t* __restrict__ skeys, int64_t* __restrict__ cptr) {
    const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q > nnz) return;
    const int32_t cur = q < nnz ? skeys[q] : static_cast<int32_t>(n);
    const int32_t prev = q > 0 ? skeys[q - 1] : -1;
    for (int32_t c = prev + 1; c <= cur; ++c) cptr[c] = q;
}

cudaError_t launch_als_init(int64_t n, int k, uint64_t seed, float* V, cudaStream_t s) {
    const int64_t tot = n * k;
    als_init_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, s>>>(n, k, seed, V);
    return cudaGetLastError();
}

template <int K>
static cudaError_t launch_gs(int64_t nitems, const int64_t* ptr, const int32_t* idx, const float* val,
                             const float* Y, float* X, float* Gout, float lambda, int wpi, int mode, int sm_count,
                             cudaStream_t s) {
    const int per_cta = 8 / wpi;
    int64_t blocks = (nitems + per_cta - 1) / per_cta;
    const int64_t cap = static_cast<int64_t>(sm_count) * 16;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    const unsigned b = static_cast<unsigned>(blocks);
    if (wpi == 1 && mode == 0) als_gram_solve_kernel<K, 1, 0><<<b, 256, 0, s>>>(nitems, ptr, idx, val, Y, X, Gout, lambda);
    else if (wpi == 8 && mode == 0) als_gram_solve_kernel<K, 8, 0><<<b, 256, 0, s>>>(nitems, ptr, idx, val, Y, X, Gout, lambda);
    else if (wpi == 1 && mode == 1) als_gram_solve_kernel<K, 1, 1><<<b, 256, 0, s>>>(nitems, ptr, idx, val, Y, X, Gout, lambda);
    else if (wpi == 8 && mode == 1) als_gram_solve_kernel<K, 8, 1><<<b, 256, 0, s>>>(nitems, ptr, idx, val, Y, X, Gout, lambda);
    else return cudaErrorInvalidValue;
    return cudaGetLastError();
}

cudaError_t launch_als_gram_solve(int k, int64_t nitems, const int64_t* ptr, const int32_t* idx, const float* val,
                                  const float* Y, float* X, float* Gout, float lambda, int wpi, int mode,
                                  int sm_count, cudaStream_t s) {
    switch (k) {
        case 8: return launch_gs<8>(nitems, ptr, idx, val, Y, X, Gout, lambda, wpi, mode, sm_count, s);
        case 16: return launch_gs<16>(nitems, ptr, idx, val, Y, X, Gout, lambda, wpi, mode, sm_count, s);
        case 32: return launch_gs<32>(nitems, ptr, idx, val, Y, X, Gout, lambda, wpi, mode, sm_count, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_als_solve_from_gram(int k, int64_t nitems, const int64_t* counts, const float* G, float* X,
                                       float lambda, int sm_count, cudaStream_t s) {
    int64_t blocks = (nitems + 7) / 8;
    if (blocks > sm_count * 16) blocks = sm_count * 16;
    if (blocks < 1) blocks = 1;
    const unsigned b = static_cast<unsigned>(blocks);
    switch (k) {
        case 8: als_solve_from_gram_kernel<8><<<b, 256, 0, s>>>(nitems, counts, G, X, lambda); break;
        case 16: als_solve_from_gram_kernel<16><<<b, 256, 0, s>>>(nitems, counts, G, X, lambda); break;
        case 32: als_solve_from_gram_kernel<32><<<b, 256, 0, s>>>(nitems, counts, G, X, lambda); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_expand_rows(int64_t m, const int64_t* ptr, int32_t* rowid, int sm_count, cudaStream_t s) {
    expand_rows_kernel<<<sm_count * 8, 256, 0, s>>>(m, ptr, rowid);
    return cudaGetLastError();
}

cudaError_t launch_gather_csc(int64_t nnz, const int32_t* perm, const int32_t* rowid, const float* val, int32_t* crow,
                              float* cval, cudaStream_t s) {
    if (nnz == 0) return cudaSuccess;
    gather_csc_kernel<<<static_cast<unsigned>((nnz + 255) / 256), 256, 0, s>>>(nnz, perm, rowid, val, crow, cval);
    return cudaGetLastError();
}

cudaError_t launch_col_ptr(int64_t nnz, int64_t n, const int32_t* skeys, int64_t* cptr, cudaStream_t s) {
    col_ptr_kernel<<<static_cast<unsigned>((nnz + 1 + 255) / 256), 256, 0, s>>>(nnz, n, skeys, cptr);
    return cudaGetLastError();
}

}  // namespace ocg
