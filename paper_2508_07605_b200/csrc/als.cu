// ALS completion kernels for ranks 8 and 16 (SIMT; ranks 32/64 run on the
// tensor cores, als_mma.cu), the segment tables both paths share, and the
// CSC-build helpers.
//
// No reference counterpart (the reference's CF is NCF only): the
// semantics are defined by oracle/ocg_oracle.c (ocgo_als_fit) — weighted-
// lambda ALS, u_i = (sum_j v_j v_j^T + lambda n_i I)^-1 sum_j r_ij v_j.
//
// Work unit = SEGMENT: at most kSeg consecutive observations of one ITEM (a
// row for the row half-sweep, a column for the column half-sweep).  Segments
// make the work uniform: C2's plan columns hold ~1M observations and its dense
// rows 4096, against ~80 for a typical row.
//
// als_seg_gram_kernel: one warp per segment.  The warp streams its
// observations 32 at a time: (index, value) pairs are read coalesced, the 32
// gathered factor rows (K floats) are copied global->shared
// with cp.async into a double-buffered stage (the next chunk's gathers are in
// flight while the current chunk is accumulated), and every lane accumulates
// a (K/8) x (K/4) block of the K x K Gram in registers (conflict-free 16-byte
// LDS inside one staged row).  A single-segment item is solved right there
// (fused K3+K4); otherwise the partial Gram + rhs goes to a slot in a global
// buffer and als_reduce_solve_kernel sums the item's partials in segment order
// (deterministic) and solves.  The solve is a compact left-looking Cholesky on
// the Gram in shared memory (lane l owns row l) + forward/back substitution.
// MODE 1 writes the reduced Gram + rhs + count instead of solving
// (multi-GPU: allreduced over ranks, then als_solve_from_gram_kernel).
#include <cuda_runtime.h>

#include <algorithm>

#include "als.h"
#include "ocg_common.cuh"

namespace ocg {

namespace {

template <int K>
struct GramShape {
    static constexpr int GS = K + 4;           // Gram row stride (floats): 16-byte rows
    static constexpr int TS = K;  // staged-row stride (floats)
    static constexpr int GSZ = K * K + K + 1;  // global Gram record: K*K, rhs K, count
};

__device__ __forceinline__ void cp_async16(float* smem, const float* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Solve (G + diag_add I) x = b on one warp.  G: K x GS shared (full
// symmetric); lane l < K holds b_l; returns x_l.  G's lower triangle is
// overwritten with L.  Left-looking: column c needs only finished columns,
// so the code stays compact (no fully unrolled K x K update).  The diagonal
// pivot is broadcast with a shuffle and every lane scales by rsqrt(pivot), so
// a column costs one shuffle + one warp barrier and no division; lane l keeps
// 1/L[l][l] for the substitutions.
template <int K>
__device__ __noinline__ float chol_solve_warp(float* G, float b, float diag_add, int lane) {
    constexpr int GS = GramShape<K>::GS;
    float* Gl = G + (lane < K ? lane : K - 1) * GS;  // lanes >= K read a valid row, results unused
    if (lane < K) Gl[lane] += diag_add;
    __syncwarp();
    float inv_diag = 1.0f;
    for (int c = 0; c < K; ++c) {
        const float* Gc = G + c * GS;
        // four independent partial sums: no serial FFMA dependency chain
        float s0 = Gl[c], s1 = 0.0f, s2 = 0.0f, s3 = 0.0f;
        int q = 0;
        for (; q + 4 <= c; q += 4) {
            const float4 a = *reinterpret_cast<const float4*>(Gl + q);
            const float4 w = *reinterpret_cast<const float4*>(Gc + q);
            s0 = fmaf(-a.x, w.x, s0);
            s1 = fmaf(-a.y, w.y, s1);
            s2 = fmaf(-a.z, w.z, s2);
            s3 = fmaf(-a.w, w.w, s3);
        }
        for (; q < c; ++q) s0 = fmaf(-Gl[q], Gc[q], s0);
        const float s = (s0 + s1) + (s2 + s3);
        const float piv = __shfl_sync(0xffffffffu, s, c);  // L[c][c]^2
        const float r = rsqrtf(piv);
        if (lane == c) inv_diag = r;
        if (lane >= c && lane < K) Gl[c] = s * r;  // lane c: sqrt(piv); below: L[l][c]
        __syncwarp();
    }
    // L y = b
    float y = b;
    for (int c = 0; c < K; ++c) {
        if (lane == c) y *= inv_diag;
        const float yc = __shfl_sync(0xffffffffu, y, c);
        if (lane > c && lane < K) y = fmaf(-Gl[c], yc, y);
    }
    // L^T x = y
    for (int c = K - 1; c >= 0; --c) {
        if (lane == c) y *= inv_diag;
        const float xc = __shfl_sync(0xffffffffu, y, c);
        if (lane < c) y = fmaf(-G[c * GS + lane], xc, y);
    }
    return y;
}

template <int N>
__device__ __forceinline__ void load_vec(float (&dst)[N], const float* src) {
    if constexpr (N % 4 == 0) {
#pragma unroll
        for (int q = 0; q < N; q += 4) {
            const float4 v = *reinterpret_cast<const float4*>(src + q);
            dst[q] = v.x;
            dst[q + 1] = v.y;
            dst[q + 2] = v.z;
            dst[q + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int q = 0; q < N; ++q) dst[q] = src[q];
    }
}

}  // namespace

// Segment table of one CSR-like side: item i with cnt observations owns
// nseg = max(1, ceil(cnt / kSeg)) consecutive segments from seg_first[i]
// (exclusive prefix sum of nseg, computed with cub on the host side).
// nmulti[i] = nseg[i] if the item needs partial Grams (nseg > 1), else 0; its
// exclusive prefix sum pfirst[] places an item's partials contiguously.
// Items with nseg > 1 are also appended (in any order) to multi_list /
// *multi_count (zeroed by the caller) so the reduce pass visits only them.
__global__ void seg_count_kernel(int64_t nitems, const int64_t* __restrict__ ptr, int32_t* __restrict__ nseg,
                                 int32_t* __restrict__ nmulti, int force_partials, int32_t* __restrict__ multi_list,
                                 int32_t* __restrict__ multi_count) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nitems) return;
    const int64_t cnt = ptr[i + 1] - ptr[i];
    const int32_t ns = cnt == 0 ? 1 : static_cast<int32_t>((cnt + kSeg - 1) / kSeg);
    nseg[i] = ns;
    nmulti[i] = (ns > 1 || force_partials) ? ns : 0;
    if (ns > 1 && multi_list) multi_list[atomicAdd(multi_count, 1)] = static_cast<int32_t>(i);
}

// column side: segment sort key = row of its first observation (the L2 band
// its factor gathers touch); padding slots sort last
__global__ void seg_key_kernel(int32_t max_segs, const int32_t* __restrict__ total, const int64_t* __restrict__ seg_beg,
                               const int32_t* __restrict__ idx, int32_t* __restrict__ key, int32_t* __restrict__ id) {
    const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= max_segs) return;
    key[s] = s < *total ? idx[seg_beg[s]] : 0x7fffffff;
    id[s] = s;
}

__global__ void seg_fill_kernel(int64_t nitems, const int64_t* __restrict__ ptr, const int32_t* __restrict__ nseg,
                                const int32_t* __restrict__ first, int32_t* __restrict__ seg_item,
                                int64_t* __restrict__ seg_beg, int32_t* __restrict__ total) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nitems) return;
    const int32_t f = first[i];
    if (i == nitems - 1) *total = f + nseg[i];
    for (int32_t s = 0; s < nseg[i]; ++s) {
        seg_item[f + s] = static_cast<int32_t>(i);
        seg_beg[f + s] = ptr[i] + static_cast<int64_t>(s) * kSeg;
    }
}

// ---- Gram accumulators ------------------------------------------------------
// Generic<K>: lane (bi, bj) owns a (K/8) x (K/4) block of the full Gram.
template <int K>
struct GramGeneric {
    static constexpr int RB = K / 8, CB = K / 4;
    float acc[RB][CB];
    float bacc;
    __device__ __forceinline__ void init() {
#pragma unroll
        for (int p = 0; p < RB; ++p)
#pragma unroll
            for (int q = 0; q < CB; ++q) acc[p][q] = 0.0f;
        bacc = 0.0f;
    }
    __device__ __forceinline__ void chunk(const float* st, const float* rs, int cnt, int lane) {
        constexpr int TS = GramShape<K>::TS;
        const int bi = lane >> 2, bj = lane & 3;
        for (int o = 0; o < cnt; ++o) {
            const float* row = st + o * TS;
            float xv[RB], yv[CB];
            load_vec(xv, row + bi * RB);
            load_vec(yv, row + bj * CB);
#pragma unroll
            for (int p = 0; p < RB; ++p)
#pragma unroll
                for (int q = 0; q < CB; ++q) acc[p][q] = fmaf(xv[p], yv[q], acc[p][q]);
            if (lane < K) bacc = fmaf(rs[o], row[lane], bacc);
        }
    }
    // full K x K into dst (row stride ld) + rhs (lane < K) into rhs_out
    __device__ __forceinline__ void store(float* dst, int ld, float* rhs_out, int lane) {
        const int bi = lane >> 2, bj = lane & 3;
#pragma unroll
        for (int p = 0; p < RB; ++p)
#pragma unroll
            for (int q = 0; q < CB; ++q) dst[(bi * RB + p) * ld + bj * CB + q] = acc[p][q];
        if (rhs_out && lane < K) rhs_out[lane] = bacc;
    }
};

template <int K>
struct GramPolicy {
    using type = GramGeneric<K>;
};

// MODE 0: fused solve of single-segment items, partials for the rest.
// MODE 1: partials for every segment (multi-GPU column side).
template <int K, int MODE>
__global__ void __launch_bounds__(256, 3) als_seg_gram_kernel(const int32_t* __restrict__ total_segs,
                                                           const int32_t* __restrict__ seg_item,
                                                           const int64_t* __restrict__ seg_beg,
                                                           const int32_t* __restrict__ nseg_of,
                                                           const int32_t* __restrict__ first,
                                                           const int32_t* __restrict__ pfirst,
                                                           const int64_t* __restrict__ ptr,
                                                           const int32_t* __restrict__ idx,
                                                           const float* __restrict__ val,
                                                           const float* __restrict__ Y, float* __restrict__ X,
                                                           float* __restrict__ partial, float lambda) {
    constexpr int GS = GramShape<K>::GS, TS = GramShape<K>::TS;
    constexpr int GSZ = GramShape<K>::GSZ;
    constexpr int CPR = K / 4;     // 16-byte chunks per factor row
    constexpr int OPI = 32 / CPR;  // observations gathered per cp.async instruction
    static_assert(K * GS <= 2 * 32 * TS, "Gram aliases the double stage");
    extern __shared__ __align__(16) float dyn[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* stage = dyn + warp * (2 * 32 * TS + 64);  // [2][32][TS] + rstage[2][32]
    float* rstage = stage + 2 * 32 * TS;
    const int c16 = lane % CPR, osub = lane / CPR;
    const int32_t nsegs = *total_segs;
    typename GramPolicy<K>::type gram;
    for (int32_t sg = blockIdx.x * 8 + warp; sg < nsegs; sg += gridDim.x * 8) {
        const int32_t item = seg_item[sg];
        const int64_t beg = seg_beg[sg];
        const int64_t iend = ptr[item + 1];
        const int64_t end = beg + kSeg < iend ? beg + kSeg : iend;
        gram.init();
        // chunk pipeline: the gathers of chunk t+1 are issued before chunk t is accumulated
        auto issue = [&](int64_t base, int buf) {
            const int cnt = static_cast<int>(end - base < 32 ? end - base : 32);
            int j = 0;
            float r = 0.0f;
            if (lane < cnt) {
                j = __ldg(idx + base + lane);
                r = __ldg(val + base + lane);
            }
            rstage[buf * 32 + lane] = r;
            float* st = stage + buf * 32 * TS;
#pragma unroll
            for (int t = 0; t < 32 / OPI; ++t) {
                const int o = t * OPI + osub;
                const int jo = __shfl_sync(0xffffffffu, j, o);
                if (o < cnt) cp_async16(st + o * TS + 4 * c16, Y + static_cast<int64_t>(jo) * K + 4 * c16);
            }
            cp_async_commit();
        };
        int buf = 0;
        if (beg < end) issue(beg, 0);
        for (int64_t base = beg; base < end; base += 32) {
            const int cnt = static_cast<int>(end - base < 32 ? end - base : 32);
            if (base + 32 < end) {
                issue(base + 32, buf ^ 1);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncwarp();
            gram.chunk(stage + buf * 32 * TS, rstage + buf * 32, cnt, lane);
            __syncwarp();
            buf ^= 1;
        }
        const bool single = MODE == 0 && nseg_of[item] == 1;
        if (single) {
            // Gram -> shared (aliases the drained stage), solve, write the factor
            float* G = stage;
            float* rhs = rstage;  // K <= 32 floats
            gram.store(G, GS, rhs, lane);
            __syncwarp();
            const int64_t cnt = iend - ptr[item];
            const float b = lane < K ? rhs[lane] : 0.0f;
            if (cnt == 0) {
                if (lane < K) X[static_cast<int64_t>(item) * K + lane] = 0.0f;
            } else {
                const float x = chol_solve_warp<K>(G, b, lambda * static_cast<float>(cnt), lane);
                if (lane < K) X[static_cast<int64_t>(item) * K + lane] = x;
            }
            __syncwarp();
        } else {
            // MODE 1 keeps every segment's partial (slot = segment index); MODE 0
            // only multi-segment items' (compact slots from pfirst)
            const int64_t slot = MODE == 1 ? sg : pfirst[item] + (sg - first[item]);
            float* out = partial + slot * GSZ;
            gram.store(out, K, out + K * K, lane);
        }
    }
}

// Sum an item's segment partials in segment order; MODE 0 solves, MODE 1
// writes the reduced record (Gram, rhs, count) to Gout[item].
// MODE 0 visits only the listed (multi-segment) items when list != nullptr.
template <int K, int MODE>
__global__ void __launch_bounds__(256) als_reduce_solve_kernel(int64_t nitems, const int32_t* __restrict__ list,
                                                               const int32_t* __restrict__ list_count,
                                                               const int64_t* __restrict__ ptr,
                                                               const int32_t* __restrict__ nseg_of,
                                                               const int32_t* __restrict__ first,
                                                               const float* __restrict__ partial,
                                                               float* __restrict__ X, float* __restrict__ Gout,
                                                               float lambda) {
    constexpr int GS = GramShape<K>::GS, GSZ = GramShape<K>::GSZ;
    __shared__ __align__(16) float G[K * GS];
    __shared__ float rhs[K];
    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t nwork = list ? static_cast<int64_t>(*list_count) : nitems;
    for (int64_t w = blockIdx.x; w < nwork; w += gridDim.x) {
        const int64_t item = list ? static_cast<int64_t>(list[w]) : w;
        const int32_t ns = nseg_of[item];
        if (MODE == 0 && ns == 1) continue;  // solved by the segment kernel
        const float* base = partial + static_cast<int64_t>(first[item]) * GSZ;  // first = pfirst here
        for (int e = tid; e < K * K + K; e += 256) {
            float s = 0.0f;
            for (int32_t q = 0; q < ns; ++q) s += base[static_cast<int64_t>(q) * GSZ + e];
            if (e < K * K) G[(e / K) * GS + (e % K)] = s;
            else rhs[e - K * K] = s;
        }
        __syncthreads();
        const int64_t cnt = ptr[item + 1] - ptr[item];
        if (MODE == 1) {
            float* out = Gout + item * GSZ;
            for (int e = tid; e < K * K; e += 256) out[e] = G[(e / K) * GS + (e % K)];
            if (tid < K) out[K * K + tid] = rhs[tid];
            if (tid == 0) out[K * K + K] = static_cast<float>(cnt);
        } else if (tid < 32) {
            const float x = chol_solve_warp<K>(G, lane < K ? rhs[lane] : 0.0f, lambda * static_cast<float>(cnt), lane);
            if (lane < K) X[item * K + lane] = x;
        }
        __syncthreads();
    }
}

// Solve from a (possibly allreduced) Gram record buffer (count in the record).
template <int K>
__global__ void __launch_bounds__(256) als_solve_from_gram_kernel(int64_t nitems, const float* __restrict__ Gin,
                                                                  float* __restrict__ X, float lambda) {
    constexpr int GS = GramShape<K>::GS, GSZ = GramShape<K>::GSZ;
    __shared__ __align__(16) float gram_all[8][K * GS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t item = static_cast<int64_t>(blockIdx.x) * 8 + warp; item < nitems;
         item += static_cast<int64_t>(gridDim.x) * 8) {
        const float* in = Gin + item * GSZ;
        float* G = gram_all[warp];
        for (int e = lane; e < K * K; e += 32) G[(e / K) * GS + (e % K)] = in[e];
        const float b = lane < K ? in[K * K + lane] : 0.0f;
        const float cnt = in[K * K + K];
        __syncwarp();
        if (cnt == 0.0f) {
            if (lane < K) X[item * K + lane] = 0.0f;
        } else {
            const float x = chol_solve_warp<K>(G, b, lambda * cnt, lane);
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

// (row << 32 | value bits) per CSR entry, the payload of the column sort
__global__ void expand_pairs_kernel(int64_t m, const int64_t* __restrict__ ptr, const uint32_t* __restrict__ vbits,
                                    uint64_t* __restrict__ pairs) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp; i < m; i += nw)
        for (int64_t q = ptr[i] + lane; q < ptr[i + 1]; q += 32)
            pairs[q] = (static_cast<uint64_t>(i) << 32) | vbits[q];
}

__global__ void split_pairs_kernel(int64_t nnz, const uint64_t* __restrict__ pairs, int32_t* __restrict__ crow,
                                   uint32_t* __restrict__ cval) {
    const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= nnz) return;
    const uint64_t p = pairs[q];
    crow[q] = static_cast<int32_t>(p >> 32);
    cval[q] = static_cast<uint32_t>(p);
}

// col_ptr from the sorted column keys (first occurrence per column)
__global__ void col_ptr_kernel(int64_t nnz, int64_t n, const int32_t* __restrict__ skeys, int64_t* __restrict__ cptr) {
    const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q > nnz) return;
    const int32_t cur = q < nnz ? skeys[q] : static_cast<int32_t>(n);
    const int32_t prev = q > 0 ? skeys[q - 1] : -1;
    for (int32_t c = prev + 1; c <= cur; ++c) cptr[c] = q;
}

// packed 32-bit CSC keys (m <= 2^rb, n <= 2^(32-rb)): key = col << rb | row, built from
// the CSR (warp per row); sorted on the column bits only (stable: rows stay ascending),
// the value words ride along as the 32-bit payload
__global__ void expand_keys_kernel(int64_t m, int rb, const int64_t* __restrict__ ptr,
                                   const int32_t* __restrict__ col, uint32_t* __restrict__ keys) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp; i < m; i += nw)
        for (int64_t q = ptr[i] + lane; q < ptr[i + 1]; q += 32)
            keys[q] = (static_cast<uint32_t>(col[q]) << rb) | static_cast<uint32_t>(i);
}
// sorted keys -> crow (row bits) and col_ptr (first occurrence of each column)
__global__ void split_keys_kernel(int64_t nnz, int64_t n, int rb, const uint32_t* __restrict__ skeys,
                                  int32_t* __restrict__ crow, int64_t* __restrict__ cptr) {
    const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q > nnz) return;
    const uint32_t rmask = (rb >= 32) ? 0xffffffffu : ((1u << rb) - 1u);
    const int64_t cur = q < nnz ? static_cast<int64_t>(skeys[q] >> rb) : n;
    const int64_t prev = q > 0 ? static_cast<int64_t>(skeys[q - 1] >> rb) : -1;
    if (q < nnz) crow[q] = static_cast<int32_t>(skeys[q] & rmask);
    for (int64_t c = prev + 1; c <= cur; ++c) cptr[c] = q;
}

cudaError_t launch_expand_keys(int64_t m, int rb, const int64_t* ptr, const int32_t* col, uint32_t* keys,
                               int sm_count, cudaStream_t s) {
    expand_keys_kernel<<<sm_count * 8, 256, 0, s>>>(m, rb, ptr, col, keys);
    return cudaGetLastError();
}
cudaError_t launch_split_keys(int64_t nnz, int64_t n, int rb, const uint32_t* skeys, int32_t* crow, int64_t* cptr,
                              cudaStream_t s) {
    split_keys_kernel<<<static_cast<unsigned>((nnz + 1 + 255) / 256), 256, 0, s>>>(nnz, n, rb, skeys, crow, cptr);
    return cudaGetLastError();
}

cudaError_t launch_als_init(int64_t n, int k, uint64_t seed, float* V, cudaStream_t s) {
    const int64_t tot = n * k;
    als_init_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, s>>>(n, k, seed, V);
    return cudaGetLastError();
}

cudaError_t launch_seg_count(int64_t nitems, const int64_t* ptr, int32_t* nseg, int32_t* nmulti, int force_partials,
                             int32_t* multi_list, int32_t* multi_count, cudaStream_t s) {
    if (multi_count) {
        const cudaError_t e = cudaMemsetAsync(multi_count, 0, sizeof(int32_t), s);
        if (e != cudaSuccess) return e;
    }
    seg_count_kernel<<<static_cast<unsigned>((nitems + 255) / 256), 256, 0, s>>>(nitems, ptr, nseg, nmulti,
                                                                                  force_partials, multi_list,
                                                                                  multi_count);
    return cudaGetLastError();
}

cudaError_t launch_seg_key(int32_t max_segs, const int32_t* total, const int64_t* seg_beg, const int32_t* idx,
                           int32_t* key, int32_t* id, cudaStream_t s) {
    seg_key_kernel<<<static_cast<unsigned>((max_segs + 255) / 256), 256, 0, s>>>(max_segs, total, seg_beg, idx, key, id);
    return cudaGetLastError();
}

cudaError_t launch_seg_fill(int64_t nitems, const int64_t* ptr, const int32_t* nseg, const int32_t* first,
                            int32_t* seg_item, int64_t* seg_beg, int32_t* total, cudaStream_t s) {
    seg_fill_kernel<<<static_cast<unsigned>((nitems + 255) / 256), 256, 0, s>>>(nitems, ptr, nseg, first, seg_item,
                                                                                 seg_beg, total);
    return cudaGetLastError();
}

// ranks 32/64 (tensor-core path): packed lower-triangle record of als_mma.cu
size_t als_gram_record_floats(int k) {
    return (k == 32 || k == 64) ? als_record_floats_mma(k) : static_cast<size_t>(k) * k + k + 1;
}

template <int K>
static cudaError_t launch_half_k(const AlsHalf& h, int mode, int sm_count, cudaStream_t s) {
    constexpr int TS = GramShape<K>::TS;
    const size_t smem = sizeof(float) * 8 * (2 * 32 * TS + 64);
    int64_t blocks = (h.max_segs + 7) / 8;
    const int64_t cap = static_cast<int64_t>(sm_count) * 32;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    const unsigned rblocks = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(h.nitems, sm_count * 8)));
    if (mode == 0) {
        cudaFuncSetAttribute(als_seg_gram_kernel<K, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
        als_seg_gram_kernel<K, 0><<<static_cast<unsigned>(blocks), 256, smem, s>>>(
            h.total_segs, h.seg_item, h.seg_beg, h.nseg, h.first, h.pfirst, h.ptr, h.idx, h.val, h.Y, h.X,
            h.partial, h.lambda);
        als_reduce_solve_kernel<K, 0><<<rblocks, 256, 0, s>>>(h.nitems, h.multi_list, h.multi_count, h.ptr, h.nseg,
                                                                 h.pfirst, h.partial, h.X, nullptr, h.lambda);
    } else {
        cudaFuncSetAttribute(als_seg_gram_kernel<K, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
        als_seg_gram_kernel<K, 1><<<static_cast<unsigned>(blocks), 256, smem, s>>>(
            h.total_segs, h.seg_item, h.seg_beg, h.nseg, h.first, h.pfirst, h.ptr, h.idx, h.val, h.Y, h.X,
            h.partial, h.lambda);
        als_reduce_solve_kernel<K, 1><<<rblocks, 256, 0, s>>>(h.nitems, nullptr, nullptr, h.ptr, h.nseg, h.first,
                                                                 h.partial, nullptr, h.gram_out, h.lambda);
    }
    return cudaGetLastError();
}

cudaError_t launch_als_half(int k, const AlsHalf& h, int mode, int sm_count, cudaStream_t s) {
    if ((k == 32 || k == 64) && h.Yh) return launch_als_mma_half(k, h, mode, sm_count, s);
    switch (k) {
        case 8: return launch_half_k<8>(h, mode, sm_count, s);
        case 16: return launch_half_k<16>(h, mode, sm_count, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_als_solve_from_gram(int k, int64_t nitems, const float* G, float* X, float lambda, int sm_count,
                                       cudaStream_t s) {
    if (k == 32 || k == 64) return launch_als_solve_records(k, nitems, G, X, lambda, sm_count, s);
    int64_t blocks = (nitems + 7) / 8;
    if (blocks > sm_count * 16) blocks = sm_count * 16;
    if (blocks < 1) blocks = 1;
    const unsigned b = static_cast<unsigned>(blocks);
    switch (k) {
        case 8: als_solve_from_gram_kernel<8><<<b, 256, 0, s>>>(nitems, G, X, lambda); break;
        case 16: als_solve_from_gram_kernel<16><<<b, 256, 0, s>>>(nitems, G, X, lambda); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_expand_pairs(int64_t m, const int64_t* ptr, const uint32_t* vbits, uint64_t* pairs, int sm_count,
                                cudaStream_t s) {
    expand_pairs_kernel<<<sm_count * 8, 256, 0, s>>>(m, ptr, vbits, pairs);
    return cudaGetLastError();
}

cudaError_t launch_split_pairs(int64_t nnz, const uint64_t* pairs, int32_t* crow, uint32_t* cval, cudaStream_t s) {
    if (nnz == 0) return cudaSuccess;
    split_pairs_kernel<<<static_cast<unsigned>((nnz + 255) / 256), 256, 0, s>>>(nnz, pairs, crow, cval);
    return cudaGetLastError();
}

cudaError_t launch_col_ptr(int64_t nnz, int64_t n, const int32_t* skeys, int64_t* cptr, cudaStream_t s) {
    col_ptr_kernel<<<static_cast<unsigned>((nnz + 1 + 255) / 256), 256, 0, s>>>(nnz, n, skeys, cptr);
    return cudaGetLastError();
}

}  // namespace ocg
