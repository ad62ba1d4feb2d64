// ALS K3 Gram accumulation on the tensor cores (rank 32) + register-resident
// Cholesky (K4), fused per segment.
//
// Semantics: oracle/ocg_oracle.c ocgo_als_fit (weighted-lambda ALS; no
// reference counterpart).  Same work decomposition as the
// SIMT kernel in als.cu (warp per <= kSeg-observation segment, single-segment
// items solved in place, multi-segment items reduced in segment order by
// als_reduce_solve_kernel), different arithmetic:
//
// * Factor rows are gathered as FP16 hi/lo pairs, written once per half-sweep
//   by als_pack_kernel: y*s = hi + lo (hi = fp16(y*s), lo = fp16(y*s - hi)),
//   s = 2^e a power-of-two scale from the factor matrix's max |y| (so y*s <=
//   2^14 and lo stays a normal fp16 for every entry that matters).  The packed
//   row is 8 x 16 B: chunk g = {hi[4g..4g+3], lo[4g..4g+3]}.
// * Gram = H^T H + H^T L + L^T H (the L^T L term is below 2^-22 relative) with
//   mma.sync m16n8k16 f16 -> f32.  A lane loads ONE 16-byte chunk g of four
//   observation rows and byte-permutes them into the B fragments of all four
//   n-tiles (MMA column 8j+g <-> factor dim 4g+j); the A fragments of the two
//   m-tiles are the same registers.  Per 16 observations: 6 MMAs for the
//   lower tiles of H^T H, 8 for S = H^T L (full; G = HH + S + S^T), 4 for the
//   rhs (B = [r_hi, r_lo, 0..]).  That replaces 18 FFMA/observation/lane.
// * Epilogue: fragments -> shared (natural dim order, mirrored), lane l builds
//   row l of G + lambda*n*I in registers, then a fully unrolled left-looking
//   Cholesky (row c of L broadcast from shared with LDS.128) with the forward
//   substitution folded into the factorisation loop, and a column-oriented
//   back substitution.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "als.h"
#include "ocg_common.cuh"

namespace ocg {

namespace {

constexpr int K = 32;
constexpr int RS = 9;      // staged packed row stride in 16-byte units (144 B: conflict-free fragment loads)
constexpr int SS = 36;     // shared Gram / S / L row stride in floats
constexpr int GSZ = K * K + K + 1;
constexpr int kWarps = 8;
// per warp: double stage [2][32][RS] uint4 + r stage [2][32] floats
constexpr int kStageU4 = 2 * 32 * RS + 16;
static_assert(2 * 32 * SS * 4 <= 2 * 32 * RS * 16, "Gram + S buffers alias the drained stage");

__device__ __forceinline__ void cp_async16_zfill(void* smem, const void* gmem, int bytes) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}

__device__ __forceinline__ uint32_t pack_h2(__half lo, __half hi) {
    return static_cast<uint32_t>(__half_as_ushort(lo)) | (static_cast<uint32_t>(__half_as_ushort(hi)) << 16);
}

// MMA index X in [0,32) <-> natural factor dim pi(X) = 4*(X%8) + X/8
__device__ __forceinline__ int pi_dim(int x) { return 4 * (x & 7) + (x >> 3); }

}  // namespace

// power-of-two scale with max|y| * s <= 2^14 (exponent clamped so s^2 and its
// inverse stay finite in FP32)
__device__ __forceinline__ int als_scale_exp(unsigned maxbits) {
    const float mx = __uint_as_float(maxbits);
    if (!(mx > 0.0f) || !isfinite(mx)) return 0;
    int e;
    frexpf(mx, &e);  // mx = f * 2^e, f in [0.5, 1)  ->  mx < 2^e
    int x = 14 - e;
    return x < -60 ? -60 : (x > 60 ? 60 : x);
}

__global__ void als_absmax_kernel(int64_t count, const float* __restrict__ x, unsigned* __restrict__ out) {
    float m = 0.0f;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        m = fmaxf(m, fabsf(x[i]));
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    __shared__ float wm[32];
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        m = threadIdx.x < (blockDim.x >> 5) ? wm[threadIdx.x] : 0.0f;
#pragma unroll
        for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (threadIdx.x == 0) atomicMax(out, __float_as_uint(m));  // non-negative floats order as unsigned
    }
}

// X (rows x 32 f32) -> packed hi/lo rows (8 x uint4 per row)
__global__ void als_pack_kernel(int64_t rows, const float* __restrict__ X, const unsigned* __restrict__ maxbits,
                                uint4* __restrict__ Xh) {
    const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;  // chunk id
    if (q >= rows * 8) return;
    const float s = ldexpf(1.0f, als_scale_exp(*maxbits));
    const float4 v = reinterpret_cast<const float4*>(X)[q];
    const float y[4] = {v.x * s, v.y * s, v.z * s, v.w * s};
    __half h[4], l[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        h[c] = __float2half_rn(y[c]);
        l[c] = __float2half_rn(y[c] - __half2float(h[c]));
    }
    Xh[q] = make_uint4(pack_h2(h[0], h[1]), pack_h2(h[2], h[3]), pack_h2(l[0], l[1]), pack_h2(l[2], l[3]));
}

// Solve A x = b on one warp; lane l holds row l of A (SPD) in a[] and b_l.
// L overwrites a[] (lane l: row l of L); Ls is a warp-private 32 x SS shared
// buffer that mirrors L row-wise so row c can be broadcast.
__device__ __forceinline__ float chol_solve_regs(float (&a)[K], float b, float* Ls, int lane) {
    float inv = 0.0f;
    float t = b;  // forward substitution residual: b_l - sum_{q<c} L[l][q] y_q
    float* Lrow = Ls + lane * SS;
#pragma unroll
    for (int c = 0; c < K; ++c) {
        const float* Lc = Ls + c * SS;
        float s0 = a[c], s1 = 0.0f, s2 = 0.0f, s3 = 0.0f;
#pragma unroll
        for (int q = 0; q + 4 <= c; q += 4) {
            const float4 w = *reinterpret_cast<const float4*>(Lc + q);
            s0 = fmaf(-a[q], w.x, s0);
            s1 = fmaf(-a[q + 1], w.y, s1);
            s2 = fmaf(-a[q + 2], w.z, s2);
            s3 = fmaf(-a[q + 3], w.w, s3);
        }
#pragma unroll
        for (int q = c & ~3; q < c; ++q) s0 = fmaf(-a[q], Lc[q], s0);
        const float s = (s0 + s1) + (s2 + s3);
        const float piv = __shfl_sync(0xffffffffu, s, c);
        const float tc = __shfl_sync(0xffffffffu, t, c);
        const float r = rsqrtf(piv);
        a[c] = s * r;  // L[l][c] (lane c: the diagonal)
        Lrow[c] = a[c];
        inv = lane == c ? r : inv;
        const float yc = tc * r;  // y_c
        t = lane == c ? yc : (lane > c ? fmaf(-a[c], yc, t) : t);
        __syncwarp();
    }
    // L^T x = y (lane l holds y_l in t)
    float y = t;
#pragma unroll
    for (int c = K - 1; c >= 0; --c) {
        const float xc = __shfl_sync(0xffffffffu, y * inv, c);
        if (lane == c) y = xc;
        else if (lane < c) y = fmaf(-Ls[c * SS + lane], xc, y);
    }
    return y;
}

// MODE 0: fused solve of single-segment items, partial records for the rest.
// MODE 1: partial records for every segment (multi-GPU column side).
template <int MODE>
__global__ void __launch_bounds__(256, 2) als_mma_gram32_kernel(
    const int32_t* __restrict__ total_segs, const int32_t* __restrict__ seg_item, const int64_t* __restrict__ seg_beg,
    const int32_t* __restrict__ nseg_of, const int32_t* __restrict__ first, const int32_t* __restrict__ pfirst,
    const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx, const float* __restrict__ val,
    const uint4* __restrict__ Yh, const unsigned* __restrict__ ymax, const unsigned* __restrict__ vmax,
    float* __restrict__ X, float* __restrict__ partial, float lambda) {
    extern __shared__ __align__(16) uint4 dyn4[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    uint4* stage = dyn4 + warp * kStageU4;
    float* rstage = reinterpret_cast<float*>(stage + 2 * 32 * RS);
    const int ey = als_scale_exp(*ymax), ev = als_scale_exp(*vmax);
    const float vsc = ldexpf(1.0f, ev);
    const float inv_s = ldexpf(1.0f, -ey), inv_sv = ldexpf(1.0f, -(ey + ev));
    const int32_t nsegs = *total_segs;
    for (int32_t sg = blockIdx.x * kWarps + warp; sg < nsegs; sg += gridDim.x * kWarps) {
        const int32_t item = seg_item[sg];
        const int64_t beg = seg_beg[sg];
        const int64_t iend = ptr[item + 1];
        const int64_t end = beg + kSeg < iend ? beg + kSeg : iend;
        float hh[6][4], sacc[8][4], racc[2][4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
#pragma unroll
            for (int q = 0; q < 6; ++q) hh[q][e] = 0.0f;
#pragma unroll
            for (int q = 0; q < 8; ++q) sacc[q][e] = 0.0f;
            racc[0][e] = racc[1][e] = 0.0f;
        }
        auto issue = [&](int64_t base, int buf) {
            const int cnt = static_cast<int>(end - base < 32 ? end - base : 32);
            int j = 0;
            float r = 0.0f;
            if (lane < cnt) {
                j = __ldg(idx + base + lane);
                r = __ldg(val + base + lane);
            }
            rstage[buf * 32 + lane] = r * vsc;
            uint4* st = stage + buf * 32 * RS;
            const int c16 = lane & 7, osub = lane >> 3;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int o = q * 4 + osub;
                const int jo = __shfl_sync(0xffffffffu, j, o);
                cp_async16_zfill(st + o * RS + c16, Yh + static_cast<int64_t>(jo) * 8 + c16, o < cnt ? 16 : 0);
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
            const uint4* st = stage + buf * 32 * RS;
            const float* rs = rstage + buf * 32;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (h == 1 && cnt <= 16) break;
                const int o0 = h * 16 + 2 * t;
                const uint4 q0 = st[o0 * RS + g], q1 = st[(o0 + 1) * RS + g];
                const uint4 q2 = st[(o0 + 8) * RS + g], q3 = st[(o0 + 9) * RS + g];
                // B fragments of n-tile j (factor dim 4g+j): [j] = {b0, b1}
                uint32_t bh0[4], bh1[4], bl0[4], bl1[4];
                bh0[0] = prmt(q0.x, q1.x, 0x5410);
                bh0[1] = prmt(q0.x, q1.x, 0x7632);
                bh0[2] = prmt(q0.y, q1.y, 0x5410);
                bh0[3] = prmt(q0.y, q1.y, 0x7632);
                bh1[0] = prmt(q2.x, q3.x, 0x5410);
                bh1[1] = prmt(q2.x, q3.x, 0x7632);
                bh1[2] = prmt(q2.y, q3.y, 0x5410);
                bh1[3] = prmt(q2.y, q3.y, 0x7632);
                bl0[0] = prmt(q0.z, q1.z, 0x5410);
                bl0[1] = prmt(q0.z, q1.z, 0x7632);
                bl0[2] = prmt(q0.w, q1.w, 0x5410);
                bl0[3] = prmt(q0.w, q1.w, 0x7632);
                bl1[0] = prmt(q2.z, q3.z, 0x5410);
                bl1[1] = prmt(q2.z, q3.z, 0x7632);
                bl1[2] = prmt(q2.w, q3.w, 0x5410);
                bl1[3] = prmt(q2.w, q3.w, 0x7632);
                // rhs B fragment: column 0 = r_hi, column 1 = r_lo
                const float2 ra = *reinterpret_cast<const float2*>(rs + o0);
                const float2 rb = *reinterpret_cast<const float2*>(rs + o0 + 8);
                const __half ha0 = __float2half_rn(ra.x), ha1 = __float2half_rn(ra.y);
                const __half hb0 = __float2half_rn(rb.x), hb1 = __float2half_rn(rb.y);
                uint32_t rb0 = 0u, rb1 = 0u;
                if (g == 0) {
                    rb0 = pack_h2(ha0, ha1);
                    rb1 = pack_h2(hb0, hb1);
                } else if (g == 1) {
                    rb0 = pack_h2(__float2half_rn(ra.x - __half2float(ha0)), __float2half_rn(ra.y - __half2float(ha1)));
                    rb1 = pack_h2(__float2half_rn(rb.x - __half2float(hb0)), __float2half_rn(rb.y - __half2float(hb1)));
                }
                // H^T H, lower tiles (i,j): (0,0) (0,1) (1,0) (1,1) (1,2) (1,3)
                mma16816(hh[0], bh0[0], bh0[1], bh1[0], bh1[1], bh0[0], bh1[0]);
                mma16816(hh[1], bh0[0], bh0[1], bh1[0], bh1[1], bh0[1], bh1[1]);
#pragma unroll
                for (int j = 0; j < 4; ++j) mma16816(hh[2 + j], bh0[2], bh0[3], bh1[2], bh1[3], bh0[j], bh1[j]);
                // S = H^T L, all tiles
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    mma16816(sacc[j], bh0[0], bh0[1], bh1[0], bh1[1], bl0[j], bl1[j]);
                    mma16816(sacc[4 + j], bh0[2], bh0[3], bh1[2], bh1[3], bl0[j], bl1[j]);
                }
                // rhs: (H + L)^T [r_hi r_lo]
                mma16816(racc[0], bh0[0], bh0[1], bh1[0], bh1[1], rb0, rb1);
                mma16816(racc[0], bl0[0], bl0[1], bl1[0], bl1[1], rb0, rb1);
                mma16816(racc[1], bh0[2], bh0[3], bh1[2], bh1[3], rb0, rb1);
                mma16816(racc[1], bl0[2], bl0[3], bl1[2], bl1[3], rb0, rb1);
            }
            __syncwarp();
            buf ^= 1;
        }
        // ---- epilogue: fragments -> shared (natural dims), rows into registers
        float* Gs = reinterpret_cast<float*>(stage);  // [32][SS]
        float* Ss = Gs + 32 * SS;                     // [32][SS]
        float* rhs = rstage;                          // [32] (drained)
        // HH lower tiles, mirrored: element e of tile (i,j) is MMA (M, N) =
        // (16i + g + 8(e>>1), 8j + 2t + (e&1)) -> natural (4g + 2i + (e>>1), 8t + 4(e&1) + j)
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            const int i = q < 2 ? 0 : 1, j = q < 2 ? q : q - 2;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int M = 16 * i + g + 8 * (e >> 1), N = 8 * j + 2 * t + (e & 1);
                if (M >= N) {
                    const int a = pi_dim(M), b = pi_dim(N);
                    Gs[a * SS + b] = hh[q][e];
                    Gs[b * SS + a] = hh[q][e];
                }
            }
        }
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int M = 16 * i + g + 8 * (e >> 1), N = 8 * j + 2 * t + (e & 1);
                    Ss[pi_dim(M) * SS + pi_dim(N)] = sacc[i * 4 + j][e];
                }
        if (t == 0) {
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                rhs[4 * g + 2 * i] = racc[i][0] + racc[i][1];
                rhs[4 * g + 2 * i + 1] = racc[i][2] + racc[i][3];
            }
        }
        __syncwarp();
        const bool single = MODE == 0 && nseg_of[item] == 1;
        const int64_t cnt_item = iend - ptr[item];
        float row[K];
        const float* Gl = Gs + lane * SS;
        const float* Sl = Ss + lane * SS;
#pragma unroll
        for (int c = 0; c < K; c += 4) {
            const float4 gv = *reinterpret_cast<const float4*>(Gl + c);
            const float4 sv = *reinterpret_cast<const float4*>(Sl + c);
            row[c] = gv.x + sv.x + Ss[c * SS + lane];
            row[c + 1] = gv.y + sv.y + Ss[(c + 1) * SS + lane];
            row[c + 2] = gv.z + sv.z + Ss[(c + 2) * SS + lane];
            row[c + 3] = gv.w + sv.w + Ss[(c + 3) * SS + lane];
        }
        const float inv_s2 = inv_s * inv_s;
#pragma unroll
        for (int c = 0; c < K; ++c) row[c] *= inv_s2;
        const float b = rhs[lane] * inv_sv;
        __syncwarp();  // Gs/Ss/rhs are dead from here; Gs becomes the L mirror
        if (single) {
            float x = 0.0f;
            if (cnt_item > 0) {
                const float diag = lambda * static_cast<float>(cnt_item);
#pragma unroll
                for (int c = 0; c < K; ++c)
                    if (c == lane) row[c] += diag;
                x = chol_solve_regs(row, b, Gs, lane);
            }
            X[static_cast<int64_t>(item) * K + lane] = x;
        } else {
            const int64_t slot = MODE == 1 ? sg : pfirst[item] + (sg - first[item]);
            float* out = partial + slot * GSZ;
#pragma unroll
            for (int c = 0; c < K; ++c) out[lane * K + c] = row[c];  // records are only 4-byte aligned
            out[K * K + lane] = b;
        }
        __syncwarp();
    }
}

size_t als_mma_smem_bytes() { return sizeof(uint4) * kWarps * kStageU4; }

cudaError_t launch_als_mma_gram(const AlsHalf& h, int mode, int sm_count, cudaStream_t s) {
    const size_t smem = als_mma_smem_bytes();
    int64_t blocks = (h.max_segs + kWarps - 1) / kWarps;
    const int64_t cap = static_cast<int64_t>(sm_count) * 2;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    if (mode == 0) {
        cudaFuncSetAttribute(als_mma_gram32_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        als_mma_gram32_kernel<0><<<static_cast<unsigned>(blocks), 256, smem, s>>>(
            h.total_segs, h.seg_item, h.seg_beg, h.nseg, h.first, h.pfirst, h.ptr, h.idx, h.val, h.Yh, h.ymax, h.vmax,
            h.X, h.partial, h.lambda);
    } else {
        cudaFuncSetAttribute(als_mma_gram32_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        als_mma_gram32_kernel<1><<<static_cast<unsigned>(blocks), 256, smem, s>>>(
            h.total_segs, h.seg_item, h.seg_beg, h.nseg, h.first, h.pfirst, h.ptr, h.idx, h.val, h.Yh, h.ymax, h.vmax,
            h.X, h.partial, h.lambda);
    }
    return cudaGetLastError();
}

// max |X| -> *maxbits (zeroed here), then X -> packed hi/lo rows
cudaError_t launch_als_pack(int64_t rows, const float* X, unsigned* maxbits, uint4* Xh, int sm_count, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(maxbits, 0, sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
    const int64_t cnt = rows * K;
    int64_t blocks = (cnt + 255) / 256;
    if (blocks > sm_count * 8) blocks = sm_count * 8;
    if (blocks < 1) blocks = 1;
    als_absmax_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(cnt, X, maxbits);
    als_pack_kernel<<<static_cast<unsigned>((rows * 8 + 255) / 256), 256, 0, s>>>(rows, X, maxbits, Xh);
    return cudaGetLastError();
}

cudaError_t launch_absmax(int64_t count, const float* x, unsigned* maxbits, int sm_count, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(maxbits, 0, sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
    int64_t blocks = (count + 255) / 256;
    if (blocks > sm_count * 8) blocks = sm_count * 8;
    if (blocks < 1) blocks = 1;
    als_absmax_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(count, x, maxbits);
    return cudaGetLastError();
}

}  // namespace ocg
