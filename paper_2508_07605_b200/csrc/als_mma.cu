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
constexpr int GSZ = K * K + K + 1;
constexpr int kWarps = 8;
// per warp: double stage [2][32 rows][8 x 16 B] + packed r stage [2][32] u32
constexpr int kStageU4 = 2 * 32 * 8 + 16;

__device__ __forceinline__ void cp_async16_zfill(void* smem, const void* gmem, int bytes) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(bytes) : "memory");
}
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
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

__device__ __forceinline__ int min32(int64_t v) { return v < 32 ? static_cast<int>(v) : 32; }

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

__device__ __forceinline__ float rsqrt_ftz(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Gram / L rows in shared memory: 32 floats per row, 16-byte chunk cc of row a
// stored at chunk cc ^ (a & 7) so that 8 lanes reading 8 different rows' same
// chunk (LDS.128) hit 8 different bank groups; broadcasts of one row and
// column reads (lane = column) stay conflict-free.
__device__ __forceinline__ int gidx(int a, int b) { return a * K + ((((b >> 2) ^ a) & 7) << 2) + (b & 3); }

// Solve A x = b on one warp; lane l holds row l of A (SPD) in a[] and b_l.
// L overwrites a[] (lane l: row l of L, entries above the diagonal are
// garbage); Ls (32 x 32 swizzled, warp-private) mirrors L row-wise so row c
// can be broadcast.  The forward substitution L y = b rides along in the
// factorisation loop (t); the back substitution is column-oriented.
__device__ __forceinline__ float chol_solve_regs(float (&a)[K], float b, float* Ls, int lane) {
    float inv = 0.0f;
    float t = b;  // b_l - sum_{q<c} L[l][q] y_q; lanes < c hold y_l
#pragma unroll
    for (int c = 0; c < K; ++c) {
        float s0 = a[c], s1 = 0.0f, s2 = 0.0f, s3 = 0.0f;
#pragma unroll
        for (int q = 0; q + 4 <= c; q += 4) {
            const float4 w = *reinterpret_cast<const float4*>(Ls + gidx(c, q));
            s0 = fmaf(-a[q], w.x, s0);
            s1 = fmaf(-a[q + 1], w.y, s1);
            s2 = fmaf(-a[q + 2], w.z, s2);
            s3 = fmaf(-a[q + 3], w.w, s3);
        }
#pragma unroll
        for (int q = c & ~3; q < c; ++q) s0 = fmaf(-a[q], Ls[gidx(c, q)], s0);
        const float s = (s0 + s1) + (s2 + s3);
        const float piv = __shfl_sync(0xffffffffu, s, c);
        const float tc = __shfl_sync(0xffffffffu, t, c);
        const float r = rsqrt_ftz(piv);
        a[c] = s * r;  // L[l][c] (lane c: the diagonal)
        Ls[gidx(lane, c)] = a[c];
        inv = lane == c ? r : inv;
        const float yc = tc * r;  // y_c
        t = lane == c ? yc : (lane > c ? fmaf(-a[c], yc, t) : t);
        __syncwarp();
    }
    // L^T x = y (lane l holds y_l in t)
    float y = t;
#pragma unroll
    for (int c = K - 1; c >= 0; --c) {
        const float lc = Ls[gidx(c, lane)];  // L[c][l]
        const float xc = __shfl_sync(0xffffffffu, y * inv, c);
        if (lane == c) y = xc;
        else if (lane < c) y = fmaf(-lc, xc, y);
    }
    return y;
}

// MODE 0: fused solve of single-segment items, partial records for the rest.
// MODE 1: partial records for every segment (multi-GPU column side).
//
// Gathers: 8 lanes copy one 128-byte factor row with 16-byte cp.async (rows
// past the chunk are zero-filled); 16-byte chunk c of stage row o sits at
// chunk c ^ (o & 7), which makes the fragment loads conflict-free.  (One TMA
// bulk copy per row was measured 1.4x slower: per-operation cost of the
// bulk-copy unit at 128 B.)  Observed values arrive pre-packed as (fp16 hi,
// fp16 lo) of val * 2^ev (als_pack_vals_kernel).
// Pipelining: a segment's first chunk is gathered into stage buffer 1 while
// the previous segment is in its Cholesky (which only uses buffer 0), its
// metadata two segments ahead, and every chunk's (index, value) pair one chunk
// ahead of its gather.
template <int MODE>
__global__ void __launch_bounds__(kWarps * 32, 3) als_mma_gram32_kernel(
    const int32_t* __restrict__ total_segs, const int32_t* __restrict__ seg_order, const int32_t* __restrict__ seg_item,
    const int64_t* __restrict__ seg_beg, const int32_t* __restrict__ nseg_of, const int32_t* __restrict__ first,
    const int32_t* __restrict__ pfirst, const int64_t* __restrict__ ptr, int64_t nitems, const int32_t* __restrict__ idx,
    const uint32_t* __restrict__ valh, const uint4* __restrict__ Yh, const unsigned* __restrict__ ymax,
    const unsigned* __restrict__ vmax, float* __restrict__ X, float* __restrict__ partial, float lambda) {
    extern __shared__ __align__(16) uint4 dyn4[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    uint4* stage = dyn4 + warp * kStageU4;  // [2][32][8] uint4
    uint32_t* rstage = reinterpret_cast<uint32_t*>(stage + 2 * 32 * 8);  // [2][32] packed r
    float* Gs = reinterpret_cast<float*>(stage);  // epilogue: Gram / L (inside buffer 0)
    const int ey = als_scale_exp(*ymax), ev = als_scale_exp(*vmax);
    const float s2 = ldexpf(1.0f, 2 * ey), inv_s2 = ldexpf(1.0f, -2 * ey), inv_sv = ldexpf(1.0f, -(ey + ev));
    const int32_t nsegs = *total_segs;
    const int64_t nnz = ptr[nitems];
    const int32_t stride = gridDim.x * kWarps;
    const uint32_t rsel = g == 0 ? 0x5410u : 0x7632u;  // rhs B column 0 = r_hi, column 1 = r_lo
    const uint32_t rmask = g < 2 ? 0xffffffffu : 0u;

    auto ldidx = [&](int64_t base, int64_t end, int& j, uint32_t& r) {
        j = 0;
        r = 0u;
        if (base + lane < end) {
            j = __ldg(idx + base + lane);
            r = __ldg(valh + base + lane);
        }
    };
    // gather a chunk of cnt rows (indices j, packed values r of lane = row) into buffer buf
    auto issue = [&](int buf, int cnt, int j, uint32_t r) {
        rstage[buf * 32 + lane] = lane < cnt ? r : 0u;
        uint4* st = stage + buf * 32 * 8;
        const int c16 = lane & 7, osub = lane >> 3;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int o = q * 4 + osub;
            const int jo = __shfl_sync(0xffffffffu, j, o);
            cp_async16_zfill(st + o * 8 + (c16 ^ (o & 7)), Yh + static_cast<int64_t>(o < cnt ? jo : 0) * 8 + c16,
                             o < cnt ? 16 : 0);
        }
        cp_async_commit();
    };

    // work index k -> segment id (seg_order: column side sorted by first row, so
    // concurrently running warps gather from one band of the factor matrix)
    auto seg_of = [&](int32_t k) { return seg_order ? seg_order[k] : k; };
    int32_t wk = blockIdx.x * kWarps + warp;
    if (wk >= nsegs) return;
    int32_t sg = seg_of(wk);
    int32_t item = seg_item[sg];
    int64_t beg = seg_beg[sg];
    int64_t end = min(beg + kSeg, ptr[item + 1]);
    {
        int j;
        uint32_t r;
        ldidx(beg, end, j, r);
        issue(1, min32(end - beg), j, r);
    }
    int32_t nwk = wk + stride;
    int32_t nsg = nwk < nsegs ? seg_of(nwk) : 0;
    int32_t nitem = nwk < nsegs ? seg_item[nsg] : 0;
    int64_t nbeg = nwk < nsegs ? seg_beg[nsg] : 0;
    while (true) {
        // per-segment scalars + the next segment's end / first indices (in flight over this segment)
        const int32_t nseg_item = nseg_of[item];
        const int64_t item_beg = ptr[item];
        const int64_t item_end = ptr[item + 1];
        int64_t slot = 0;
        if (MODE == 1) slot = sg;
        else if (nseg_item > 1) slot = pfirst[item] + (sg - first[item]);
        int64_t nend = 0;
        int j0n = 0;
        uint32_t r0n = 0u;
        if (nwk < nsegs) {
            nend = min(nbeg + kSeg, ptr[nitem + 1]);
            ldidx(nbeg, nnz, j0n, r0n);  // speculative: masked to the segment when issued
        }
        const int32_t nnwk = nwk + stride;
        const int32_t nnsg = nnwk < nsegs ? seg_of(nnwk) : 0;
        const int32_t nnitem = nnwk < nsegs ? seg_item[nnsg] : 0;
        const int64_t nnbeg = nnwk < nsegs ? seg_beg[nnsg] : 0;

        float acc[6][4], racc[2][4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
#pragma unroll
            for (int q = 0; q < 6; ++q) acc[q][e] = 0.0f;
            racc[0][e] = racc[1][e] = 0.0f;
        }
        int jn = 0;
        uint32_t rn = 0u;
        if (beg + 32 < end) ldidx(beg + 32, end, jn, rn);
        int buf = 1;
        for (int64_t base = beg; base < end; base += 32) {
            const int cnt = min32(end - base);
            if (base + 32 < end) {
                issue(buf ^ 1, min32(end - base - 32), jn, rn);
                if (base + 64 < end) ldidx(base + 64, end, jn, rn);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncwarp();
            const uint4* st = stage + buf * 32 * 8;
            const uint32_t* rs = rstage + buf * 32;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (h == 1 && cnt <= 16) break;
                const int o0 = h * 16 + 2 * t;  // rows o0, o0+1, o0+8, o0+9 have (row & 7) = (2t, 2t+1, 2t, 2t+1)
                const uint4 q0 = st[o0 * 8 + (g ^ (2 * t))], q1 = st[(o0 + 1) * 8 + (g ^ (2 * t + 1))];
                const uint4 q2 = st[(o0 + 8) * 8 + (g ^ (2 * t))], q3 = st[(o0 + 9) * 8 + (g ^ (2 * t + 1))];
                // B fragments of n-tile j (factor dim 4g+j): {b0, b1} for hi (h) and lo (l)
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
                // rhs B fragment from the packed (hi, lo) values of observations o0, o0+1 / o0+8, o0+9
                const uint2 ra = *reinterpret_cast<const uint2*>(rs + o0);
                const uint2 rb = *reinterpret_cast<const uint2*>(rs + o0 + 8);
                const uint32_t rb0 = prmt(ra.x, ra.y, rsel) & rmask, rb1 = prmt(rb.x, rb.y, rsel) & rmask;
                // G lower tiles (i,j) = (0,0) (0,1) (1,0) (1,1) (1,2) (1,3): H^T H + H^T L + L^T H
                mma16816(acc[0], bh0[0], bh0[1], bh1[0], bh1[1], bh0[0], bh1[0]);
                mma16816(acc[0], bh0[0], bh0[1], bh1[0], bh1[1], bl0[0], bl1[0]);
                mma16816(acc[0], bl0[0], bl0[1], bl1[0], bl1[1], bh0[0], bh1[0]);
                mma16816(acc[1], bh0[0], bh0[1], bh1[0], bh1[1], bh0[1], bh1[1]);
                mma16816(acc[1], bh0[0], bh0[1], bh1[0], bh1[1], bl0[1], bl1[1]);
                mma16816(acc[1], bl0[0], bl0[1], bl1[0], bl1[1], bh0[1], bh1[1]);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    mma16816(acc[2 + j], bh0[2], bh0[3], bh1[2], bh1[3], bh0[j], bh1[j]);
                    mma16816(acc[2 + j], bh0[2], bh0[3], bh1[2], bh1[3], bl0[j], bl1[j]);
                    mma16816(acc[2 + j], bl0[2], bl0[3], bl1[2], bl1[3], bh0[j], bh1[j]);
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
        // ---- epilogue: lower tiles -> shared (natural dims, mirrored), rows into registers.
        // Element e of tile (i,j) is MMA (M, N) = (16i + g + 8(e>>1), 8j + 2t + (e&1)).
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            const int i = q < 2 ? 0 : 1, j = q < 2 ? q : q - 2;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int M = 16 * i + g + 8 * (e >> 1), N = 8 * j + 2 * t + (e & 1);
                if (M >= N) {
                    const int a = pi_dim(M), b = pi_dim(N);
                    Gs[gidx(a, b)] = acc[q][e];
                    Gs[gidx(b, a)] = acc[q][e];
                }
            }
        }
        float* rhs = reinterpret_cast<float*>(rstage);  // buffer 0's r slots (drained)
        if (t == 0) {
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                rhs[4 * g + 2 * i] = racc[i][0] + racc[i][1];
                rhs[4 * g + 2 * i + 1] = racc[i][2] + racc[i][3];
            }
        }
        const bool single = MODE == 0 && nseg_item == 1;
        const int64_t cnt_item = item_end - item_beg;
        __syncwarp();
        if (single && cnt_item > 0) Gs[gidx(lane, lane)] += lambda * static_cast<float>(cnt_item) * s2;
        __syncwarp();
        float row[K];
#pragma unroll
        for (int c = 0; c < K; c += 4) {
            const float4 gv = *reinterpret_cast<const float4*>(Gs + gidx(lane, c));
            row[c] = gv.x * inv_s2;
            row[c + 1] = gv.y * inv_s2;
            row[c + 2] = gv.z * inv_s2;
            row[c + 3] = gv.w * inv_s2;
        }
        const float b = rhs[lane] * inv_sv;
        __syncwarp();  // Gs / rhs dead: buffer 1 takes the next segment's first chunk, buffer 0 the L mirror
        if (nwk < nsegs) issue(1, min32(nend - nbeg), j0n, r0n);
        if (single) {
            const float x = cnt_item > 0 ? chol_solve_regs(row, b, Gs, lane) : 0.0f;
            X[static_cast<int64_t>(item) * K + lane] = x;
        } else {
            float* out = partial + slot * GSZ;
#pragma unroll
            for (int c = 0; c < K; ++c) out[lane * K + c] = row[c];  // records are only 4-byte aligned
            out[K * K + lane] = b;
        }
        __syncwarp();
        if (nwk >= nsegs) break;
        wk = nwk;
        sg = nsg;
        item = nitem;
        beg = nbeg;
        end = nend;
        nwk = nnwk;
        nsg = nnsg;
        nitem = nnitem;
        nbeg = nnbeg;
    }
}

// observed values -> packed (fp16 hi, fp16 lo) of val * 2^ev
__global__ void als_pack_vals_kernel(int64_t n, const float* __restrict__ val, const unsigned* __restrict__ vmax,
                                     uint32_t* __restrict__ out) {
    const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const float y = val[q] * ldexpf(1.0f, als_scale_exp(*vmax));
    const __half h = __float2half_rn(y);
    out[q] = pack_h2(h, __float2half_rn(y - __half2float(h)));
}

cudaError_t launch_als_pack_vals(int64_t n, const float* val, const unsigned* vmax, uint32_t* out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    als_pack_vals_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(n, val, vmax, out);
    return cudaGetLastError();
}

// Multi-segment items: sum the partial records in segment order
// (deterministic), then one warp solves with the register Cholesky.
__global__ void __launch_bounds__(256) als_reduce_solve32_kernel(const int32_t* __restrict__ list,
                                                                 const int32_t* __restrict__ list_count,
                                                                 const int64_t* __restrict__ ptr,
                                                                 const int32_t* __restrict__ nseg_of,
                                                                 const int32_t* __restrict__ pfirst,
                                                                 const float* __restrict__ partial,
                                                                 float* __restrict__ X, float lambda) {
    __shared__ __align__(16) float Gs[K * K];
    __shared__ float rhs[K];
    const int tid = threadIdx.x, lane = tid & 31;
    const int32_t nwork = *list_count;
    for (int32_t w = blockIdx.x; w < nwork; w += gridDim.x) {
        const int32_t item = list[w];
        const int32_t ns = nseg_of[item];
        const float* base = partial + static_cast<int64_t>(pfirst[item]) * GSZ;
        for (int e = tid; e < K * K + K; e += 256) {
            float s = 0.0f;
            for (int32_t q = 0; q < ns; ++q) s += base[static_cast<int64_t>(q) * GSZ + e];
            if (e < K * K) Gs[gidx(e / K, e % K)] = s;
            else rhs[e - K * K] = s;
        }
        __syncthreads();
        if (tid < 32) {
            const int64_t cnt = ptr[item + 1] - ptr[item];
            if (cnt > 0) Gs[gidx(lane, lane)] += lambda * static_cast<float>(cnt);
            __syncwarp();
            float row[K];
#pragma unroll
            for (int c = 0; c < K; c += 4) {
                const float4 gv = *reinterpret_cast<const float4*>(Gs + gidx(lane, c));
                row[c] = gv.x;
                row[c + 1] = gv.y;
                row[c + 2] = gv.z;
                row[c + 3] = gv.w;
            }
            const float b = rhs[lane];
            __syncwarp();
            X[static_cast<int64_t>(item) * K + lane] = cnt > 0 ? chol_solve_regs(row, b, Gs, lane) : 0.0f;
        }
        __syncthreads();
    }
}

cudaError_t launch_als_reduce_solve32(const AlsHalf& h, int sm_count, cudaStream_t s) {
    const int64_t cap = static_cast<int64_t>(sm_count) * 8;
    const unsigned blocks = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(h.nitems, cap)));
    als_reduce_solve32_kernel<<<blocks, 256, 0, s>>>(h.multi_list, h.multi_count, h.ptr, h.nseg, h.pfirst, h.partial,
                                                     h.X, h.lambda);
    return cudaGetLastError();
}

size_t als_mma_smem_bytes() { return sizeof(uint4) * kWarps * kStageU4; }

cudaError_t launch_als_mma_gram(const AlsHalf& h, int mode, int sm_count, cudaStream_t s) {
    const size_t smem = als_mma_smem_bytes();
    int64_t blocks = (h.max_segs + kWarps - 1) / kWarps;
    const int64_t cap = static_cast<int64_t>(sm_count) * 3;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    if (mode == 0) {
        cudaFuncSetAttribute(als_mma_gram32_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        als_mma_gram32_kernel<0><<<static_cast<unsigned>(blocks), kWarps * 32, smem, s>>>(
            h.total_segs, h.seg_order, h.seg_item, h.seg_beg, h.nseg, h.first, h.pfirst, h.ptr, h.nitems, h.idx, h.valh, h.Yh,
            h.ymax, h.vmax,
            h.X, h.partial, h.lambda);
    } else {
        cudaFuncSetAttribute(als_mma_gram32_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        als_mma_gram32_kernel<1><<<static_cast<unsigned>(blocks), kWarps * 32, smem, s>>>(
            h.total_segs, h.seg_order, h.seg_item, h.seg_beg, h.nseg, h.first, h.pfirst, h.ptr, h.nitems, h.idx, h.valh, h.Yh,
            h.ymax, h.vmax,
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
