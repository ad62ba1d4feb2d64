// ALS half-sweep on B200 at ranks 32 and 64: K3 Gram accumulation on the
// tensor cores, K4 batched Cholesky.
//
// Semantics: oracle/ocg_oracle.c ocgo_als_fit (weighted-lambda ALS; no
// reference counterpart): x_i = (G_i + lambda n_i I)^-1 b_i,
// G_i = sum_j y_j y_j^T and b_i = sum_j r_ij y_j over item i's observations.
//
// K3 als_mma_gram_kernel<K>: warp per <= kSeg-observation segment.
// * Factor rows are gathered as FP16 hi/lo pairs written once per half-sweep
//   by als_pack_kernel: y*s = hi + lo (hi = fp16(y*s), lo = fp16(y*s - hi)),
//   s = 2^e from the factor matrix's max |y| (y*s <= 2^14, lo stays normal for
//   every entry that matters).  Packed row = [hi dims 0..K-1 | lo dims 0..K-1].
//   Observed values are packed the same way once per plan.
// * G = H^T H + H^T L + L^T H (L^T L is below 2^-22 relative) with mma.sync
//   m16n8k16 f16 -> f32 on the lower tiles of the KxK Gram.  The B fragments
//   come straight from the staged rows by ldmatrix.x4.trans; the A fragments of
//   the m-tiles are the same registers.  rhs: (H + L)^T [r_hi r_lo].  Rank 32:
//   22 MMAs per 16 observations, or 18 on the column side (SPLIT: H^T L on all
//   tiles, its transpose folded in the epilogue).
// * Output: one RECORD per segment (layout below), unscaled FP32, written from
//   the accumulator fragments through shared memory with 16-byte stores.
// Reduce (multi-segment items): records summed in segment order into the
// item's first slot (deterministic).
// K4: als_solve_rows_kernel<K> (register-resident rows, 4 / 16 lanes per
// system, paired FP32 FMAs); rank 64 als_solve_records_kernel (records staged
// in shared memory, 8 lanes per system).  Left-looking Cholesky with the rhs
// carried as an extra row (forward substitution folded in), then L^T x = y.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <utility>

#include "als.h"
#include "ocg_common.cuh"

namespace ocg {

namespace {

constexpr int kWarps = 8;

__device__ __forceinline__ void cp_async16_zfill(void* smem, const void* gmem, int bytes) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem) : "memory");
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

// compile-time loop: f(integral_constant<int, 0>) ... f(<N-1>) -- forces full unrolling where
// #pragma unroll gives up (rank 64), so register arrays stay register arrays
template <class F, int... J>
__device__ __forceinline__ void static_for_impl(F&& f, std::integer_sequence<int, J...>) {
    (f(std::integral_constant<int, J>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
    static_for_impl(f, std::make_integer_sequence<int, N>{});
}

}  // namespace

// ---- record layout (floats): padded lower triangle, row i at T(i) with its
// length rounded up to 4 (16-byte aligned rows), then rhs (K), count (1).
__host__ __device__ constexpr int tri_off(int i) { return 4 * ((i >> 2) + 1) * (2 * (i >> 2) + (i & 3)); }

// Per-rank constants of the tensor-core path (K = 32 or 64).
//  D   factor dims per lane group (= MMA n-tiles), MT m-tiles, NLT lower tiles
//  RU4 packed factor row in 16-byte units: [hi dims 0..K-1 | lo dims 0..K-1]
//  RS  stage row stride (16-byte units): conflict-free fragment loads, and at K=64 a
//      record fits one stage buffer
template <int K>
struct Cfg {
    static_assert(K == 32 || K == 64, "tensor-core ALS ranks");
    static constexpr int D = K / 8, MT = K / 16, NLT = MT * (MT + 1);
    static constexpr int RU4 = K / 4;
    static constexpr int RS = K == 32 ? 9 : 19;
    static constexpr int kStageU4 = 2 * 32 * RS + (8 * 32 * 2 * 4) / 16;  // + index/value ring [8][32] x 2
    static constexpr int kRhs = tri_off(K), kCnt = kRhs + K, kRec = (kCnt + 1 + 3) & ~3;
    static constexpr int kMinBlocks = K == 32 ? 2 : 1;
};
static_assert(Cfg<32>::kRec == 612 && Cfg<32>::kRhs == 576, "rank-32 record layout");
static_assert(Cfg<64>::kRec * 4 <= 32 * Cfg<64>::RS * 16, "rank-64 record fits a stage buffer");

// T(i + LPS) - T(i) for i = 4a + p (padded row lengths 4((r >> 2) + 1))
template <int LPS>
__device__ __forceinline__ int row_step(int a, int p) {
    return LPS == 4 ? 16 * a + 16 + 4 * p : 32 * a + 48 + 8 * p;
}


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

// X (rows x K f32) -> packed hi/lo rows: [hi dims 0..K-1 | lo dims 0..K-1] (Cfg<K>::RU4 x
// uint4 per row); thread = (row, group of 8 dims)
template <int K>
__global__ void als_pack_kernel(int64_t rows, const float* __restrict__ X, const unsigned* __restrict__ maxbits,
                                uint4* __restrict__ Xh) {
    constexpr int G = K / 8, RU4 = Cfg<K>::RU4;
    const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= rows * G) return;
    const int64_t r = q / G;
    const int c = static_cast<int>(q % G);
    const float s = ldexpf(1.0f, als_scale_exp(*maxbits));
    const float* x = X + r * K + 8 * c;
    uint32_t hw[4], lw[4];
#pragma unroll
    for (int e = 0; e < 8; e += 2) {
        const float y0 = x[e] * s, y1 = x[e + 1] * s;
        const __half h0 = __float2half_rn(y0), h1 = __float2half_rn(y1);
        hw[e / 2] = pack_h2(h0, h1);
        lw[e / 2] = pack_h2(__float2half_rn(y0 - __half2float(h0)), __float2half_rn(y1 - __half2float(h1)));
    }
    Xh[r * RU4 + c] = make_uint4(hw[0], hw[1], hw[2], hw[3]);
    Xh[r * RU4 + RU4 / 2 + c] = make_uint4(lw[0], lw[1], lw[2], lw[3]);
}

__device__ __forceinline__ void ldsm_x4_trans(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3,
                                              const void* smem_row) {
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(smem_row));
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(a));
}

__device__ __forceinline__ float rsqrt_ftz(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}


// K3.  One record per segment, slot = segment id (the reduce step decides
// what happens to it).
//
// Work: blocks of 32 consecutive work indices (segments; column side in
// seg_order, i.e. sorted by first row) handed out by an atomic counter; a warp
// walks its blocks chunk by chunk (chunk = <= 32 observations of one segment;
// an empty segment is one empty chunk).  Two cursors walk the same chunk
// sequence:
//  * the refill cursor, kAhead chunks ahead, copies each chunk's (index,
//    packed value) pairs into a kRC-slot ring in shared memory (4-byte
//    cp.async, no register round trip), crossing segment and block
//    boundaries freely, so no global-load latency is ever exposed at a
//    segment start;
//  * the consumer issues the factor-row gathers of chunk c+1 from the ring
//    (8 lanes per 128-byte row, 16-byte cp.async, zero-filled past the chunk;
//    stage rows padded to 144 B: conflict-free fragment loads, and the copy
//    addresses are immediate offsets), runs the MMAs of chunk c, and writes the segment's record
//    after its last chunk (assembled in the drained stage buffer, stored with
//    16-byte coalesced writes).
// (One TMA bulk copy per factor row was measured 1.4x slower than the cp.async
// gathers: per-operation cost of the bulk-copy unit at 128 B.)

constexpr int kRC = 8;     // ring slots (chunks)
constexpr int kAhead = 5;  // refill distance (chunks); < kRC - 1
// SPLIT (rank 32, column side: long segments, MMA-bound): H^T L accumulated apart
// on all tiles, 18 instead of 22 MMAs per 16 observations, at 56 more accumulator
// registers (12 warps per SM instead of 16; the row side's short segments want
// the occupancy and the cheaper epilogue)
template <int K, bool SPLIT = false>
__host__ __device__ constexpr int gram_warps() { return SPLIT ? 6 : kWarps; }

template <int K, bool SPLIT>
__global__ void __launch_bounds__(gram_warps<K, SPLIT>() * 32, Cfg<K>::kMinBlocks) als_mma_gram_kernel(
    const int32_t* __restrict__ total_segs, const int32_t* __restrict__ seg_order, const int32_t* __restrict__ seg_item,
    const int64_t* __restrict__ seg_beg, const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
    const uint32_t* __restrict__ valh, const uint4* __restrict__ Yh, const unsigned* __restrict__ ymax,
    const unsigned* __restrict__ vmax, float* __restrict__ rec, int32_t* __restrict__ blk_ctr,
    const int32_t* /*unused*/) {
    using C = Cfg<K>;
    constexpr int D = C::D, MT = C::MT, NLT = C::NLT, RU4 = C::RU4, RS = C::RS;
    constexpr int kRec = C::kRec, kRhs = C::kRhs, kCnt = C::kCnt;
    constexpr int W = gram_warps<K, SPLIT>();
    extern __shared__ __align__(16) uint4 dyn4[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    uint4* stage = dyn4 + warp * C::kStageU4;                               // [2][32][RS] uint4
    int32_t* ring_j = reinterpret_cast<int32_t*>(stage + 2 * 32 * RS);     // [kRC][32]
    uint32_t* ring_r = reinterpret_cast<uint32_t*>(ring_j + kRC * 32);     // [kRC][32]
    const int ey = als_scale_exp(*ymax), ev = als_scale_exp(*vmax);
    const float inv_s2 = ldexpf(1.0f, -2 * ey), inv_sv = ldexpf(1.0f, -(ey + ev));
    const int32_t nsegs = *total_segs;
    const int32_t nblk = (nsegs + 31) / 32;
    (void)W;
    const uint32_t rsel = g == 0 ? 0x5410u : 0x7632u;  // rhs B column 0 = r_hi, column 1 = r_lo
    const uint32_t rmask = g < 2 ? 0xffffffffu : 0u;

    auto grab = [&]() {
        int32_t b = 0;
        if (lane == 0) b = atomicAdd(blk_ctr, 1);
        return __shfl_sync(0xffffffffu, b, 0);
    };
    // lane i <- segment of work index 32 b + i, or b + i * nblk when the work
    // order is sorted by band (column side: the warps active at any moment then
    // gather from one band of the factor matrix); sg < 0: none
    auto load_meta = [&](int32_t b, int32_t& sg, int64_t& beg, int64_t& end) {
        const int32_t k = seg_order ? b + lane * nblk : b * 32 + lane;
        sg = -1;
        beg = end = 0;
        if (b < nblk && k < nsegs) {
            sg = seg_order ? seg_order[k] : k;
            const int32_t it = seg_item[sg];
            beg = seg_beg[sg];
            end = min(beg + kSeg, ptr[it + 1]);
        }
    };
    auto bcast64 = [&](int64_t v, int src) {
        return static_cast<int64_t>(__shfl_sync(0xffffffffu, static_cast<unsigned long long>(v), src));
    };

    // ---- refill cursor (producer of ring slots)
    int32_t rb = grab();
    if (rb >= nblk) return;
    int32_t r_sg;
    int64_t r_beg, r_end;
    load_meta(rb, r_sg, r_beg, r_end);
    // consumer block = the refill's first block
    int32_t cb = rb, c_sg = r_sg;
    int64_t c_beg = r_beg, c_end = r_end;
    int rk = 0;
    int64_t rpos = bcast64(r_beg, 0), r_e = bcast64(r_end, 0);  // refill segment: position, end
    bool rex = false;   // refill block exhausted
    bool rdone = false;
    int prod = 0;  // chunks produced
    auto refill = [&]() {
        if (rdone) return;
        if (rex) {
            if (rb != cb) return;  // the consumer still needs the pending block's metadata: wait
            rb = grab();
            load_meta(rb, r_sg, r_beg, r_end);
            rk = 0;
            if (rb >= nblk || __shfl_sync(0xffffffffu, r_sg, 0) < 0) {
                rdone = true;
                return;
            }
            rex = false;
            rpos = bcast64(r_beg, 0);
            r_e = bcast64(r_end, 0);
        }
        const int cnt = min32(r_e - rpos < 0 ? 0 : r_e - rpos);
        const int slot = (prod % kRC) * 32 + lane;
        if (lane < cnt) {
            cp_async4(ring_j + slot, idx + rpos + lane);
            cp_async4(ring_r + slot, valh + rpos + lane);
        } else {
            ring_j[slot] = 0;
            ring_r[slot] = 0u;
        }
        ++prod;
        rpos += 32;
        if (rpos >= r_e) {  // next segment (shuffles only at segment transitions)
            ++rk;
            rex = rk == 32 || __shfl_sync(0xffffffffu, r_sg, rk & 31) < 0;
            if (!rex) {
                rpos = bcast64(r_beg, rk);
                r_e = bcast64(r_end, rk);
            }
        }
    };

    // ---- consumer cursor: current chunk (ck, cpos, cend)
    int ck = 0;
    int64_t cpos = bcast64(c_beg, 0), cend = bcast64(c_end, 0);
    // gathers of a chunk (segment lane k of the consumer block, position pos) from ring slot cons
    // lane = 8 * rg + c16 copies 16-byte chunk c16 of rows 8 rg + q (q = 0..7): its 8 row
    // indices are two 16-byte ring loads (0 past the chunk: a valid address, zero-filled)
    auto gather = [&](int buf, int cons, int64_t pos, int64_t e) {
        const int cnt = min32(e - pos < 0 ? 0 : e - pos);
        const int c16 = lane & 7, rg = lane >> 3;
        uint4* st = stage + buf * 32 * RS + rg * 8 * RS + c16;
        const int4* rj = reinterpret_cast<const int4*>(ring_j + (cons % kRC) * 32 + rg * 8);
        const int4 j0 = rj[0], j1 = rj[1];
        const int jj[8] = {j0.x, j0.y, j0.z, j0.w, j1.x, j1.y, j1.z, j1.w};
        const uint4* src = Yh + c16;
        const int nv = cnt - rg * 8;  // rows of this lane group inside the chunk
#pragma unroll
        for (int q = 0; q < 8; ++q) {
#pragma unroll
            for (int h = 0; h < RU4 / 8; ++h)  // K=64: the lane's second 16-byte chunk of the row
                cp_async16_zfill(st + q * RS + 8 * h, src + static_cast<uint32_t>(jj[q]) * RU4 + 8 * h,
                                 q < nv ? 16 : 0);
        }
    };

    for (int i = 0; i < kAhead; ++i) {
        refill();
        cp_async_commit();
    }
    cp_async_wait<0>();
    __syncwarp();
    gather(0, 0, cpos, cend);
    cp_async_commit();

    // SPLIT: H^T L kept apart on all MT x D tiles (14 + 4 MMAs per 16 observations instead of
    // 18 + 4); rank 64 has no registers for it
    static_assert(!SPLIT || K == 32, "split H^T L: rank 32");
    constexpr bool kSplitHL = SPLIT;
    constexpr int NHL = kSplitHL ? MT * D : 1;
    float acc[NLT][4], racc[MT][4], hl[NHL][4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
#pragma unroll
        for (int q = 0; q < NLT; ++q) acc[q][e] = 0.0f;
#pragma unroll
        for (int q = 0; q < NHL; ++q) hl[q][e] = 0.0f;
#pragma unroll
        for (int q = 0; q < MT; ++q) racc[q][e] = 0.0f;
    }
    int buf = 0;
    for (int cons = 0;; ++cons) {
        const bool last_of_seg = cpos + 32 >= cend;
        // locate the next chunk (shuffles only at segment transitions)
        int nk = ck;
        int64_t npos = cpos + 32, nend = cend;
        bool nblock = false, finished = false;
        if (last_of_seg) {
            nk = ck + 1;
            if (nk == 32 || __shfl_sync(0xffffffffu, c_sg, nk & 31) < 0) {
                // a starved refill cursor (it paused on a short block) may not have
                // fetched the next block yet: let it, before deciding the warp is done
                while (rb == cb && !rdone) {
                    refill();
                    cp_async_commit();
                    cp_async_wait<0>();
                    __syncwarp();
                }
                // next block: the refill cursor holds its metadata (or the warp is done)
                if (rb == cb || rb >= nblk) finished = true;
                else nblock = true;
                nk = 0;
            }
            if (!finished) {
                npos = nblock ? bcast64(r_beg, 0) : bcast64(c_beg, nk);
                nend = nblock ? bcast64(r_end, 0) : bcast64(c_end, nk);
            }
        }
        if (!finished) gather(buf ^ 1, cons + 1, npos, nend);
        refill();
        cp_async_commit();
        cp_async_wait<1>();
        __syncwarp();
        const int cnt = min32(cend - cpos < 0 ? 0 : cend - cpos);
        const uint4* st = stage + buf * 32 * RS;
        const uint32_t* rs = ring_r + (cons % kRC) * 32;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (h * 16 >= cnt) break;
            const int o0 = h * 16 + 2 * t;
            // B fragments of n-tile j (factor dims 8j..8j+7): b0 = observations 2t, 2t+1, b1 =
            // 2t+8, 2t+9 (hi / lo) -- the transposing ldmatrix of the 8x8 blocks (8 observation rows
            // x 16 bytes) hands every lane exactly its pair; the A fragment of m-tile i is
            // {B0(2i), B0(2i+1), B1(2i), B1(2i+1)}.  Lane l addresses row (l & 7) of block l >> 3 =
            // (k-half (l>>3) & 1, n-tile j + (l >> 4)).
            uint32_t bh0[D], bh1[D], bl0[D], bl1[D];
            {
                const uint4* rowp = st + (h * 16 + 8 * ((lane >> 3) & 1) + (lane & 7)) * RS + (lane >> 4);
#pragma unroll
                for (int j = 0; j < D; j += 2) {
                    ldsm_x4_trans(bh0[j], bh1[j], bh0[j + 1], bh1[j + 1], rowp + j);
                    ldsm_x4_trans(bl0[j], bl1[j], bl0[j + 1], bl1[j + 1], rowp + RU4 / 2 + j);
                }
            }
            // rhs B fragment from the packed (hi, lo) values of observations o0, o0+1 / o0+8, o0+9
            // (ring entries past the chunk are 0)
            const uint2 ra = *reinterpret_cast<const uint2*>(rs + o0);
            const uint2 rb2 = *reinterpret_cast<const uint2*>(rs + o0 + 8);
            const uint32_t rb0 = prmt(ra.x, ra.y, rsel) & rmask, rb1 = prmt(rb2.x, rb2.y, rsel) & rmask;
            if constexpr (kSplitHL) {
                // H^T H on the lower tiles, H^T L on all tiles (L^T H = (H^T L)^T, folded in the epilogue)
#pragma unroll
                for (int i = 0; i < MT; ++i)
#pragma unroll
                    for (int j = 0; j < D; ++j) {
                        if (j <= 2 * i + 1)
                            mma16816(acc[i * (i + 1) + j], bh0[2 * i], bh0[2 * i + 1], bh1[2 * i], bh1[2 * i + 1],
                                     bh0[j], bh1[j]);
                        mma16816(hl[i * D + j], bh0[2 * i], bh0[2 * i + 1], bh1[2 * i], bh1[2 * i + 1], bl0[j],
                                 bl1[j]);
                    }
            } else {
                // G lower tiles (i, j <= 2i+1), tile index i(i+1)+j: H^T H + H^T L + L^T H
#pragma unroll
                for (int i = 0; i < MT; ++i)
#pragma unroll
                    for (int j = 0; j <= 2 * i + 1; ++j) {
                        float (&a)[4] = acc[i * (i + 1) + j];
                        mma16816(a, bh0[2 * i], bh0[2 * i + 1], bh1[2 * i], bh1[2 * i + 1], bh0[j], bh1[j]);
                        mma16816(a, bh0[2 * i], bh0[2 * i + 1], bh1[2 * i], bh1[2 * i + 1], bl0[j], bl1[j]);
                        mma16816(a, bl0[2 * i], bl0[2 * i + 1], bl1[2 * i], bl1[2 * i + 1], bh0[j], bh1[j]);
                    }
            }
            // rhs: (H + L)^T [r_hi r_lo]
#pragma unroll
            for (int i = 0; i < MT; ++i) {
                mma16816(racc[i], bh0[2 * i], bh0[2 * i + 1], bh1[2 * i], bh1[2 * i + 1], rb0, rb1);
                mma16816(racc[i], bl0[2 * i], bl0[2 * i + 1], bl1[2 * i], bl1[2 * i + 1], rb0, rb1);
            }
        }
        __syncwarp();
        if (last_of_seg) {
            // ---- record, assembled in the drained buffer, stored with 16-byte coalesced writes.
            // Element e of lower tile (i,j) is MMA (M, N) = (16i + g + 8(e>>1), 8j + 2t + (e&1)) = factor
            // dims (M, N); each unordered pair is owned by exactly one (M >= N) element.
            float* rs_ = reinterpret_cast<float*>(stage + buf * 32 * RS);
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int j = 0; j <= 2 * i + 1; ++j)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int M = 16 * i + g + 8 * (e >> 1), N = 8 * j + 2 * t + (e & 1);
                        float& v = acc[i * (i + 1) + j][e];
                        if (M >= N) {
                            rs_[tri_off(M) + N] = (kSplitHL ? v + hl[i * D + j][e] : v) * inv_s2;
                        }
                        v = 0.0f;
                    }
            if constexpr (kSplitHL) {  // + (H^T L)(N, M) at (M, N): element (M <= N) of H^T L -> (N, M)
                __syncwarp();
#pragma unroll
                for (int i = 0; i < MT; ++i)
#pragma unroll
                    for (int j = 0; j < D; ++j)
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int M = 16 * i + g + 8 * (e >> 1), N = 8 * j + 2 * t + (e & 1);
                            float& v = hl[i * D + j][e];
                            if (M <= N) rs_[tri_off(N) + M] += v * inv_s2;
                            v = 0.0f;
                        }
            }
            if (t == 0) {  // lane (g, 0) holds the rhs of dims 16i + g and 16i + g + 8
#pragma unroll
                for (int i = 0; i < MT; ++i) {
                    rs_[kRhs + 16 * i + g] = (racc[i][0] + racc[i][1]) * inv_sv;
                    rs_[kRhs + 16 * i + g + 8] = (racc[i][2] + racc[i][3]) * inv_sv;
                }
            }
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int e = 0; e < 4; ++e) racc[i][e] = 0.0f;
            const int32_t sg = __shfl_sync(0xffffffffu, c_sg, ck);
            const int64_t sbeg = bcast64(c_beg, ck);  // (outside the lane-0 branch: full-warp shuffle)
            if (lane == 0) rs_[kCnt] = static_cast<float>(cend - sbeg);
            __syncwarp();
            float4* out = reinterpret_cast<float4*>(rec + static_cast<int64_t>(sg) * kRec);
            const float4* src = reinterpret_cast<const float4*>(rs_);
#pragma unroll
            for (int c = lane; c < kRec / 4; c += 32) out[c] = src[c];  // padding slots: stale, never read
            __syncwarp();
        }
        if (finished) break;
        if (nblock) {
            cb = rb;
            c_sg = r_sg;
            c_beg = r_beg;
            c_end = r_end;
        }
        ck = nk;
        cpos = npos;
        cend = nend;
        buf ^= 1;
    }
    cp_async_wait<0>();
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

// Sum each multi-segment item's segment records, in two levels so that a very
// long item (e.g. the always-profiled baseline column: ~1000 segments at C2) is
// not one block's serial chain: level 1 sums each group of kRG consecutive
// records in order into the group's first slot (blocks (x, y) take items x mod
// gridDim.x and groups y mod gridDim.y); level 2 sums an item's group partials
// in order.  list == nullptr: every item, result to out[item] (multi-GPU Gram
// records); else the listed items, result to rec[first[item]] in place.  The
// order is fixed, so the result is deterministic.
constexpr int kRG = 16;
template <int K>
__device__ __forceinline__ float4 sum_records(const float4* src, int32_t n, int64_t stride4) {
    float4 s = src[0];
    int32_t q = 1;
    for (; q + 4 <= n; q += 4) {  // four loads in flight; the sum order stays q = 0, 1, 2, ...
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = src[static_cast<int64_t>(q + u) * stride4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            s.x += v[u].x;
            s.y += v[u].y;
            s.z += v[u].z;
            s.w += v[u].w;
        }
    }
    for (; q < n; ++q) {
        const float4 v = src[static_cast<int64_t>(q) * stride4];
        s.x += v.x;
        s.y += v.y;
        s.z += v.z;
        s.w += v.w;
    }
    return s;
}
template <int K>
__global__ void __launch_bounds__(160) als_reduce_groups_kernel(int64_t nitems, const int32_t* __restrict__ list,
                                                                const int32_t* __restrict__ list_count,
                                                                const int32_t* __restrict__ nseg_of,
                                                                const int32_t* __restrict__ first,
                                                                float* __restrict__ rec) {
    constexpr int kRec = Cfg<K>::kRec;
    const int64_t nwork = list ? static_cast<int64_t>(*list_count) : nitems;
    for (int64_t w = blockIdx.x; w < nwork; w += gridDim.x) {
        const int64_t item = list ? static_cast<int64_t>(list[w]) : w;
        const int32_t ns = nseg_of[item];
        if (ns < 2) continue;
        for (int32_t gq = blockIdx.y; gq * kRG < ns; gq += gridDim.y) {
            const int32_t n = min(kRG, ns - gq * kRG);
            if (n < 2) continue;
            float4* base = reinterpret_cast<float4*>(rec + (static_cast<int64_t>(first[item]) + gq * kRG) * kRec);
            for (int c = threadIdx.x; c < kRec / 4; c += blockDim.x) base[c] = sum_records<K>(base + c, n, kRec / 4);
        }
    }
}
template <int K>
__global__ void __launch_bounds__(160) als_reduce_records_kernel(int64_t nitems, const int32_t* __restrict__ list,
                                                                 const int32_t* __restrict__ list_count,
                                                                 const int32_t* __restrict__ nseg_of,
                                                                 const int32_t* __restrict__ first,
                                                                 float* __restrict__ rec, float* __restrict__ out) {
    constexpr int kRec = Cfg<K>::kRec;
    const int64_t nwork = list ? static_cast<int64_t>(*list_count) : nitems;
    for (int64_t w = blockIdx.x; w < nwork; w += gridDim.x) {
        const int64_t item = list ? static_cast<int64_t>(list[w]) : w;
        const int32_t ng = (nseg_of[item] + kRG - 1) / kRG;
        if (list && ng < 2) continue;  // in place: level 1 already left the sum in the first slot
        for (int c = threadIdx.x; c < kRec / 4; c += blockDim.x) {  // float4 chunk of the record
            const float4* src = reinterpret_cast<const float4*>(rec + static_cast<int64_t>(first[item]) * kRec) + c;
            const float4 s = sum_records<K>(src, ng, static_cast<int64_t>(kRG) * (kRec / 4));
            float4* dst = list ? reinterpret_cast<float4*>(rec + static_cast<int64_t>(first[item]) * kRec) + c
                               : reinterpret_cast<float4*>(out + item * kRec) + c;
            *dst = s;
        }
    }
}


// register-row K4: lanes per system (rank 32: 4 lanes x 8 rows, rank 64: 16 lanes x 4 rows)
template <int K>
__host__ __device__ constexpr int rows_lps() { return K == 32 ? 4 : 16; }

// element i of a row stored as column pairs (i compile-time after unrolling)
template <int N>
__device__ __forceinline__ float& el(float2 (&r)[N], int i) {
    return (i & 1) ? r[i >> 1].y : r[i >> 1].x;
}

// K4 at rank 32 with register-resident rows: lane (sys = lane & 7, par = lane >> 3)
// holds rows i = 4m + par (m = 0..7, row m = columns 0..4m+3) of system sys in
// registers, loaded straight from the record.  Left-looking: at column j the
// owner of row j (par == j & 3) publishes it through shared memory; every lane
// reads it once (float4, broadcast over the item's 4 lanes) and updates its rows
// m >= j/4 with register operands only -- 8 independent chains, no shared-memory
// operand per FMA.  The rhs is carried as row K by all four lanes (forward
// substitution folded in); the published rows plus 1/L[j][j]
// then serve the column-oriented back substitution L^T x = y.
template <int K>
__global__ void __launch_bounds__(32) als_solve_rows_kernel(int64_t nitems, const int32_t* __restrict__ first,
                                                            const float* __restrict__ rec, float* __restrict__ X,
                                                            float lambda, const int32_t* __restrict__ list,
                                                            const int32_t* __restrict__ list_count,
                                                            unsigned* __restrict__ xmax) {
    constexpr int kRec = Cfg<K>::kRec, kRhs = Cfg<K>::kRhs, kCnt = Cfg<K>::kCnt;
    constexpr int LPS = rows_lps<K>(), kSys = 32 / LPS, R = K / LPS;  // lanes per system, systems, rows per lane
    // rank 64: the rhs / solution is distributed (lane p keeps the column pairs p, p + LPS, ...;
    // row-K dot products reduced over the system's lanes by shuffles) -- 64 fewer registers
    constexpr bool DY = K == 64;
    constexpr int NP = DY ? K / 2 / LPS : K / 2;
    // per-system strides = 4 (mod 32) words: the 8 systems' 16-byte reads at one offset hit
    // 8 distinct bank groups
    constexpr int kTri = tri_off(K) + 4, kDiag = K + 1, kTail = kRec - kRhs;  // tail = rhs, count, pad
    static_assert(kTail % 4 == 0 && kTri % 32 == 4, "record tail / bank stride");
    __shared__ __align__(16) float srow[kSys * kTri];
    __shared__ float sdiag[kSys * kDiag];
    __shared__ __align__(16) float stail[kSys * kTail];
    const int lane = threadIdx.x, sys = lane % kSys, par = lane / kSys;
    float* S = srow + sys * kTri;
    float* Rd = sdiag + sys * kDiag;
    float* T = stail + sys * kTail;
    const int64_t nwork = list ? static_cast<int64_t>(*list_count) : nitems;
    const int64_t nbatch = (nwork + kSys - 1) / kSys;
    int64_t bt = blockIdx.x;
    if (bt >= nbatch) return;
    float2 L[R][K / 2];  // column pairs; row m = LPS m + par uses (m + 1) LPS columns
    bool live;
    int64_t item;
    auto fetch = [&](int64_t b) {  // batch b -> L registers, tail -> T (cp.async)
        const int64_t i0 = b * kSys;
        const int nb = static_cast<int>(nwork - i0 < kSys ? nwork - i0 : kSys);
        live = sys < nb;
        const int64_t w = i0 + (live ? sys : nb - 1);  // dead lanes redo the last system, unstored
        item = list ? static_cast<int64_t>(list[w]) : w;
        const int64_t slot = first ? static_cast<int64_t>(first[item]) : item;
        const float* Rp = rec + slot * kRec;
        static_for<R>([&](auto mc) {
            constexpr int m = decltype(mc)::value;
            // (rank 64: past a row's padded length the loads read the next rows -- entries
            // above the diagonal, never used; the last row ends at the rhs)
            const float4* src = reinterpret_cast<const float4*>(Rp + tri_off(LPS * m + par));
#pragma unroll
            for (int c = 0; c < (m + 1) * LPS / 4; ++c) {
                const float4 v = __ldg(src + c);
                L[m][2 * c] = make_float2(v.x, v.y);
                L[m][2 * c + 1] = make_float2(v.z, v.w);
            }
        });
        for (int c = par; c < kTail / 4; c += LPS) {
            const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(T + 4 * c));
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(Rp + kRhs + 4 * c) : "memory");
        }
        cp_async_commit();
    };
    float lmax = 0.0f;  // max |x| of the rows this lane stored (xmax: the next packing's scale)
    fetch(bt);
    for (;;) {
        cp_async_wait<0>();
        __syncwarp();
        float2 y[NP];
        if constexpr (DY) {
#pragma unroll
            for (int q = 0; q < NP; ++q) y[q] = *reinterpret_cast<const float2*>(T + 2 * (par + LPS * q));
        } else {
#pragma unroll
            for (int c = 0; c < K / 4; ++c) {
                const float4 v = *reinterpret_cast<const float4*>(T + 4 * c);
                y[2 * c] = make_float2(v.x, v.y);
                y[2 * c + 1] = make_float2(v.z, v.w);
            }
        }
        const float cnt = T[kCnt - kRhs];
        const float diag = lambda * cnt;
#pragma unroll
        for (int m = 0; m < R; ++m)
#pragma unroll
            for (int p = 0; p < LPS; ++p)
                if (par == p) el(L[m], LPS * m + p) += diag;
        static_for<K>([&](auto jc) {
            constexpr int j = decltype(jc)::value, mo = j / LPS;
            constexpr int tj = tri_off(j);
            if (par == j % LPS) {  // publish row j: columns < j final, column j = A_jj
#pragma unroll
                for (int c = 0; c <= j / 4; ++c)
                    *reinterpret_cast<float4*>(S + tj + 4 * c) =
                        make_float4(L[mo][2 * c].x, L[mo][2 * c].y, L[mo][2 * c + 1].x, L[mo][2 * c + 1].y);
            }
            __syncwarp();
            // rows m >= mo (rows <= j of block mo compute unused entries above the diagonal);
            // paired FP32 FMAs over column pairs (q, q+1), .x / .y the two partial sums.  Finished
            // entries are kept NEGATED (N = -L), so every update is a plain FMA:
            //   -L[i][j] / r = -A[i][j] + sum_q N[i][q] N[j][q],   A_jj - L_jj^2 = A_jj - sum N[j][q]^2,
            //   y_j / r = b_j + sum_q N[j][q] y_q
            float2 acc[R];
#pragma unroll
            for (int m = mo; m < R; ++m) acc[m] = make_float2(-el(L[m], j), 0.0f);
            float2 ss = make_float2(0.0f, 0.0f), yy = make_float2(DY ? 0.0f : el(y, j), 0.0f);
#pragma unroll
            for (int c = 0; 4 * c < j; ++c) {
                const float4 v = *reinterpret_cast<const float4*>(S + tj + 4 * c);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int p = 2 * c + h;  // column pair (2p, 2p+1)
                    const float2 nv = h ? make_float2(v.z, v.w) : make_float2(v.x, v.y);
                    if (2 * p + 1 < j) {
                        ss = __ffma2_rn(nv, nv, ss);
                        if constexpr (!DY) yy = __ffma2_rn(nv, y[p], yy);
#pragma unroll
                        for (int m = mo; m < R; ++m) acc[m] = __ffma2_rn(L[m][p], nv, acc[m]);
                    } else if (2 * p < j) {  // odd j: the single column j-1
                        ss.x = fmaf(nv.x, nv.x, ss.x);
                        if constexpr (!DY) yy.x = fmaf(nv.x, y[p].x, yy.x);
#pragma unroll
                        for (int m = mo; m < R; ++m) acc[m].x = fmaf(L[m][p].x, nv.x, acc[m].x);
                    }
                }
            }
            const float r = rsqrt_ftz(S[tj + j] - (ss.x + ss.y));
#pragma unroll
            for (int m = mo; m < R; ++m) el(L[m], j) = (acc[m].x + acc[m].y) * r;
            if constexpr (DY) {  // the lane's pairs' share of sum_q N[j][q] y_q, reduced over the system
                float tot = 0.0f;
#pragma unroll
                for (int q = 0; q < NP; ++q) {
                    const int pp = par + LPS * q;  // (entries past the row are masked, never multiplied)
                    const float2 w = *reinterpret_cast<const float2*>(S + tj + 2 * pp);
                    tot = fmaf(2 * pp < j ? w.x : 0.0f, y[q].x, tot);
                    tot = fmaf(2 * pp + 1 < j ? w.y : 0.0f, y[q].y, tot);
                }
#pragma unroll
                for (int o = kSys; o < 32; o <<= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
                constexpr int pj = j / 2;
                if (par == pj % LPS) {
                    float& yj = (j & 1) ? y[pj / LPS].y : y[pj / LPS].x;
                    yj = (yj + tot) * r;
                }
            } else {
                el(y, j) = (yy.x + yy.y) * r;
            }
            if (par == 0) Rd[j] = r;
        });
        __syncwarp();
        const bool cur_live = live;
        const int64_t cur_item = item;
        const int64_t nbt = bt + gridDim.x;
        // L^T x = y, column-oriented over the published rows, all lanes of the item
        if constexpr (DY) static_for<K>([&](auto qc) {  // x_q from its owner, then every lane's pairs
            constexpr int q = K - 1 - decltype(qc)::value, pq = q / 2;
            const float* Rq = S + tri_off(q);
            float& yo = (q & 1) ? y[pq / LPS].y : y[pq / LPS].x;
            const float xq = __shfl_sync(0xffffffffu, yo * Rd[q], (pq % LPS) * kSys + sys);
            if (par == pq % LPS) yo = xq;
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                const int pp = par + LPS * i;
                const float2 w = *reinterpret_cast<const float2*>(Rq + 2 * pp);
                y[i] = __ffma2_rn(make_float2(2 * pp < q ? w.x : 0.0f, 2 * pp + 1 < q ? w.y : 0.0f),
                                  make_float2(xq, xq), y[i]);
            }
        });
        else static_for<K>([&](auto qc) {
            constexpr int q = K - 1 - decltype(qc)::value;
            const float* Rq = S + tri_off(q);
            el(y, q) *= Rd[q];
            const float yq = el(y, q);
            const float2 yq2 = make_float2(yq, yq);
#pragma unroll
            for (int i = 0; i + 4 <= q; i += 4) {  // y_i -= L[q][i] x_q = y_i + N[q][i] x_q
                const float4 v = *reinterpret_cast<const float4*>(Rq + i);
                y[i / 2] = __ffma2_rn(make_float2(v.x, v.y), yq2, y[i / 2]);
                y[i / 2 + 1] = __ffma2_rn(make_float2(v.z, v.w), yq2, y[i / 2 + 1]);
            }
#pragma unroll
            for (int i = q & ~3; i < q; ++i) el(y, i) = fmaf(Rq[i], yq, el(y, i));
        });
        if (DY && cur_live) {
            const bool empty = cnt == 0.0f;  // item without observations: x = 0 (ocgo_als_fit)
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                *reinterpret_cast<float2*>(X + cur_item * K + 2 * (par + LPS * i)) =
                    empty ? make_float2(0.0f, 0.0f) : y[i];
                if (!empty) lmax = fmaxf(lmax, fmaxf(fabsf(y[i].x), fabsf(y[i].y)));
            }
        } else if (!DY && cur_live && par == 0) {
            float4* xo = reinterpret_cast<float4*>(X + cur_item * K);
            const bool empty = cnt == 0.0f;  // item without observations: x = 0 (ocgo_als_fit)
#pragma unroll
            for (int q = 0; q < K / 4; ++q)
                xo[q] = empty ? make_float4(0.0f, 0.0f, 0.0f, 0.0f)
                              : make_float4(y[2 * q].x, y[2 * q].y, y[2 * q + 1].x, y[2 * q + 1].y);
            if (!empty)
#pragma unroll
                for (int q = 0; q < K / 2; ++q) lmax = fmaxf(lmax, fmaxf(fabsf(y[q].x), fabsf(y[q].y)));
        }
        __syncwarp();
        if (nbt >= nbatch) break;
        fetch(nbt);
        bt = nbt;
    }
    if (xmax) {
#pragma unroll
        for (int o = 16; o; o >>= 1) lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
        if (lane == 0) atomicMax(xmax, __float_as_uint(lmax));  // non-negative floats order as unsigned
    }
}

template <int K>
static cudaError_t launch_solve_k(int64_t nitems, const int32_t* first, const float* rec, float* X, float lambda,
                                  int sm_count, cudaStream_t s, const int32_t* list = nullptr,
                                  const int32_t* list_count = nullptr, unsigned* xmax = nullptr) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, als_solve_rows_kernel<K>, 32, 0);
    constexpr int kSys = 32 / rows_lps<K>();
    int64_t blocks = (nitems + kSys - 1) / kSys;
    const int64_t cap = static_cast<int64_t>(sm_count) * std::max(per_sm, 1);
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    als_solve_rows_kernel<K><<<static_cast<unsigned>(blocks), 32, 0, s>>>(nitems, first, rec, X, lambda, list,
                                                                          list_count, xmax);
    return cudaGetLastError();
}

// one tensor-core half-sweep: K3 records per segment -> reduce -> K4 (mode 0), or
// -> per-item Gram records in h.gram_out (mode 1, multi-GPU column side)
template <int K, bool SPLIT = false>
static cudaError_t launch_gram_k(const AlsHalf& h, int sm_count, cudaStream_t s) {
    constexpr int W = gram_warps<K, SPLIT>();
    const size_t smem = sizeof(uint4) * W * Cfg<K>::kStageU4;
    int64_t blocks = (h.max_segs + W - 1) / W;
    const int64_t cap = static_cast<int64_t>(sm_count) * Cfg<K>::kMinBlocks;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    cudaFuncSetAttribute(als_mma_gram_kernel<K, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    if (h.ev_gram0) cudaEventRecord(h.ev_gram0, s);
    als_mma_gram_kernel<K, SPLIT><<<static_cast<unsigned>(blocks), W * 32, smem, s>>>(
        h.total_segs, h.seg_order, h.seg_item, h.seg_beg, h.ptr, h.idx, h.valh, h.Yh, h.ymax, h.vmax, h.partial,
        h.blk_ctr, h.nseg);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (h.ev_gram1) cudaEventRecord(h.ev_gram1, s);
    return cudaSuccess;
}

template <int K>
static cudaError_t launch_half_k(const AlsHalf& h, int mode, int sm_count, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(h.blk_ctr, 0, sizeof(int32_t), s);
    if (e != cudaSuccess) return e;
    unsigned* xmax = (mode == 0 && h.xmax) ? h.xmax : nullptr;
    if (xmax && (e = cudaMemsetAsync(xmax, 0, sizeof(unsigned), s)) != cudaSuccess) return e;
    if (K == 32 && h.seg_order) e = launch_gram_k<32, true>(h, sm_count, s);  // column side
    else e = launch_gram_k<K>(h, sm_count, s);
    if (e != cudaSuccess) return e;
    const unsigned rblocks = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(h.nitems, sm_count * 12)));
    // column side: a few items with many segments (y spreads their groups); row side: many short items
    const dim3 gblocks(static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(h.nitems, sm_count * 2))),
                       h.seg_order ? 32 : 2);
    if (mode == 1) {
        als_reduce_groups_kernel<K><<<gblocks, 160, 0, s>>>(h.nitems, nullptr, nullptr, h.nseg, h.first, h.partial);
        als_reduce_records_kernel<K><<<rblocks, 160, 0, s>>>(h.nitems, nullptr, nullptr, h.nseg, h.first, h.partial,
                                                             h.gram_out);
        return cudaGetLastError();
    }
    als_reduce_groups_kernel<K><<<gblocks, 160, 0, s>>>(h.nitems, h.multi_list, h.multi_count, h.nseg, h.first,
                                                        h.partial);
    als_reduce_records_kernel<K><<<rblocks, 160, 0, s>>>(h.nitems, h.multi_list, h.multi_count, h.nseg, h.first,
                                                         h.partial, nullptr);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_solve_k<K>(h.nitems, h.first, h.partial, h.X, h.lambda, sm_count, s, nullptr, nullptr, xmax);
}

cudaError_t launch_als_mma_half(int k, const AlsHalf& h, int mode, int sm_count, cudaStream_t s) {
    if (k == 32) return launch_half_k<32>(h, mode, sm_count, s);
    if (k == 64) return launch_half_k<64>(h, mode, sm_count, s);
    return cudaErrorInvalidValue;
}

cudaError_t launch_als_solve_records(int k, int64_t nitems, const float* G, float* X, float lambda, int sm_count,
                                     cudaStream_t s) {
    if (k == 32) return launch_solve_k<32>(nitems, nullptr, G, X, lambda, sm_count, s);
    if (k == 64) return launch_solve_k<64>(nitems, nullptr, G, X, lambda, sm_count, s);
    return cudaErrorInvalidValue;
}

size_t als_record_floats_mma(int k) { return k == 64 ? Cfg<64>::kRec : Cfg<32>::kRec; }

// max |X| -> *maxbits (zeroed here), then X -> packed hi/lo rows
cudaError_t launch_als_pack(int k, int64_t rows, const float* X, unsigned* maxbits, uint4* Xh, int sm_count,
                            cudaStream_t s, bool have_max) {
    if (!have_max) {  // (else the K4 that wrote X left max |X| in *maxbits)
        cudaError_t e = cudaMemsetAsync(maxbits, 0, sizeof(unsigned), s);
        if (e != cudaSuccess) return e;
        const int64_t cnt = rows * k;
        int64_t blocks = (cnt + 255) / 256;
        if (blocks > sm_count * 8) blocks = sm_count * 8;
        if (blocks < 1) blocks = 1;
        als_absmax_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(cnt, X, maxbits);
    }
    const unsigned pb = static_cast<unsigned>((rows * (k / 8) + 255) / 256);
    if (k == 32) als_pack_kernel<32><<<pb, 256, 0, s>>>(rows, X, maxbits, Xh);
    else if (k == 64) als_pack_kernel<64><<<pb, 256, 0, s>>>(rows, X, maxbits, Xh);
    else return cudaErrorInvalidValue;
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

cudaError_t launch_als_pack_vals(int64_t n, const float* val, const unsigned* vmax, uint32_t* out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    als_pack_vals_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(n, val, vmax, out);
    return cudaGetLastError();
}

}  // namespace ocg
