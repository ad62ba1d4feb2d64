// Rank-32 fused ALS imputation + Algorithm-2 selection on the tensor cores.
//
// Same contract as als_select_kernel (als_select.cu): for every row i the
// completed row is p_ij = r_ij (observed, verbatim) or clamp(u_i . v_j, 0.01,
// 1.25) (cf::complete semantics, cfcomplete.cpp:198-213), and
// policy::select_caps (policy.cpp:17-64) picks the setting, bit-exact given
// the completed row.  What changes is how u_i . v_j is formed and how the
// epilogue is organised:
//
// * The m x n product is a GEMM with K = 32.  U and V are split into FP16
//   hi/lo pairs (power-of-two scales su, sv; als_pack*), and
//   u.v * su*sv = Uh.Vh + Uh.Vl + Ul.Vh  (the Ul.Vl term is below 2^-21
//   relative) runs as mma.sync m16n8k16 f16 -> f32: 6 MMAs per 16x8 cell
//   tile (2 k-steps x 3).  The completed value of an unobserved cell is the
//   FP32 accumulator times 2^-(eu+ev) (exact).
// * A warp owns 16 rows; a CTA (8 warps, 128 rows) streams V in 256-column
//   tiles (32 KB, cp.async double buffer) stored per column as 8 x 16 B
//   chunks ordered so that one LDS.128 yields a lane's B fragments for both
//   k-steps (hi or lo); hi/lo chunk halves swap on odd columns so the 8 lanes
//   of a shared-memory phase hit 8 different bank groups.
// * Each lane holds 2 rows x 64 columns of a tile in the accumulator layout
//   (rows g, g+8; columns 8nt + 2t + e).  Observed cells are skipped through
//   a per-tile bit mask (bits permuted so a lane's 64 bits are two words) and
//   evaluated afterwards from the CSR entries (observed pass); the two passes
//   feed the same per-row selection state.
// * Per unobserved cell the epilogue is branch-free FP32: validity
//   loss <= gamma as an exact compare against the row's FP32 threshold, the
//   candidate count, and the 2^-18 band test of c_sum/p against the lane's
//   best (as a multiply); only cells inside the band take the out-of-line
//   FP64 path (exact saving + the 4-key order).
// * The baseline p_base = p_{i,n-1} is produced first by the same MMA
//   sequence on the tile holding column n-1, so thresholds use the very value
//   the row completes to.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <type_traits>

#include "als.h"
#include "ocg_common.cuh"
#include "select_dev.cuh"

namespace ocg {

namespace {

constexpr int kW = 8;          // warps per CTA
constexpr int kTile = 256;     // V columns per tile
constexpr int kNT = kTile / 8;  // n-tiles per tile
constexpr float kBand = 1.0f + 0x1p-18f;
constexpr int kList = 96;      // observed columns kept in shared memory per row (longer rows: global)

struct BestX {
    double s, p;
    int j, sum;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_h2(__half lo, __half hi) {
    return static_cast<uint32_t>(__half_as_ushort(lo)) | (static_cast<uint32_t>(__half_as_ushort(hi)) << 16);
}
// (a, b) -> packed hi pair and lo pair of a*s, b*s
__device__ __forceinline__ void split2(float a, float b, float s, uint32_t& hi, uint32_t& lo) {
    const float ya = a * s, yb = b * s;
    const __half ha = __float2half_rn(ya), hb = __float2half_rn(yb);
    hi = pack_h2(ha, hb);
    lo = pack_h2(__float2half_rn(ya - __half2float(ha)), __float2half_rn(yb - __half2float(hb)));
}

__device__ __forceinline__ int scale_exp(unsigned maxbits) {
    const float mx = __uint_as_float(maxbits);
    if (!(mx > 0.0f) || !isfinite(mx)) return 0;
    int e;
    frexpf(mx, &e);
    const int x = 14 - e;
    return x < -60 ? -60 : (x > 60 ? 60 : x);
}

// loss(p) = fl(1 - fl(p / p_base)) <= gamma, exactly as policy.cpp:34-35
__device__ __forceinline__ bool valid_exact(double p, double p_base, double gamma) {
    return !(dsub(1.0, ddiv(p, p_base)) > gamma);
}
__device__ __forceinline__ double next_up(double x) { return u2d(d2u(x) + 1); }
__device__ __forceinline__ double next_down(double x) { return u2d(d2u(x) - 1); }
__device__ double valid_threshold(double p_base, double gamma) {
    double x = dmul(p_base, dsub(1.0, gamma));
    if (valid_exact(x, p_base, gamma)) {
        for (int it = 0; it < 64; ++it) {
            const double y = next_down(x);
            if (!valid_exact(y, p_base, gamma)) break;
            x = y;
        }
    } else {
        for (int it = 0; it < 64 && !valid_exact(x, p_base, gamma); ++it) x = next_up(x);
    }
    return x;
}

// FP64 evaluation of one cell (policy.cpp:37-38) + the 4-key compare
__device__ __noinline__ void exact_update(BestX* b, double pd, int cs, int j, double e_base) {
    const double e_pred = ddiv(static_cast<double>(cs), pd);
    const double s = ddiv(dsub(e_base, e_pred), e_base);
    bool better;
    if (b->j < 0) better = true;
    else if (s != b->s) better = s > b->s;
    else if (pd != b->p) better = pd > b->p;
    else if (cs != b->sum) better = cs < b->sum;
    else better = j < b->j;
    if (better) {
        b->s = s;
        b->p = pd;
        b->j = j;
        b->sum = cs;
    }
}

// V (n x 32 f32) -> per column 8 x 16 B: chunk t of the hi (lo) half holds dims
// {2t, 2t+1, 2t+8, 2t+9, 2t+16, 2t+17, 2t+24, 2t+25}; hi chunks sit at
// positions 0-3 on even columns and 4-7 on odd columns (lo the other half)
// (rank 64: the same per block p of 32 dims, chunks 8p .. 8p+7)
template <int K>
__global__ void pack_vsel_kernel(int64_t n, const float* __restrict__ V, const unsigned* __restrict__ vmaxbits,
                                 uint4* __restrict__ out) {
    const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;  // (column, t)
    if (q >= n * 4) return;
    const int64_t c = q >> 2;
    const int t = static_cast<int>(q & 3);
    const float s = ldexpf(1.0f, scale_exp(*vmaxbits));
    const int odd = static_cast<int>(c & 1);
#pragma unroll
    for (int p = 0; p < K / 32; ++p) {
        const float* v = V + c * K + 32 * p;
        const int d[8] = {2 * t, 2 * t + 1, 2 * t + 8, 2 * t + 9, 2 * t + 16, 2 * t + 17, 2 * t + 24, 2 * t + 25};
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) split2(v[d[2 * u]], v[d[2 * u + 1]], s, hi[u], lo[u]);
        out[c * (K / 4) + 8 * p + t + 4 * odd] = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        out[c * (K / 4) + 8 * p + t + 4 * (1 - odd)] = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    }
}

}  // namespace

struct AlsSelMmaArgs {
    AlsSelectArgs a;
    const uint4* Vsel;         // packed V (pack_vsel_kernel)
    const unsigned* umax;      // max |U| bits
    const unsigned* vmax;      // max |V| bits
};

template <int K, bool WRITE_COMPLETED>
__global__ void __launch_bounds__(kW * 32, K == 32 ? 2 : 1) als_select_mma_kernel(AlsSelMmaArgs P) {
    constexpr int KS = K / 16, CPC = K / 4;  // k-steps, 16-byte chunks per V column
    const AlsSelectArgs& a = P.a;
    extern __shared__ __align__(16) uint4 sdyn[];
    uint4* Vs = sdyn;                                                     // [2][kTile][8]
    float* csum = reinterpret_cast<float*>(Vs + 2 * kTile * CPC);         // [2][kTile] c+g per column
    uint32_t* maskw = reinterpret_cast<uint32_t*>(csum + 2 * kTile);      // [kW][16][8]
    BestX* bx = reinterpret_cast<BestX*>(maskw + kW * 16 * 8);            // [kW][32 lanes][2 rows]
    BestX* obest = bx + kW * 32 * 2;                                      // [kW][16 rows] observed best
    int32_t* ocnt = reinterpret_cast<int32_t*>(obest + kW * 16);          // [kW][16] valid observed
    int32_t* caps = ocnt + kW * 16;                                       // [512]
    uint16_t* olist = reinterpret_cast<uint16_t*>(caps + 512);            // [kW][16][kList] columns
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, t = lane & 3;
    const int64_t n = a.n;
    const int ngpu = a.ngpu, ncpu = static_cast<int>(n / ngpu);
    const int ntiles = static_cast<int>((n + kTile - 1) / kTile);
    for (int e = tid; e < ncpu + ngpu; e += blockDim.x) caps[e] = e < ncpu ? a.cpu_caps[e] : a.gpu_caps[e - ncpu];
    const int eu = scale_exp(*P.umax), ev = scale_exp(*P.vmax);
    const float su = ldexpf(1.0f, eu), inv_s = ldexpf(1.0f, -(eu + ev));
    uint32_t* mymask = maskw + warp * 16 * 8;
    BestX* myb = bx + (warp * 32 + lane) * 2;
    BestX* myob = obest + warp * 16;
    int32_t* myoc = ocnt + warp * 16;
    uint16_t* mylist = olist + warp * 16 * kList;
    __syncthreads();  // caps

    auto load_tile = [&](int tt, int buf) {
        const int64_t c0 = static_cast<int64_t>(tt) * kTile;
        for (int e = tid; e < kTile * CPC; e += blockDim.x) {
            const int64_t c = c0 + e / CPC;
            uint4* dst = Vs + buf * kTile * CPC + e;
            if (c < n) cp_async16(dst, P.Vsel + c * CPC + (e % CPC));
            else *dst = make_uint4(0u, 0u, 0u, 0u);
        }
        for (int e = tid; e < kTile; e += blockDim.x) {
            const int64_t j = c0 + e;
            int cs = 1;
            if (j < n) {
                const int ci = static_cast<int>(j / ngpu);
                cs = caps[ci] + caps[ncpu + static_cast<int>(j - static_cast<int64_t>(ci) * ngpu)];
            }
            csum[buf * kTile + e] = static_cast<float>(cs);  // small integer: exact
        }
        cp_async_commit();
    };

    for (int64_t rb = static_cast<int64_t>(blockIdx.x) * (kW * 16); rb < a.m;
         rb += static_cast<int64_t>(gridDim.x) * (kW * 16)) {
        __syncthreads();  // previous block's tile buffers are free
        load_tile(0, 0);
        const int64_t r0 = rb + warp * 16;
        const int64_t rowg[2] = {r0 + g, r0 + g + 8};
        const bool live[2] = {rowg[0] < a.m, rowg[1] < a.m};
        // A fragments (rows g, g+8; k-step ks: dims 16ks + {2t,2t+1} / {2t+8,2t+9})
        uint32_t ah[KS][4], al[KS][4];
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            float2 v[2][2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const float* u = a.U + (live[q] ? rowg[q] : 0) * K + 16 * ks + 2 * t;
                v[q][0] = live[q] ? *reinterpret_cast<const float2*>(u) : make_float2(0.f, 0.f);
                v[q][1] = live[q] ? *reinterpret_cast<const float2*>(u + 8) : make_float2(0.f, 0.f);
            }
            split2(v[0][0].x, v[0][0].y, su, ah[ks][0], al[ks][0]);  // row g,   k 2t..
            split2(v[1][0].x, v[1][0].y, su, ah[ks][1], al[ks][1]);  // row g+8, k 2t..
            split2(v[0][1].x, v[0][1].y, su, ah[ks][2], al[ks][2]);  // row g,   k 2t+8..
            split2(v[1][1].x, v[1][1].y, su, ah[ks][3], al[ks][3]);  // row g+8, k 2t+8..
        }
        // bh/bl[p]: the lane's hi/lo chunk of block p (k-steps 2p, 2p+1)
        auto mma_cell = [&](float (&d)[4], const uint4 (&bh)[K / 32], const uint4 (&bl)[K / 32]) {
            d[0] = d[1] = d[2] = d[3] = 0.0f;
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                const uint4& h = bh[ks >> 1];
                const uint4& l = bl[ks >> 1];
                const uint32_t h0 = (ks & 1) ? h.z : h.x, h1 = (ks & 1) ? h.w : h.y;
                const uint32_t l0 = (ks & 1) ? l.z : l.x, l1 = (ks & 1) ? l.w : l.y;
                mma16816(d, ah[ks][0], ah[ks][1], ah[ks][2], ah[ks][3], h0, h1);
                mma16816(d, ah[ks][0], ah[ks][1], ah[ks][2], ah[ks][3], l0, l1);
                mma16816(d, al[ks][0], al[ks][1], al[ks][2], al[ks][3], h0, h1);
            }
        };
        // ---- baseline p_{i,n-1}: the n-tile holding column n-1, same MMA sequence
        double pbase[2];
        {
            const int64_t cb = (n - 1) & ~static_cast<int64_t>(7);  // n-tile base column
            const int64_t col = cb + g;                              // this lane's B column
            uint4 bh[K / 32], bl[K / 32];
#pragma unroll
            for (int p = 0; p < K / 32; ++p) {
                bh[p] = bl[p] = make_uint4(0u, 0u, 0u, 0u);
                if (col < n) {
                    const int odd = static_cast<int>(col & 1);
                    bh[p] = P.Vsel[col * CPC + 8 * p + t + 4 * odd];
                    bl[p] = P.Vsel[col * CPC + 8 * p + t + 4 * (1 - odd)];
                }
            }
            float d[4];
            mma_cell(d, bh, bl);
            const int jl = static_cast<int>((n - 1) - cb);  // 0..7: column within the n-tile
            const int src = jl >> 1;                                 // lane t of the quad holding it
            const float v0 = (jl & 1) ? d[1] : d[0], v1 = (jl & 1) ? d[3] : d[2];
            float pb[2];
            pb[0] = __shfl_sync(0xffffffffu, v0, (lane & ~3) | src) * inv_s;
            pb[1] = __shfl_sync(0xffffffffu, v1, (lane & ~3) | src) * inv_s;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                double p = 1.0;
                if (live[q]) {
                    const int64_t e = a.row_ptr[rowg[q] + 1] - 1;  // baseline = last column n-1
                    if (e >= a.row_ptr[rowg[q]] && a.col[e] == n - 1) p = static_cast<double>(a.val[e]);
                    else p = pb[q] <= 0.01f ? 0.01 : (pb[q] > 1.25f ? 1.25 : static_cast<double>(pb[q]));
                }
                pbase[q] = p;
            }
        }
        float fthr[2], lov[2], tbest[2], tband[2];
        int ncand[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const double thr = valid_threshold(pbase[q], a.gamma);
            float f = static_cast<float>(thr);
            if (static_cast<double>(f) < thr) f = __uint_as_float(__float_as_uint(f) + 1u);
            fthr[q] = live[q] ? f : INFINITY;  // float p valid <=> p >= fthr (dead rows: nothing valid)
            lov[q] = live[q] && 0.01 >= thr ? INFINITY : -INFINITY;  // cells clamped to 0.01: valid iff 0.01 >= thr
            ncand[q] = 0;
            myb[q] = BestX{0.0, 0.0, -1, 0};
        }
        // ---- observed pass: the whole warp walks each row's CSR entries (coalesced),
        // evaluates the valid ones exactly, keeps the columns for the tile masks, and
        // seeds the row's band with the best observed cell.
#pragma unroll 1
        for (int rr = 0; rr < 16; ++rr) {
            const int64_t i = r0 + rr;
            if (i >= a.m) break;
            const int src = (rr & 7) * 4;
            const float fth = __shfl_sync(0xffffffffu, (rr >> 3) ? fthr[1] : fthr[0], src);
            const int64_t rbeg = a.row_ptr[i];
            const int rl = static_cast<int>(a.row_ptr[i + 1] - rbeg);
            SelResult sr{-1, 0.0, 0.0, 0.0, 0, 0};
            bool have = false;
            int oc = 0;
            for (int e = lane; e < rl; e += 32) {
                const int j = a.col[rbeg + e];
                const float v = a.val[rbeg + e];
                if (e < kList) mylist[rr * kList + e] = static_cast<uint16_t>(j);
                if (WRITE_COMPLETED) a.completed[i * n + j] = static_cast<double>(v);
                if (v >= fth) {
                    ++oc;
                    const int ci = j / ngpu;
                    const int cs = caps[ci] + caps[ncpu + (j - ci * ngpu)];
                    const double pd = static_cast<double>(v);
                    const double sv = ddiv(dsub(a.e_base, ddiv(static_cast<double>(cs), pd)), a.e_base);
                    if (!have || sel_better(sv, pd, cs, j, sr)) {
                        sr = SelResult{j, sv, 0.0, pd, cs, 0};
                        have = true;
                    }
                }
            }
            const SelResult w = sel_warp_reduce(sr, have, oc);
            if (lane == 0) {
                myob[rr] = BestX{w.saving, w.perf, w.idx, w.sum};
                myoc[rr] = w.ncand;
            }
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const BestX ob = myob[(g + 8 * q) & 15];
            tbest[q] = ob.j >= 0 ? __fdividef(static_cast<float>(ob.sum), static_cast<float>(ob.p)) : INFINITY;
            tband[q] = tbest[q] * kBand;
        }
        // mask owner: lane r < 16 walks row r0 + r's columns tile by tile
        int mcur = 0, mend = 0;
        int64_t mbeg = 0;
        bool mfull = false, mglob = false;
        if (lane < 16 && r0 + lane < a.m) {
            mbeg = a.row_ptr[r0 + lane];
            mend = static_cast<int>(a.row_ptr[r0 + lane + 1] - mbeg);
            mfull = mend == n;        // fully observed (offline dense rows)
            mglob = mend > kList;     // list overflow: read the columns from global memory
        }
        // every row of the warp has p_thr > 0.01 (the common case): the cheaper epilogue
        const bool fast = !__any_sync(0xffffffffu, lov[0] > 0.0f || lov[1] > 0.0f);
        // ---- dense pass over the tiles (unobserved cells)
        for (int tt = 0; tt < ntiles; ++tt) {
            const int buf = tt & 1;
            const int64_t c0 = static_cast<int64_t>(tt) * kTile;
            // observed-cell mask of this tile: column cc -> word 2*((cc&7)>>1) + (cc>>7),
            // bit (((cc>>3)&15)<<1) | (cc&1)  (a lane's 64 bits are 2 words per row)
            __syncwarp();  // every lane has read the previous tile's mask words
            if (lane < 16) {
                uint32_t* mw = mymask + lane * 8;
                const uint32_t fill = mfull ? 0xffffffffu : 0u;
#pragma unroll
                for (int w = 0; w < 8; ++w) mw[w] = fill;
                if (!mfull) {
                    while (mcur < mend) {
                        const int c = mglob ? a.col[mbeg + mcur] : mylist[lane * kList + mcur];
                        if (c >= c0 + kTile) break;
                        const int cc = static_cast<int>(c - c0);
                        mw[2 * ((cc & 7) >> 1) + (cc >> 7)] |= 1u << ((((cc >> 3) & 15) << 1) | (cc & 1));
                        ++mcur;
                    }
                }
            }
            cp_async_wait_all();
            __syncthreads();  // tile tt landed, masks written
            if (tt + 1 < ntiles) load_tile(tt + 1, buf ^ 1);
            const uint4* vt = Vs + buf * kTile * CPC;
            const float* cst = csum + buf * kTile;
            uint32_t mk[2][2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const uint2 w = *reinterpret_cast<const uint2*>(mymask + (g + 8 * q) * 8 + 2 * t);
                mk[q][0] = w.x;
                mk[q][1] = w.y;
            }
            if (n - c0 < kTile) {  // ragged last tile: columns >= n count as observed
#pragma unroll
                for (int nt = 0; nt < kNT; ++nt)
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        if (nt * 8 + 2 * t + e >= n - c0) {
                            const uint32_t b = 1u << (((nt & 15) << 1) | e);
                            mk[0][nt >> 4] |= b;
                            mk[1][nt >> 4] |= b;
                        }
            }
            // Epilogue in the accumulator's scale S = 2^(eu+ev) (all comparisons against
            // thresholds multiplied by S are exact); branch-free over 2 n-tiles (8 cells),
            // then one branch into the rare exact path if any cell is inside the band.
            const float S = ldexpf(1.0f, eu + ev);
            const float lo_s = 0.01f * S, hi_s = 1.25f * S;
            // validity of an unobserved cell as ONE compare: if 0.01 >= p_thr every completed
            // value (>= 0.01) is valid; otherwise cells clamped to 0.01 are invalid and
            // min(x, 1.25 S) >= fthr S decides (fthr > 0.01f, and 1.25 is a float)
            const float fth_s[2] = {lov[0] > 0.0f ? -INFINITY : fthr[0] * S, lov[1] > 0.0f ? -INFINITY : fthr[1] * S};
            float tb_s[2] = {tband[0] * inv_s, tband[1] * inv_s};
            const float fthp[2] = {fth_s[0] <= hi_s ? fth_s[0] : INFINITY, fth_s[1] <= hi_s ? fth_s[1] : INFINITY};
            auto tiles = [&](auto FAST) {
#pragma unroll 2
            for (int nt = 0; nt < kNT; nt += 2) {
                float d[2][4];
                float2 cs2[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int cc = (nt + u) * 8;
                    const int odd = g & 1;
                    uint4 bh[K / 32], bl[K / 32];
#pragma unroll
                    for (int p = 0; p < K / 32; ++p) {
                        bh[p] = vt[(cc + g) * CPC + 8 * p + t + 4 * odd];
                        bl[p] = vt[(cc + g) * CPC + 8 * p + t + 4 * (1 - odd)];
                    }
                    mma_cell(d[u], bh, bl);
                    cs2[u] = *reinterpret_cast<const float2*>(cst + cc + 2 * t);
                }
                // per row q, cell c = 2u + e of the group: validity and band-candidate bits;
                // the lane's observed bits of the group are 4 consecutive mask bits
                unsigned hit = 0;
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    unsigned vb = 0u, hb = 0u;
#pragma unroll
                    for (int u = 0; u < 2; ++u)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const float csf = e ? cs2[u].y : cs2[u].x;
                            const float x = d[u][2 * q + e];
                            if constexpr (decltype(FAST)::value) {
                                // no row of the warp has p_thr <= 0.01: valid cells have x > 0.01 S,
                                // min(x, 1.25 S) >= fth <=> x >= fthp, and the band test on the raw
                                // x is a superset of the clamped one (the exact path re-checks)
                                vb |= x >= fthp[q] ? 1u << (2 * u + e) : 0u;
                                hb |= csf <= tb_s[q] * x ? 1u << (2 * u + e) : 0u;
                            } else {
                                const float pc = fminf(x, hi_s);
                                vb |= pc >= fth_s[q] ? 1u << (2 * u + e) : 0u;
                                hb |= csf <= tb_s[q] * fmaxf(pc, lo_s) ? 1u << (2 * u + e) : 0u;
                            }
                        }
                    const unsigned ob4 = (mk[q][nt >> 4] >> ((nt & 15) * 2)) & 0xFu;
                    vb &= ~ob4;
                    ncand[q] += __popc(vb);
                    hit |= (hb & vb) << (4 * q);
                    if (WRITE_COMPLETED && live[q]) {
#pragma unroll
                        for (int u = 0; u < 2; ++u)
#pragma unroll
                            for (int e = 0; e < 2; ++e) {
                                if ((ob4 >> (2 * u + e)) & 1u) continue;
                                const float x = d[u][2 * q + e];
                                const float pf = x * inv_s;
                                a.completed[rowg[q] * n + c0 + (nt + u) * 8 + 2 * t + e] =
                                    x <= lo_s ? 0.01 : (pf > 1.25f ? 1.25 : static_cast<double>(pf));
                            }
                    }
                }
                if (hit) {  // rare: exact FP64 evaluation of the cells inside the band
#pragma unroll
                    for (int u = 0; u < 2; ++u)
#pragma unroll
                        for (int e = 0; e < 2; ++e)
#pragma unroll
                            for (int q = 0; q < 2; ++q) {
                                if (!((hit >> (4 * q + 2 * u + e)) & 1u)) continue;
                                const float csf = e ? cs2[u].y : cs2[u].x;
                                const float pf = d[u][2 * q + e] * inv_s;
                                const bool lo = pf <= 0.01f;
                                if (csf > tb_s[q] * fmaxf(fminf(d[u][2 * q + e], hi_s), lo_s)) continue;  // band moved
                                const double pd = lo ? 0.01 : (pf > 1.25f ? 1.25 : static_cast<double>(pf));
                                exact_update(myb + q, pd, static_cast<int>(csf),
                                             static_cast<int>(c0) + (nt + u) * 8 + 2 * t + e, a.e_base);
                                const float pe = fmaxf(fminf(pf, 1.25f), 0.01f);
                                tbest[q] = fminf(tbest[q], __fdividef(csf, pe));
                                tband[q] = tbest[q] * kBand;
                                tb_s[q] = tband[q] * inv_s;
                            }
                }
            }
            };
            if (fast) tiles(std::true_type{});
            else tiles(std::false_type{});
            // share the running best within the quad (the 4 lanes holding a row)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                tbest[q] = fminf(tbest[q], __shfl_xor_sync(0xffffffffu, tbest[q], 1));
                tbest[q] = fminf(tbest[q], __shfl_xor_sync(0xffffffffu, tbest[q], 2));
                tband[q] = tbest[q] * kBand;
            }
        }
        // ---- merge per row: the quad's dense candidates + the observed best
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            BestX b = myb[q];
            int cnt = ncand[q];
#pragma unroll
            for (int off = 1; off <= 2; off <<= 1) {
                BestX o;
                o.s = __shfl_xor_sync(0xffffffffu, b.s, off);
                o.p = __shfl_xor_sync(0xffffffffu, b.p, off);
                o.j = __shfl_xor_sync(0xffffffffu, b.j, off);
                o.sum = __shfl_xor_sync(0xffffffffu, b.sum, off);
                cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
                bool better;
                if (o.j < 0) better = false;
                else if (b.j < 0) better = true;
                else if (o.s != b.s) better = o.s > b.s;
                else if (o.p != b.p) better = o.p > b.p;
                else if (o.sum != b.sum) better = o.sum < b.sum;
                else better = o.j < b.j;
                if (better) b = o;
            }
            const int rr = g + 8 * q;
            if (t == 0 && live[q]) {
                const BestX o = myob[rr];
                bool better;
                if (o.j < 0) better = false;
                else if (b.j < 0) better = true;
                else if (o.s != b.s) better = o.s > b.s;
                else if (o.p != b.p) better = o.p > b.p;
                else if (o.sum != b.sum) better = o.sum < b.sum;
                else better = o.j < b.j;
                if (better) b = o;
                const int64_t i = rowg[q];
                a.idx[i] = b.j;
                a.saving[i] = b.j >= 0 ? b.s : 0.0;
                a.loss[i] = b.j >= 0 ? dsub(1.0, ddiv(b.p, pbase[q])) : 0.0;
                a.ncand[i] = cnt + myoc[rr];
            }
        }
    }
}

template <int K>
static size_t select_smem() {
    return sizeof(uint4) * 2 * kTile * (K / 4) + sizeof(float) * 2 * kTile + sizeof(uint32_t) * kW * 16 * 8 +
           sizeof(BestX) * (kW * 32 * 2 + kW * 16) + sizeof(int32_t) * (kW * 16 + 512) +
           sizeof(uint16_t) * kW * 16 * kList;
}

template <int K>
static cudaError_t launch_select_k(const AlsSelectArgs& a, uint4* Vsel, const unsigned* umax, const unsigned* vmax,
                                   int sm_count, cudaStream_t s) {
    pack_vsel_kernel<K><<<static_cast<unsigned>((a.n * 4 + 255) / 256), 256, 0, s>>>(a.n, a.V, vmax, Vsel);
    AlsSelMmaArgs P{a, Vsel, umax, vmax};
    const size_t smem = select_smem<K>();
    int64_t blocks = (a.m + kW * 16 - 1) / (kW * 16);
    const int64_t cap = static_cast<int64_t>(sm_count) * (K == 32 ? 2 : 1);
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        kern<<<static_cast<unsigned>(blocks), kW * 32, smem, s>>>(P);
    };
    if (a.completed) go(als_select_mma_kernel<K, true>);
    else go(als_select_mma_kernel<K, false>);
    return cudaGetLastError();
}

// V -> packed select layout; U's and V's scales come from the Gram packing
// (maxbits[0] = max |U|, maxbits[1] = max |V|, refreshed after every half-sweep)
cudaError_t launch_als_select_mma(const AlsSelectArgs& a, uint4* Vsel, const unsigned* umax, const unsigned* vmax,
                                  int sm_count, cudaStream_t s) {
    if (static_cast<int64_t>(a.n / a.ngpu) + a.ngpu > 512) return cudaErrorInvalidValue;
    if (a.k == 32) return launch_select_k<32>(a, Vsel, umax, vmax, sm_count, s);
    if (a.k == 64) return launch_select_k<64>(a, Vsel, umax, vmax, sm_count, s);
    return cudaErrorInvalidValue;
}

}  // namespace ocg
