// Fused ALS imputation + Algorithm-2 selection (K2 for the MF model).
//
// For every row i the completed row is  p_ij = r_ij (observed, verbatim) or
// clamp(u_i . v_j, 0.01, 1.25) (cf::complete semantics, cfcomplete.cpp:198-
// 213), and policy::select_caps (policy.cpp:17-64) picks the setting.  The
// m x n completed matrix is never materialised: a CTA owns 32 rows, streams
// V^T in 128-column tiles through shared memory (cp.async double buffer) and
// each lane computes a 4-row x 4-column register tile of dot products, then
// runs the selection epilogue on its 16 cells.
//
// Exactness without FP64 divisions per cell:
//  * validity  loss = 1 - p/p_base <= gamma is monotone in p, so per row the
//    smallest valid double p_thr is found once (FP64, a few ulp steps around
//    p_base*(1-gamma)); a cell is valid iff p >= p_thr — an exact compare.
//  * ranking   saving = (E - c_sum/p)/E is monotone in the real c_sum/p, so a
//    lane tracks its best FP32 estimate t = c_sum/p and evaluates the exact
//    FP64 saving only for cells within a 2^-18 relative band of it; cells
//    outside the band are provably worse.  The exact 4-key order
//    (saving, p, c+g, index) then decides, and a warp reduction with the same
//    key merges lanes.  ncand counts valid cells exactly.
#include <cuda_runtime.h>

#include "als.h"
#include "ocg_common.cuh"
#include "select_dev.cuh"

namespace ocg {

namespace {

constexpr int kRows = 32;      // rows per CTA (8 warps x 4)
constexpr int kRPW = 4;        // rows per warp
constexpr int kTC = 128;       // columns per V tile (32 lanes x 4)
constexpr float kBand = 1.0f + 0x1p-18f;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// loss(p) = fl(1 - fl(p / p_base)) <= gamma, exactly as policy.cpp:34-35
__device__ __forceinline__ bool valid_exact(double p, double p_base, double gamma) {
    return !(dsub(1.0, ddiv(p, p_base)) > gamma);
}

// neighbours of a positive finite double / float
__device__ __forceinline__ double next_up(double x) { return u2d(d2u(x) + 1); }
__device__ __forceinline__ double next_down(double x) { return u2d(d2u(x) - 1); }

// smallest double p with valid_exact(p) (the valid set is an up-set in p)
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

// exact state of a lane's best cell for one row (shared memory; touched only
// on the rare exact-evaluation path)
struct BestExact {
    double s, p;  // exact saving and completed value
    int j, sum;   // column (-1: none), c+g
};

// Rare path: FP64 evaluation of one cell (policy.cpp:37-38) and the 4-key
// compare against the lane's current best.  Kept out of line so the unrolled
// hot loop stays small.
__device__ __noinline__ void exact_update(BestExact* b, double pd, int cs, int j, double e_base) {
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

}  // namespace

template <int K, bool WRITE_COMPLETED>
__global__ void __launch_bounds__(256, 2) als_select_kernel(AlsSelectArgs a) {
    static_assert(K % 4 == 0 && K <= 32, "rank");
    __shared__ __align__(16) float Ut[K][kRows];
    __shared__ double pbase_s[kRows], pthr_s[kRows];
    __shared__ float fthr_s[kRows];
    __shared__ int32_t caps_s[512];  // cpu caps then gpu caps
    extern __shared__ __align__(16) float dyn[];
    float (*Vt)[K][kTC] = reinterpret_cast<float (*)[K][kTC]>(dyn);                      // [2][K][kTC]
    float (*obs)[kRPW][kTC] = reinterpret_cast<float (*)[kRPW][kTC]>(dyn + 2 * K * kTC);  // [8][kRPW][kTC]
    BestExact* bex = reinterpret_cast<BestExact*>(dyn + 2 * K * kTC + 8 * kRPW * kTC);     // [8][kRPW][32]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t n = a.n;
    const int ntiles = static_cast<int>((n + kTC - 1) / kTC);
    const int ncpu = static_cast<int>(n / a.ngpu);
    for (int e = tid; e < ncpu + a.ngpu; e += 256) caps_s[e] = e < ncpu ? a.cpu_caps[e] : a.gpu_caps[e - ncpu];
    for (int64_t rb = static_cast<int64_t>(blockIdx.x) * kRows; rb < a.m; rb += static_cast<int64_t>(gridDim.x) * kRows) {
        __syncthreads();
        // ---- U block (transposed) + p_base / p_thr per row --------------
        for (int e = tid; e < kRows * K; e += 256) {
            const int r = e % kRows, k = e / kRows;
            const int64_t i = rb + r;
            Ut[k][r] = i < a.m ? a.U[i * K + k] : 0.0f;
        }
        __syncthreads();
        if (tid < kRows) {
            const int r = tid;
            const int64_t i = rb + r;
            double pb = 1.0;
            if (i < a.m) {
                const int64_t q = a.row_ptr[i + 1] - 1;  // baseline = last column n-1
                if (q >= a.row_ptr[i] && a.col[q] == n - 1) {
                    pb = static_cast<double>(a.val[q]);
                } else {
                    float acc = 0.0f;
#pragma unroll
                    for (int k = 0; k < K; ++k) acc = fmaf(Ut[k][r], a.V[(n - 1) * K + k], acc);
                    pb = fmin(fmax(static_cast<double>(acc), 0.01), 1.25);
                }
            }
            pbase_s[r] = pb;
            const double thr = valid_threshold(pb, a.gamma);
            pthr_s[r] = thr;
            // smallest float >= thr: float p valid  <=>  p >= fthr
            float f = static_cast<float>(thr);
            if (static_cast<double>(f) < thr) f = __uint_as_float(__float_as_uint(f) + 1u);
            fthr_s[r] = f;
        }
        __syncthreads();
        const int r0 = warp * kRPW;
        float tbest[kRPW];   // FP32 estimate of c_sum/p of the lane's best, per row
        int ncand[kRPW];
        bool lo_ok[kRPW], hi_ok[kRPW];  // clamp floor 0.01 / ceiling 1.25 valid for this row
        const int32_t* rcol[kRPW];  // the row's CSR columns / values (32-bit cursors)
        const float* rval[kRPW];
        int cursor[kRPW], rend[kRPW];
        bool rowlive[kRPW];
        float fthr[kRPW];
        BestExact* myb = bex + (warp * kRPW) * 32 + lane;  // row q at myb[q * 32]
#pragma unroll
        for (int q = 0; q < kRPW; ++q) {
            tbest[q] = INFINITY;
            ncand[q] = 0;
            myb[q * 32] = BestExact{0.0, 0.0, -1, 0};
            const int64_t i = rb + r0 + q;
            rowlive[q] = i < a.m;
            const int64_t rbeg = rowlive[q] ? a.row_ptr[i] : 0;
            rcol[q] = a.col + rbeg;
            rval[q] = a.val + rbeg;
            cursor[q] = 0;
            rend[q] = rowlive[q] ? static_cast<int>(a.row_ptr[i + 1] - rbeg) : 0;
            fthr[q] = fthr_s[r0 + q];
            lo_ok[q] = 0.01 >= pthr_s[r0 + q];
            hi_ok[q] = 1.25 >= pthr_s[r0 + q];
        }
        // ---- prefetch tile 0 ---------------------------------------------
        auto load_tile = [&](int t, int buf) {
            const int64_t c0 = static_cast<int64_t>(t) * kTC;
            for (int e = tid; e < K * (kTC / 4); e += 256) {
                const int k = e / (kTC / 4), c4 = (e % (kTC / 4)) * 4;
                float* dst = &Vt[buf][k][c4];
                if (c0 + c4 + 3 < n) {
                    cp_async16(dst, a.Vt + static_cast<int64_t>(k) * n + c0 + c4);
                } else {
                    for (int u = 0; u < 4; ++u) dst[u] = c0 + c4 + u < n ? a.Vt[static_cast<int64_t>(k) * n + c0 + c4 + u] : 0.0f;
                }
            }
            cp_async_commit();
        };
        load_tile(0, 0);
        for (int t = 0; t < ntiles; ++t) {
            const int buf = t & 1;
            cp_async_wait_all();
            __syncthreads();
            if (t + 1 < ntiles) load_tile(t + 1, buf ^ 1);
            const int64_t c0 = static_cast<int64_t>(t) * kTC;
            // observed entries of this tile for the warp's rows -> obs[warp]
#pragma unroll
            for (int q = 0; q < kRPW; ++q) {
                float4* o4 = reinterpret_cast<float4*>(&obs[warp][q][0]);
                o4[lane] = make_float4(-1.f, -1.f, -1.f, -1.f);
            }
            __syncwarp();
            const int c0i = static_cast<int>(c0);
#pragma unroll
            for (int q = 0; q < kRPW; ++q) {
                while (cursor[q] < rend[q]) {
                    const int e = cursor[q] + lane;
                    const int c = e < rend[q] ? __ldg(rcol[q] + e) : INT32_MAX;
                    const bool in = c < c0i + kTC;
                    if (in) obs[warp][q][c - c0i] = __ldg(rval[q] + e);
                    const unsigned bal = __ballot_sync(0xffffffffu, in);
                    cursor[q] += __popc(bal);
                    if (bal != 0xffffffffu) break;
                }
            }
            __syncwarp();
            // register tile: rows r0..r0+3 x columns c0+4*lane..+3
            float acc[kRPW][4];
#pragma unroll
            for (int q = 0; q < kRPW; ++q)
#pragma unroll
                for (int u = 0; u < 4; ++u) acc[q][u] = 0.0f;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const float4 uu = *reinterpret_cast<const float4*>(&Ut[k][r0]);
                const float4 vv = *reinterpret_cast<const float4*>(&Vt[buf][k][lane * 4]);
                const float us[4] = {uu.x, uu.y, uu.z, uu.w}, vs[4] = {vv.x, vv.y, vv.z, vv.w};
#pragma unroll
                for (int q = 0; q < kRPW; ++q)
#pragma unroll
                    for (int u = 0; u < 4; ++u) acc[q][u] = fmaf(us[q], vs[u], acc[q][u]);
            }
            // selection epilogue on the 16 cells (branch-free hot path; the
            // exact FP64 path runs only for cells within the band of the best)
            const int jb = c0i + lane * 4;
            int ci = jb / a.ngpu;
            int gi = jb - ci * a.ngpu;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int j = jb + u;
                if (u > 0 && ++gi == a.ngpu) {
                    gi = 0;
                    ++ci;
                }
                const bool jin = j < n;
                const int cs = jin ? caps_s[ci] + caps_s[ncpu + gi] : 1;
                const float csf = static_cast<float>(cs);
#pragma unroll
                for (int q = 0; q < kRPW; ++q) {
                    const bool live = jin && rowlive[q];
                    const float ov = obs[warp][q][lane * 4 + u];
                    const bool is_obs = ov > 0.0f;
                    const float pf = is_obs ? ov : acc[q][u];
                    // clamp(p, 0.01, 1.25) in the double domain: float p <= 0.01f <=> (double)p < 0.01
                    const bool lo = !is_obs && pf <= 0.01f;
                    const bool hi = !is_obs && pf > 1.25f;
                    const float pe = lo ? 0.01f : (hi ? 1.25f : pf);
                    const bool valid = live && (lo ? lo_ok[q] : (hi ? hi_ok[q] : pf >= fthr[q]));
                    if (WRITE_COMPLETED && live)
                        a.completed[(rb + r0 + q) * n + j] = lo ? 0.01 : (hi ? 1.25 : static_cast<double>(pf));
                    ncand[q] += valid ? 1 : 0;
                    const float tf = __fdividef(csf, pe);
                    if (valid && tf <= tbest[q] * kBand) {
                        const double pd = lo ? 0.01 : (hi ? 1.25 : static_cast<double>(pf));
                        exact_update(myb + q * 32, pd, cs, j, a.e_base);
                        tbest[q] = fminf(tbest[q], tf);
                    }
                }
            }
        }
        // ---- warp reduction per row + outputs ------------------------------
#pragma unroll
        for (int q = 0; q < kRPW; ++q) {
            const int64_t i = rb + r0 + q;
            const BestExact b = myb[q * 32];
            SelResult sr{b.j, b.s, 0.0, b.p, b.sum, 0};
            const SelResult w = sel_warp_reduce(sr, b.j >= 0, ncand[q]);
            if (lane == 0 && i < a.m) {
                a.idx[i] = w.idx;
                a.saving[i] = w.saving;
                a.loss[i] = w.idx >= 0 ? dsub(1.0, ddiv(w.perf, pbase_s[r0 + q])) : 0.0;
                a.ncand[i] = w.ncand;
            }
        }
    }
}

__global__ void transpose_kernel(int64_t n, int k, const float* __restrict__ V, float* __restrict__ Vt) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= n * k) return;
    const int64_t j = e / k;
    const int f = static_cast<int>(e - j * k);
    Vt[static_cast<int64_t>(f) * n + j] = V[e];
}

cudaError_t launch_als_select(const AlsSelectArgs& a, int sm_count, cudaStream_t s) {
    int64_t blocks = (a.m + kRows - 1) / kRows;
    const int64_t cap = static_cast<int64_t>(sm_count) * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    const unsigned b = static_cast<unsigned>(blocks);
    const size_t smem = sizeof(float) * (2 * static_cast<size_t>(a.k) * kTC + 8 * kRPW * kTC) +
                        sizeof(BestExact) * 8 * kRPW * 32;
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        kern<<<b, 256, smem, s>>>(a);
    };
    const bool wc = a.completed != nullptr;
    switch (a.k) {
        case 8: wc ? go(als_select_kernel<8, true>) : go(als_select_kernel<8, false>); break;
        case 16: wc ? go(als_select_kernel<16, true>) : go(als_select_kernel<16, false>); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_transpose(int64_t n, int k, const float* V, float* Vt, cudaStream_t s) {
    const int64_t tot = n * k;
    transpose_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, s>>>(n, k, V, Vt);
    return cudaGetLastError();
}

}  // namespace ocg
