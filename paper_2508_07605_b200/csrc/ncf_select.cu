// Fused NCF imputation + Algorithm-2 selection (SURVEY §8a rows a9 + a10 at
// scale; north star item 2): for every row i of a sparse matrix and a fitted
// NCF model, the completed row is
//     p_ij = r_ij                                   (observed: kept verbatim)
//     p_ij = clamp(mlp([u_i ; v_j]), 0.01, 1.25)    (NcfModel::predict, cfcomplete.cpp:47-58)
// (cf::complete's imputation, cfcomplete.cpp:208-211), and policy::select_caps
// (policy.cpp:17-64) picks the row's setting.  The completed matrix is never
// materialised (a test hook writes requested rows).
//
// Passes:
//  * ncf_base_kernel (thread per row): the baseline p_{i,n-1} when it is not
//    observed — FP64, lane-exact (both modes), so every row's thresholds use
//    the reference's own baseline value.
//  * ncf_rowprep_kernel (warp per row): the row's error status (row without
//    observations -> invalid_argument, cfcomplete.cpp:199-205; cold app ->
//    runtime_error, :50-52), the exact float threshold of loss <= gamma, and
//    every observed cell + the baseline cell evaluated in FP64 (policy.cpp:30-60).
//  * dense pass over the unobserved cells, two precisions:
//      EXACT (ncf_exact_kernel): FP64 in the operation order of the chosen
//        reference kernel lane (lane_ops.cuh) with glibc's exp — predictions and
//        selections bit-identical to the reference.  Warp per row, lane per cell;
//        the u-part of layer 0's dot is precomputed once per row (the lane's
//        partial sums after the first ka inputs are exactly the state the
//        reference's dot has reached there).
//      FAST (ncf_fast_kernel): FP32 + tensor cores.  Layer 0 is additive,
//        W0 [u;v] + b0 = A_i + B_j, and its exp factorises, exp(A+B) =
//        exp(A) exp(B), so SELU needs no MUFU op; the 32 -> 16 layer runs on
//        the 5th-gen tensor cores (tcgen05.mma kind::f16, M = 128 rows x N = 16
//        x K = 32, FP16 hi/lo split: Ah.Wh + Ah.Wl + (-Al).(-Wh), FP32 accumulate
//        in TMEM); B_j tiles arrive by TMA.  |dp|/p ~ 1e-6; selections exact
//        wherever the row's margin exceeds that.
#include <algorithm>
#include <type_traits>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "../../include/ocg.h"
#include "lane_ops.cuh"
#include "ncf_select.h"
#include "ocg_common.cuh"
#include "select_dev.cuh"

namespace ocg {

namespace {

constexpr float kBandF = 1.0f + 0x1p-18f;

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ double clamp_perf(double y) { return y < 0.01 ? 0.01 : (1.25 < y ? 1.25 : y); }

// loss(p) = fl(1 - fl(p / p_base)) <= gamma  (policy.cpp:34-35)
__device__ __forceinline__ bool valid_exact(double p, double p_base, double gamma) {
    return !(dsub(1.0, ddiv(p, p_base)) > gamma);
}
__device__ __forceinline__ double next_up(double x) { return u2d(d2u(x) + 1); }
__device__ __forceinline__ double next_down(double x) { return u2d(d2u(x) - 1); }
// smallest double p with valid_exact(p) (valid is monotone in p)
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

struct Best {
    double s, p;
    int j, sum;
};
// 4-key order of select_caps (policy.cpp:44-52): saving desc, perf desc, c+g asc, column asc
__device__ __forceinline__ bool better(double s, double p, int sum, int j, const Best& b) {
    if (b.j < 0) return true;
    if (s != b.s) return s > b.s;
    if (p != b.p) return p > b.p;
    if (sum != b.sum) return sum < b.sum;
    return j < b.j;
}
__device__ __forceinline__ void merge(Best& b, const Best& o) {
    if (o.j >= 0 && better(o.s, o.p, o.sum, o.j, b)) b = o;
}
// FP64 evaluation of a valid cell (policy.cpp:37-38) + the 4-key compare; out of line for the
// dense kernels (a rare band path), inline for the observed-cell pass
__device__ __forceinline__ void exact_consider_inl(Best& b, double pd, int cs, int j, double e_base) {
    const double e_pred = ddiv(static_cast<double>(cs), pd);
    const double s = ddiv(dsub(e_base, e_pred), e_base);
    if (better(s, pd, cs, j, b)) b = Best{s, pd, j, cs};
}
__device__ __noinline__ void exact_consider(Best* b, double pd, int cs, int j, double e_base) {
    exact_consider_inl(*b, pd, cs, j, e_base);
}
__device__ __forceinline__ Best warp_best(Best b) {
    for (int off = 16; off > 0; off >>= 1) {
        Best o;
        o.s = __shfl_xor_sync(0xffffffffu, b.s, off);
        o.p = __shfl_xor_sync(0xffffffffu, b.p, off);
        o.j = __shfl_xor_sync(0xffffffffu, b.j, off);
        o.sum = __shfl_xor_sync(0xffffffffu, b.sum, off);
        merge(b, o);
    }
    return b;
}
__device__ __forceinline__ int capsum(const NcfSelArgs& a, int64_t j) {
    const int64_t ci = j / a.ngpu;
    return a.cpu[ci] + a.gpu[j - ci * a.ngpu];
}

// generic FP64 lane-exact forward (nnkit.cpp:74-89) of one cell, any layer stack
// within the per-app limits (local arrays); W = the flat MLP block (W0 b0 W1 b1 ...)
template <int LANE, class Tab>
__device__ double cell_generic(const NcfSelArgs& g, const double* W, const double* u, const double* v, Tab tab) {
    double a[64], z[64];
    for (int q = 0; q < g.ka; ++q) a[q] = u[q];
    for (int q = 0; q < g.ks; ++q) a[g.ka + q] = v[q];
    const int64_t base = g.off_w[0];
    for (int l = 0; l < g.L; ++l) {
        const int in = g.dims[l], outd = g.dims[l + 1];
        const double* Wl = W + (g.off_w[l] - base);
        const double* bl = W + (g.off_b[l] - base);
        for (int o = 0; o < outd; ++o) z[o] = dadd(LaneOps<LANE>::dot(Wl + o * in, a, in), bl[o]);
        const bool hidden = l + 1 < g.L;
        for (int o = 0; o < outd; ++o) {
            double val = z[o], gf;
            if (hidden) selu_fwd(z[o], val, gf, tab);
            a[o] = val;
        }
    }
    return clamp_perf(a[0]);
}

// compile-time dot over a register array, the lane's FP order (kernels_*.cpp dot)
template <int LANE, int N>
__device__ __forceinline__ double dotN(const double* w, const double* x) {
    if constexpr (LANE == 0) {
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < N; ++i) acc = dadd(acc, dmul(w[i], x[i]));
        return acc;
    } else {
        static_assert(N % 4 == 0, "full chunks only");
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
        for (int i = 0; i < N; i += 4) {
            a0 = dfma(w[i], x[i], a0);
            a1 = dfma(w[i + 1], x[i + 1], a1);
            a2 = dfma(w[i + 2], x[i + 2], a2);
            a3 = dfma(w[i + 3], x[i + 3], a3);
        }
        return dadd(dadd(dadd(a0, a2), dadd(a1, a3)), 0.0);  // + the (empty) scalar tail
    }
}

// ============================================================ base kernel
// p_{i,n-1} for rows whose baseline is unobserved (thread per row).
template <int LANE>
__global__ void __launch_bounds__(128) ncf_base_kernel(NcfSelArgs a) {
    extern __shared__ __align__(16) double sw[];  // MLP block | v_{n-1} | exp table
    const int64_t nw = a.off_b[a.L - 1] + a.dims[a.L] - a.off_w[0];
    double* sv = sw + nw;
    uint64_t* stab = reinterpret_cast<uint64_t*>(sv + a.ks);
    for (int64_t e = threadIdx.x; e < nw; e += blockDim.x) sw[e] = a.P[a.off_w[0] + e];
    for (int e = threadIdx.x; e < a.ks; e += blockDim.x) sv[e] = a.P[a.set_off + (a.n - 1) * a.ks + e];
    for (int e = threadIdx.x; e < 256; e += blockDim.x) stab[e] = exp_tab(e);
    __syncthreads();
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= a.m) return;
    const int64_t rb = a.row_ptr[i], re = a.row_ptr[i + 1];
    if (re > rb && a.col[re - 1] == a.n - 1) return;  // observed baseline: the row prep takes it verbatim
    a.rows[i].pbase = cell_generic<LANE>(a, sw, a.P + i * a.ka, sv, ExpTabPtr{stab});
}

// ======================================================== row prep kernel
// warp per row: status, thresholds, observed cells + the baseline cell (exact FP64)
__global__ void __launch_bounds__(256) ncf_rowprep_kernel(NcfSelArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    const int64_t n = a.n;
    for (int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < a.m; i += nwarps) {
        const int64_t rb = a.row_ptr[i], re = a.row_ptr[i + 1];
        const int64_t cnt = re - rb;
        NcfRowState st{};
        st.best_j = -1;
        st.status = OCG_OK;
        if (cnt <= 0) st.status = OCG_E_INVALID;                          // cfcomplete.cpp:199-205
        else if (cnt < n && !a.app_seen[i]) st.status = OCG_E_COLD;      // :50-52 (a cell needs predict)
        const bool base_obs = cnt > 0 && a.col[re - 1] == n - 1;
        const double pbase = base_obs ? a.val[re - 1] : (st.status == OCG_OK ? a.rows[i].pbase : 1.0);
        st.pbase = pbase;
        const double thr = valid_threshold(pbase, a.gamma);
        // valid is monotone in p, so a verified threshold turns each cell's exact test (an FP64
        // divide) into one compare
        st.thr = thr;
        st.thr_ok = valid_exact(thr, pbase, a.gamma) && !valid_exact(next_down(thr), pbase, a.gamma) ? 1 : 0;
        float f = static_cast<float>(thr);
        if (static_cast<double>(f) < thr) f = __uint_as_float(__float_as_uint(f) + 1u);
        st.fthr = f;
        st.lov = 0.01 >= thr ? 1 : 0;
        // observed cells (the baseline cell included when observed), then the predicted baseline
        Best b{0.0, 0.0, -1, 0};
        int oc = 0;
        for (int64_t e = rb + lane; e < re; e += 32) {
            const int j = a.col[e];
            const double p = a.val[e];
            if (st.thr_ok ? !(p >= thr) : !valid_exact(p, pbase, a.gamma)) continue;
            ++oc;
            exact_consider_inl(b, p, capsum(a, j), j, a.e_base);
        }
        b = warp_best(b);
        for (int off = 16; off > 0; off >>= 1) oc += __shfl_xor_sync(0xffffffffu, oc, off);
        if (!base_obs && st.status == OCG_OK) {  // the predicted baseline cell: loss 0, always valid
            ++oc;
            if (lane == 0) exact_consider_inl(b, pbase, capsum(a, n - 1), static_cast<int>(n - 1), a.e_base);
        }
        st.best_s = b.s;
        st.best_p = b.p;
        st.best_j = b.j;
        st.best_sum = b.sum;
        st.ocnt = oc;
        if (lane == 0) {
            a.rows[i] = st;
            if (st.status != OCG_OK) atomicOr(a.err, 1 << st.status);
        }
    }
}

// completed-row hook: observed values + baseline of the listed rows
__global__ void ncf_list_observed_kernel(NcfSelArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (r >= a.nlist) return;
    const int64_t i = a.row_list[r];
    const int64_t rb = a.row_ptr[i], re = a.row_ptr[i + 1];
    double* out = a.completed + r * a.n;
    for (int64_t e = rb + lane; e < re; e += 32) out[a.col[e]] = a.val[e];
    if (lane == 0 && !(re > rb && a.col[re - 1] == a.n - 1)) out[a.n - 1] = a.rows[i].pbase;
}

// final merge of a row's dense best with its observed best
__device__ __forceinline__ void write_row(const NcfSelArgs& a, int64_t i, const NcfRowState& st, Best b, int cnt) {
    merge(b, Best{st.best_s, st.best_p, st.best_j, st.best_sum});
    if (st.status != OCG_OK) b.j = -1;
    a.idx[i] = b.j;
    a.saving[i] = b.j >= 0 ? b.s : 0.0;
    a.loss[i] = b.j >= 0 ? dsub(1.0, ddiv(b.p, st.pbase)) : 0.0;
    a.ncand[i] = st.status == OCG_OK ? cnt + st.ocnt : 0;
}

// ===================================================== exact dense kernel
// warp per row, lane per column.  Reference default layer stack (2k -> 32 -> 16
// -> 1, SELU) with k = ka = ks; layer 0's dot continues from the row state
// (the lane's partial sums over u_i), layer 1 is accumulated as layer 0's
// outputs stream out (same per-accumulator order as the reference's dot).
constexpr int kExW = 4;  // warps per CTA

template <int LANE, int K, bool LIST>
__global__ void __launch_bounds__(kExW * 32) ncf_exact_kernel(NcfSelArgs a) {
    constexpr int H0 = kNsH0, H1 = kNsH1, IN = 2 * K, NACC = LANE == 0 ? 1 : 4;
    extern __shared__ __align__(16) double sh[];
    // W0 v-part transposed per output: wv[o][q] = W0[o][K + q]; then b0, W1, b1, W2, b2
    double* wv = sh;
    double* b0 = wv + H0 * K;
    double* w1 = b0 + H0;
    double* b1 = w1 + H1 * H0;
    double* w2 = b1 + H1;
    double* b2 = w2 + H1;
    uint64_t* stab = reinterpret_cast<uint64_t*>(b2 + 2);
    double* rstate = reinterpret_cast<double*>(stab + 256);  // [kExW][H0 * NACC]
    uint32_t* obits = reinterpret_cast<uint32_t*>(rstate + kExW * H0 * NACC);  // [kExW][n/32 + 1]
    const int64_t n = a.n;
    const int nwords = static_cast<int>((n + 31) >> 5);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const double* P = a.P;
    const int64_t ow = a.off_w[0];
    for (int e = tid; e < H0 * K; e += blockDim.x) {
        const int o = e / K, q = e - o * K;
        wv[e] = P[ow + o * IN + K + q];
    }
    for (int e = tid; e < H0; e += blockDim.x) b0[e] = P[a.off_b[0] + e];
    for (int e = tid; e < H1 * H0; e += blockDim.x) w1[e] = P[a.off_w[1] + e];
    for (int e = tid; e < H1; e += blockDim.x) {
        b1[e] = P[a.off_b[1] + e];
        w2[e] = P[a.off_w[2] + e];
    }
    if (tid == 0) b2[0] = P[a.off_b[2]];
    for (int e = tid; e < 256; e += blockDim.x) stab[e] = exp_tab(e);
    __syncthreads();
    const ExpTabPtr tab{stab};
    double* myst = rstate + warp * H0 * NACC;
    uint32_t* mybits = obits + warp * (nwords + 1);
    const int64_t nrows = LIST ? a.nlist : a.m;
    const int64_t gw = static_cast<int64_t>(gridDim.x) * kExW;
    for (int64_t r = static_cast<int64_t>(blockIdx.x) * kExW + warp; r < nrows; r += gw) {
        const int64_t i = LIST ? a.row_list[r] : r;
        const NcfRowState st = a.rows[i];
        if (st.status != OCG_OK) {
            if (!LIST && lane == 0) write_row(a, i, st, Best{0.0, 0.0, -1, 0}, 0);
            continue;
        }
        // row state: the lane's partial sums of W0[o] . x over x[0..K) = u_i
        const double* u = P + i * K;
        for (int e = lane; e < H0 * NACC; e += 32) {
            const int o = e / NACC, c = e - o * NACC;
            const double* w = P + ow + o * IN;
            double acc = 0.0;
            if (LANE == 0) {
                for (int q = 0; q < K; ++q) acc = dadd(acc, dmul(w[q], u[q]));
            } else {
                for (int q = c; q < K; q += 4) acc = dfma(w[q], u[q], acc);
            }
            myst[e] = acc;
        }
        // observed columns of the row (+ the baseline column) as a bit set
        for (int w = lane; w < nwords; w += 32) mybits[w] = 0u;
        __syncwarp();
        const int64_t rb = a.row_ptr[i], re = a.row_ptr[i + 1];
        for (int64_t e = rb + lane; e < re; e += 32) {
            const int j = a.col[e];
            atomicOr(mybits + (j >> 5), 1u << (j & 31));
        }
        __syncwarp();
        if (lane == 0) mybits[(n - 1) >> 5] |= 1u << ((n - 1) & 31);
        __syncwarp();
        Best b{0.0, 0.0, -1, 0};
        int cnt = 0;
        for (int64_t j = lane; j < n; j += 32) {
            if ((mybits[j >> 5] >> (j & 31)) & 1u) continue;
            double v[K];
            const double* vp = P + a.set_off + j * K;
#pragma unroll
            for (int q = 0; q < K; q += 2) {
                const double2 t = *reinterpret_cast<const double2*>(vp + q);
                v[q] = t.x;
                v[q + 1] = t.y;
            }
            double h1[H1];
            if constexpr (K <= 32) {
                // layer 0 (continued over v) -> SELU into registers, then layer 1 one output at a
                // time: v's registers die as h0's fill, and layer 1 needs 4 accumulators instead of
                // 64 -- the same operation order (dotN = the lane's dot), half the registers
                double h0[H0];
#pragma unroll
                for (int o = 0; o < H0; ++o) {
                    const double* w = wv + o * K;
                    double z;
                    if (LANE == 0) {
                        double acc = myst[o];
#pragma unroll
                        for (int q = 0; q < K; ++q) acc = dadd(acc, dmul(w[q], v[q]));
                        z = acc;
                    } else {
                        double c0 = myst[4 * o], c1 = myst[4 * o + 1], c2 = myst[4 * o + 2], c3 = myst[4 * o + 3];
#pragma unroll
                        for (int q = 0; q < K; q += 4) {
                            c0 = dfma(w[q], v[q], c0);
                            c1 = dfma(w[q + 1], v[q + 1], c1);
                            c2 = dfma(w[q + 2], v[q + 2], c2);
                            c3 = dfma(w[q + 3], v[q + 3], c3);
                        }
                        z = dadd(dadd(dadd(c0, c2), dadd(c1, c3)), 0.0);  // IN % 4 == 0: empty tail
                    }
                    z = dadd(z, b0[o]);
                    double gf;
                    selu_fwd(z, h0[o], gf, tab);
                }
#pragma unroll
                for (int p = 0; p < H1; ++p) {
                    const double z = dadd(dotN<LANE, H0>(w1 + p * H0, h0), b1[p]);
                    double gf;
                    selu_fwd(z, h1[p], gf, tab);
                }
            } else {
                // layer 0 (continued over v) -> SELU -> streamed into layer 1's accumulators
                double acc1[H1][NACC];
#pragma unroll
                for (int p = 0; p < H1; ++p)
#pragma unroll
                    for (int c = 0; c < NACC; ++c) acc1[p][c] = 0.0;
#pragma unroll 1
                for (int o0 = 0; o0 < H0; o0 += NACC) {
#pragma unroll
                    for (int oo = 0; oo < NACC; ++oo) {
                        const int o = o0 + oo;
                        const double* w = wv + o * K;
                        double z;
                        if (LANE == 0) {
                            double acc = myst[o];
#pragma unroll
                            for (int q = 0; q < K; ++q) acc = dadd(acc, dmul(w[q], v[q]));
                            z = acc;
                        } else {
                            double c0 = myst[4 * o], c1 = myst[4 * o + 1], c2 = myst[4 * o + 2], c3 = myst[4 * o + 3];
#pragma unroll
                            for (int q = 0; q < K; q += 4) {
                                c0 = dfma(w[q], v[q], c0);
                                c1 = dfma(w[q + 1], v[q + 1], c1);
                                c2 = dfma(w[q + 2], v[q + 2], c2);
                                c3 = dfma(w[q + 3], v[q + 3], c3);
                            }
                            z = dadd(dadd(dadd(c0, c2), dadd(c1, c3)), 0.0);  // IN % 4 == 0: empty tail
                        }
                        z = dadd(z, b0[o]);
                        double h, gf;
                        selu_fwd(z, h, gf, tab);
#pragma unroll
                        for (int p = 0; p < H1; ++p) {
                            if (LANE == 0) acc1[p][0] = dadd(acc1[p][0], dmul(w1[p * H0 + o], h));
                            else acc1[p][oo] = dfma(w1[p * H0 + o], h, acc1[p][oo]);
                        }
                    }
                }
#pragma unroll
                for (int p = 0; p < H1; ++p) {
                    double z = LANE == 0 ? acc1[p][0]
                                         : dadd(dadd(dadd(acc1[p][0], acc1[p][NACC > 2 ? 2 : 0]),
                                                     dadd(acc1[p][NACC > 1 ? 1 : 0], acc1[p][NACC > 3 ? 3 : 0])),
                                                0.0);
                    z = dadd(z, b1[p]);
                    double gf;
                    selu_fwd(z, h1[p], gf, tab);
                }
            }
            const double pd = clamp_perf(dadd(dotN<LANE, H1>(w2, h1), b2[0]));
            if (LIST) a.completed[r * n + j] = pd;
            if (st.thr_ok ? !(pd >= st.thr) : !valid_exact(pd, st.pbase, a.gamma)) continue;
            ++cnt;
            exact_consider(&b, pd, capsum(a, j), static_cast<int>(j), a.e_base);
        }
        if (!LIST) {
            b = warp_best(b);
            for (int off = 16; off > 0; off >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
            if (lane == 0) write_row(a, i, st, b, cnt);
        }
        __syncwarp();
    }
}

// generic-shape exact dense kernel (any layer stack within the per-app limits)
template <int LANE, bool LIST>
__global__ void __launch_bounds__(kExW * 32) ncf_exact_generic_kernel(NcfSelArgs a) {
    extern __shared__ __align__(16) double sh[];
    const int64_t nw = a.off_b[a.L - 1] + a.dims[a.L] - a.off_w[0];
    double* sw = sh;
    uint64_t* stab = reinterpret_cast<uint64_t*>(sw + nw);
    uint32_t* obits = reinterpret_cast<uint32_t*>(stab + 256);
    const int64_t n = a.n;
    const int nwords = static_cast<int>((n + 31) >> 5);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int64_t e = tid; e < nw; e += blockDim.x) sw[e] = a.P[a.off_w[0] + e];
    for (int e = tid; e < 256; e += blockDim.x) stab[e] = exp_tab(e);
    __syncthreads();
    uint32_t* mybits = obits + warp * (nwords + 1);
    const int64_t nrows = LIST ? a.nlist : a.m;
    const int64_t gw = static_cast<int64_t>(gridDim.x) * kExW;
    for (int64_t r = static_cast<int64_t>(blockIdx.x) * kExW + warp; r < nrows; r += gw) {
        const int64_t i = LIST ? a.row_list[r] : r;
        const NcfRowState st = a.rows[i];
        if (st.status != OCG_OK) {
            if (!LIST && lane == 0) write_row(a, i, st, Best{0.0, 0.0, -1, 0}, 0);
            continue;
        }
        for (int w = lane; w < nwords; w += 32) mybits[w] = 0u;
        __syncwarp();
        const int64_t rb = a.row_ptr[i], re = a.row_ptr[i + 1];
        for (int64_t e = rb + lane; e < re; e += 32) atomicOr(mybits + (a.col[e] >> 5), 1u << (a.col[e] & 31));
        __syncwarp();
        if (lane == 0) mybits[(n - 1) >> 5] |= 1u << ((n - 1) & 31);
        __syncwarp();
        Best b{0.0, 0.0, -1, 0};
        int cnt = 0;
        for (int64_t j = lane; j < n; j += 32) {
            if ((mybits[j >> 5] >> (j & 31)) & 1u) continue;
            const double pd = cell_generic<LANE>(a, sw, a.P + i * a.ka, a.P + a.set_off + j * a.ks, ExpTabPtr{stab});
            if (LIST) a.completed[r * n + j] = pd;
            if (st.thr_ok ? !(pd >= st.thr) : !valid_exact(pd, st.pbase, a.gamma)) continue;
            ++cnt;
            exact_consider(&b, pd, capsum(a, j), static_cast<int>(j), a.e_base);
        }
        if (!LIST) {
            b = warp_best(b);
            for (int off = 16; off > 0; off >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
            if (lane == 0) write_row(a, i, st, b, cnt);
        }
        __syncwarp();
    }
}

// ====================================================== fast path: prep
// A_i = W0[:, :ka] . u_i + b0 and B_j = W0[:, ka:] . v_j (FP64, rounded once),
// their exps, and the max magnitudes that set the FP16 split's scale.
// warp max of |v| first, then one atomic per warp (a single-address atomic per thread
// serialises ~32M updates at C2 in L2)
__device__ __forceinline__ void atomic_max_f(unsigned* addr, float v) {
    unsigned b = __float_as_uint(fabsf(v));  // non-negative floats order like their bits
    b = __reduce_max_sync(__activemask(), b);
    if ((threadIdx.x & 31) == (__ffs(__activemask()) - 1)) atomicMax(addr, b);
}

// warp per row, lane o = layer-0 output; W0[:, :ka] staged transposed in shared memory
// (Wt[q][o]: the 32 lanes read 32 consecutive doubles, not 32 rows 512 B apart)
__global__ void __launch_bounds__(256) ncf_fast_rows_kernel(NcfFastArgs f) {
    const NcfSelArgs& a = f.s;
    extern __shared__ double wt[];  // [ka][32]
    for (int e = threadIdx.x; e < a.ka * kNsH0; e += blockDim.x) {
        const int q = e / kNsH0, o = e - q * kNsH0;
        wt[e] = a.P[a.off_w[0] + static_cast<int64_t>(o) * (a.ka + a.ks) + q];
    }
    __syncthreads();
    const int o = threadIdx.x & 31;
    const double bo = a.P[a.off_b[0] + o];
    float amax = 0.0f;
    const int64_t nw = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < a.m; i += nw) {
        const double* u = a.P + i * a.ka;
        double acc = bo;
        for (int q = 0; q < a.ka; ++q) acc = fma(wt[q * kNsH0 + o], u[q], acc);
        const float av = static_cast<float>(acc);
        f.A[i * kNsH0 + o] = av;
        f.EA[i * kNsH0 + o] = static_cast<float>(exp(acc));
        amax = fmaxf(amax, fabsf(av));
    }
    atomic_max_f(&f.scale->maxA, amax);
}

__global__ void ncf_fast_cols_kernel(NcfFastArgs f) {
    const NcfSelArgs& a = f.s;
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;  // (column, o)
    if (t >= a.n * kNsH0) return;
    const int64_t j = t >> 5;
    const int o = static_cast<int>(t & 31);
    const double* w = a.P + a.off_w[0] + static_cast<int64_t>(o) * (a.ka + a.ks) + a.ka;
    const double* v = a.P + a.set_off + j * a.ks;
    double acc = 0.0;
    for (int q = 0; q < a.ks; ++q) acc = fma(w[q], v[q], acc);
    const float bv = static_cast<float>(acc);
    float* col = f.BE + j * kNsColFloats;
    col[o] = bv;  // scaled by s_h in ncf_fast_scale_kernel
    col[32 + o] = static_cast<float>(exp(acc));
    if (o == 0) {
        col[64] = static_cast<float>(capsum(a, j));
        col[65] = col[66] = col[67] = 0.0f;
    }
    atomic_max_f(&f.scale->maxB, bv);
}

__global__ void ncf_fast_scale_kernel(NcfFastArgs f) {
    const NcfSelArgs& a = f.s;
    const float ma = __uint_as_float(f.scale->maxA), mb = __uint_as_float(f.scale->maxB);
    // |z| <= max|A| + max|B|; SELU' output lies in [-alpha, max z]
    const float bound = fmaxf(ma + mb, 1.6732632423543772f);
    int e;
    frexpf(bound, &e);  // bound < 2^e
    const int eh = 14 - e;
    const float s_h = ldexpf(1.0f, eh);
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < a.n * kNsH0) {
        const int64_t j = t >> 5;
        f.BE[j * kNsColFloats + (t & 31)] *= s_h;
    }
    if (t == 0) {
        f.scale->s_h = s_h;
        f.scale->sd = ldexpf(1.0f, -(eh + f.e_w)) * 1.4426950408889634f;  // z1 log2(e) per accumulator unit
        f.scale->alpha_s = 1.6732632423543772f * s_h;
        // exp(A) exp(B) needs both factors finite and normal
        f.scale->bad = !(ma < 80.0f && mb < 80.0f) ? 1 : 0;
    }
}

// ====================================================== fast path: dense
// PTX wrappers (tcgen05 / TMA / mbarrier)
__device__ __forceinline__ uint32_t saddr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(saddr(b)), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            saddr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(saddr(bar))
        : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// SMEM matrix descriptor, K-major, no swizzle: 8-row x 16-byte core matrices; lbo = byte
// step between the two K-adjacent core matrices, sbo = byte step between 8-row groups
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return static_cast<uint64_t>((addr & 0x3FFFFu) >> 4) | (static_cast<uint64_t>(lbo >> 4) << 16) |
           (static_cast<uint64_t>(sbo >> 4) << 32) | (1ull << 46);
}
// kind::f16 instruction descriptor: F16 x F16 -> F32, both K-major, M = 128, N = 16
constexpr uint32_t kIdesc = (1u << 4) | ((16u >> 3) << 17) | ((128u >> 4) << 24);
__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t ad, uint64_t bd, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(
            d_tmem),
        "l"(ad), "l"(bd), "r"(kIdesc), "r"(accum)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&d)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int q = 0; q < 16; ++q) d[q] = __uint_as_float(r[q]);
}
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }

constexpr int kFT = 128;                       // threads = rows per CTA = UMMA M = TMEM lanes
constexpr int kABytes = 128 * 32 * 2;          // one operand (hi or lo): 128 rows x K 32 fp16
constexpr int kBufBytes = 2 * kABytes;         // hi + lo
constexpr int kStageBytes = kNsTileCols * kNsColFloats * 4;
constexpr int kWImgBytes = 3072;  // W1 image: lambda W1 s_w as fp16 hi | lo | -hi (1 KB each)
constexpr int kFastSmem = 2 * kBufBytes + 2 * kStageBytes + kWImgBytes + 64;

// operand byte offset of (row t, 8-element chunk q) inside one hi/lo operand:
// slab s = q >> 1 (K 16s..16s+15) at s * 4096; within a slab, 8-row group g at g * 256,
// K-chunk c = q & 1 at c * 128, row r at r * 16
__device__ __forceinline__ uint32_t aoff(int t, int q) {
    return static_cast<uint32_t>((q >> 1) * 4096 + (t >> 3) * 256 + (q & 1) * 128 + (t & 7) * 16);
}

template <bool LIST>
__global__ void __launch_bounds__(kFT, 4) ncf_fast_kernel(const __grid_constant__ CUtensorMap tmap, NcfFastArgs f) {
    const NcfSelArgs& a = f.s;
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* abuf = sm;                                                  // [2][hi|lo]
    float* stage = reinterpret_cast<float*>(sm + 2 * kBufBytes);         // [2][kNsTileCols][68]
    uint8_t* wimg = sm + 2 * kBufBytes + 2 * kStageBytes;                // W1 hi | lo | -hi (3 KB)
    uint64_t* bars = reinterpret_cast<uint64_t*>(wimg + kWImgBytes);     // [0,1] TMA, [2,3] MMA
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 4);
    const int t = threadIdx.x, warp = t >> 5;
    const int64_t n = a.n;
    const int ntiles = static_cast<int>((n + kNsTileCols - 1) / kNsTileCols);

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(saddr(tslot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (t == 0) {
        for (int q = 0; q < 4; ++q) mbar_init(bars + q, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    reinterpret_cast<uint4*>(wimg)[t] = f.w1img[t];  // 192 x 16 B
    if (t < 64) reinterpret_cast<uint4*>(wimg)[128 + t] = f.w1img[128 + t];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const NcfFastScale sc = *f.scale;

    const int64_t nrows = LIST ? a.nlist : a.m;
    const int64_t r = static_cast<int64_t>(blockIdx.x) * kFT + t;
    const bool live = r < nrows;
    const int64_t i = live ? (LIST ? a.row_list[r] : r) : 0;
    NcfRowState st = a.rows[i];
    const bool work = live && st.status == OCG_OK && !sc.bad;
    // row operands: s_h A_i and exp(A_i)
    float As[32], EA[32];
#pragma unroll
    for (int q = 0; q < 32; q += 4) {
        const float4 x = work ? *reinterpret_cast<const float4*>(f.A + i * 32 + q) : make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 y = work ? *reinterpret_cast<const float4*>(f.EA + i * 32 + q) : make_float4(0.f, 0.f, 0.f, 0.f);
        As[q] = x.x * sc.s_h;
        As[q + 1] = x.y * sc.s_h;
        As[q + 2] = x.z * sc.s_h;
        As[q + 3] = x.w * sc.s_h;
        EA[q] = y.x * sc.alpha_s;  // alpha s_h exp(A_i): the negative branch is one FFMA per unit
        EA[q + 1] = y.y * sc.alpha_s;
        EA[q + 2] = y.z * sc.alpha_s;
        EA[q + 3] = y.w * sc.alpha_s;
    }
    // observed-column cursor (ascending CSR columns; the thread sweeps j ascending)
    int64_t cur = work ? a.row_ptr[i] : 0;
    const int64_t cend = work ? a.row_ptr[i + 1] : 0;
    int nxt = cur < cend ? a.col[cur] : 0x7fffffff;
    const float fthr = st.fthr;
    const bool lov = st.lov != 0;
    Best best{0.0, 0.0, -1, 0};
    float tbest = INFINITY;  // c/p of the best valid dense cell so far (band anchor)
    if (st.best_j >= 0) tbest = static_cast<float>(st.best_sum) / static_cast<float>(st.best_p);
    float tb = tbest * kBandF;
    int cnt = 0;
    const float sd = sc.sd, as = sc.alpha_s;
    constexpr float kAlphaL = 1.6732632423543772f * 1.4426950408889634f;
    const uint32_t a_base = saddr(abuf), w_base = saddr(wimg);
    const uint64_t adesc0 = umma_desc(a_base, 128, 256), wdesc0 = umma_desc(w_base, 128, 256);

    if (t == 0) {
        mbar_expect_tx(bars + 0, kStageBytes);
        tma_load_2d(stage, &tmap, 0, 0, bars + 0);
        if (ntiles > 1) {
            mbar_expect_tx(bars + 1, kStageBytes);
            tma_load_2d(stage + kNsTileCols * kNsColFloats, &tmap, 0, kNsTileCols, bars + 1);
        }
    }
    uint32_t tph = 0u, mph = 0u;  // mbarrier phase bits per buffer (registers, not a local array)

    float cs_prev = 0.0f;  // c+g of the column whose epilogue is pending (read while its tile is staged)
    auto epilogue = [&](int64_t jc, int b, float csf) {
        mbar_wait(bars + 2 + b, (mph >> b) & 1u);
        mph ^= 1u << b;
        tc_fence_after();
        float d[16];
        tmem_ld16(tmem + ((static_cast<uint32_t>(warp) * 32u) << 16) + static_cast<uint32_t>(b * 16), d);
        tc_fence_before();
        float out = f.b2;
#pragma unroll
        for (int p = 0; p < 16; ++p) {
            // in log2 units: zl = z1 log2(e) (sd and b1 carry the factor), hl = SELU(z1)/lambda log2(e),
            // and w2 carries lambda ln(2)
            const float zl = fmaf(d[p], sd, f.b1[p]);
            const float e = ex2_approx(zl);
            const float hl = zl > 0.0f ? zl : fmaf(kAlphaL, e, -kAlphaL);
            out = fmaf(f.w2[p], hl, out);
        }
        const bool obs = jc == nxt;
        if (obs) {
            ++cur;
            nxt = cur < cend ? a.col[cur] : 0x7fffffff;
        }
        if (!work || obs || jc == n - 1) return;
        const float xm = fminf(out, 1.25f);
        const bool valid = lov || xm >= fthr;
        cnt += valid ? 1 : 0;
        if (LIST) {
            a.completed[r * n + jc] = out < 0.01f ? 0.01 : static_cast<double>(xm);
        }
        if (valid && csf <= tb * fmaxf(xm, 0.01f)) {
            const double pd = out <= 0.01f ? 0.01 : static_cast<double>(xm);
            exact_consider(&best, pd, static_cast<int>(csf), static_cast<int>(jc), a.e_base);
            tbest = fminf(tbest, csf / fmaxf(xm, 0.01f));
            tb = tbest * kBandF;
        }
    };

    // one column: operand -> barrier -> MMA issue -> the previous column's epilogue.  The loop
    // runs column pairs so the buffer index B is a compile-time constant (and a tile, 32
    // columns, always starts on an even column)
    auto step = [&](int64_t j, auto Bc) {
        constexpr int b = decltype(Bc)::value;
        const int T = static_cast<int>(j / kNsTileCols), jj = static_cast<int>(j % kNsTileCols), stg = T & 1;
        if (b == 0 && jj == 0) {
            mbar_wait(bars + stg, (tph >> stg) & 1u);
            tph ^= 1u << stg;
        }
        // ---- operand: h'(z) = s_h SELU(z)/lambda for the 32 layer-0 outputs, as fp16 hi/lo
        const float* bcol = stage + stg * kNsTileCols * kNsColFloats + jj * kNsColFloats;
        const float4* bj = reinterpret_cast<const float4*>(bcol);
        const float cs_cur = bcol[64];
        uint8_t* hi = abuf + b * kBufBytes;
        uint8_t* lo = hi + kABytes;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float4 b0 = bj[2 * q], b1v = bj[2 * q + 1], e0 = bj[8 + 2 * q], e1 = bj[8 + 2 * q + 1];
            const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1v.x, b1v.y, b1v.z, b1v.w};
            const float eb[8] = {e0.x, e0.y, e0.z, e0.w, e1.x, e1.y, e1.z, e1.w};
            uint32_t hw[4], lw[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                float h2[2];
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    const int k = 8 * q + 2 * u + v;
                    const float z = As[k] + bb[2 * u + v];
                    h2[v] = z > 0.0f ? z : fmaf(EA[k], eb[2 * u + v], -as);
                }
                const __half2 hh = __floats2half2_rn(h2[0], h2[1]);
                // the split's residual as hi - h (exact), one mixed-precision FHADD per unit; the
                // lo product then runs against -W_hi (third W image block)
                float r0, r1;
                asm("{\n\t.reg .f16 a, b;\n\tmov.b32 {a, b}, %2;\n\tsub.rn.f32.f16 %0, a, %3;\n\t"
                    "sub.rn.f32.f16 %1, b, %4;\n\t}"
                    : "=f"(r0), "=f"(r1)
                    : "r"(h2u(hh)), "f"(h2[0]), "f"(h2[1]));
                const __half2 ll = __floats2half2_rn(r0, r1);
                hw[u] = h2u(hh);
                lw[u] = h2u(ll);
            }
            *reinterpret_cast<uint4*>(hi + aoff(t, q)) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
            *reinterpret_cast<uint4*>(lo + aoff(t, q)) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc_fence_before();
        __syncthreads();
        if (t == 0) {
            tc_fence_after();
            if (b == 0 && jj == 0 && T >= 1 && T + 1 < ntiles) {  // stage (T+1)&1 held tile T-1: all are past it
                const int s2 = (T + 1) & 1;
                mbar_expect_tx(bars + s2, kStageBytes);
                tma_load_2d(stage + s2 * kNsTileCols * kNsColFloats, &tmap, 0, (T + 1) * kNsTileCols, bars + s2);
            }
            // descriptors = the base descriptors + (byte offset >> 4) in the start-address field
            const uint64_t ah = adesc0 + static_cast<uint64_t>((b * kBufBytes) >> 4), al = ah + (kABytes >> 4);
            const uint32_t d = tmem + static_cast<uint32_t>(b * 16);
            // D = Ah.Wh + Ah.Wl + (-Al).(-Wh) over K = 32 (2 slabs of 16); the operand's lo
            // half holds hi - h = -Al
            umma_f16(d, ah, wdesc0, 0u);
            umma_f16(d, ah + (4096 >> 4), wdesc0 + (512 >> 4), 1u);
            umma_f16(d, ah, wdesc0 + (1024 >> 4), 1u);
            umma_f16(d, ah + (4096 >> 4), wdesc0 + (1536 >> 4), 1u);
            umma_f16(d, al, wdesc0 + (2048 >> 4), 1u);
            umma_f16(d, al + (4096 >> 4), wdesc0 + (2560 >> 4), 1u);
            umma_commit(bars + 2 + b);
        }
        __syncwarp();
        if (b == 1 || j > 0) epilogue(j - 1, b ^ 1, cs_prev);
        cs_prev = cs_cur;
    };
    int64_t j = 0;
    for (; j + 1 < n; j += 2) {
        step(j, std::integral_constant<int, 0>{});
        step(j + 1, std::integral_constant<int, 1>{});
    }
    if (j < n) step(j, std::integral_constant<int, 0>{});
    epilogue(n - 1, static_cast<int>((n - 1) & 1), cs_prev);

    if (!LIST && live) {
        if (sc.bad && st.status == OCG_OK) {
            st.status = OCG_E_UNSUPPORTED;
            atomicOr(a.err, 1 << OCG_E_UNSUPPORTED);
        }
        write_row(a, i, st, best, cnt);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem) : "memory");
}

}  // namespace

// ------------------------------------------------------------ launchers
static int64_t mlp_block_len(const NcfSelArgs& a) { return a.off_b[a.L - 1] + a.dims[a.L] - a.off_w[0]; }

bool ncf_fast_shape_ok(const NcfSelArgs& a) {
    return a.L == 3 && a.dims[1] == kNsH0 && a.dims[2] == kNsH1 && a.dims[3] == 1;
}
static bool exact_default(const NcfSelArgs& a) {
    return ncf_fast_shape_ok(a) && a.ka == a.ks && (a.ka == 8 || a.ka == 16 || a.ka == 32 || a.ka == 64);
}

cudaError_t ncf_launch_base(const NcfSelArgs& a, int lane, cudaStream_t s) {
    if (a.m == 0) return cudaSuccess;
    const size_t smem = sizeof(double) * (mlp_block_len(a) + a.ks) + sizeof(uint64_t) * 256;
    const unsigned grid = static_cast<unsigned>((a.m + 127) / 128);
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        kern<<<grid, 128, smem, s>>>(a);
    };
    if (lane == 0) go(ncf_base_kernel<0>);
    else go(ncf_base_kernel<1>);
    return cudaGetLastError();
}

cudaError_t ncf_launch_rowprep(const NcfSelArgs& a, int sm_count, cudaStream_t s) {
    if (a.m > 0) ncf_rowprep_kernel<<<sm_count * 8, 256, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t ncf_launch_list_observed(const NcfSelArgs& a, cudaStream_t s) {
    if (a.row_list && a.nlist > 0)
        ncf_list_observed_kernel<<<static_cast<unsigned>((a.nlist * 32 + 255) / 256), 256, 0, s>>>(a);
    return cudaGetLastError();
}

template <int LANE, int K>
static cudaError_t exact_go(const NcfSelArgs& a, int sm_count, cudaStream_t s) {
    const int nwords = static_cast<int>((a.n + 31) >> 5);
    const int nacc = LANE == 0 ? 1 : 4;
    const size_t smem = sizeof(double) * (kNsH0 * K + kNsH0 + kNsH1 * kNsH0 + 2 * kNsH1 + 2) + sizeof(uint64_t) * 256 +
                        sizeof(double) * kExW * kNsH0 * nacc + sizeof(uint32_t) * kExW * (nwords + 1);
    const bool list = a.row_list != nullptr;
    const int64_t rows = list ? a.nlist : a.m;
    int64_t grid = (rows + kExW - 1) / kExW;
    const int64_t cap = static_cast<int64_t>(sm_count) * 16;
    if (grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        kern<<<static_cast<unsigned>(grid), kExW * 32, smem, s>>>(a);
    };
    if (list) go(ncf_exact_kernel<LANE, K, true>);
    else go(ncf_exact_kernel<LANE, K, false>);
    return cudaGetLastError();
}

template <int LANE>
static cudaError_t exact_generic_go(const NcfSelArgs& a, int sm_count, cudaStream_t s) {
    const int nwords = static_cast<int>((a.n + 31) >> 5);
    const size_t smem = sizeof(double) * mlp_block_len(a) + sizeof(uint64_t) * 256 + sizeof(uint32_t) * kExW * (nwords + 1);
    const bool list = a.row_list != nullptr;
    const int64_t rows = list ? a.nlist : a.m;
    int64_t grid = (rows + kExW - 1) / kExW;
    const int64_t cap = static_cast<int64_t>(sm_count) * 16;
    if (grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        kern<<<static_cast<unsigned>(grid), kExW * 32, smem, s>>>(a);
    };
    if (list) go(ncf_exact_generic_kernel<LANE, true>);
    else go(ncf_exact_generic_kernel<LANE, false>);
    return cudaGetLastError();
}

cudaError_t ncf_launch_exact(const NcfSelArgs& a, int lane, int sm_count, cudaStream_t s) {
    if ((a.row_list ? a.nlist : a.m) == 0) return cudaSuccess;
    if (exact_default(a)) {
        switch (a.ka * 2 + lane) {
            case 16: return exact_go<0, 8>(a, sm_count, s);
            case 17: return exact_go<1, 8>(a, sm_count, s);
            case 32: return exact_go<0, 16>(a, sm_count, s);
            case 33: return exact_go<1, 16>(a, sm_count, s);
            case 64: return exact_go<0, 32>(a, sm_count, s);
            case 65: return exact_go<1, 32>(a, sm_count, s);
            case 128: return exact_go<0, 64>(a, sm_count, s);
            case 129: return exact_go<1, 64>(a, sm_count, s);
            default: break;
        }
    }
    return lane == 0 ? exact_generic_go<0>(a, sm_count, s) : exact_generic_go<1>(a, sm_count, s);
}

cudaError_t ncf_launch_fast_prep(const NcfFastArgs& f, cudaStream_t s) {
    const NcfSelArgs& a = f.s;
    cudaError_t e = cudaMemsetAsync(f.scale, 0, sizeof(NcfFastScale), s);
    if (e != cudaSuccess) return e;
    if (a.m > 0) {
        const int64_t blocks = std::min<int64_t>((a.m + 7) / 8, 148 * 16);
        ncf_fast_rows_kernel<<<static_cast<unsigned>(blocks), 256, sizeof(double) * a.ka * kNsH0, s>>>(f);
    }
    ncf_fast_cols_kernel<<<static_cast<unsigned>((a.n * kNsH0 + 255) / 256), 256, 0, s>>>(f);
    ncf_fast_scale_kernel<<<static_cast<unsigned>((a.n * kNsH0 + 255) / 256), 256, 0, s>>>(f);
    return cudaGetLastError();
}

cudaError_t ncf_launch_fast(const NcfFastArgs& f, const CUtensorMap* tmap, cudaStream_t s) {
    const NcfSelArgs& a = f.s;
    const bool list = a.row_list != nullptr;
    const int64_t rows = list ? a.nlist : a.m;
    if (rows == 0) return cudaSuccess;
    const unsigned grid = static_cast<unsigned>((rows + kFT - 1) / kFT);
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kFastSmem);
        kern<<<grid, kFT, kFastSmem, s>>>(*tmap, f);
    };
    if (list) go(ncf_fast_kernel<true>);
    else go(ncf_fast_kernel<false>);
    return cudaGetLastError();
}

}  // namespace ocg
