// Probe ingest: pred::predict_perf (predictor.cpp:151-157) batched over many
// counter samples — validate_counters (core.cpp:97-106), standardize
// (predictor.cpp:74-79), MlpModel::forward (nnkit.cpp:74-89: 7 -> 64 -> 64 -> 1,
// SELU hidden, identity out) and clamp to [kPredictMin, kPerfMax].  FP64 in
// the operation order of the chosen reference kernel lane, so every estimate
// is bit-identical to the reference's.
//
// One warp per sample: lane o computes outputs o, o+32, ... of a layer as a
// dot product over the previous layer's activations (broadcast from shared
// memory) and the layer's weights stored transposed in shared memory (lanes
// read consecutive addresses).  The MLP weights are staged once per CTA.
#include <cuda_runtime.h>

#include "lane_ops.cuh"
#include "predictor.h"

namespace ocg {

namespace {

constexpr int kWarps = 8;

// dot over i of w[i*ws] * x[i] in the lane's FP order (see LaneOps::dot)
template <int LANE>
__device__ __forceinline__ double dot_strided(const double* w, int ws, const double* x, int n) {
    if (LANE == 0) {
        double acc = 0.0;
        for (int i = 0; i < n; ++i) acc = dadd(acc, dmul(w[i * ws], x[i]));
        return acc;
    }
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int i = 0;
    for (; i + 4 <= n; i += 4) {
        a0 = dfma(w[i * ws], x[i], a0);
        a1 = dfma(w[(i + 1) * ws], x[i + 1], a1);
        a2 = dfma(w[(i + 2) * ws], x[i + 2], a2);
        a3 = dfma(w[(i + 3) * ws], x[i + 3], a3);
    }
    double tail = 0.0;
    const int r = n - i;
    if (r >= 2) {
        tail = dadd(tail, dmul(w[i * ws], x[i]));
        tail = dadd(tail, dmul(w[(i + 1) * ws], x[i + 1]));
        if (r == 3) tail = dfma(w[(i + 2) * ws], x[i + 2], tail);
    } else if (r == 1) {
        tail = dfma(w[i * ws], x[i], tail);
    }
    return dadd(dadd(dadd(a0, a2), dadd(a1, a3)), tail);
}

// dot of N compile-time-sized smem weights (16B aligned when ALIGNED) with a
// register array, in the lane's FP order (LaneOps::dot)
template <int LANE, int N, bool ALIGNED>
__device__ __forceinline__ double dot_regs(const double* w, const double (&x)[N]) {
    // weights are consumed as they arrive (pairs when 16B aligned) so that at
    // most a few weight registers are live next to the 64 activations
    auto wpair = [&](int i, double& w0, double& w1) {
        if constexpr (ALIGNED) {
            const double2 t = *reinterpret_cast<const double2*>(w + i);
            w0 = t.x;
            w1 = t.y;
        } else {
            w0 = w[i];
            w1 = w[i + 1];
        }
    };
    if constexpr (LANE == 0) {
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i + 1 < N; i += 2) {
            double w0, w1;
            wpair(i, w0, w1);
            acc = dadd(acc, dmul(w0, x[i]));
            acc = dadd(acc, dmul(w1, x[i + 1]));
        }
        if constexpr (N % 2) acc = dadd(acc, dmul(w[N - 1], x[N - 1]));
        return acc;
    } else {
        double a[4] = {0.0, 0.0, 0.0, 0.0};
        constexpr int full = N / 4 * 4;
#pragma unroll
        for (int i = 0; i < full; i += 2) {
            double w0, w1;
            wpair(i, w0, w1);
            a[i & 3] = dfma(w0, x[i], a[i & 3]);
            a[(i + 1) & 3] = dfma(w1, x[i + 1], a[(i + 1) & 3]);
        }
        double tail = 0.0;
        constexpr int r = N - full;
        if constexpr (r >= 2) {
            tail = dadd(tail, dmul(w[full], x[full]));
            tail = dadd(tail, dmul(w[full + 1], x[full + 1]));
            if constexpr (r == 3) tail = dfma(w[full + 2], x[full + 2], tail);
        } else if constexpr (r == 1) {
            tail = dfma(w[full], x[full], tail);
        }
        return dadd(dadd(dadd(a[0], a[2]), dadd(a[1], a[3])), tail);
    }
}

// SELU split around the exp table loads: exp_pre(selu_exp_arg(z)) early,
// selu_finish later.  Positive z takes the lambda*z branch (its exp argument is
// a harmless -1); the result equals selu_fwd's bit for bit.
__device__ __forceinline__ double selu_exp_arg(double z) { return z > 0 ? -1.0 : z; }

// per-lane copy of the interleaved exp table (entry i of copy r at (i/2*8 + r)*2 + i%2)
struct ExpTabLanes {
    const uint64_t* p;  // already offset by this lane's copy
    __device__ __forceinline__ void pair(int entry, uint64_t& tail, uint64_t& hi) const {
        const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(p + entry * 16);
        tail = v.x;
        hi = v.y;
    }
};

template <class Tab>
__device__ __forceinline__ double selu_finish(double z, const ExpPre& e, Tab tab) {
    const double ev = exp_post(e, tab);
    return z > 0 ? dmul(kLambda, z) : dmul(kLA, dsub(ev, 1.0));
}

__device__ __forceinline__ bool counter_ok(int q, double v) {
    bool ok = isfinite(v);
    if (q >= 2 && q <= 4) ok = ok && !(v < 0.0);
    if (q >= 5) ok = ok && !(v < 0.0 || v > 1.0);
    return ok;
}

}  // namespace

// The reference predictor's own architecture (PredictorHyper defaults: 7 -> 64
// SELU -> 64 SELU -> 1 identity): one THREAD per sample.  Layer-1 activations
// live in 64 FP64 registers; layer 2 streams its outputs one at a time into
// layer 3's (lane-order) partial sums, so nothing but the weights touches
// shared memory — weight rows are warp-uniform broadcast LDS.128.
constexpr int kFixIn = 7, kFixH = 64;
constexpr int kFixOffB1 = kFixH * kFixIn, kFixOffW2 = kFixOffB1 + kFixH, kFixOffB2 = kFixOffW2 + kFixH * kFixH;
constexpr int kFixOffW3 = kFixOffB2 + kFixH, kFixOffB3 = kFixOffW3 + kFixH, kFixT = kFixOffB3 + 1;
constexpr int kFixThreads = 128, kFixStage = kFixH / 2, kFixTPad = (kFixT + 1) / 2 * 2;
constexpr size_t kFixSmem = sizeof(double) * (kFixTPad + kFixStage * kFixThreads + 256);

template <int LANE>
__global__ void __launch_bounds__(kFixThreads, 3) predict_fixed_kernel(PredGeom g, const double* __restrict__ params,
                                                                        const double* __restrict__ counters,
                                                                        int64_t count, double* __restrict__ out,
                                                                        int* __restrict__ bad) {
    extern __shared__ __align__(16) double sm[];
    for (int e = threadIdx.x; e < kFixT; e += blockDim.x) sm[e] = params[e];
    double* stage = sm + kFixTPad + threadIdx.x;  // this thread's column of the layer-1 stage
    uint64_t* tab_s = reinterpret_cast<uint64_t*>(sm + kFixTPad + kFixStage * kFixThreads);
    for (int e = threadIdx.x; e < 256; e += blockDim.x) tab_s[e] = exp_tab(e);
    const ExpTabPtr tab{tab_s};
    __syncthreads();
    for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < count;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        // opaque per-sample base: keeps ptxas from hoisting the (sample-invariant)
        // weight loads out of the loop into spilled registers
        int zero = 0;
        asm volatile("" : "+r"(zero));
        const double* W = sm + zero;
        // validate_counters (core.cpp:97-106) + standardize (predictor.cpp:74-79)
        double x[kFixIn];
        bool ok = true;
#pragma unroll
        for (int q = 0; q < kFixIn; ++q) {
            const double v = counters[k * kFixIn + q];
            ok = ok && counter_ok(q, v);
            x[q] = ddiv(dsub(v, g.mean[q]), g.std[q]);
        }
        if (!ok) atomicExch(bad, 1);
        // layer 1: a rolled loop (one copy of the exp code — fully unrolled it
        // is 60 KB of straight-line SASS that misses the instruction cache)
        // through a per-thread shared-memory column, half the outputs at a time
        double h[kFixH];
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const int o0 = half * kFixStage;
            double zc = dadd(dot_regs<LANE, kFixIn, false>(W + o0 * kFixIn, x), W[kFixOffB1 + o0]);
            ExpPre ec = exp_pre(selu_exp_arg(zc), tab);
#pragma unroll 1
            for (int j = 0; j < kFixStage; ++j) {
                const int o = o0 + j;
                double zn = 0.0;
                if (j + 1 < kFixStage) zn = dadd(dot_regs<LANE, kFixIn, false>(W + (o + 1) * kFixIn, x), W[kFixOffB1 + o + 1]);
                stage[j * kFixThreads] = selu_finish(zc, ec, tab);
                zc = zn;
                ec = exp_pre(selu_exp_arg(zn), tab);
            }
#pragma unroll
            for (int j = 0; j < kFixStage; ++j) h[o0 + j] = stage[j * kFixThreads];
        }
        // layer-3 dot partials: LANE 1 updates the partial of residue o%4,
        // kept in p0 by rotating (p0..p3) after every output
        double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
        // software-pipelined: output o+1's dot runs while o's exp table loads land
        double zc = dadd(dot_regs<LANE, kFixH, true>(W + kFixOffW2, h), W[kFixOffB2]);
        ExpPre ec = exp_pre(selu_exp_arg(zc), tab);
#pragma unroll 1
        for (int o = 0; o < kFixH; ++o) {
            double zn = 0.0;
            if (o + 1 < kFixH) zn = dadd(dot_regs<LANE, kFixH, true>(W + kFixOffW2 + (o + 1) * kFixH, h), W[kFixOffB2 + o + 1]);
            const double a = selu_finish(zc, ec, tab);
            if constexpr (LANE == 0) {
                p0 = dadd(p0, dmul(W[kFixOffW3 + o], a));
            } else {
                const double t = dfma(W[kFixOffW3 + o], a, p0);
                p0 = p1;
                p1 = p2;
                p2 = p3;
                p3 = t;
            }
            zc = zn;
            ec = exp_pre(selu_exp_arg(zn), tab);
        }
        const double p[4] = {p0, p1, p2, p3};  // kFixH % 4 == 0: back in residue order
        double y = LANE == 0 ? p[0] : dadd(dadd(dadd(p[0], p[2]), dadd(p[1], p[3])), 0.0);
        y = dadd(y, W[kFixOffB3]);
        out[k] = y < 0.01 ? 0.01 : (1.25 < y ? 1.25 : y);  // std::clamp(kPredictMin, kPerfMax)
    }
}


// AVX2 lane, reference architecture: a PAIR of threads per sample.  The lane's
// dot keeps four partial chains (i % 4); thread c of the pair owns chains c and
// c+2, i.e. only the 32 layer-1 activations those chains read (half the
// registers of one-thread-per-sample, so twice the warps to hide latency), and
// the pair combines (a0+a2) + (a1+a3) with one shuffle.  Layer 2 runs two
// outputs per step: thread c applies SELU to output 2u+c only and accumulates
// layer 3's chains of the residues it owns ((2u+c) % 4 alternates c, c+2), so
// no FP64 work is duplicated beyond the standardisation.
constexpr int kPairThreads = 256, kPairSamples = kPairThreads / 2, kPairStage = 16;
// W2 rows permuted: [chains 0,2 (32) | pad 2 | chains 1,3 (32)], stride 66 so the
// two halves a warp reads at once start in different banks
constexpr int kPairRow = 66, kPairHalf = 34;
constexpr int kPairOffW2 = kFixOffW2, kPairW2Size = kFixH * kPairRow;
constexpr int kPairOffB2 = kPairOffW2 + kPairW2Size, kPairOffW3 = kPairOffB2 + kFixH, kPairOffB3 = kPairOffW3 + kFixH;
constexpr int kPairT = (kPairOffB3 + 2) / 2 * 2;
// exp table: 8 interleaved copies of the 128 (tail, sbits) pairs; lane l reads
// copy l % 8, so the 8 lanes of a 128-bit shared-load phase hit 8 distinct
// bank groups whatever entries they need (conflict-free lookups)
constexpr int kPairTab = 8 * 128 * 2;
constexpr size_t kPairSmem = sizeof(double) * (kPairT + kPairStage * kPairThreads) + 8 * kPairTab;

__global__ void __launch_bounds__(kPairThreads, 2) predict_pair_kernel(PredGeom g, const double* __restrict__ params,
                                                                       const double* __restrict__ counters,
                                                                       int64_t count, double* __restrict__ out,
                                                                       int* __restrict__ bad) {
    extern __shared__ __align__(16) double sm[];
    // stage parameters; W2 row o is stored as 32 pairs: for c in {0,1}, q < 16:
    // (w[4q+c], w[4q+c+2]) at o*64 + c*32 + 2q
    for (int e = threadIdx.x; e < kFixT; e += blockDim.x) {
        const double v = params[e];
        if (e >= kFixOffW2 && e < kFixOffB2) {
            const int o = (e - kFixOffW2) / kFixH, i = (e - kFixOffW2) % kFixH;
            const int c = i & 1, r = (i >> 1) & 1, q = i >> 2;
            sm[kPairOffW2 + o * kPairRow + c * kPairHalf + 2 * q + r] = v;
        } else {
            sm[e < kFixOffW2 ? e : e - kFixOffB2 + kPairOffB2] = v;  // W1, b1 | b2, W3, b3
        }
    }
    double* stage = sm + kPairT + threadIdx.x;
    uint64_t* tab_s = reinterpret_cast<uint64_t*>(sm + kPairT + kPairStage * kPairThreads);
    for (int e = threadIdx.x; e < kPairTab; e += blockDim.x) {
        const int entry = e >> 4, half = e & 1;  // e = (entry*8 + copy)*2 + half
        tab_s[e] = exp_tab(2 * entry + half);
    }
    const ExpTabLanes tab{tab_s + 2 * (threadIdx.x & 7)};
    __syncthreads();
    const int c = threadIdx.x & 1;
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * kPairSamples; base < count;
         base += static_cast<int64_t>(gridDim.x) * kPairSamples) {
        const int64_t k = base + (threadIdx.x >> 1);
        const int64_t kk = k < count ? k : count - 1;  // both threads of a pair stay for the shuffles
        int zero = 0;
        asm volatile("" : "+r"(zero));
        const double* W = sm + zero;
        double x[kFixIn];
        bool ok = true;
#pragma unroll
        for (int q = 0; q < kFixIn; ++q) {
            const double v = counters[kk * kFixIn + q];
            ok = ok && counter_ok(q, v);
            x[q] = ddiv(dsub(v, g.mean[q]), g.std[q]);
        }
        if (!ok && c == 0) atomicExch(bad, 1);
        // layer 1, this thread's 32 activations: hh[2q + r] = h[4q + c + 2r]
        double hh[32];
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            auto unit = [&](int m) { return 4 * (m >> 1) + c + 2 * (m & 1); };
            const int m0 = half * kPairStage;
            double zc = dadd(dot_regs<1, kFixIn, false>(W + unit(m0) * kFixIn, x), W[kFixOffB1 + unit(m0)]);
            ExpPre ec = exp_pre(selu_exp_arg(zc), tab);
#pragma unroll 1
            for (int j = 0; j < kPairStage; ++j) {
                const int m = m0 + j;
                double zn = 0.0;
                if (j + 1 < kPairStage) {
                    const int o = unit(m + 1);
                    zn = dadd(dot_regs<1, kFixIn, false>(W + o * kFixIn, x), W[kFixOffB1 + o]);
                }
                stage[j * kPairThreads] = selu_finish(zc, ec, tab);
                zc = zn;
                ec = exp_pre(selu_exp_arg(zn), tab);
            }
#pragma unroll
            for (int j = 0; j < kPairStage; ++j) hh[m0 + j] = stage[j * kPairThreads];
        }
        // layer 2 (+ streamed layer 3), two outputs per step, exp loads pipelined one step
        auto zpair = [&](int o) {
            const double* row = W + kPairOffW2 + o * kPairRow + c * kPairHalf;
            double alo = 0.0, ahi = 0.0;
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const double2 w = *reinterpret_cast<const double2*>(row + 2 * q);
                alo = dfma(w.x, hh[2 * q], alo);
                ahi = dfma(w.y, hh[2 * q + 1], ahi);
            }
            const double mine = dadd(alo, ahi);  // c=0: a0+a2, c=1: a1+a3
            const double other = __shfl_xor_sync(0xffffffffu, mine, 1);
            return dadd(dadd(dadd(mine, other), 0.0), W[kPairOffB2 + o]);  // (a0+a2)+(a1+a3) (+ empty tail) + b
        };
        double qa = 0.0, qb = 0.0;  // layer-3 chains of residues c (qa) and c+2 (qb), rotated per step
        double zc;
        {
            const double z0 = zpair(0), z1 = zpair(1);
            zc = c ? z1 : z0;
        }
        ExpPre ec = exp_pre(selu_exp_arg(zc), tab);
#pragma unroll 1
        for (int u = 0; u < kFixH / 2; ++u) {
            double zn = 0.0;
            if (u + 1 < kFixH / 2) {
                const double z0 = zpair(2 * u + 2), z1 = zpair(2 * u + 3);
                zn = c ? z1 : z0;
            }
            const double a = selu_finish(zc, ec, tab);
            const double t = dfma(W[kPairOffW3 + 2 * u + c], a, qa);
            qa = qb;
            qb = t;
            zc = zn;
            ec = exp_pre(selu_exp_arg(zn), tab);
        }
        const double mine = dadd(qa, qb);  // c=0: p0+p2, c=1: p1+p3
        const double other = __shfl_xor_sync(0xffffffffu, mine, 1);
        double y = dadd(dadd(mine, other), 0.0);
        y = dadd(y, W[kPairOffB3]);
        if (c == 0 && k < count) out[k] = y < 0.01 ? 0.01 : (1.25 < y ? 1.25 : y);
    }
}

bool predictor_is_fixed(const PredGeom& g) {
    return g.L == 3 && g.dims[0] == kFixIn && g.dims[1] == kFixH && g.dims[2] == kFixH && g.dims[3] == 1 &&
           g.acts[0] == 0 && g.acts[1] == 0 && g.acts[2] == 2;
}

template <int LANE>
__global__ void __launch_bounds__(256, 4) predict_perf_kernel(PredGeom g, const double* __restrict__ params,
                                                           const double* __restrict__ counters, int64_t count,
                                                           double* __restrict__ out, int* __restrict__ bad) {
    extern __shared__ __align__(16) double sm[];
    double* Wt = sm;                                  // transposed weights + biases, layer by layer
    double* act = sm + g.T + (threadIdx.x >> 5) * 2 * kPredMaxWidth;  // per warp: 2 x width
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // stage parameters: W_l (out x in, row-major) -> Wt_l (in x out), biases after
    for (int l = 0; l < g.L; ++l) {
        const int in = g.dims[l], outd = g.dims[l + 1];
        for (int e = threadIdx.x; e < in * outd; e += blockDim.x) {
            const int o = e / in, i = e - o * in;
            Wt[g.off_w[l] + i * outd + o] = params[g.off_w[l] + e];
        }
        for (int e = threadIdx.x; e < outd; e += blockDim.x) Wt[g.off_b[l] + e] = params[g.off_b[l] + e];
    }
    __syncthreads();
    for (int64_t k = static_cast<int64_t>(blockIdx.x) * kWarps + warp; k < count;
         k += static_cast<int64_t>(gridDim.x) * kWarps) {
        const double* c = counters + k * 7;
        // validate_counters (core.cpp:97-106) + standardize (predictor.cpp:74-79)
        if (lane < 7) {
            const double v = c[lane];
            if (!counter_ok(lane, v)) atomicExch(bad, 1);
            act[lane] = ddiv(dsub(v, g.mean[lane]), g.std[lane]);
        }
        __syncwarp();
        double* cur = act;
        double* nxt = act + kPredMaxWidth;
        for (int l = 0; l < g.L; ++l) {
            const int in = g.dims[l], outd = g.dims[l + 1];
            for (int o = lane; o < outd; o += 32) {
                double z = dadd(dot_strided<LANE>(Wt + g.off_w[l] + o, outd, cur, in), Wt[g.off_b[l] + o]);
                const int a = g.acts[l];
                if (a == 0) {
                    double gf;
                    selu_fwd(z, z, gf);
                } else if (a == 1) {
                    z = z > 0 ? z : 0.0;
                }
                nxt[o] = z;
            }
            __syncwarp();
            double* t = cur;
            cur = nxt;
            nxt = t;
        }
        if (lane == 0) {
            const double v = cur[0];
            out[k] = v < 0.01 ? 0.01 : (1.25 < v ? 1.25 : v);  // std::clamp(kPredictMin, kPerfMax)
        }
        __syncwarp();
    }
}

size_t predictor_smem_bytes(const PredGeom& g) { return sizeof(double) * (g.T + kWarps * 2 * kPredMaxWidth); }

cudaError_t launch_predict_perf(const PredGeom& g, const double* params, const double* counters, int64_t count,
                                double* out, int* bad, int lane, int sm_count, cudaStream_t s, bool allow_fixed) {
    if (count == 0) return cudaSuccess;
    if (allow_fixed && predictor_is_fixed(g)) {
        const size_t smem = kFixSmem;
        int64_t blocks = (count + kFixThreads - 1) / kFixThreads;
        if (blocks > static_cast<int64_t>(sm_count) * 3) blocks = static_cast<int64_t>(sm_count) * 3;
        auto go = [&](auto kern) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
            kern<<<static_cast<unsigned>(blocks), kFixThreads, smem, s>>>(g, params, counters, count, out, bad);
        };
        if (lane == 0) {
            go(predict_fixed_kernel<0>);
        } else {
            int64_t pb = (count + kPairSamples - 1) / kPairSamples;
            if (pb > static_cast<int64_t>(sm_count) * 2) pb = static_cast<int64_t>(sm_count) * 2;
            cudaFuncSetAttribute(predict_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(kPairSmem));
            predict_pair_kernel<<<static_cast<unsigned>(pb), kPairThreads, kPairSmem, s>>>(g, params, counters, count,
                                                                                          out, bad);
        }
        return cudaGetLastError();
    }
    const size_t smem = predictor_smem_bytes(g);
    int64_t blocks = (count + kWarps - 1) / kWarps;
    if (blocks > static_cast<int64_t>(sm_count) * 8) blocks = static_cast<int64_t>(sm_count) * 8;
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        kern<<<static_cast<unsigned>(blocks), 256, smem, s>>>(g, params, counters, count, out, bad);
    };
    if (lane == 0) go(predict_perf_kernel<0>);
    else go(predict_perf_kernel<1>);
    return cudaGetLastError();
}

}  // namespace ocg
