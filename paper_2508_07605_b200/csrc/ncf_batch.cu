// Per-app batched NCF completion + selection — the reference's online phase
// (run_open_online steps 3-4, policy.cpp:178-189) for many independent apps.
//
// One CTA owns one app's entire cf::complete (cfcomplete.cpp:198-213):
//   init (cfcomplete.cpp:74-86) -> validation split (:92-103) -> epochs of
//   shuffled minibatches with dense Adam (:150-178) -> validation MSE + early
//   stop + best snapshot (:179-190) -> impute the app's missing cells with
//   NcfModel::predict (:47-58) -> policy::select_caps (policy.cpp:17-64).
// Everything runs in FP64 with the operation order of the chosen reference
// kernel lane (scalar: kernels_scalar.cpp, AVX2: kernels_avx2.cpp), so the
// result is bit-identical to the reference on the same inputs.
//
// CTA layout: 8 compute warps + 1 RNG warp.  The RNG warp owns the app's
// mt19937_64 stream (rng.hpp) in shared memory: it draws the parameter init,
// the validation split and, one epoch ahead, the next epoch's Fisher-Yates
// permutation while the compute warps train on the current one (the shuffle
// of epoch e+1 depends only on epoch e's permutation, never on parameters).
//
// Within a minibatch step lanes map to samples (<=32) and warps to neurons,
// so every weight read is a shared-memory broadcast and every activation read
// hits a padded (odd-stride) per-sample row.  Parameters live in shared
// memory; Adam moments and the best snapshot live in the registers of the
// thread that owns each parameter (owner-computes: the owner reduces its
// gradient over the batch in sample order — the reference's accumulation
// order — then applies Adam immediately).
//
// Two instantiations of one body: FixArch<8,8,32,16> (the reference default
// NcfHyper: every layer width a compile-time constant, all layer loops
// unrolled, shared-memory pointers resolved statically) and RtArch (any
// other shape within the limits of ncf_batch.h, dims read at run time).
#include <cuda_runtime.h>

#include "lane_ops.cuh"
#include "ncf_batch.h"
#include "ocg_common.cuh"
#include "select_dev.cuh"

namespace ocg {

namespace {

constexpr int kCW = 8;              // compute warps
constexpr int kCT = kCW * 32;       // compute threads
constexpr int kThreads = kCT + 32;  // + RNG warp

__device__ __forceinline__ void bar_compute() { asm volatile("bar.sync 1, %0;" ::"n"(kCT) : "memory"); }

// ---- architecture policies ------------------------------------------------
struct RtArch {
    static constexpr bool kStatic = false;
    static constexpr int kEPT = kMaxParams / kCT;
    const BatchGeom& g;
    __device__ __forceinline__ int L() const { return g.L; }
    __device__ __forceinline__ int dim(int l) const { return g.dims[l]; }
    __device__ __forceinline__ int stride(int l) const { return g.stride[l]; }
    __device__ __forceinline__ int ka() const { return g.ka; }
    __device__ __forceinline__ int ks() const { return g.ks; }
};

template <int KA, int KS, int H0, int H1>
struct FixArch {
    static constexpr bool kStatic = true;
    static constexpr int kEPT = kFixMaxParams / kCT;
    const BatchGeom& g;
    __device__ __forceinline__ static constexpr int L() { return 3; }
    __device__ __forceinline__ static constexpr int dim(int l) {
        return l == 0 ? KA + KS : (l == 1 ? H0 : (l == 2 ? H1 : 1));
    }
    __device__ __forceinline__ static constexpr int stride(int l) { return dim(l) | 1; }
    __device__ __forceinline__ static constexpr int ka() { return KA; }
    __device__ __forceinline__ static constexpr int ks() { return KS; }
};

// ---- shared-memory carve-up ---------------------------------------------
// Regions are kept as 32-bit byte offsets into the dynamic shared-memory
// window and turned into pointers at the point of use, so every access is a
// 32-bit-addressed LDS/STS and the layout costs one register per region.
extern __shared__ __align__(16) char g_smem[];

template <typename T>
__device__ __forceinline__ T* smp(uint32_t off) {
    return reinterpret_cast<T*>(g_smem + off);
}

struct Smem {
    uint32_t oP;                    // [T] parameters
    uint32_t oact[kMaxLayers + 1];  // act[0] = gathered inputs X; act[l+1] = layer l output
    uint32_t odel[kMaxLayers];      // del[l]: act-grad factors, then deltas, of layer l output
    uint32_t oig, ocval, ocrc, otset, ovset, operm[2], odraw, omt, orow, os_app, os_set, os_y, octrl, otab, omask;
    __device__ __forceinline__ double* P() const { return smp<double>(oP); }
    __device__ __forceinline__ double* act(int l) const { return smp<double>(oact[l]); }
    __device__ __forceinline__ double* del(int l) const { return smp<double>(odel[l]); }
    __device__ __forceinline__ double* ig() const { return smp<double>(oig); }        // input grads
    __device__ __forceinline__ double* cval() const { return smp<double>(ocval); }    // cell values
    __device__ __forceinline__ uint32_t* crc() const { return smp<uint32_t>(ocrc); }  // (row<<16 | col)
    __device__ __forceinline__ uint16_t* tset() const { return smp<uint16_t>(otset); }  // train cell ids
    __device__ __forceinline__ uint16_t* vset() const { return smp<uint16_t>(ovset); }  // validation ids
    __device__ __forceinline__ uint16_t* perm(int k) const { return smp<uint16_t>(operm[k]); }
    __device__ __forceinline__ uint32_t* draw() const { return smp<uint32_t>(odraw); }
    __device__ __forceinline__ uint64_t* mt() const { return smp<uint64_t>(omt); }
    __device__ __forceinline__ double* row() const { return smp<double>(orow); }  // completed app row
    // per embedding row (apps 0..m-1, then settings): bit s = minibatch sample s touches it
    __device__ __forceinline__ uint32_t* mask() const { return smp<uint32_t>(omask); }
    __device__ __forceinline__ int* s_app() const { return smp<int>(os_app); }
    __device__ __forceinline__ int* s_set() const { return smp<int>(os_set); }
    __device__ __forceinline__ double* s_y() const { return smp<double>(os_y); }
    __device__ __forceinline__ int* ctrl() const { return smp<int>(octrl); }
    // glibc exp table: SELU's exp runs on per-lane (divergent) arguments
    __device__ __forceinline__ ExpTabPtr tab() const { return ExpTabPtr{smp<uint64_t>(otab)}; }
};

__device__ __forceinline__ uint32_t carve(uint32_t& p, size_t bytes) {
    const uint32_t r = p;
    p += static_cast<uint32_t>((bytes + 15) & ~size_t(15));
    return r;
}

// Fixed-size regions first: with FixArch every layer stride is a compile-time constant,
// so the offsets of the hot per-step regions (activations, deltas, sample ids, control,
// exp table) fold to immediates and cost no registers; the app-sized regions follow.
template <class A>
__device__ __forceinline__ void setup_smem(Smem& S, const A& a, const BatchGeom& g) {
    uint32_t p = 0;
#pragma unroll
    for (int l = 0; l <= kMaxLayers; ++l)
        if (l <= a.L()) S.oact[l] = carve(p, sizeof(double) * 32 * a.stride(l));
#pragma unroll
    for (int l = 0; l < kMaxLayers; ++l)
        if (l < a.L()) S.odel[l] = carve(p, sizeof(double) * 32 * a.stride(l + 1));
    S.oig = carve(p, sizeof(double) * 32 * a.stride(0));
    S.os_app = carve(p, sizeof(int) * 32);
    S.os_set = carve(p, sizeof(int) * 32);
    S.os_y = carve(p, sizeof(double) * 32);
    S.octrl = carve(p, sizeof(int) * 16);
    S.otab = carve(p, sizeof(uint64_t) * 256);
    S.omt = carve(p, sizeof(uint64_t) * 313);
    S.oP = carve(p, sizeof(double) * g.T);
    S.ocval = carve(p, sizeof(double) * g.max_cells);
    S.ocrc = carve(p, sizeof(uint32_t) * g.max_cells);
    S.otset = carve(p, sizeof(uint16_t) * g.max_cells);
    S.ovset = carve(p, sizeof(uint16_t) * g.max_cells);
    S.operm[0] = carve(p, sizeof(uint16_t) * g.max_cells);
    S.operm[1] = carve(p, sizeof(uint16_t) * g.max_cells);
    S.odraw = carve(p, sizeof(uint32_t) * g.max_cells);
    S.orow = carve(p, sizeof(double) * g.n);
    S.omask = carve(p, sizeof(uint32_t) * (g.m + g.n));
}

enum Ctrl { kMtIdx = 0, kStop = 1, kImproved = 2, kNt = 3, kNv = 4, kNc = 5, kDiverged = 6 };

// ---- RNG warp helpers ---------------------------------------------------
// Fisher-Yates over a[0..len): for i = len..2: swap(a[i-1], a[uniform_int(0, i-1)])
// (cfcomplete.cpp:98-99, :153-154).  Draws in parallel, swaps on lane 0.
__device__ void shuffle_warp(uint16_t* a, int len, uint32_t* draw, MtWarp& mt, int lane) {
    const int nd = len > 1 ? len - 1 : 0;
    for (int base = 0; base < nd; base += 32) {
        const int cnt = min(32, nd - base);
        const uint64_t r = mt.take(cnt, lane);
        if (lane < cnt) {
            const uint64_t span = static_cast<uint64_t>(len - (base + lane));  // i for this draw
            draw[base + lane] = static_cast<uint32_t>(r % span);
        }
    }
    __syncwarp();
    if (lane == 0) {
        for (int k = 0; k < nd; ++k) {
            const int i = len - k;
            const uint32_t j = draw[k];
            const uint16_t t = a[i - 1];
            a[i - 1] = a[j];
            a[j] = t;
        }
    }
    __syncwarp();
}

// uniform(lo, hi) draws into dst[0..cnt) (rng.hpp:22-24)
__device__ void uniform_fill(double* dst, int cnt, double lo, double hi, MtWarp& mt, int lane) {
    const double span = dsub(hi, lo);
    for (int base = 0; base < cnt; base += 32) {
        const int c = min(32, cnt - base);
        const uint64_t r = mt.take(c, lane);
        if (lane < c) {
            const double u = static_cast<double>(r >> 11) * 0x1.0p-53;
            dst[base + lane] = dadd(lo, dmul(span, u));
        }
    }
}

// ---- compute-warp helpers -----------------------------------------------
// forward() / forward_tape() (nnkit.cpp:74-89, :124-138) for cnt <= 32 cells
// whose (app, setting) ids are in s_app/s_set.  Leaves layer outputs in act[],
// and (tape) SELU derivative factors in del[].
// compile-time layer (FixArch): the warp's NO outputs are formed together, so their dot
// chains and SELU exps are independent instruction streams (ILP) instead of a loop
template <int LANE, class A, int LAY>
__device__ __forceinline__ void forward_layer_fix(const Smem& S, const A& a, const BatchGeom& g, int cnt, bool tape,
                                                  double scale, int warp, int lane) {
    constexpr int in = A::dim(LAY), out = A::dim(LAY + 1), NO = (out + kCW - 1) / kCW;
    constexpr bool hidden = LAY + 1 < A::L();
    const double* W = S.P() + g.off_w[LAY];
    const double* b = S.P() + g.off_b[LAY];
    const double* ain = S.act(LAY) + lane * A::stride(LAY);
    if (lane < cnt) {
        double z[NO];
#pragma unroll
        for (int q = 0; q < NO; ++q) {
            const int o = warp + q * kCW;
            if (out % kCW == 0 || o < out) z[q] = dadd(LaneOps<LANE>::dot(W + o * in, ain, in), b[o]);
        }
#pragma unroll
        for (int q = 0; q < NO; ++q) {
            const int o = warp + q * kCW;
            if (out % kCW == 0 || o < out) {
                double v = z[q], gf = 1.0;
                if (hidden) selu_fwd(z[q], v, gf, S.tab());
                S.act(LAY + 1)[lane * A::stride(LAY + 1) + o] = v;
                // output layer with tape: backprop's first delta here (2 err scale * 1), saving a barrier
                if (tape) S.del(LAY)[lane * A::stride(LAY + 1) + o] =
                    hidden ? gf : dmul(dmul(dmul(2.0, dsub(v, S.s_y()[lane])), scale), 1.0);
            }
        }
    }
    bar_compute();
}

// forward() / forward_tape(); with tape the output layer also writes backprop's first delta
// (2 err scale, identity grad 1) so backward_chunk starts at the output layer's matvec_t
template <int LANE, class A>
__device__ __forceinline__ void forward_chunk(const Smem& S, const A& a, const BatchGeom& g, int cnt, bool tape,
                                              int warp, int lane, int ctid, double scale = 0.0) {
    const int in0 = a.dim(0);
    for (int w = ctid; w < cnt * in0; w += kCT) {
        const int s = w / in0, i = w - s * in0;
        const double v = i < a.ka() ? S.P()[S.s_app()[s] * a.ka() + i]
                                    : S.P()[g.set_off + S.s_set()[s] * a.ks() + (i - a.ka())];
        S.act(0)[s * a.stride(0) + i] = v;
    }
    bar_compute();
    if constexpr (A::kStatic && LANE == 0) {  // (the AVX2 lane's 4-accumulator dots would spill)
        static_assert(A::L() == 3, "FixArch is the 3-layer default stack");
        forward_layer_fix<LANE, A, 0>(S, a, g, cnt, tape, scale, warp, lane);
        forward_layer_fix<LANE, A, 1>(S, a, g, cnt, tape, scale, warp, lane);
        forward_layer_fix<LANE, A, 2>(S, a, g, cnt, tape, scale, warp, lane);
    } else {
#pragma unroll
        for (int l = 0; l < kMaxLayers; ++l) {
            if (l >= a.L()) break;
            const int in = a.dim(l), out = a.dim(l + 1);
            const double* W = S.P() + g.off_w[l];
            const double* b = S.P() + g.off_b[l];
            const double* ain = S.act(l) + lane * a.stride(l);
            const bool hidden = l + 1 < a.L();
            if (lane < cnt) {
                for (int o = warp; o < out; o += kCW) {
                    const double z = dadd(LaneOps<LANE>::dot(W + o * in, ain, in), b[o]);
                    double v = z, gf = 1.0;
                    if (hidden) selu_fwd(z, v, gf, S.tab());
                    S.act(l + 1)[lane * a.stride(l + 1) + o] = v;
                    if (tape) S.del(l)[lane * a.stride(l + 1) + o] =
                        hidden ? gf : dmul(dmul(dmul(2.0, dsub(v, S.s_y()[lane])), scale), 1.0);
                }
            }
            bar_compute();
        }
    }
}

// backprop_sample (nnkit.cpp:184-212) deltas for a minibatch already
// forwarded with tape; writes del[l] = deltas and ig = input gradients.
// compile-time layer (FixArch): the warp's NC input columns' matvec_t chains side by side
template <int LANE, class A, int LAY>
__device__ __forceinline__ void backward_layer_fix(const Smem& S, const A& a, const BatchGeom& g, int cnt, int warp,
                                                   int lane) {
    constexpr int in = A::dim(LAY), out = A::dim(LAY + 1), NC = (in + kCW - 1) / kCW;
    const double* W = S.P() + g.off_w[LAY];
    const double* d = S.del(LAY) + lane * A::stride(LAY + 1);
    if (lane < cnt) {
        double nd[NC];
#pragma unroll
        for (int q = 0; q < NC; ++q) nd[q] = 0.0;  // matvec_t: out[c] = 0; out[c] += d[r]*w[r][c]
        for (int r = 0; r < out; ++r) {
            const double dr = d[r];
#pragma unroll
            for (int q = 0; q < NC; ++q) {
                const int c = warp + q * kCW;
                if (in % kCW == 0 || c < in) nd[q] = LaneOps<LANE>::axpy(nd[q], dr, W[r * in + c]);
            }
        }
#pragma unroll
        for (int q = 0; q < NC; ++q) {
            const int c = warp + q * kCW;
            if (in % kCW == 0 || c < in) {
                if (LAY > 0) {
                    double* gf = S.del(LAY > 0 ? LAY - 1 : 0) + lane * A::stride(LAY) + c;
                    *gf = dmul(nd[q], *gf);  // delta[o] *= activate_grad
                } else {
                    S.ig()[lane * A::stride(0) + c] = nd[q];
                }
            }
        }
    }
    bar_compute();
}

template <int LANE, class A>
__device__ __forceinline__ void backward_chunk(const Smem& S, const A& a, const BatchGeom& g, int cnt,
                                               double scale, int warp, int lane) {
    (void)scale;  // the output delta was written by forward_chunk (tape)
    if constexpr (A::kStatic && LANE == 1) {  // (with the scalar lane's ILP forward this would spill)
        backward_layer_fix<LANE, A, 2>(S, a, g, cnt, warp, lane);
        backward_layer_fix<LANE, A, 1>(S, a, g, cnt, warp, lane);
        backward_layer_fix<LANE, A, 0>(S, a, g, cnt, warp, lane);
    } else {
        const int L = a.L();
#pragma unroll
        for (int l = kMaxLayers - 1; l >= 0; --l) {
            if (l >= L) continue;
            const int in = a.dim(l), out = a.dim(l + 1);
            const double* W = S.P() + g.off_w[l];
            const double* d = S.del(l) + lane * a.stride(l + 1);
            if (lane < cnt) {
                for (int c = warp; c < in; c += kCW) {
                    double nd = 0.0;  // matvec_t: out[c] = 0; out[c] += d[r]*w[r][c]
                    for (int r = 0; r < out; ++r) nd = LaneOps<LANE>::axpy(nd, d[r], W[r * in + c]);
                    if (l > 0) {
                        double* gf = S.del(l > 0 ? l - 1 : 0) + lane * a.stride(l) + c;
                        *gf = dmul(nd, *gf);  // delta[o] *= activate_grad
                    } else {
                        S.ig()[lane * a.stride(0) + c] = nd;
                    }
                }
            }
            bar_compute();
        }
    }
}

// the network output row (act[L]) without a run-time array index
template <class A>
__device__ __forceinline__ const double* out_act(const Smem& S, const A& a) {
    if constexpr (A::kStatic) return S.act(A::L());
    switch (a.L()) {
        case 1: return S.act(1);
        case 2: return S.act(2);
        case 3: return S.act(3);
        default: return S.act(4);
    }
}

// sequential MSE over a list of cells (cells_mse, cfcomplete.cpp:34-43)
template <int LANE, class A>
__device__ __forceinline__ double cells_mse(const Smem& S, const A& a, const BatchGeom& g, const uint16_t* ids,
                                            int count, int warp, int lane, int ctid) {
    double acc = 0.0;  // meaningful on ctid 0 only
    for (int base = 0; base < count; base += 32) {
        const int cnt = min(32, count - base);
        if (ctid < cnt) {
            const int c = ids[base + ctid];
            const uint32_t rc = S.crc()[c];
            S.s_app()[ctid] = static_cast<int>(rc >> 16);
            S.s_set()[ctid] = static_cast<int>(rc & 0xffff);
            S.s_y()[ctid] = S.cval()[c];
        }
        bar_compute();
        forward_chunk<LANE>(S, a, g, cnt, false, warp, lane, ctid);
        if (ctid == 0) {
            const double* out = out_act(S, a);
            const int so = a.stride(a.L());
            for (int s = 0; s < cnt; ++s) {
                const double err = dsub(out[s * so], S.s_y()[s]);
                acc = dadd(acc, dmul(err, err));
            }
        }
        bar_compute();
    }
    return count == 0 ? 0.0 : ddiv(acc, static_cast<double>(count));
}

// An owned parameter, packed: c[0,12) r[12,24) kind[24,26) layer[26,29) vec[29] valid[31]
// kind: 0 app emb, 1 setting emb, 2 weight, 3 bias
__device__ __forceinline__ int own_c(uint32_t d) { return d & 0xfff; }
__device__ __forceinline__ int own_r(uint32_t d) { return (d >> 12) & 0xfff; }
__device__ __forceinline__ int own_kind(uint32_t d) { return (d >> 24) & 3; }
__device__ __forceinline__ int own_layer(uint32_t d) { return (d >> 26) & 7; }
__device__ __forceinline__ bool own_vec(uint32_t d) { return (d >> 29) & 1; }
__device__ __forceinline__ bool own_valid(uint32_t d) { return (d >> 31) & 1; }

__device__ inline uint32_t describe(const BatchGeom& g, int e) {
    if (e >= g.T) return 0u;
    int kind, layer = 0, r, c = 0, start, size;
    if (e < g.set_off) {
        kind = 0;
        r = e / g.ka;
        c = e - r * g.ka;
        start = 0;
        size = g.set_off;
    } else if (e < g.off_w[0]) {
        kind = 1;
        const int q = e - g.set_off;
        r = q / g.ks;
        c = q - r * g.ks;
        start = g.set_off;
        size = g.off_w[0] - g.set_off;
    } else {
        while (layer + 1 < g.L && e >= g.off_w[layer + 1]) ++layer;
        if (e < g.off_b[layer]) {
            kind = 2;
            const int q = e - g.off_w[layer];
            r = q / g.dims[layer];
            c = q - r * g.dims[layer];
            start = g.off_w[layer];
            size = g.off_b[layer] - g.off_w[layer];
        } else {
            kind = 3;
            r = e - g.off_b[layer];
            start = g.off_b[layer];
            size = g.dims[layer + 1];
        }
    }
    const uint32_t vec = (e - start) < (size & ~3) ? 1u : 0u;
    return 0x80000000u | (vec << 29) | (static_cast<uint32_t>(layer) << 26) |
           (static_cast<uint32_t>(kind) << 24) | (static_cast<uint32_t>(r) << 12) | static_cast<uint32_t>(c);
}

// weight / bias gradient of layer LAY summed over the batch in sample order
template <int LANE, int LAY, class A>
__device__ __forceinline__ double layer_grad(const Smem& S, const A& a, bool is_weight, int r, int c, int cnt) {
    const double* dl = S.del(LAY) + r;
    const int sd = a.stride(LAY + 1);
    double gsum = 0.0;
    if (is_weight) {  // outer_acc: G[r][c] += d[r] * x[c]
        const double* al = S.act(LAY) + c;
        const int sa = a.stride(LAY);
        for (int s = 0; s < cnt; ++s) gsum = LaneOps<LANE>::axpy(gsum, dl[s * sd], al[s * sa]);
    } else {  // bias: G[o] += delta[o]
        for (int s = 0; s < cnt; ++s) gsum = dadd(gsum, dl[s * sd]);
    }
    return gsum;
}

template <int LANE, class A>
__device__ __forceinline__ double param_grad(const Smem& S, const A& a, uint32_t o, int cnt) {
    const int kind = own_kind(o), orow = own_r(o), ocol = own_c(o);
    if (kind >= 2) {
        const bool w = kind == 2;
        switch (own_layer(o)) {
            case 0: return layer_grad<LANE, 0>(S, a, w, orow, ocol, cnt);
            case 1: return layer_grad<LANE, 1>(S, a, w, orow, ocol, cnt);
            case 2: return layer_grad<LANE, 2>(S, a, w, orow, ocol, cnt);
            default: return layer_grad<LANE, 3>(S, a, w, orow, ocol, cnt);
        }
    }
    double gsum = 0.0;
    const int st0 = a.stride(0);
    // embedding scatter (cfcomplete.cpp:171-174): the samples that touch the row, in sample
    // order, from the step's row mask (built by warp 0 when it loads the minibatch)
    const double* ig = S.ig() + (kind == 0 ? ocol : a.ka() + ocol);
    uint32_t mk = S.mask()[kind == 0 ? orow : a.g.m + orow];
    while (mk) {
        const int s = __ffs(mk) - 1;
        mk &= mk - 1;
        gsum = dadd(gsum, ig[s * st0]);
    }
    (void)cnt;
    return gsum;
}

// Parameter ownership.  Run-time shapes: thread ctid owns parameters ctid + k kCT.
// Compile-time shape (FixArch<8,8,32,16>): slots 0-3 are a 2x2 tile of W0 (threads 0-127)
// or W1 (128-255), whose gradients share their operand loads (4 shared-memory loads per
// 4 FMAs instead of 8); slots 4-5 take the remaining parameters in block order
// (embeddings, b0, b1, W2, b2).  Each parameter still sums its gradient over the samples
// in the reference's order.
template <class ARCH>
__device__ __forceinline__ int owned_index(const BatchGeom& g, int k, int ctid) {
    if constexpr (!ARCH::kStatic) {
        return ctid + k * kCT;
    } else {
        constexpr int in0 = ARCH::dim(0), h0 = ARCH::dim(1), h1 = ARCH::dim(2);
        if (k < 4) {
            if (ctid < 128) {  // W0: h0 x in0, tiles of 2 rows x 2 cols
                const int r = 2 * (ctid / (in0 / 2)) + (k >> 1), c = 2 * (ctid % (in0 / 2)) + (k & 1);
                return g.off_w[0] + r * in0 + c;
            }
            const int tt = ctid - 128;  // W1: h1 x h0
            const int r = 2 * (tt / (h0 / 2)) + (k >> 1), c = 2 * (tt % (h0 / 2)) + (k & 1);
            return g.off_w[1] + r * h0 + c;
        }
        int q = ctid + (k - 4) * kCT;
        if (q < g.off_w[0]) return q;  // embedding tables
        q -= g.off_w[0];
        if (q < h0) return g.off_b[0] + q;
        q -= h0;
        if (q < h1) return g.off_b[1] + q;
        q -= h1;
        if (q < h1) return g.off_w[2] + q;
        q -= h1;
        if (q < 1) return g.off_b[2];
        return g.T;  // no parameter
    }
}

// gradients of the 2x2 tile W_LAY[r..r+1][c..c+1], each summed over the batch in sample order
template <int LANE, int LAY, class A>
__device__ __forceinline__ void tile_grad(const Smem& S, const A& a, int r, int c, int cnt, double (&gt)[4]) {
    const double* dl = S.del(LAY) + r;
    const double* al = S.act(LAY) + c;
    constexpr int sd = A::stride(LAY + 1), sa = A::stride(LAY);
    double g0 = 0.0, g1 = 0.0, g2 = 0.0, g3 = 0.0;
    for (int q = 0; q < cnt; ++q) {
        const double d0 = dl[q * sd], d1 = dl[q * sd + 1], x0 = al[q * sa], x1 = al[q * sa + 1];
        g0 = LaneOps<LANE>::axpy(g0, d0, x0);
        g1 = LaneOps<LANE>::axpy(g1, d0, x1);
        g2 = LaneOps<LANE>::axpy(g2, d1, x0);
        g3 = LaneOps<LANE>::axpy(g3, d1, x1);
    }
    gt[0] = g0;
    gt[1] = g1;
    gt[2] = g2;
    gt[3] = g3;
}

template <int LANE, class ARCH>
__device__ __forceinline__ void app_batch_body(const BatchGeom& g, const BatchIO& io) {
    const ARCH a{g};
    constexpr int kEPT = ARCH::kEPT;
    Smem S;
    setup_smem(S, a, g);
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const bool is_rng = warp == kCW;
    const int ctid = tid;  // valid for compute threads
    MtWarp mt{S.mt(), S.ctrl() + kMtIdx};
    for (int e = tid; e < 256; e += blockDim.x) smp<uint64_t>(S.otab)[e] = exp_tab(e);  // first app's sync publishes it

    // owned parameters (compile-time indexed so moments stay in registers)
    // (compile-time shape: the 2x2 weight tile of slots 0-3 is implied by ctid and kept as
    // its first index only; descriptors are stored for the remaining slots)
    constexpr int kK0 = ARCH::kStatic ? 4 : 0;  // slots [0, kK0) are the tile
    uint32_t own[kEPT - kK0];
    int eidx[kEPT - kK0];
    double M1[kEPT], V1[kEPT];
    int tile_r = 0, tile_c = 0, tile_e = 0;
    if constexpr (ARCH::kStatic) {
        constexpr int in0 = ARCH::dim(0), h0 = ARCH::dim(1);
        if (ctid < 128) {
            tile_r = 2 * (ctid / (in0 / 2));
            tile_c = 2 * (ctid % (in0 / 2));
            tile_e = g.off_w[0] + tile_r * in0 + tile_c;
        } else {
            tile_r = 2 * ((ctid - 128) / (h0 / 2));
            tile_c = 2 * ((ctid - 128) % (h0 / 2));
            tile_e = g.off_w[1] + tile_r * h0 + tile_c;
        }
    }
#pragma unroll
    for (int k = kK0; k < kEPT; ++k) {
        eidx[k - kK0] = is_rng ? g.T : owned_index<ARCH>(g, k, ctid);
        own[k - kK0] = is_rng ? 0u : describe(g, eidx[k - kK0]);
    }
#pragma unroll
    for (int k = 0; k < kEPT; ++k) M1[k] = V1[k] = 0.0;
    // best snapshot in global scratch (L2-resident): written when validation improves,
    // read once at restore; keeping it in registers cost the hot loops their spills
    double* const bestbuf = io.best + static_cast<int64_t>(blockIdx.x) * io.best_stride;

    const double lr = g.lr, b1 = 0.9, b2 = 0.999, eps = 1e-8;  // nnkit.hpp:95
    const double omb1 = dsub(1.0, b1), omb2 = dsub(1.0, b2);

    for (int64_t app = blockIdx.x; app < io.napps; app += gridDim.x) {
        // ---------------- load cells: block rows, then the app row ---------
        const double* prow = io.probe_vals + app * g.n;
        const uint8_t* pmask = io.probe_mask + app * g.n;
        const int D = g.m - 1;
        if (tid < 16) S.ctrl()[tid] = 0;
        __syncthreads();
        if (tid == 0) {
            S.ctrl()[kMtIdx] = 312;
            int napp = 0;
            for (int j = 0; j < g.n; ++j) napp += pmask[j] != 0;
            S.ctrl()[kNc] = g.block_nnz + napp;
        }
        for (int q = tid; q < g.block_nnz; q += kThreads) {
            S.cval()[q] = io.block_val[q];
            S.crc()[q] = io.block_rc[q];
        }
        if (tid < 32) {  // app row cells in column order (ballot compaction)
            int base = g.block_nnz;
            for (int j0 = 0; j0 < g.n; j0 += 32) {
                const int j = j0 + lane;
                const bool obs = j < g.n && pmask[j] != 0;
                const unsigned bal = __ballot_sync(0xffffffffu, obs);
                if (obs) {
                    const int pos = base + __popc(bal & ((1u << lane) - 1));
                    S.cval()[pos] = prow[j];
                    S.crc()[pos] = (static_cast<uint32_t>(D) << 16) | static_cast<uint32_t>(j);
                }
                base += __popc(bal);
            }
        }
        for (int j = tid; j < g.n; j += kThreads) S.row()[j] = prow[j];
        for (int q = tid; q < g.m + g.n; q += kThreads) S.mask()[q] = 0u;
        __syncthreads();
        const int nc = S.ctrl()[kNc];
        const int napp_obs = nc - g.block_nnz;

        int status = OCG_OK;
        if (napp_obs == 0) status = OCG_E_INVALID;  // complete(): row without probes (:199-205)
        bool cold = false;
        if (status == OCG_OK && napp_obs < g.n) {
            for (int j = 0; j < g.n; ++j)
                if (!io.block_col_seen[j] && pmask[j] == 0) cold = true;
        }
        const bool full = status == OCG_OK && napp_obs == g.n && g.block_full;
        if (status == OCG_OK && full) {
            // fully observed -> returned unchanged, no fit (:206)
        } else if (status == OCG_OK) {
            const uint64_t seed = io.seeds[app];
            // ------------- init + split (RNG warp) -----------------------
            if (is_rng) {
                mt.seed(derive_seed_h(seed, g.fit_tag_mix, 0), lane);
                const double ba = dsqrt(ddiv(6.0, static_cast<double>(g.m + a.ka())));
                uniform_fill(S.P(), g.m * a.ka(), -ba, ba, mt, lane);
                const double bs = dsqrt(ddiv(6.0, static_cast<double>(g.n + a.ks())));
                uniform_fill(S.P() + g.set_off, g.n * a.ks(), -bs, bs, mt, lane);
                for (int l = 0; l < a.L(); ++l) {
                    const double bw = dsqrt(ddiv(6.0, static_cast<double>(a.dim(l) + a.dim(l + 1))));
                    uniform_fill(S.P() + g.off_w[l], a.dim(l) * a.dim(l + 1), -bw, bw, mt, lane);
                    for (int q = lane; q < a.dim(l + 1); q += 32) S.P()[g.off_b[l] + q] = 0.0;
                }
                // validation split: order = shuffled iota(nc)
                uint16_t* order = S.perm(1);
                for (int q = lane; q < nc; q += 32) order[q] = static_cast<uint16_t>(q);
                __syncwarp();
                shuffle_warp(order, nc, S.draw(), mt, lane);
                const int val_count = static_cast<int>(g.val_fraction * static_cast<double>(nc));
                for (int q = lane; q < nc; q += 32) {
                    if (q < val_count) S.vset()[q] = order[q];
                    else S.tset()[q - val_count] = order[q];
                }
                int nv = val_count, nt = nc - val_count;
                __syncwarp();
                if (nt == 0) {  // std::swap(train, val)
                    for (int q = lane; q < nv; q += 32) S.tset()[q] = S.vset()[q];
                    nt = nv;
                    nv = 0;
                }
                if (lane == 0) {
                    S.ctrl()[kNt] = nt;
                    S.ctrl()[kNv] = nv;
                }
                __syncwarp();
            }
            __syncthreads();
            const int nt = S.ctrl()[kNt], nv = S.ctrl()[kNv];
            const uint16_t* mon = nv == 0 ? S.tset() : S.vset();
            const int nmon = nv == 0 ? nt : nv;

            double init_train = 0.0, best_val = 0.0;
            if (!is_rng) {
#pragma unroll
                for (int k = 0; k < kEPT; ++k) M1[k] = V1[k] = 0.0;
                for (int q = ctid; q < g.T; q += kCT) bestbuf[q] = S.P()[q];
                init_train = cells_mse<LANE>(S, a, g, S.tset(), nt, warp, lane, ctid);
                best_val = cells_mse<LANE>(S, a, g, mon, nmon, warp, lane, ctid);
            } else {
                // epoch-0 permutation of train positions
                for (int q = lane; q < nt; q += 32) S.perm(0)[q] = static_cast<uint16_t>(q);
                __syncwarp();
                shuffle_warp(S.perm(0), nt, S.draw(), mt, lane);
            }
            __syncthreads();

            int stale = 0, epoch = 0;
            double b1p = 1.0, b2p = 1.0;
            bool diverged = false;
            for (; epoch < g.max_epochs; ++epoch) {
                const uint16_t* perm = S.perm(epoch & 1);
                if (is_rng) {
                    uint16_t* nxt = S.perm((epoch + 1) & 1);
                    for (int q = lane; q < nt; q += 32) nxt[q] = perm[q];
                    __syncwarp();
                    shuffle_warp(nxt, nt, S.draw(), mt, lane);
                } else {
                    for (int start = 0; start < nt; start += g.batch) {
                        const int cnt = min(g.batch, nt - start);
                        const double scale = ddiv(1.0, static_cast<double>(cnt));
                        if (warp == 0) {  // (cnt <= 32: the minibatch is warp 0's)
                            if (start > 0 && lane < g.batch) {  // the previous step's rows: masks back to 0
                                S.mask()[S.s_app()[lane]] = 0u;
                                S.mask()[g.m + S.s_set()[lane]] = 0u;
                            }
                            __syncwarp();
                            if (lane < cnt) {
                                const int c = S.tset()[perm[start + lane]];
                                const uint32_t rc = S.crc()[c];
                                const int ra = static_cast<int>(rc >> 16), rs = static_cast<int>(rc & 0xffff);
                                S.s_app()[lane] = ra;
                                S.s_set()[lane] = rs;
                                S.s_y()[lane] = S.cval()[c];
                                atomicOr(S.mask() + ra, 1u << lane);
                                atomicOr(S.mask() + g.m + rs, 1u << lane);
                            }
                        }
                        bar_compute();
                        forward_chunk<LANE>(S, a, g, cnt, true, warp, lane, ctid, scale);
                        backward_chunk<LANE>(S, a, g, cnt, scale, warp, lane);
                        // AdamState::step (nnkit.cpp:239-251): dense over every block
                        b1p = dmul(b1p, b1);
                        b2p = dmul(b2p, b2);
                        const double mc = ddiv(1.0, dsub(1.0, b1p)), vc = ddiv(1.0, dsub(1.0, b2p));
                        double gt[4] = {0.0, 0.0, 0.0, 0.0};
                        if constexpr (ARCH::kStatic) {
                            if (!is_rng) {
                                if (ctid < 128) tile_grad<LANE, 0>(S, a, tile_r, tile_c, cnt, gt);
                                else tile_grad<LANE, 1>(S, a, tile_r, tile_c, cnt, gt);
                                const int rstep = ctid < 128 ? ARCH::dim(0) : ARCH::dim(1);
#pragma unroll
                                for (int k = 0; k < 4; ++k) {  // W0 / W1 sizes are multiples of 4: vector part
                                    const int e = tile_e + (k >> 1) * rstep + (k & 1);
                                    double p = S.P()[e];
                                    LaneOps<LANE>::adam(p, M1[k], V1[k], gt[k], lr, b1, omb1, b2, omb2, eps, mc, vc,
                                                        true);
                                    S.P()[e] = p;
                                }
                            }
                        }
#pragma unroll
                        for (int k = kK0; k < kEPT; ++k) {
                            const uint32_t o = own[k - kK0];
                            if (!own_valid(o)) continue;
                            const int e = eidx[k - kK0];
                            const double gsum = param_grad<LANE>(S, a, o, cnt);
                            double p = S.P()[e];
                            LaneOps<LANE>::adam(p, M1[k], V1[k], gsum, lr, b1, omb1, b2, omb2, eps, mc, vc,
                                                own_vec(o));
                            S.P()[e] = p;
                        }
                        bar_compute();
                    }
                    if (warp == 0 && nt > 0) {  // the epoch's last step: masks back to 0 (before validation reuses s_app)
                        const int last = nt - ((nt - 1) / g.batch) * g.batch;
                        if (lane < last) {
                            S.mask()[S.s_app()[lane]] = 0u;
                            S.mask()[g.m + S.s_set()[lane]] = 0u;
                        }
                        __syncwarp();
                    }
                    const double vl = cells_mse<LANE>(S, a, g, mon, nmon, warp, lane, ctid);
                    if (ctid == 0) {
                        int improved = 0, stop = 0, div = 0;
                        if (!isfinite(vl)) {
                            div = 1;
                            stop = 1;
                        } else if (vl < best_val) {
                            best_val = vl;
                            improved = 1;
                            stale = 0;
                        } else if (++stale > g.patience) {
                            stop = 1;
                        }
                        S.ctrl()[kImproved] = improved;
                        S.ctrl()[kStop] = stop;
                        S.ctrl()[kDiverged] = div;
                    }
                }
                __syncthreads();
                const bool stop = S.ctrl()[kStop] != 0;
                if (S.ctrl()[kDiverged]) {
                    diverged = true;
                    break;
                }
                if (!is_rng && S.ctrl()[kImproved])
                    for (int q = ctid; q < g.T; q += kCT) bestbuf[q] = S.P()[q];
                if (stop) {
                    ++epoch;
                    break;
                }
            }
            if (diverged) {
                status = OCG_E_DIVERGE;
            } else {
                // restore(best) (:190)
                if (!is_rng)
                    for (int q = ctid; q < g.T; q += kCT) S.P()[q] = bestbuf[q];
                __syncthreads();
                double final_train = 0.0;
                if (!is_rng) final_train = cells_mse<LANE>(S, a, g, S.tset(), nt, warp, lane, ctid);
                if (tid == 0) {
                    for (int q = g.off_w[0]; q < g.T; ++q)  // check_finite (nnkit.cpp:106-113)
                        if (!isfinite(S.P()[q])) {
                            S.ctrl()[kDiverged] = 2;
                            break;
                        }
                    if (io.meta) {
                        OcgMetaDev m;
                        m.seed = seed;
                        m.epochs_run = epoch;
                        m.initial_train_mse = init_train;
                        m.final_train_mse = final_train;
                        m.best_val_mse = best_val;
                        io.meta[app] = m;
                    }
                }
                if (io.params) {
                    __syncthreads();
                    for (int q = tid; q < g.T; q += kThreads) io.params[app * io.params_stride + q] = S.P()[q];
                }
                __syncthreads();
                if (S.ctrl()[kDiverged] == 2) status = OCG_E_LOGIC;
                else if (cold) status = OCG_E_COLD;
                // ------------ impute the app's missing cells ---------------
                if (status == OCG_OK && !is_rng) {
                    for (int j0 = 0; j0 < g.n; j0 += 32) {
                        if (ctid < 32) {
                            const int j = j0 + ctid;
                            S.s_app()[ctid] = D;
                            S.s_set()[ctid] = j < g.n ? j : 0;
                        }
                        bar_compute();
                        const int cnt = min(32, g.n - j0);
                        forward_chunk<LANE>(S, a, g, cnt, false, warp, lane, ctid);
                        if (ctid < cnt && pmask[j0 + ctid] == 0) {
                            const double v = out_act(S, a)[ctid * a.stride(a.L())];
                            S.row()[j0 + ctid] = v < 0.01 ? 0.01 : (1.25 < v ? 1.25 : v);  // std::clamp
                        }
                        bar_compute();
                    }
                }
            }
        }
        __syncthreads();
        // ---------------- select_caps on the completed row -----------------
        if (warp == 0) {
            SelResult r{};
            if (status == OCG_OK && io.cpu_caps != nullptr) {
                r = select_row_warp(S.row(), g.n, io.cpu_caps, io.gpu_caps, g.ngpu, g.e_base, g.gamma, lane);
                if (r.idx < 0) status = OCG_E_LOGIC;
            }
            if (lane == 0) {
                io.status[app] = status;
                if (io.sel_idx) io.sel_idx[app] = status == OCG_OK ? r.idx : -1;
                if (io.sel_saving) io.sel_saving[app] = r.saving;
                if (io.sel_loss) io.sel_loss[app] = r.loss;
                if (io.sel_ncand) io.sel_ncand[app] = r.ncand;
            }
        }
        if (io.completed)
            for (int j = tid; j < g.n; j += kThreads) io.completed[app * g.n + j] = S.row()[j];
        __syncthreads();
    }
}

}  // namespace

template <int LANE>
__global__ void __launch_bounds__(kThreads, 2) ncf_app_batch_kernel(BatchGeom g, BatchIO io) {
    app_batch_body<LANE, RtArch>(g, io);
}

// reference-default architecture: app/setting dim 8, hidden {32, 16}
template <int LANE>
__global__ void __launch_bounds__(kThreads, 3) ncf_app_batch_kernel_k8(BatchGeom g, BatchIO io) {
    app_batch_body<LANE, FixArch<8, 8, 32, 16>>(g, io);
}

size_t batch_smem_bytes(const BatchGeom& g) {
    size_t b = 0;
    auto add = [&](size_t x) { b += (x + 15) & ~size_t(15); };
    add(sizeof(double) * g.T);
    for (int l = 0; l <= g.L; ++l) add(sizeof(double) * 32 * g.stride[l]);
    for (int l = 0; l < g.L; ++l) add(sizeof(double) * 32 * g.stride[l + 1]);
    add(sizeof(double) * 32 * g.stride[0]);
    add(sizeof(double) * g.max_cells);
    add(sizeof(uint32_t) * g.max_cells);
    for (int k = 0; k < 4; ++k) add(sizeof(uint16_t) * g.max_cells);
    add(sizeof(uint32_t) * g.max_cells);
    add(sizeof(uint64_t) * 313);
    add(sizeof(double) * g.n);
    add(sizeof(int) * 32);
    add(sizeof(int) * 32);
    add(sizeof(double) * 32);
    add(sizeof(int) * 16);
    add(sizeof(uint64_t) * 256);
    add(sizeof(uint32_t) * (g.m + g.n));
    return b;
}

int batch_threads() { return kThreads; }

bool batch_is_fixed_k8(const BatchGeom& g) {
    return g.L == 3 && g.ka == 8 && g.ks == 8 && g.dims[1] == 32 && g.dims[2] == 16 && g.T <= kFixMaxParams;
}

namespace {
using KernelFn = void (*)(BatchGeom, BatchIO);
KernelFn pick(const BatchGeom& g, int lane) {
    if (batch_is_fixed_k8(g)) return lane == 0 ? ncf_app_batch_kernel_k8<0> : ncf_app_batch_kernel_k8<1>;
    return lane == 0 ? ncf_app_batch_kernel<0> : ncf_app_batch_kernel<1>;
}
}  // namespace

cudaError_t launch_app_batch(const BatchGeom& g, const BatchIO& io, int lane, int grid, cudaStream_t stream) {
    const size_t smem = batch_smem_bytes(g);
    const KernelFn k = pick(g, lane);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k<<<grid, kThreads, smem, stream>>>(g, io);
    return cudaGetLastError();
}

int batch_max_active_per_sm(const BatchGeom& g, int lane) {
    int n = 0;
    const size_t smem = batch_smem_bytes(g);
    const KernelFn k = pick(g, lane);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, kThreads, smem);
    return n;
}

}  // namespace ocg
