// Joint-mode NCF fit — cf::fit (cfcomplete.cpp:63-196) over ONE whole sparse
// matrix (the C1/C2 "joint" configs), on one GPU, with the
// reference's own schedule: minibatches of 32 shuffled observed cells, each
// followed by a dense Adam step over every parameter (nnkit.cpp:239-251).
//
// The reference spends >99.9 % of the online phase here and is strictly
// sequential (each minibatch reads the parameters the previous one wrote), so
// the design question is how to make one step short and keep the dense Adam
// off the critical path:
//
//  * Leader CTA (blockIdx 0, 8 warps) runs the step chain: gather the <= 64
//    embedding rows the minibatch touches ("slots"), forward with tape and
//    backprop_sample for <= 32 samples (lanes = samples, warps = neurons,
//    nnkit.cpp:124-212), owner-computes gradient sums in sample order (the
//    reference's += order, cfcomplete.cpp:166-175), Adam on the MLP and on the
//    touched rows, write-back, then publish `progress = s`.
//  * Every other CTA is a replay helper.  A row that no minibatch touches
//    still moves at every step (its Adam moments decay: with g = 0 both lanes
//    compute m = round(b1 m), v = round(b2 v), and p moves by lr m^/(sqrt v^ +
//    eps)).  Because those zero-gradient steps depend only on the row's own
//    state and the step's bias corrections, they are replayed lazily and
//    EXACTLY (same lane operations, same per-step mc/vc) by helper warps:
//    the host knows the epoch's whole schedule (the shuffle depends only on
//    the RNG, never on parameters), so for each (row, step) where a row is
//    touched again it emits a task "wait until the leader has finished the
//    row's previous touch, replay the steps in between, signal ready[step]".
//    Rows touched in consecutive steps stay in the leader's shared memory.
//    The leader therefore never waits on HBM-bound dense Adam; per step it
//    only spins on one counter that helpers have usually filled long before.
//  * Epoch end (one cooperative grid.sync() per phase): every row is flushed
//    to the last step, the monitor MSE is computed in parallel and summed in
//    the reference's sequential order (cells_mse, cfcomplete.cpp:34-43),
//    early stopping / best snapshot (:179-190) decided on the device.
//
// The host side of the schedule (mt19937_64 init draws, the validation split
// and each epoch's Fisher-Yates shuffle, rng.hpp / cfcomplete.cpp:74-105,
// :153-154) is generated one epoch ahead while the device runs the current
// epoch: it is the same RNG stream the reference draws, produced where the
// reference produces it.  No parameter arithmetic happens on the host.
//
// Precision: ExactNum<LANE> = FP64 in the operation order of the reference's
// kernel lane (lane_ops.cuh; glibc-exact exp) -> parameters and meta bit-
// identical to the reference.  FastNum = FP32 on the same schedule.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "lane_ops.cuh"
#include "ncf_joint.h"
#include "ocg_common.cuh"

namespace cg = cooperative_groups;

namespace ocg {

namespace {

constexpr int kJT = 512;  // threads per CTA (leader: 16 warps over neurons)
constexpr int kJW = kJT / 32;
constexpr int kJMaxK = 64;        // embedding dim
constexpr int kJMaxIn = 2 * kJMaxK;
constexpr int kJMaxHid = 64;      // hidden widths
constexpr int kJMaxL = 4;         // layers (hidden + output)
constexpr int kJMaxB = 32;        // minibatch (one sample per lane)
constexpr int kJMaxSlots = 2 * kJMaxB;
constexpr int kRC = 8;  // parameters per replay lane: independent Adam chains (ILP)
constexpr double kB1 = 0.9, kB2 = 0.999, kEps = 1e-8;  // AdamState defaults (nnkit.hpp:95)

struct JointCtl {
    double best_val;
    double last_val;
    int stale, stop, improved, diverged;
};

// shared-memory carve-up (byte offsets), computed on the host
struct JLayout {
    uint32_t P, M, V, slot[2], act[kJMaxL + 1], del[kJMaxL], ig, sy, ssa, sss, tab, smask, ones, srow;
    uint32_t bytes;
};

template <typename T>
struct JointArgs {
    int64_t m, n;
    int ka, ks, L, kmax, lpt;  // lpt: replay lanes per row (kRC parameters each)
    int dims[kJMaxL + 1], stride[kJMaxL + 1];
    int off_w[kJMaxL], off_b[kJMaxL];  // within the MLP block
    int T_mlp;
    T lr;
    JLayout lay;
    // resident state: per row [p(k) | m(k) | v(k)]
    T* app_rec;
    T* set_rec;
    int64_t* row_last;  // global Adam step through which the row's state is current
    T* mlp;             // [p | m | v] of the MLP block
    const uint32_t* dec;  // per MLP parameter: col | row << 8 | layer << 16 | weight << 20 | vec << 21
    int64_t app_vec, set_vec;  // (m*ka) & ~3, (n*ks) & ~3: AVX2-lane vector/tail split
    const double* tab_mc;
    const double* tab_vc;
    int64_t tab_len;  // steps t >= tab_len have mc = vc = 1 exactly
    // this epoch's schedule
    int64_t epoch_base;  // Adam step count before the epoch
    int S, nt, B;
    const double* smp_y;
    const uint16_t* smp_slot;  // app slot | setting slot << 8
    const int32_t* slot_off;   // [S+1]
    const int32_t* slot_row;   // global row: app i, or m + setting j
    const int16_t* slot_prev;  // slot index in step s-1 holding the row's state, or -1
    // replay tasks (row touched at step s, previously at leader step w, -1: none this epoch),
    // grouped in SIMD bundles of similar availability and length, claimed in availability order
    const int32_t* task_row;
    const int32_t* task_step;
    const int32_t* task_wait;
    const int32_t* b_off;   // [nbundle + 1]
    const int32_t* b_wait;  // leader step the bundle waits for
    int nbundle;
    int* bundle_next;
    const int32_t* need;  // tasks per step
    int* progress;
    int* ready;
    // monitor cells (validation, or train when the split left none)
    const int32_t* mon_app;
    const int32_t* mon_set;
    const double* mon_y;
    int64_t nmon;
    double* err2;
    T* best_app;
    T* best_set;
    T* best_mlp;
    JointCtl* ctl;
    int patience;
    unsigned long long* prof;  // optional leader phase cycle counters (OCG_JOINT_PROFILE)
};

// ---------------------------------------------------------------- numerics
template <int LANE>
struct ExactNum {
    using T = double;
    static constexpr bool kExact = true;
    __device__ static T add(T a, T b) { return dadd(a, b); }
    __device__ static T sub(T a, T b) { return dsub(a, b); }
    __device__ static T mul(T a, T b) { return dmul(a, b); }
    __device__ static T dot(const T* w, const T* x, int n) { return LaneOps<LANE>::dot(w, x, n); }
    __device__ static T axpy(T y, T a, T x) { return LaneOps<LANE>::axpy(y, a, x); }
    __device__ static void adam(T& p, T& m, T& v, T g, T lr, double mc, double vc, bool vec) {
        LaneOps<LANE>::adam(p, m, v, g, lr, kB1, dsub(1.0, kB1), kB2, dsub(1.0, kB2), kEps, mc, vc, vec);
    }
    __device__ static void selu(T z, T& a, T& gf, ExpTabPtr tab) { selu_fwd(z, a, gf, tab); }
    __device__ static double sq(T e) { return dmul(e, e); }
    // a zero-gradient step, the reference lane's exact operations (g = +0)
    __device__ static void zadam(T& p, T& m, T& v, T lr, double mc, double vc, bool vec) {
        adam(p, m, v, T(0), lr, mc, vc, vec);
    }
};

// FP32 on the reference schedule (FastNumT<double>: the same formulas in FP64,
// a diagnostic that separates FP32 rounding from the code path)
template <typename TT>
struct FastNumT {
    using T = TT;
    static constexpr bool kExact = false;
    __device__ static T add(T a, T b) { return a + b; }
    __device__ static T sub(T a, T b) { return a - b; }
    __device__ static T mul(T a, T b) { return a * b; }
    __device__ static T fma_(T a, T b, T c) { return fma(a, b, c); }
    __device__ static T dot(const T* w, const T* x, int n) {
        T a0 = 0, a1 = 0, a2 = 0, a3 = 0;
        int i = 0;
        for (; i + 4 <= n; i += 4) {
            a0 = fma_(w[i], x[i], a0);
            a1 = fma_(w[i + 1], x[i + 1], a1);
            a2 = fma_(w[i + 2], x[i + 2], a2);
            a3 = fma_(w[i + 3], x[i + 3], a3);
        }
        for (; i < n; ++i) a0 = fma_(w[i], x[i], a0);
        return (a0 + a2) + (a1 + a3);
    }
    __device__ static T axpy(T y, T a, T x) { return fma_(a, x, y); }
    __device__ static void adam(T& p, T& m, T& v, T g, T lr, double mc, double vc, bool) {
        m = fma_(T(0.9), m, T(0.1) * g);
        v = fma_(T(0.999), v, T(0.001) * (g * g));
        const T num = m * static_cast<T>(mc);
        const T den = sqrt(v * static_cast<T>(vc)) + T(1e-8);
        p = fma_(-lr, num / den, p);
    }
    __device__ static void selu(T z, T& a, T& gf, ExpTabPtr) {
        const T l = T(1.0507009873554805), la = T(1.0507009873554805 * 1.6732632423543772);
        if (z > T(0)) {
            a = l * z;
            gf = l;
        } else {
            const T e = exp(z);
            a = la * (e - T(1));
            gf = la * e;
        }
    }
    __device__ static double sq(T e) { return static_cast<double>(e) * static_cast<double>(e); }
    // a zero-gradient step: the g terms vanish; FP32 mode uses the approximate sqrt / divide
    // (a few ulp, like any FP32 Adam) on this replay path
    __device__ static void zadam(T& p, T& m, T& v, T lr, double mc, double vc, bool) {
        if constexpr (sizeof(T) == 4) {
            m = m * 0.9f;
            v = v * 0.999f;
            float r;
            asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(v * static_cast<float>(vc)));
            p = __fmaf_rn(-lr, __fdividef(m * static_cast<float>(mc), r + 1e-8f), p);
        } else {
            adam(p, m, v, T(0), lr, mc, vc, false);  // (the FP64 diagnostic build keeps the full step)
        }
    }
};
using FastNum = FastNumT<float>;

template <typename T>
__device__ __forceinline__ T* sp(char* base, uint32_t off) {
    return reinterpret_cast<T*>(base + off);
}

extern __shared__ __align__(16) char g_jsmem[];

// Spin with relaxed loads and acquire once: an ld.acquire compiles to a load plus an
// L1 invalidation (CCTL.IVALL), which inside a spin loop evicts the waiting SM's L1
// on every iteration (76 % of the epoch kernel's stall samples in the first capture).
__device__ __forceinline__ int ld_relaxed(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void wait_geq(const int* p, int want, bool sleep) {
    if (ld_relaxed(p) < want) {
        do {
            if (sleep) __nanosleep(32);
        } while (ld_relaxed(p) < want);
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void step_corr(const double* mc_tab, const double* vc_tab, int64_t len, int64_t t, double& mc,
                                          double& vc) {
    if (t < len) {
        mc = __ldg(mc_tab + t);
        vc = __ldg(vc_tab + t);
    } else {
        mc = 1.0;
        vc = 1.0;
    }
}

// zero-gradient Adam steps t0..t1 (inclusive) of parameters [ch*kRC, ch*kRC + kRC)
// of one embedding row: kRC independent chains per lane (exact lane arithmetic)
template <class NUM, typename T>
__device__ __forceinline__ void replay_chunk(const JointArgs<T>& a, int64_t row, int ch, int64_t t0, int64_t t1) {
    const bool is_app = row < a.m;
    const int k = is_app ? a.ka : a.ks;
    const int c0 = ch * kRC;
    if (t0 > t1 || c0 >= k) return;
    const int64_t r = is_app ? row : row - a.m;
    T* rec = (is_app ? a.app_rec : a.set_rec) + r * 3 * k;
    const int64_t vlim = (is_app ? a.app_vec : a.set_vec) - r * k;  // column c < vlim: AVX2 vector body
    T p[kRC], mm[kRC], vv[kRC];
#pragma unroll
    for (int j = 0; j < kRC; ++j) {
        const int c = c0 + j;
        p[j] = c < k ? __ldcg(rec + c) : T(0);
        mm[j] = c < k ? __ldcg(rec + k + c) : T(0);
        vv[j] = c < k ? __ldcg(rec + 2 * k + c) : T(0);
    }
    // bias corrections of step t + 1 are loaded while step t computes; once both reach 1.0
    // (t >= tab_len: ~37K steps into a fit) the loop needs no table at all
    double mc, vc;
    step_corr(a.tab_mc, a.tab_vc, a.tab_len, t0, mc, vc);
    int64_t t = t0;
    for (; t <= t1 && t < a.tab_len; ++t) {
        double mcn, vcn;
        step_corr(a.tab_mc, a.tab_vc, a.tab_len, t + 1, mcn, vcn);
#pragma unroll
        for (int j = 0; j < kRC; ++j) NUM::zadam(p[j], mm[j], vv[j], a.lr, mc, vc, c0 + j < vlim);
        mc = mcn;
        vc = vcn;
    }
    for (; t <= t1; ++t) {
#pragma unroll
        for (int j = 0; j < kRC; ++j) NUM::zadam(p[j], mm[j], vv[j], a.lr, 1.0, 1.0, c0 + j < vlim);
    }
#pragma unroll
    for (int j = 0; j < kRC; ++j) {
        const int c = c0 + j;
        if (c < k) {
            __stcg(rec + c, p[j]);
            __stcg(rec + k + c, mm[j]);
            __stcg(rec + 2 * k + c, vv[j]);
        }
    }
}

// MLP parameter e (offset in the MLP block) -> layer, row, col, kind, vector flag
struct MlpParam {
    int layer, r, c;
    bool weight, vec;
};
template <typename T>
__device__ __forceinline__ MlpParam decode_mlp(const JointArgs<T>& a, int e) {
    MlpParam d;
    int l = 0;
    while (l + 1 < a.L && e >= a.off_w[l + 1]) ++l;
    d.layer = l;
    const int in = a.dims[l], out = a.dims[l + 1];
    if (e < a.off_b[l]) {
        const int q = e - a.off_w[l];
        d.weight = true;
        d.r = q / in;
        d.c = q - d.r * in;
        d.vec = q < ((out * in) & ~3);
    } else {
        d.weight = false;
        d.r = e - a.off_b[l];
        d.c = 0;
        d.vec = d.r < (out & ~3);
    }
    return d;
}

// ------------------------------------------------------------- leader CTA
// Layer shapes: run-time (any NcfHyper within the kernel's limits) or compile-time
// (FixShape: every layer loop unrolled, every index product folded).
struct RtShape {
    int L_, ka_, ks_, kmax_, dims_[kJMaxL + 1], stride_[kJMaxL + 1], offw_[kJMaxL], offb_[kJMaxL];
    template <typename T>
    __device__ explicit RtShape(const JointArgs<T>& a) : L_(a.L), ka_(a.ka), ks_(a.ks), kmax_(a.kmax) {
#pragma unroll
        for (int l = 0; l <= kJMaxL; ++l) {
            dims_[l] = l <= a.L ? a.dims[l] : 0;
            stride_[l] = l <= a.L ? a.stride[l] : 0;
        }
#pragma unroll
        for (int l = 0; l < kJMaxL; ++l) {
            offw_[l] = l < a.L ? a.off_w[l] : 0;
            offb_[l] = l < a.L ? a.off_b[l] : 0;
        }
    }
    __device__ int L() const { return L_; }
    __device__ int ka() const { return ka_; }
    __device__ int ks() const { return ks_; }
    __device__ int kmax() const { return kmax_; }
    __device__ int dim(int l) const { return dims_[l]; }
    __device__ int stride(int l) const { return stride_[l]; }
    __device__ int off_w(int l) const { return offw_[l]; }
    __device__ int off_b(int l) const { return offb_[l]; }
};

template <int KA, int KS, int H0, int H1>
struct FixShape {
    template <typename T>
    __device__ explicit FixShape(const JointArgs<T>&) {}
    __device__ static constexpr int L() { return 3; }
    __device__ static constexpr int ka() { return KA; }
    __device__ static constexpr int ks() { return KS; }
    __device__ static constexpr int kmax() { return KA > KS ? KA : KS; }
    __device__ static constexpr int dim(int l) { return l == 0 ? KA + KS : (l == 1 ? H0 : (l == 2 ? H1 : 1)); }
    __device__ static constexpr int stride(int l) { return dim(l) | 1; }
    __device__ static constexpr int off_w(int l) {
        return l == 0 ? 0 : (l == 1 ? (KA + KS) * H0 + H0 : (KA + KS) * H0 + H0 + H0 * H1 + H1);
    }
    __device__ static constexpr int off_b(int l) { return off_w(l) + dim(l) * dim(l + 1); }
};
using DefaultShape = FixShape<8, 8, 32, 16>;  // NcfHyper{} (cfcomplete.hpp:11-20)

template <class NUM, class SH, typename T>
__device__ void leader_epoch(const JointArgs<T>& a) {
    const SH sh(a);
    char* sm = g_jsmem;
    const JLayout& ly = a.lay;
    T* P = sp<T>(sm, ly.P);
    T* M = sp<T>(sm, ly.M);
    T* V = sp<T>(sm, ly.V);
    double* sy = sp<double>(sm, ly.sy);
    int* ssa = sp<int>(sm, ly.ssa);
    int* sss = sp<int>(sm, ly.sss);
    // per slot, bit q = minibatch sample q touches the slot's row; double-buffered by step parity
    uint32_t* smask = sp<uint32_t>(sm, ly.smask);
    const ExpTabPtr tab{sp<uint64_t>(sm, ly.tab)};
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int L = sh.L(), kmax = sh.kmax(), rs = 3 * kmax;
    const int in0 = sh.dim(0), st0 = sh.stride(0);

    const uint32_t* dec = a.dec;
    for (int e = tid; e < a.T_mlp; e += kJT) {
        P[e] = __ldcg(a.mlp + e);
        M[e] = __ldcg(a.mlp + a.T_mlp + e);
        V[e] = __ldcg(a.mlp + 2 * a.T_mlp + e);
    }
    for (int q = tid; q < 2 * kJMaxSlots; q += kJT) smask[q] = 0u;
    if (tid == 0) *sp<T>(sm, ly.ones) = T(1);
    __syncthreads();

    int64_t* srow = sp<int64_t>(sm, ly.srow);
    // the host-built schedule of step s + 1 is read during step s (off the critical path)
    int so_n = a.S > 0 ? a.slot_off[0] : 0, so1_n = a.S > 0 ? a.slot_off[1] : 0;
    int need_n = tid == 0 && a.S > 0 ? a.need[0] : 0;
    uint16_t smp_n = 0;
    double y_n = 0.0;
    if (a.S > 0 && tid < min(a.B, a.nt)) {
        smp_n = a.smp_slot[tid];
        y_n = a.smp_y[tid];
    }
    for (int s = 0; s < a.S; ++s) {
        const int cnt = min(a.B, a.nt - s * a.B);
        const int64_t t = a.epoch_base + s + 1;
        double mc, vc;
        step_corr(a.tab_mc, a.tab_vc, a.tab_len, t, mc, vc);
        const int so = so_n, nsl = so1_n - so_n;
        const int want_s = need_n;
        const uint16_t smp_s = smp_n;
        const double y_s = y_n;
        if (s + 1 < a.S) {
            so_n = so1_n;
            so1_n = a.slot_off[s + 2];
            if (tid == 0) need_n = a.need[s + 1];
            if (tid < min(a.B, a.nt - (s + 1) * a.B)) {
                smp_n = a.smp_slot[static_cast<int64_t>(s + 1) * a.B + tid];
                y_n = a.smp_y[static_cast<int64_t>(s + 1) * a.B + tid];
            }
        }
        T* cur = sp<T>(sm, ly.slot[s & 1]);
        const T* prv = sp<T>(sm, ly.slot[(s + 1) & 1]);
        long long c0 = 0, c1 = 0;
        if (tid == 0) {
            c0 = clock64();
            wait_geq(a.ready + s, want_s, false);
            c1 = clock64();
        }
        uint32_t* mk_cur = smask + (s & 1) * kJMaxSlots;
        if (tid < cnt) {
            const uint16_t sl = smp_s;
            ssa[tid] = sl & 0xff;
            sss[tid] = sl >> 8;
            sy[tid] = y_s;
            atomicOr(mk_cur + (sl & 0xff), 1u << tid);
            atomicOr(mk_cur + (sl >> 8), 1u << tid);
        }
        // the other buffer was last read in step s - 1 (finished): clear it for step s + 1
        if (tid >= kJT - kJMaxSlots) smask[((s + 1) & 1) * kJMaxSlots + tid - (kJT - kJMaxSlots)] = 0u;
        __syncthreads();
        // ---- slots: from the previous step's smem, or (replayed) from HBM
        for (int q = tid; q < nsl * kmax; q += kJT) {
            const int sl = q / kmax, c = q - sl * kmax;
            const int64_t row = a.slot_row[so + sl];
            if (c == 0) srow[sl] = row;  // for the Adam and write-back phases (no second HBM/L2 trip)
            const bool is_app = row < a.m;
            const int k = is_app ? sh.ka() : sh.ks();
            if (c >= k) continue;
            const int ps = a.slot_prev[so + sl];
            T* d = cur + sl * rs;
            if (ps >= 0) {
                const T* src = prv + ps * rs;
                d[c] = src[c];
                d[kmax + c] = src[kmax + c];
                d[2 * kmax + c] = src[2 * kmax + c];
            } else {
                const T* rec = is_app ? a.app_rec + row * 3 * k : a.set_rec + (row - a.m) * 3 * k;
                d[c] = __ldcg(rec + c);
                d[kmax + c] = __ldcg(rec + k + c);
                d[2 * kmax + c] = __ldcg(rec + 2 * k + c);
            }
        }
        __syncthreads();
        long long c2 = tid == 0 ? clock64() : 0;
        // ---- concat_embed (cfcomplete.cpp:23-32)
        T* X = sp<T>(sm, ly.act[0]);
        for (int w = tid; w < cnt * in0; w += kJT) {
            const int smp = w / in0, i = w - smp * in0;
            X[smp * st0 + i] = i < sh.ka() ? cur[ssa[smp] * rs + i] : cur[sss[smp] * rs + (i - sh.ka())];
        }
        __syncthreads();
        // ---- forward_tape (nnkit.cpp:124-138)
#pragma unroll
        for (int l = 0; l < kJMaxL; ++l) {
            if (l >= L) break;
            const int in = sh.dim(l), out = sh.dim(l + 1);
            const T* W = P + sh.off_w(l);
            const T* b = P + sh.off_b(l);
            const T* ain = sp<T>(sm, ly.act[l]) + lane * sh.stride(l);
            T* aout = sp<T>(sm, ly.act[l + 1]) + lane * sh.stride(l + 1);
            T* gfo = sp<T>(sm, ly.del[l]) + lane * sh.stride(l + 1);
            const bool hidden = l + 1 < L;
            if (lane < cnt) {
                for (int o = warp; o < out; o += kJW) {
                    const T z = NUM::add(NUM::dot(W + o * in, ain, in), b[o]);
                    T v = z, gf = T(1);
                    if (hidden) NUM::selu(z, v, gf, tab);
                    aout[o] = v;
                    gfo[o] = gf;
                }
            }
            __syncthreads();
        }
        // ---- backprop_sample (nnkit.cpp:184-212)
        const T scale = NUM::kExact ? T(ddiv(1.0, static_cast<double>(cnt))) : T(1) / T(cnt);
        if (warp == 0 && lane < cnt) {
            const T err = NUM::sub(sp<T>(sm, ly.act[L])[lane * sh.stride(L)], T(sy[lane]));
            sp<T>(sm, ly.del[L - 1])[lane * sh.stride(L)] = NUM::mul(NUM::mul(NUM::mul(T(2), err), scale), T(1));
        }
        __syncthreads();
#pragma unroll
        for (int l = kJMaxL - 1; l >= 0; --l) {
            if (l >= L) continue;
            const int in = sh.dim(l), out = sh.dim(l + 1);
            const T* W = P + sh.off_w(l);
            const T* d = sp<T>(sm, ly.del[l]) + lane * sh.stride(l + 1);
            if (lane < cnt) {
                for (int c = warp; c < in; c += kJW) {
                    T nd = T(0);  // matvec_t: out[c] = 0; out[c] += d[r] * w[r][c]
                    for (int r = 0; r < out; ++r) nd = NUM::axpy(nd, d[r], W[r * in + c]);
                    if (l > 0) {
                        T* gf = sp<T>(sm, ly.del[l - 1]) + lane * sh.stride(l) + c;
                        *gf = NUM::mul(nd, *gf);  // delta *= activate_grad
                    } else {
                        sp<T>(sm, ly.ig)[lane * st0 + c] = nd;
                    }
                }
            }
            __syncthreads();
        }
        long long c3 = tid == 0 ? clock64() : 0;
        // ---- gradient sums in sample order + Adam (nnkit.cpp:239-251)
        if (cnt == kJMaxB) {
            // full minibatch: two parameters per pass, their 32-sample chains side by side.  A bias
            // chain is the weight chain against x = 1 (fma(d, 1, g) and g + d*1 both round d + g
            // once, exactly the reference's add), so both chains are the same straight-line code.
            const T* ones = sp<T>(sm, ly.ones);
            for (int e0 = tid; e0 < a.T_mlp; e0 += 2 * kJT) {
                const int e1 = e0 + kJT;
                const bool has1 = e1 < a.T_mlp;
                const uint32_t d0 = __ldg(dec + e0), d1 = has1 ? __ldg(dec + e1) : d0;
                const int l0 = (d0 >> 16) & 15, l1 = (d1 >> 16) & 15;
                const T* dl0 = sp<T>(sm, ly.del[l0]) + ((d0 >> 8) & 255);
                const T* dl1 = sp<T>(sm, ly.del[l1]) + ((d1 >> 8) & 255);
                const int sd0 = sh.stride(l0 + 1), sd1 = sh.stride(l1 + 1);
                const bool w0 = d0 & (1u << 20), w1 = d1 & (1u << 20);
                const T* al0 = w0 ? sp<T>(sm, ly.act[l0]) + (d0 & 255) : ones;
                const T* al1 = w1 ? sp<T>(sm, ly.act[l1]) + (d1 & 255) : ones;
                const int sa0 = w0 ? sh.stride(l0) : 0, sa1 = w1 ? sh.stride(l1) : 0;
                T g0 = T(0), g1 = T(0);
#pragma unroll
                for (int q2 = 0; q2 < kJMaxB; ++q2) {
                    g0 = NUM::axpy(g0, dl0[q2 * sd0], al0[q2 * sa0]);
                    g1 = NUM::axpy(g1, dl1[q2 * sd1], al1[q2 * sa1]);
                }
                NUM::adam(P[e0], M[e0], V[e0], g0, a.lr, mc, vc, (d0 >> 21) & 1);
                if (has1) NUM::adam(P[e1], M[e1], V[e1], g1, a.lr, mc, vc, (d1 >> 21) & 1);
            }
        } else {
            for (int e = tid; e < a.T_mlp; e += kJT) {
                const uint32_t d = __ldg(dec + e);
                const int layer = (d >> 16) & 15, r = (d >> 8) & 255, c = d & 255;
                const T* dl = sp<T>(sm, ly.del[layer]) + r;
                const int sd = sh.stride(layer + 1);
                T g = T(0);
                if (d & (1u << 20)) {  // outer_acc: G[r][c] += d[r] * x[c], samples in order
                    const T* al = sp<T>(sm, ly.act[layer]) + c;
                    const int sa = sh.stride(layer);
                    for (int q = 0; q < cnt; ++q) g = NUM::axpy(g, dl[q * sd], al[q * sa]);
                } else {
                    for (int q = 0; q < cnt; ++q) g = NUM::add(g, dl[q * sd]);
                }
                NUM::adam(P[e], M[e], V[e], g, a.lr, mc, vc, (d >> 21) & 1);
            }
        }
        const T* ig = sp<T>(sm, ly.ig);
        for (int q = tid; q < nsl * kmax; q += kJT) {
            const int sl = q / kmax, c = q - sl * kmax;
            const int64_t row = srow[sl];
            const bool is_app = row < a.m;
            const int k = is_app ? sh.ka() : sh.ks();
            if (c >= k) continue;
            T g = T(0);  // embedding-gradient scatter (cfcomplete.cpp:171-174), samples in order
            const T* igc = ig + (is_app ? c : sh.ka() + c);
            for (uint32_t mk = mk_cur[sl]; mk; mk &= mk - 1) g = NUM::add(g, igc[(__ffs(mk) - 1) * st0]);
            T* d = cur + sl * rs;
            const int64_t r = is_app ? row : row - a.m;
            const bool vec = r * k + c < (is_app ? a.app_vec : a.set_vec);
            NUM::adam(d[c], d[kmax + c], d[2 * kmax + c], g, a.lr, mc, vc, vec);
        }
        __syncthreads();
        long long c4 = tid == 0 ? clock64() : 0;
        // ---- write the touched rows back, then publish the step
        for (int q = tid; q < nsl * kmax; q += kJT) {
            const int sl = q / kmax, c = q - sl * kmax;
            const int64_t row = srow[sl];
            const bool is_app = row < a.m;
            const int k = is_app ? sh.ka() : sh.ks();
            if (c >= k) continue;
            T* rec = is_app ? a.app_rec + row * 3 * k : a.set_rec + (row - a.m) * 3 * k;
            const T* d = cur + sl * rs;
            __stcg(rec + c, d[c]);
            __stcg(rec + k + c, d[kmax + c]);
            __stcg(rec + 2 * k + c, d[2 * kmax + c]);
            if (c == 0) __stcg(a.row_last + row, t);
        }
        __syncthreads();
        if (tid == kJT - 1) {
            __threadfence();
            st_release(a.progress, s);
        }
        if (tid == 0 && a.prof) {
            const long long c5 = clock64();
            a.prof[0] += c1 - c0;  // waiting for replays
            a.prof[1] += c2 - c1;  // slot loads
            a.prof[2] += c3 - c2;  // forward + backward
            a.prof[3] += c4 - c3;  // gradients + Adam
            a.prof[4] += c5 - c4;  // write-back + publish
            a.prof[5] += 1;
        }
    }
    for (int e = tid; e < a.T_mlp; e += kJT) {
        __stcg(a.mlp + e, P[e]);
        __stcg(a.mlp + a.T_mlp + e, M[e]);
        __stcg(a.mlp + 2 * a.T_mlp + e, V[e]);
    }
}

// ----------------------------------------------------------- helper warps
// A warp claims the next bundle (tasks of similar availability and replay
// length), waits until the leader has finished the bundle's latest previous
// touch, replays every task's rows in SIMD, then counts each task into ready[s].
template <class NUM, typename T>
__device__ void helper_epoch(const JointArgs<T>& a) {
    const int lane = threadIdx.x & 31;
    const int tl = lane / a.lpt, ch = lane - tl * a.lpt;
    for (;;) {
        int bi = 0;
        if (lane == 0) bi = atomicAdd(a.bundle_next, 1);
        bi = __shfl_sync(0xffffffffu, bi, 0);
        if (bi >= a.nbundle) break;
        const int wait = a.b_wait[bi];
        if (lane == 0 && wait >= 0)
            wait_geq(a.progress, wait, true);
        __syncwarp();
        const int q0 = a.b_off[bi], cnt = a.b_off[bi + 1] - q0;
        int s = 0;
        if (tl < cnt) {
            const int q = q0 + tl;
            const int64_t row = a.task_row[q];
            s = a.task_step[q];
            const int w = a.task_wait[q];
            const int64_t t = a.epoch_base + s + 1;
            const int64_t last = w >= 0 ? a.epoch_base + w + 1 : a.epoch_base;
            replay_chunk<NUM>(a, row, ch, last + 1, t - 1);
        }
        __threadfence();
        __syncwarp();
        if (tl < cnt && ch == 0) atomicAdd(a.ready + s, 1);
    }
}

// ------------------------------------------------------------ evaluation
template <typename T>
struct PView {
    const T* app;
    int64_t sa;
    const T* set;
    int64_t ss;
};

// squared error of one cell with the MLP in shared memory (forward,
// nnkit.cpp:74-89; cells_mse's err*err, cfcomplete.cpp:38-40)
template <class NUM, typename T, class Arg>
__device__ double cell_sqerr(const Arg& a, const T* W, const PView<T>& pv, int64_t app, int64_t set, double y,
                             ExpTabPtr tab) {
    T b0[kJMaxIn], b1[kJMaxIn];
    T* x = b0;
    T* z = b1;
    for (int i = 0; i < a.ka; ++i) x[i] = pv.app[app * pv.sa + i];
    for (int i = 0; i < a.ks; ++i) x[a.ka + i] = pv.set[set * pv.ss + i];
    for (int l = 0; l < a.L; ++l) {
        const int in = a.dims[l], out = a.dims[l + 1];
        const bool hidden = l + 1 < a.L;
        for (int o = 0; o < out; ++o) {
            T v = NUM::add(NUM::dot(W + a.off_w[l] + o * in, x, in), W[a.off_b[l] + o]);
            if (hidden) {
                T gf;
                NUM::selu(v, v, gf, tab);
            }
            z[o] = v;
        }
        T* tmp = x;
        x = z;
        z = tmp;
    }
    return NUM::sq(NUM::sub(x[0], T(y)));
}

template <class NUM, typename T, class Arg>
__device__ void eval_cells(const Arg& a, const T* mlp_p, const PView<T>& pv, const int32_t* capp, const int32_t* cset,
                           const double* cy, int64_t count, double* err2, const JLayout& ly) {
    char* sm = g_jsmem;
    T* W = sp<T>(sm, ly.P);
    uint64_t* tb = sp<uint64_t>(sm, ly.tab);
    for (int e = threadIdx.x; e < a.T_mlp; e += blockDim.x) W[e] = __ldcg(mlp_p + e);
    for (int e = threadIdx.x; e < 256; e += blockDim.x) tb[e] = exp_tab(e);
    __syncthreads();
    const ExpTabPtr tab{tb};
    const int64_t nth = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += nth)
        err2[i] = cell_sqerr<NUM>(a, W, pv, capp[i], cset[i], cy[i], tab);
}

template <class NUM, class SH>
__global__ void __launch_bounds__(kJT, 1) joint_epoch_kernel(JointArgs<typename NUM::T> a) {
    using T = typename NUM::T;
    cg::grid_group grid = cg::this_grid();
    if (blockIdx.x == 0) {
        for (int e = threadIdx.x; e < 256; e += kJT) sp<uint64_t>(g_jsmem, a.lay.tab)[e] = exp_tab(e);
        __syncthreads();
        leader_epoch<NUM, SH>(a);
    } else {
        helper_epoch<NUM>(a);
    }
    grid.sync();
    // ---- flush every row to the epoch's last step
    const int64_t tend = a.epoch_base + a.S;
    {
        const int64_t gt = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
        const int64_t slot = gt / a.lpt, nslot = static_cast<int64_t>(gridDim.x) * blockDim.x / a.lpt;
        const int ch = static_cast<int>(gt - slot * a.lpt);
        for (int64_t row = slot; row < a.m + a.n; row += nslot)
            replay_chunk<NUM>(a, row, ch, __ldcg(a.row_last + row) + 1, tend);
    }
    grid.sync();
    {
        const int64_t nth = static_cast<int64_t>(gridDim.x) * blockDim.x;
        for (int64_t row = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; row < a.m + a.n; row += nth)
            a.row_last[row] = tend;
    }
    // ---- monitor MSE
    const PView<T> cur{a.app_rec, 3 * a.ka, a.set_rec, 3 * a.ks};
    eval_cells<NUM>(a, a.mlp, cur, a.mon_app, a.mon_set, a.mon_y, a.nmon, a.err2, a.lay);
    grid.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        double acc = 0.0;  // sequential, in the monitor list's order
        for (int64_t i = 0; i < a.nmon; ++i) acc = dadd(acc, __ldcg(a.err2 + i));
        const double vl = a.nmon == 0 ? 0.0 : ddiv(acc, static_cast<double>(a.nmon));
        JointCtl c = *a.ctl;
        c.last_val = vl;
        c.improved = 0;
        if (!isfinite(vl)) {
            c.diverged = 1;
            c.stop = 1;
        } else if (vl < c.best_val) {
            c.best_val = vl;
            c.stale = 0;
            c.improved = 1;
        } else if (++c.stale > a.patience) {
            c.stop = 1;
        }
        *a.ctl = c;
        __threadfence();
    }
    grid.sync();
    // ---- best snapshot (cfcomplete.cpp:183-185)
    if (__ldcg(&a.ctl->improved)) {
        const int64_t nth = static_cast<int64_t>(gridDim.x) * blockDim.x;
        const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
        for (int64_t q = tid; q < a.m * a.ka; q += nth) {
            const int64_t r = q / a.ka;
            a.best_app[q] = __ldcg(a.app_rec + r * 3 * a.ka + (q - r * a.ka));
        }
        for (int64_t q = tid; q < a.n * a.ks; q += nth) {
            const int64_t r = q / a.ks;
            a.best_set[q] = __ldcg(a.set_rec + r * 3 * a.ks + (q - r * a.ks));
        }
        for (int64_t q = tid; q < a.T_mlp; q += nth) a.best_mlp[q] = __ldcg(a.mlp + q);
    }
}

// standalone evaluation (initial / final MSE) and the sequential sum
template <class NUM>
__global__ void __launch_bounds__(kJT) joint_eval_kernel(JointArgs<typename NUM::T> a, PView<typename NUM::T> pv,
                                                         const typename NUM::T* mlp_p, const int32_t* capp,
                                                         const int32_t* cset, const double* cy, int64_t count,
                                                         double* err2) {
    eval_cells<NUM>(a, mlp_p, pv, capp, cset, cy, count, err2, a.lay);
}

__global__ void joint_sum_kernel(const double* err2, int64_t count, double* out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double acc = 0.0;
    for (int64_t i = 0; i < count; ++i) acc = dadd(acc, err2[i]);
    *out = count == 0 ? 0.0 : ddiv(acc, static_cast<double>(count));
}

template <typename T>
__global__ void joint_scatter_init_kernel(const T* flat, int64_t rows, int k, T* rec) {
    const int64_t nth = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < rows * k; q += nth) {
        const int64_t r = q / k, c = q - r * k;
        rec[r * 3 * k + c] = flat[q];
        rec[r * 3 * k + k + c] = T(0);
        rec[r * 3 * k + 2 * k + c] = T(0);
    }
}

__global__ void joint_check_finite_kernel(const double* p, int64_t count, int* bad) {
    const int64_t nth = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < count; q += nth)
        if (!isfinite(p[q])) atomicOr(bad, 1);
}

template <typename T>
__global__ void joint_widen_kernel(const T* src, double* dst, int64_t count) {
    const int64_t nth = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < count; q += nth)
        dst[q] = static_cast<double>(src[q]);
}

// ================================================================== host
template <typename T>
struct JBuf {
    T* p = nullptr;
    size_t n = 0;
    JBuf() = default;
    JBuf(const JBuf&) = delete;
    JBuf& operator=(const JBuf&) = delete;
    ~JBuf() {
        if (p) cudaFree(p);
    }
    cudaError_t alloc(size_t count) {
        if (p) cudaFree(p);
        p = nullptr;
        n = count;
        return cudaMalloc(&p, sizeof(T) * std::max<size_t>(count, 1));
    }
};

template <typename T>
struct PinBuf {
    T* p = nullptr;
    size_t n = 0;
    PinBuf() = default;
    PinBuf(const PinBuf&) = delete;
    PinBuf& operator=(const PinBuf&) = delete;
    ~PinBuf() {
        if (p) cudaFreeHost(p);
    }
    cudaError_t reserve(size_t count) {
        if (count <= n && p) return cudaSuccess;
        if (p) cudaFreeHost(p);
        p = nullptr;
        n = std::max<size_t>(count, 1);
        return cudaMallocHost(&p, sizeof(T) * n);
    }
};

#define JCU(call)                                                                   \
    do {                                                                            \
        cudaError_t e_ = (call);                                                    \
        if (e_ != cudaSuccess) {                                                    \
            err = std::string(#call) + ": " + cudaGetErrorString(e_);               \
            return OCG_E_CUDA;                                                      \
        }                                                                           \
    } while (0)

struct Cell {
    int32_t app, set;
    double y;
};

// one epoch's schedule, built on the host from the shuffled train order
struct Sched {
    PinBuf<double> y;
    PinBuf<uint16_t> slot;
    PinBuf<int32_t> slot_off, slot_row, task_row, task_step, task_wait, need, b_off, b_wait;
    PinBuf<int16_t> slot_prev;
    int64_t nslots = 0, ntask = 0, nbundle = 0;
};
struct DSched {
    JBuf<double> y;
    JBuf<uint16_t> slot;
    JBuf<int32_t> slot_off, slot_row, task_row, task_step, task_wait, need, ready, b_off, b_wait;
    JBuf<int16_t> slot_prev;
};

class ScheduleBuilder {
  public:
    ScheduleBuilder(int64_t m, int64_t n, int B, int lpt, const std::vector<Cell>& train)
        : m_(m), B_(B), tpb_(32 / lpt), train_(train), stamp_(static_cast<size_t>(m + n), -1), slot_of_(static_cast<size_t>(m + n), 0),
          last_(static_cast<size_t>(m + n), -1), lastslot_(static_cast<size_t>(m + n), 0) {}

    cudaError_t build(const std::vector<int64_t>& idx, Sched& sc) {
        const int64_t nt = static_cast<int64_t>(idx.size());
        const int S = static_cast<int>((nt + B_ - 1) / B_);
        cudaError_t e;
        if ((e = sc.y.reserve(static_cast<size_t>(nt))) != cudaSuccess) return e;
        if ((e = sc.slot.reserve(static_cast<size_t>(nt))) != cudaSuccess) return e;
        if ((e = sc.slot_off.reserve(static_cast<size_t>(S) + 1)) != cudaSuccess) return e;
        if ((e = sc.need.reserve(static_cast<size_t>(S))) != cudaSuccess) return e;
        const size_t cap = static_cast<size_t>(S) * 2 * B_;
        if ((e = sc.slot_row.reserve(cap)) != cudaSuccess) return e;
        if ((e = sc.slot_prev.reserve(cap)) != cudaSuccess) return e;
        if ((e = sc.task_row.reserve(cap)) != cudaSuccess) return e;
        if ((e = sc.task_step.reserve(cap)) != cudaSuccess) return e;
        if ((e = sc.task_wait.reserve(cap)) != cudaSuccess) return e;
        if ((e = sc.b_off.reserve(cap + 1)) != cudaSuccess) return e;
        if ((e = sc.b_wait.reserve(cap)) != cudaSuccess) return e;
        trow_.resize(cap);
        tstep_.resize(cap);
        twait_.resize(cap);
        std::fill(last_.begin(), last_.end(), -1);
        std::fill(stamp_.begin(), stamp_.end(), -1);
        int64_t nsl = 0, ntk = 0;
        for (int s = 0; s < S; ++s) {
            sc.slot_off.p[s] = static_cast<int32_t>(nsl);
            const int64_t base = nsl;
            int need = 0;
            const int64_t q0 = static_cast<int64_t>(s) * B_, q1 = std::min<int64_t>(nt, q0 + B_);
            auto slot_for = [&](int64_t row) -> int {
                if (stamp_[row] == s) return slot_of_[row];
                const int q = static_cast<int>(nsl - base);
                stamp_[row] = s;
                slot_of_[row] = q;
                sc.slot_row.p[nsl] = static_cast<int32_t>(row);
                const int prev = last_[row];
                if (prev == s - 1 && s > 0) {
                    sc.slot_prev.p[nsl] = static_cast<int16_t>(lastslot_[row]);
                } else {
                    sc.slot_prev.p[nsl] = -1;
                    trow_[ntk] = static_cast<int32_t>(row);
                    tstep_[ntk] = s;
                    twait_[ntk] = prev;
                    ++ntk;
                    ++need;
                }
                ++nsl;
                return q;
            };
            for (int64_t q = q0; q < q1; ++q) {
                const Cell& c = train_[static_cast<size_t>(idx[static_cast<size_t>(q)])];
                const int sa = slot_for(c.app);
                const int ss = slot_for(m_ + c.set);
                sc.slot.p[q] = static_cast<uint16_t>(sa | (ss << 8));
                sc.y.p[q] = c.y;
            }
            for (int64_t q = base; q < nsl; ++q) {
                const int32_t row = sc.slot_row.p[q];
                last_[row] = s;
                lastslot_[row] = static_cast<int>(q - base);
            }
            sc.need.p[s] = need;
        }
        sc.slot_off.p[S] = static_cast<int32_t>(nsl);
        sc.nslots = nsl;
        sc.ntask = ntk;
        bundle(sc, S);
        return cudaSuccess;
    }

  private:
    // SIMD bundles of <= tpb_ tasks: same replay-length octave (r in [2^b, 2^(b+1)))
    // and availability (previous touch w) within a quarter of that length, so a
    // bundle's lanes run similar trip counts and its waits do not delay its
    // deadlines; bundles ordered by availability (LSD counting sorts, O(tasks + S)).
    void bundle(Sched& sc, int S) {
        const int64_t nt = sc.ntask;
        auto rlen = [&](int64_t i) -> int64_t { return twait_[i] >= 0 ? tstep_[i] - twait_[i] - 1 : tstep_[i]; };
        auto oct = [&](int64_t i) -> int {
            const int64_t r = rlen(i);
            return r <= 1 ? 0 : 63 - __builtin_clzll(static_cast<unsigned long long>(r));
        };
        ord_.resize(static_cast<size_t>(nt));
        tmp_.resize(static_cast<size_t>(nt));
        cnt_.assign(static_cast<size_t>(S) + 2, 0);
        for (int64_t i = 0; i < nt; ++i) ++cnt_[static_cast<size_t>(twait_[i] + 1) + 1];
        for (size_t k = 1; k < cnt_.size(); ++k) cnt_[k] += cnt_[k - 1];
        for (int64_t i = 0; i < nt; ++i) tmp_[static_cast<size_t>(cnt_[static_cast<size_t>(twait_[i] + 1)]++)] = i;
        int64_t oc[66] = {};
        for (int64_t i = 0; i < nt; ++i) ++oc[oct(i) + 1];
        for (int k = 1; k < 66; ++k) oc[k] += oc[k - 1];
        for (int64_t q = 0; q < nt; ++q) {
            const int64_t i = tmp_[static_cast<size_t>(q)];
            ord_[static_cast<size_t>(oc[oct(i)]++)] = i;
        }
        // bundles over the (octave, availability)-sorted list
        bstart_.clear();
        bwait_.clear();
        int cur_oct = -1, cur_cnt = 0, first_w = 0, max_w = -1;
        auto close = [&]() {
            if (cur_cnt) bwait_.push_back(max_w);
        };
        for (int64_t q = 0; q < nt; ++q) {
            const int64_t i = ord_[static_cast<size_t>(q)];
            const int o = oct(i), w = twait_[i];
            const int delta = o < 2 ? 1 : (1 << o) / 4;
            if (o != cur_oct || cur_cnt == tpb_ || w - first_w >= delta) {
                close();
                bstart_.push_back(q);
                cur_oct = o;
                cur_cnt = 0;
                first_w = w;
                max_w = w;
            }
            ++cur_cnt;
            max_w = std::max(max_w, w);
        }
        close();
        const int64_t nb = static_cast<int64_t>(bstart_.size());
        bstart_.push_back(nt);
        // bundles by availability (stable: shorter octaves first on ties)
        cnt_.assign(static_cast<size_t>(S) + 2, 0);
        for (int64_t b = 0; b < nb; ++b) ++cnt_[static_cast<size_t>(bwait_[b] + 1) + 1];
        for (size_t k = 1; k < cnt_.size(); ++k) cnt_[k] += cnt_[k - 1];
        border_.resize(static_cast<size_t>(nb));
        for (int64_t b = 0; b < nb; ++b) border_[static_cast<size_t>(cnt_[static_cast<size_t>(bwait_[b] + 1)]++)] = b;
        int64_t q = 0;
        for (int64_t k = 0; k < nb; ++k) {
            const int64_t b = border_[static_cast<size_t>(k)];
            sc.b_off.p[k] = static_cast<int32_t>(q);
            sc.b_wait.p[k] = bwait_[b];
            for (int64_t j = bstart_[b]; j < bstart_[b + 1]; ++j, ++q) {
                const int64_t i = ord_[static_cast<size_t>(j)];
                sc.task_row.p[q] = trow_[i];
                sc.task_step.p[q] = tstep_[i];
                sc.task_wait.p[q] = twait_[i];
            }
        }
        sc.b_off.p[nb] = static_cast<int32_t>(q);
        sc.nbundle = nb;
    }

    int64_t m_;
    int B_, tpb_;
    std::vector<int32_t> trow_, tstep_, twait_;
    std::vector<int64_t> ord_, tmp_, cnt_, bstart_, border_;
    std::vector<int32_t> bwait_;
    const std::vector<Cell>& train_;
    std::vector<int> stamp_, slot_of_, last_, lastslot_;
};

template <typename T>
cudaError_t upload(JBuf<T>& d, const PinBuf<T>& h, size_t count, cudaStream_t s) {
    if (d.n < count || !d.p) {
        cudaError_t e = d.alloc(count);
        if (e != cudaSuccess) return e;
    }
    if (count == 0) return cudaSuccess;
    return cudaMemcpyAsync(d.p, h.p, sizeof(T) * count, cudaMemcpyHostToDevice, s);
}

template <typename T>
cudaError_t upload_vec(JBuf<T>& d, const std::vector<T>& h, cudaStream_t s) {
    cudaError_t e = d.alloc(h.size());
    if (e != cudaSuccess || h.empty()) return e;
    return cudaMemcpyAsync(d.p, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice, s);
}

JLayout make_layout(int T_mlp, int kmax, int L, const int* stride, size_t tsz) {
    JLayout ly{};
    uint32_t p = 0;
    auto carve = [&](size_t bytes) {
        const uint32_t r = p;
        p += static_cast<uint32_t>((bytes + 15) & ~size_t(15));
        return r;
    };
    ly.P = carve(tsz * T_mlp);
    ly.M = carve(tsz * T_mlp);
    ly.V = carve(tsz * T_mlp);
    ly.slot[0] = carve(tsz * kJMaxSlots * 3 * kmax);
    ly.slot[1] = carve(tsz * kJMaxSlots * 3 * kmax);
    for (int l = 0; l <= L; ++l) ly.act[l] = carve(tsz * kJMaxB * stride[l]);
    for (int l = 0; l < L; ++l) ly.del[l] = carve(tsz * kJMaxB * stride[l + 1]);
    ly.ig = carve(tsz * kJMaxB * stride[0]);
    ly.sy = carve(sizeof(double) * kJMaxB);
    ly.ssa = carve(sizeof(int) * kJMaxB);
    ly.sss = carve(sizeof(int) * kJMaxB);
    ly.tab = carve(sizeof(uint64_t) * 256);
    ly.smask = carve(sizeof(uint32_t) * 2 * kJMaxSlots);
    ly.ones = carve(tsz);  // one element = 1 (bias chains)
    ly.srow = carve(sizeof(int64_t) * kJMaxSlots);  // the step's slot rows
    ly.bytes = p;
    return ly;
}

struct Shape {
    int ka, ks, L, dims[kJMaxL + 1], stride[kJMaxL + 1], off_w[kJMaxL], off_b[kJMaxL], T_mlp;
};

int shape_of(const ocg_ncf_hyper& h, Shape& sh, std::string& err) {
    if (h.app_dim > kJMaxK || h.setting_dim > kJMaxK) {
        err = "joint ncf fit: embedding dims up to " + std::to_string(kJMaxK);
        return OCG_E_UNSUPPORTED;
    }
    if (h.n_hidden + 1 > kJMaxL) {
        err = "joint ncf fit: at most " + std::to_string(kJMaxL - 1) + " hidden layers";
        return OCG_E_UNSUPPORTED;
    }
    if (h.batch_size > kJMaxB) {
        err = "joint ncf fit: batch_size up to " + std::to_string(kJMaxB);
        return OCG_E_UNSUPPORTED;
    }
    sh.ka = static_cast<int>(h.app_dim);
    sh.ks = static_cast<int>(h.setting_dim);
    sh.L = static_cast<int>(h.n_hidden) + 1;
    sh.dims[0] = sh.ka + sh.ks;
    for (int l = 0; l < h.n_hidden; ++l) {
        if (h.hidden[l] > kJMaxHid) {
            err = "joint ncf fit: hidden widths up to " + std::to_string(kJMaxHid);
            return OCG_E_UNSUPPORTED;
        }
        sh.dims[l + 1] = static_cast<int>(h.hidden[l]);
    }
    sh.dims[sh.L] = 1;
    int off = 0;
    for (int l = 0; l < sh.L; ++l) {
        sh.off_w[l] = off;
        off += sh.dims[l] * sh.dims[l + 1];
        sh.off_b[l] = off;
        off += sh.dims[l + 1];
    }
    sh.T_mlp = off;
    for (int l = 0; l <= sh.L; ++l) sh.stride[l] = sh.dims[l] | 1;
    return OCG_OK;
}

template <class NUM>
int run_fit(cudaStream_t st, int sm_count, int64_t m, int64_t n, const int64_t* rp, const int32_t* col,
            const double* val, const ocg_ncf_hyper& h, const Shape& sh, uint64_t seed, double* params_out,
            uint8_t* app_seen, uint8_t* setting_seen, ocg_ncf_meta* meta, JointFitStats* stats, std::string& err) {
    using T = typename NUM::T;
    // ---- observed cells, row-major (cfcomplete.cpp:68-71)
    const int64_t nc = rp[m];
    std::vector<Cell> cells(static_cast<size_t>(nc));
    std::vector<uint8_t> aseen(static_cast<size_t>(m), 0), sseen(static_cast<size_t>(n), 0);
    for (int64_t i = 0; i < m; ++i)
        for (int64_t q = rp[i]; q < rp[i + 1]; ++q) {
            cells[static_cast<size_t>(q)] = Cell{static_cast<int32_t>(i), col[q], val[q]};
            aseen[static_cast<size_t>(i)] = 1;
            sseen[static_cast<size_t>(col[q])] = 1;
        }
    // ---- init draws (EmbeddingTable::random nnkit.cpp:258-266, MlpModel nnkit.cpp:47-62)
    std::mt19937_64 eng(derive_seed_h(seed, splitmix64(fnv1a("ncf.fit")), 0));
    auto uniform = [&](double lo, double hi) {
        const double u = static_cast<double>(eng() >> 11) * 0x1.0p-53;
        return dadd(lo, dmul(dsub(hi, lo), u));
    };
    const int ka = sh.ka, ks = sh.ks;
    std::vector<T> app0(static_cast<size_t>(m * ka)), set0(static_cast<size_t>(n * ks)), mlp0(static_cast<size_t>(sh.T_mlp), T(0));
    {
        const double b = std::sqrt(6.0 / static_cast<double>(m + ka));
        for (auto& v : app0) v = static_cast<T>(uniform(-b, b));
        const double bs = std::sqrt(6.0 / static_cast<double>(n + ks));
        for (auto& v : set0) v = static_cast<T>(uniform(-bs, bs));
        for (int l = 0; l < sh.L; ++l) {
            const double bw = std::sqrt(6.0 / static_cast<double>(sh.dims[l] + sh.dims[l + 1]));
            for (int q = 0; q < sh.dims[l] * sh.dims[l + 1]; ++q) mlp0[sh.off_w[l] + q] = static_cast<T>(uniform(-bw, bw));
        }
    }
    // ---- held-out split (cfcomplete.cpp:95-105)
    std::vector<int64_t> order(static_cast<size_t>(nc));
    for (int64_t i = 0; i < nc; ++i) order[static_cast<size_t>(i)] = i;
    for (int64_t i = nc; i > 1; --i)
        std::swap(order[static_cast<size_t>(i - 1)], order[static_cast<size_t>(eng() % static_cast<uint64_t>(i))]);
    const auto val_count = static_cast<int64_t>(h.val_fraction * static_cast<double>(nc));
    std::vector<Cell> vcell, train;
    vcell.reserve(static_cast<size_t>(val_count));
    train.reserve(static_cast<size_t>(nc - val_count));
    for (int64_t i = 0; i < nc; ++i)
        (i < val_count ? vcell : train).push_back(cells[static_cast<size_t>(order[static_cast<size_t>(i)])]);
    if (train.empty()) std::swap(train, vcell);
    const std::vector<Cell>& mon = vcell.empty() ? train : vcell;
    std::vector<Cell>().swap(cells);
    std::vector<int64_t>().swap(order);
    const int64_t nt = static_cast<int64_t>(train.size()), nmon = static_cast<int64_t>(mon.size());
    const int B = static_cast<int>(h.batch_size);
    const int S = static_cast<int>((nt + B - 1) / B);

    // ---- Adam bias-correction table: mc_t = 1/(1 - b1^t) with b1^t by repeated
    // multiplication (nnkit.cpp:242-244, kernels_*.cpp); constant 1.0 once 1 - b^t == 1
    std::vector<double> tmc(1, 0.0), tvc(1, 0.0);
    {
        double b1p = 1.0, b2p = 1.0;
        for (;;) {
            b1p = dmul(b1p, kB1);
            b2p = dmul(b2p, kB2);
            const double om1 = dsub(1.0, b1p), om2 = dsub(1.0, b2p);
            tmc.push_back(ddiv(1.0, om1));
            tvc.push_back(ddiv(1.0, om2));
            if (om1 == 1.0 && om2 == 1.0) break;
        }
    }

    // ---- device state
    JBuf<T> d_app0, d_set0, app_rec, set_rec, mlp, best_app, best_set, best_mlp;
    JBuf<int64_t> row_last;
    JBuf<double> d_tmc, d_tvc, err2, d_out, mon_y, tr_y;
    JBuf<int32_t> mon_app, mon_set, tr_app, tr_set;
    JBuf<int> progress, bad;
    JBuf<JointCtl> ctl;
    JCU(upload_vec(d_app0, app0, st));
    JCU(upload_vec(d_set0, set0, st));
    JCU(app_rec.alloc(static_cast<size_t>(m * 3 * ka)));
    JCU(set_rec.alloc(static_cast<size_t>(n * 3 * ks)));
    JCU(mlp.alloc(static_cast<size_t>(3 * sh.T_mlp)));
    JCU(cudaMemsetAsync(mlp.p, 0, sizeof(T) * 3 * sh.T_mlp, st));
    JCU(cudaMemcpyAsync(mlp.p, mlp0.data(), sizeof(T) * sh.T_mlp, cudaMemcpyHostToDevice, st));
    joint_scatter_init_kernel<T><<<sm_count * 4, 256, 0, st>>>(d_app0.p, m, ka, app_rec.p);
    joint_scatter_init_kernel<T><<<sm_count, 256, 0, st>>>(d_set0.p, n, ks, set_rec.p);
    JCU(cudaGetLastError());
    JCU(row_last.alloc(static_cast<size_t>(m + n)));
    JCU(cudaMemsetAsync(row_last.p, 0, sizeof(int64_t) * static_cast<size_t>(m + n), st));
    // best = snapshot() of the initial parameters (cfcomplete.cpp:138)
    JCU(best_app.alloc(static_cast<size_t>(m * ka)));
    JCU(best_set.alloc(static_cast<size_t>(n * ks)));
    JCU(best_mlp.alloc(static_cast<size_t>(sh.T_mlp)));
    JCU(cudaMemcpyAsync(best_app.p, d_app0.p, sizeof(T) * m * ka, cudaMemcpyDeviceToDevice, st));
    JCU(cudaMemcpyAsync(best_set.p, d_set0.p, sizeof(T) * n * ks, cudaMemcpyDeviceToDevice, st));
    JCU(cudaMemcpyAsync(best_mlp.p, mlp0.data(), sizeof(T) * sh.T_mlp, cudaMemcpyHostToDevice, st));
    JCU(upload_vec(d_tmc, tmc, st));
    JCU(upload_vec(d_tvc, tvc, st));
    {
        std::vector<int32_t> a1(static_cast<size_t>(nmon)), s1(static_cast<size_t>(nmon));
        std::vector<double> y1(static_cast<size_t>(nmon));
        for (int64_t i = 0; i < nmon; ++i) {
            a1[i] = mon[i].app;
            s1[i] = mon[i].set;
            y1[i] = mon[i].y;
        }
        JCU(upload_vec(mon_app, a1, st));
        JCU(upload_vec(mon_set, s1, st));
        JCU(upload_vec(mon_y, y1, st));
        a1.resize(static_cast<size_t>(nt));
        s1.resize(static_cast<size_t>(nt));
        y1.resize(static_cast<size_t>(nt));
        for (int64_t i = 0; i < nt; ++i) {
            a1[i] = train[i].app;
            s1[i] = train[i].set;
            y1[i] = train[i].y;
        }
        JCU(upload_vec(tr_app, a1, st));
        JCU(upload_vec(tr_set, s1, st));
        JCU(upload_vec(tr_y, y1, st));
        JCU(cudaStreamSynchronize(st));  // the host vectors above go out of scope
    }
    JCU(err2.alloc(static_cast<size_t>(std::max(nt, nmon))));
    JCU(d_out.alloc(2));
    JCU(progress.alloc(1));
    JBuf<int> bundle_next;
    JCU(bundle_next.alloc(1));
    JCU(bad.alloc(1));
    JCU(ctl.alloc(1));

    JointArgs<T> a{};
    a.m = m;
    a.n = n;
    a.ka = ka;
    a.ks = ks;
    a.L = sh.L;
    a.kmax = std::max(ka, ks);
    a.lpt = a.kmax <= 8 ? 1 : (a.kmax <= 16 ? 2 : (a.kmax <= 32 ? 4 : 8));
    for (int l = 0; l <= sh.L; ++l) {
        a.dims[l] = sh.dims[l];
        a.stride[l] = sh.stride[l];
    }
    for (int l = 0; l < sh.L; ++l) {
        a.off_w[l] = sh.off_w[l];
        a.off_b[l] = sh.off_b[l];
    }
    a.T_mlp = sh.T_mlp;
    std::vector<uint32_t> hdec(static_cast<size_t>(sh.T_mlp));
    for (int e = 0; e < sh.T_mlp; ++e) {
        int l = 0;
        while (l + 1 < sh.L && e >= sh.off_w[l + 1]) ++l;
        const int in = sh.dims[l], out = sh.dims[l + 1];
        uint32_t d = static_cast<uint32_t>(l) << 16;
        if (e < sh.off_b[l]) {
            const int q = e - sh.off_w[l], r = q / in, c = q - r * in;
            d |= static_cast<uint32_t>(c) | (static_cast<uint32_t>(r) << 8) | (1u << 20) |
                 (q < ((out * in) & ~3) ? 1u << 21 : 0u);
        } else {
            const int r = e - sh.off_b[l];
            d |= (static_cast<uint32_t>(r) << 8) | (r < (out & ~3) ? 1u << 21 : 0u);
        }
        hdec[static_cast<size_t>(e)] = d;
    }
    JBuf<uint32_t> d_dec;
    JCU(upload_vec(d_dec, hdec, st));
    a.dec = d_dec.p;
    a.lr = static_cast<T>(h.lr);
    a.lay = make_layout(sh.T_mlp, a.kmax, sh.L, sh.stride, sizeof(T));
    if (a.lay.bytes > 227u * 1024u) {
        err = "joint ncf fit: working set " + std::to_string(a.lay.bytes) + " B exceeds shared memory";
        return OCG_E_UNSUPPORTED;
    }
    a.app_rec = app_rec.p;
    a.set_rec = set_rec.p;
    a.row_last = row_last.p;
    a.mlp = mlp.p;
    a.app_vec = (m * ka) & ~int64_t(3);
    a.set_vec = (n * ks) & ~int64_t(3);
    a.tab_mc = d_tmc.p;
    a.tab_vc = d_tvc.p;
    a.tab_len = static_cast<int64_t>(tmc.size());
    a.S = S;
    a.nt = static_cast<int>(nt);
    a.B = B;
    a.progress = progress.p;
    a.bundle_next = bundle_next.p;
    a.mon_app = mon_app.p;
    a.mon_set = mon_set.p;
    a.mon_y = mon_y.p;
    a.nmon = nmon;
    a.err2 = err2.p;
    a.best_app = best_app.p;
    a.best_set = best_set.p;
    a.best_mlp = best_mlp.p;
    a.ctl = ctl.p;
    a.patience = h.patience;
    JBuf<unsigned long long> prof;
    const bool profile = std::getenv("OCG_JOINT_PROFILE") != nullptr;
    if (profile) {
        JCU(prof.alloc(8));
        JCU(cudaMemsetAsync(prof.p, 0, sizeof(unsigned long long) * 8, st));
        a.prof = prof.p;
    }

    const bool h3216 = sh.L == 3 && sh.dims[1] == 32 && sh.dims[2] == 16 && h.batch_size == 32;
    auto kep = (h3216 && sh.ka == 8 && sh.ks == 8)     ? joint_epoch_kernel<NUM, DefaultShape>
               : (h3216 && sh.ka == 32 && sh.ks == 32) ? joint_epoch_kernel<NUM, FixShape<32, 32, 32, 16>>
                                                       : joint_epoch_kernel<NUM, RtShape>;
    auto kev = joint_eval_kernel<NUM>;
    JCU(cudaFuncSetAttribute(kep, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(a.lay.bytes)));
    JCU(cudaFuncSetAttribute(kev, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(a.lay.bytes)));
    int per_sm = 0;
    JCU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kep, kJT, a.lay.bytes));
    if (per_sm < 1) {
        err = "joint ncf fit: epoch kernel cannot be resident";
        return OCG_E_CUDA;
    }
    const int grid = sm_count;  // one CTA per SM: leader + helpers, co-resident (cooperative launch)
    if (grid < 2) {
        err = "joint ncf fit: needs at least 2 SMs";
        return OCG_E_CUDA;
    }
    cudaEvent_t ev0, ev1;
    JCU(cudaEventCreate(&ev0));
    JCU(cudaEventCreate(&ev1));
    struct EvGuard {
        cudaEvent_t a, b;
        ~EvGuard() {
            cudaEventDestroy(a);
            cudaEventDestroy(b);
        }
    } evguard{ev0, ev1};
    JCU(cudaEventRecord(ev0, st));

    // ---- meta.initial_train_mse and the initial best_val (cfcomplete.cpp:137-139)
    const PView<T> init_view{app_rec.p, 3 * ka, set_rec.p, 3 * ks};
    kev<<<sm_count, kJT, a.lay.bytes, st>>>(a, init_view, mlp.p, tr_app.p, tr_set.p, tr_y.p, nt, err2.p);
    joint_sum_kernel<<<1, 32, 0, st>>>(err2.p, nt, d_out.p);
    kev<<<sm_count, kJT, a.lay.bytes, st>>>(a, init_view, mlp.p, mon_app.p, mon_set.p, mon_y.p, nmon, err2.p);
    joint_sum_kernel<<<1, 32, 0, st>>>(err2.p, nmon, d_out.p + 1);
    JCU(cudaGetLastError());
    double h_out[2];
    JCU(cudaMemcpyAsync(h_out, d_out.p, sizeof h_out, cudaMemcpyDeviceToHost, st));
    JCU(cudaStreamSynchronize(st));
    const double init_train = h_out[0];
    JointCtl hc{};
    hc.best_val = h_out[1];
    JCU(cudaMemcpyAsync(ctl.p, &hc, sizeof hc, cudaMemcpyHostToDevice, st));

    // ---- epochs: the host builds epoch e+1's schedule while the device runs epoch e
    ScheduleBuilder builder(m, n, B, a.lpt, train);
    std::vector<int64_t> idx(static_cast<size_t>(nt));
    for (int64_t i = 0; i < nt; ++i) idx[static_cast<size_t>(i)] = i;
    auto shuffle = [&]() {  // cfcomplete.cpp:153-154
        for (int64_t i = nt; i > 1; --i)
            std::swap(idx[static_cast<size_t>(i - 1)], idx[static_cast<size_t>(eng() % static_cast<uint64_t>(i))]);
    };
    Sched hs[2];
    DSched ds[2];
    auto push = [&](int b) -> cudaError_t {
        cudaError_t e;
        Sched& h2 = hs[b];
        DSched& d2 = ds[b];
        if ((e = upload(d2.y, h2.y, static_cast<size_t>(nt), st)) != cudaSuccess) return e;
        if ((e = upload(d2.slot, h2.slot, static_cast<size_t>(nt), st)) != cudaSuccess) return e;
        if ((e = upload(d2.slot_off, h2.slot_off, static_cast<size_t>(S) + 1, st)) != cudaSuccess) return e;
        if ((e = upload(d2.slot_row, h2.slot_row, static_cast<size_t>(h2.nslots), st)) != cudaSuccess) return e;
        if ((e = upload(d2.slot_prev, h2.slot_prev, static_cast<size_t>(h2.nslots), st)) != cudaSuccess) return e;
        if ((e = upload(d2.task_row, h2.task_row, static_cast<size_t>(h2.ntask), st)) != cudaSuccess) return e;
        if ((e = upload(d2.task_step, h2.task_step, static_cast<size_t>(h2.ntask), st)) != cudaSuccess) return e;
        if ((e = upload(d2.task_wait, h2.task_wait, static_cast<size_t>(h2.ntask), st)) != cudaSuccess) return e;
        if ((e = upload(d2.need, h2.need, static_cast<size_t>(S), st)) != cudaSuccess) return e;
        if ((e = upload(d2.b_off, h2.b_off, static_cast<size_t>(h2.nbundle) + 1, st)) != cudaSuccess) return e;
        if ((e = upload(d2.b_wait, h2.b_wait, static_cast<size_t>(h2.nbundle), st)) != cudaSuccess) return e;
        if (d2.ready.n < static_cast<size_t>(S) || !d2.ready.p)
            if ((e = d2.ready.alloc(static_cast<size_t>(S))) != cudaSuccess) return e;
        return cudaSuccess;
    };
    shuffle();
    JCU(builder.build(idx, hs[0]));
    JCU(push(0));
    PinBuf<JointCtl> hctl;
    JCU(hctl.reserve(1));
    int epoch = 0;
    int64_t tasks = 0, steps = 0;
    bool diverged = false;
    for (; epoch < h.max_epochs; ++epoch) {
        const int b = epoch & 1;
        JCU(cudaMemsetAsync(ds[b].ready.p, 0, sizeof(int) * S, st));
        JCU(cudaMemsetAsync(progress.p, 0xff, sizeof(int), st));
        a.epoch_base = static_cast<int64_t>(epoch) * S;
        a.smp_y = ds[b].y.p;
        a.smp_slot = ds[b].slot.p;
        a.slot_off = ds[b].slot_off.p;
        a.slot_row = ds[b].slot_row.p;
        a.slot_prev = ds[b].slot_prev.p;
        a.task_row = ds[b].task_row.p;
        a.task_step = ds[b].task_step.p;
        a.task_wait = ds[b].task_wait.p;
        a.b_off = ds[b].b_off.p;
        a.b_wait = ds[b].b_wait.p;
        a.nbundle = static_cast<int>(hs[b].nbundle);
        JCU(cudaMemsetAsync(bundle_next.p, 0, sizeof(int), st));
        a.need = ds[b].need.p;
        a.ready = ds[b].ready.p;
        void* kargs[] = {&a};
        JCU(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kep), dim3(grid), dim3(kJT), kargs, a.lay.bytes, st));
        JCU(cudaMemcpyAsync(hctl.p, ctl.p, sizeof(JointCtl), cudaMemcpyDeviceToHost, st));
        tasks += hs[b].ntask;
        steps += S;
        if (epoch + 1 < h.max_epochs) {
            shuffle();
            JCU(builder.build(idx, hs[b ^ 1]));
            JCU(push(b ^ 1));
        }
        JCU(cudaStreamSynchronize(st));
        if (hctl.p->diverged) {
            diverged = true;
            break;
        }
        if (hctl.p->stop) {
            ++epoch;
            break;
        }
    }
    if (diverged) {
        err = "ncf: divergence";
        return OCG_E_DIVERGE;
    }
    const double best_val = hctl.p->best_val;
    // ---- restore(best) (:190), final_train_mse (:193), check_finite (:194)
    const PView<T> best_view{best_app.p, ka, best_set.p, ks};
    kev<<<sm_count, kJT, a.lay.bytes, st>>>(a, best_view, best_mlp.p, tr_app.p, tr_set.p, tr_y.p, nt, err2.p);
    joint_sum_kernel<<<1, 32, 0, st>>>(err2.p, nt, d_out.p);
    JCU(cudaGetLastError());
    JCU(cudaEventRecord(ev1, st));
    // flat parameters, widened to FP64
    JBuf<double> flat;
    const int64_t total = m * ka + n * ks + sh.T_mlp;
    JCU(flat.alloc(static_cast<size_t>(total)));
    joint_widen_kernel<T><<<sm_count * 4, 256, 0, st>>>(best_app.p, flat.p, m * ka);
    joint_widen_kernel<T><<<sm_count, 256, 0, st>>>(best_set.p, flat.p + m * ka, n * ks);
    joint_widen_kernel<T><<<1, 256, 0, st>>>(best_mlp.p, flat.p + m * ka + n * ks, sh.T_mlp);
    JCU(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
    joint_check_finite_kernel<<<1, 256, 0, st>>>(flat.p + m * ka + n * ks, sh.T_mlp, bad.p);
    JCU(cudaGetLastError());
    int hbad = 0;
    JCU(cudaMemcpyAsync(h_out, d_out.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    JCU(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    if (params_out) JCU(cudaMemcpyAsync(params_out, flat.p, sizeof(double) * total, cudaMemcpyDeviceToHost, st));
    JCU(cudaStreamSynchronize(st));
    float ms = 0.f;
    JCU(cudaEventElapsedTime(&ms, ev0, ev1));
    if (profile) {
        unsigned long long hp[8];
        JCU(cudaMemcpy(hp, prof.p, sizeof hp, cudaMemcpyDeviceToHost));
        const double ns = hp[5] ? 1.0 / hp[5] : 0.0;
        std::fprintf(stderr, "[joint profile] steps %llu, cycles/step: wait %.0f load %.0f fwd+bwd %.0f adam %.0f wb %.0f\n",
                     hp[5], hp[0] * ns, hp[1] * ns, hp[2] * ns, hp[3] * ns, hp[4] * ns);
    }
    if (hbad) {
        err = "non-finite weight";
        return OCG_E_LOGIC;
    }
    if (app_seen) std::memcpy(app_seen, aseen.data(), aseen.size());
    if (setting_seen) std::memcpy(setting_seen, sseen.data(), sseen.size());
    if (meta) {
        meta->seed = seed;
        meta->epochs_run = epoch;
        meta->initial_train_mse = init_train;
        meta->final_train_mse = h_out[0];
        meta->best_val_mse = best_val;
    }
    if (stats) {
        stats->steps = steps;
        stats->replay_tasks = tasks;
        stats->device_ms = ms;
    }
    return OCG_OK;
}

}  // namespace

int joint_ncf_supported(const ocg_ncf_hyper& h, int precision, std::string& err) {
    Shape sh{};
    int rc = shape_of(h, sh, err);
    if (rc) return rc;
    const int kmax = std::max(sh.ka, sh.ks);
    const JLayout ly = make_layout(sh.T_mlp, kmax, sh.L, sh.stride, precision == OCG_NCF_FAST ? 4 : 8);
    if (ly.bytes > 227u * 1024u) {
        err = "joint ncf fit: working set " + std::to_string(ly.bytes) + " B exceeds shared memory";
        return OCG_E_UNSUPPORTED;
    }
    return OCG_OK;
}

int joint_ncf_fit(cudaStream_t stream, int sm_count, int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col,
                  const double* val, const ocg_ncf_hyper& h, uint64_t seed, int precision, int lane, double* params,
                  uint8_t* app_seen, uint8_t* setting_seen, ocg_ncf_meta* meta, JointFitStats* stats,
                  std::string& err) {
    Shape sh{};
    int rc = shape_of(h, sh, err);
    if (rc) return rc;
    if ((rc = joint_ncf_supported(h, precision, err))) return rc;
    if (m + n >= (int64_t(1) << 31) || row_ptr[m] >= (int64_t(1) << 31)) {
        err = "joint ncf fit: more than 2^31 rows or observed cells";
        return OCG_E_UNSUPPORTED;
    }
    if (precision == OCG_NCF_FAST && std::getenv("OCG_JOINT_FAST64"))
        return run_fit<FastNumT<double>>(stream, sm_count, m, n, row_ptr, col, val, h, sh, seed, params, app_seen,
                                         setting_seen, meta, stats, err);
    if (precision == OCG_NCF_FAST)
        return run_fit<FastNum>(stream, sm_count, m, n, row_ptr, col, val, h, sh, seed, params, app_seen,
                                setting_seen, meta, stats, err);
    if (lane == OCG_LANE_SCALAR)
        return run_fit<ExactNum<0>>(stream, sm_count, m, n, row_ptr, col, val, h, sh, seed, params, app_seen,
                                    setting_seen, meta, stats, err);
    return run_fit<ExactNum<1>>(stream, sm_count, m, n, row_ptr, col, val, h, sh, seed, params, app_seen,
                                setting_seen, meta, stats, err);
}

}  // namespace ocg
