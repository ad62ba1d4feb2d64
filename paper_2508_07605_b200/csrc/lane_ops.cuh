// The reference's two FP64 kernel lanes (kern::Ops, kernels.hpp:12-26) as
// device code with explicit rounding, so a kernel templated on LANE repeats
// the reference's floating-point operation order exactly:
//   LANE 0 = scalar lane (kernels_scalar.cpp, baseline x86-64: no FMA)
//   LANE 1 = AVX2/FMA lane (kernels_avx2.cpp as g++ 13 -O3 -mavx2 -mfma emits it,
//            incl. the contractions -ffp-contract=fast adds; see the
//            disassembly notes in DESIGN.md)
#pragma once

#include "ocg_common.cuh"

namespace ocg {

constexpr double kLambda = 1.0507009873554805;                     // nnkit.hpp:20
constexpr double kLA = 1.0507009873554805 * 1.6732632423543772;   // lambda*alpha, folded as g++ does

template <int LANE>
struct LaneOps;

template <>
struct LaneOps<0> {
    // dot_scalar: acc += x[i]*y[i]
    __device__ static double dot(const double* w, const double* x, int n) {
        double acc = 0.0;
        for (int i = 0; i < n; ++i) acc = dadd(acc, dmul(w[i], x[i]));
        return acc;
    }
    // axpy_scalar element: y += a*x
    __device__ static double axpy(double y, double a, double x) { return dadd(y, dmul(a, x)); }
    __device__ static void adam(double& p, double& m, double& v, double g, double lr, double b1,
                                double omb1, double b2, double omb2, double eps, double mc, double vc,
                                bool /*vec*/) {
        m = dadd(dmul(b1, m), dmul(omb1, g));
        v = dadd(dmul(b2, v), dmul(dmul(omb2, g), g));
        p = dsub(p, ddiv(dmul(lr, dmul(m, mc)), dadd(dsqrt(dmul(v, vc)), eps)));
    }
};

template <>
struct LaneOps<1> {
    // dot_avx2: four FMA partial sums over full 4-chunks, hsum (a0+a2)+(a1+a3),
    // plus an FMA-contracted scalar tail
    __device__ static double dot(const double* w, const double* x, int n) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int i = 0;
        for (; i + 4 <= n; i += 4) {
            a0 = dfma(w[i], x[i], a0);
            a1 = dfma(w[i + 1], x[i + 1], a1);
            a2 = dfma(w[i + 2], x[i + 2], a2);
            a3 = dfma(w[i + 3], x[i + 3], a3);
        }
        // scalar tail as g++ vectorises it: the first two leftovers as unfused
        // products added in order, a third (or lone) leftover fused
        double tail = 0.0;
        const int r = n - i;
        if (r >= 2) {
            tail = dadd(tail, dmul(w[i], x[i]));
            tail = dadd(tail, dmul(w[i + 1], x[i + 1]));
            if (r == 3) tail = dfma(w[i + 2], x[i + 2], tail);
        } else if (r == 1) {
            tail = dfma(w[i], x[i], tail);
        }
        return dadd(dadd(dadd(a0, a2), dadd(a1, a3)), tail);
    }
    __device__ static double axpy(double y, double a, double x) { return dfma(a, x, y); }
    __device__ static void adam(double& p, double& m, double& v, double g, double lr, double b1,
                                double omb1, double b2, double omb2, double eps, double mc, double vc,
                                bool vec) {
        if (!vec) {  // block tail -> scalar lane (kernels_avx2.cpp:75-76)
            LaneOps<0>::adam(p, m, v, g, lr, b1, omb1, b2, omb2, eps, mc, vc, false);
            return;
        }
        m = dfma(b1, m, dmul(omb1, g));
        v = dfma(b2, v, dmul(omb2, dmul(g, g)));
        const double num = dmul(m, mc);
        const double den = dadd(dsqrt(dmul(v, vc)), eps);
        p = dfma(-lr, ddiv(num, den), p);  // g++ fuses _mm256_sub_pd(p, _mm256_mul_pd(lr, q)) -> vfnmadd
    }
};


// SELU value and derivative from one exp (nnkit.cpp:27-45)
template <class Tab = ExpTabConst>
__device__ __forceinline__ void selu_fwd(double z, double& a, double& gf, Tab tab = Tab{}) {
    if (z > 0) {
        a = dmul(kLambda, z);
        gf = kLambda;
    } else {
        const double e = glibc_exp_with(z, tab);
        a = dmul(kLA, dsub(e, 1.0));
        gf = dmul(kLA, e);
    }
}

}  // namespace ocg
