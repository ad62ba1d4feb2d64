// Algorithm 2 selection (policy::select_caps, policy.cpp:17-64) as warp-level
// device code.  FP64 arithmetic in the reference's operation order:
//   loss = 1 - p/p_base; skip if loss > gamma; e_pred = (c+g)/p;
//   saving = (E_base - e_pred)/E_base.
// The reference scans settings in grid order keeping the first best under
// "saving desc, then p desc, then c+g asc, then (c,g) lexicographic asc"
// (:44-52).  That key is a strict total order over distinct settings, so a
// parallel argmax under the same key returns the identical setting.  Grid
// columns are lexicographic (cpu, gpu) (core.cpp:59-65), hence the final key
// compares column indices.
#pragma once

#include "ocg_common.cuh"

namespace ocg {

struct SelResult {
    int idx;
    double saving, loss, perf;
    int sum;
    int ncand;
};

__device__ __forceinline__ bool sel_better(double s, double p, int sum, int j, const SelResult& b) {
    if (s != b.saving) return s > b.saving;
    if (p != b.perf) return p > b.perf;
    if (sum != b.sum) return sum < b.sum;
    return j < b.idx;
}

// one candidate evaluation; returns false when the setting breaches gamma
__device__ __forceinline__ bool sel_eval(double p, double p_base, int capsum, double e_base,
                                         double gamma, double& loss, double& saving) {
    loss = dsub(1.0, ddiv(p, p_base));
    if (loss > gamma) return false;
    const double e_pred = ddiv(static_cast<double>(capsum), p);
    saving = ddiv(dsub(e_base, e_pred), e_base);
    return true;
}

__device__ __forceinline__ void sel_consider(SelResult& best, bool& have, double p, int capsum, int j,
                                             double loss, double saving) {
    if (!have || sel_better(saving, p, capsum, j, best)) {
        best.idx = j;
        best.saving = saving;
        best.loss = loss;
        best.perf = p;
        best.sum = capsum;
        have = true;
    }
}

// warp-wide merge of per-lane bests; every lane returns the winner
__device__ __forceinline__ SelResult sel_warp_reduce(SelResult best, bool have, int cnt) {
    for (int off = 16; off > 0; off >>= 1) {
        SelResult o;
        o.idx = __shfl_xor_sync(0xffffffffu, best.idx, off);
        o.saving = __shfl_xor_sync(0xffffffffu, best.saving, off);
        o.loss = __shfl_xor_sync(0xffffffffu, best.loss, off);
        o.perf = __shfl_xor_sync(0xffffffffu, best.perf, off);
        o.sum = __shfl_xor_sync(0xffffffffu, best.sum, off);
        const bool ohave = __shfl_xor_sync(0xffffffffu, have ? 1 : 0, off) != 0;
        cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
        if (ohave && (!have || sel_better(o.saving, o.perf, o.sum, o.idx, best))) {
            best = o;
            have = true;
        }
    }
    if (!have) best.idx = -1;
    best.ncand = cnt;
    return best;
}

// select over one row held in shared or global memory; whole warp participates
template <typename T>
__device__ __forceinline__ SelResult select_row_warp(const T* row, int n, const int32_t* cpu,
                                                     const int32_t* gpu, int ngpu, double e_base,
                                                     double gamma, int lane) {
    const double p_base = static_cast<double>(row[n - 1]);
    SelResult best{-1, 0.0, 0.0, 0.0, 0, 0};
    bool have = false;
    int cnt = 0;
    for (int j = lane; j < n; j += 32) {
        const double p = static_cast<double>(row[j]);
        const int ci = j / ngpu;
        const int capsum = cpu[ci] + gpu[j - ci * ngpu];
        double loss, saving;
        if (!sel_eval(p, p_base, capsum, e_base, gamma, loss, saving)) continue;
        ++cnt;
        sel_consider(best, have, p, capsum, j, loss, saving);
    }
    return sel_warp_reduce(best, have, cnt);
}

}  // namespace ocg
