// Evaluation harness on the GPU: policy::evaluate_suite's table
// and policy logic (policy.cpp:213-405) for many apps at once, from the
// simulator's repetition runs (sim::run stays on the host: it is the simulator).
//   * truth_kernel  (thread per (app, setting)): measure_truth (policy.cpp:213-256) —
//     paired repetitions against the baseline, the slowest then the fastest repetition
//     dropped, the rest averaged in order; FP64 in the reference's operation order.
//   * choose_kernel (thread per (app, policy)): candidate_set + choose_exhaustive
//     (policy.cpp:271-320; max measured efficiency subject to measured loss <= gamma,
//     the reference's tie order) and row_from_truth (:322-337); the open policy's row
//     takes the setting and pred_saving of its run_open_online decision.
//   * aggregates (:384-403): per policy, sequential over the apps in order.
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../../include/ocg.h"
#include "ocg_common.cuh"

int ocg_internal_fail(int code, const std::string& msg);
cudaStream_t ocg_internal_stream(ocg_ctx* ctx);

namespace {

struct Truth {
    double perf, power, eff, energy, avg_power;
};

__global__ void truth_kernel(int64_t napps, int n, int reps, const ocg_run_result* __restrict__ base,
                             const ocg_run_result* __restrict__ runs, Truth* __restrict__ table) {
    const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= napps * n) return;
    const int64_t a = q / n;
    constexpr int kMaxReps = 64;
    double rt[kMaxReps], pf[kMaxReps], pw[kMaxReps], ef[kMaxReps], en[kMaxReps], ap[kMaxReps];
    bool keep[kMaxReps];
    for (int r = 0; r < reps; ++r) {
        const ocg_run_result b = base[a * reps + r], c = runs[q * reps + r];
        rt[r] = c.runtime_s;
        pf[r] = ocg::ddiv(b.runtime_s, c.runtime_s);
        pw[r] = ocg::ddiv(c.avg_power_w, b.avg_power_w);
        ef[r] = ocg::ddiv(pf[r], pw[r]);
        en[r] = c.energy_j;
        ap[r] = c.avg_power_w;
        keep[r] = true;
    }
    if (reps >= 3) {  // max_element (first of equal maxima), then min_element of the rest
        int slow = 0;
        for (int r = 1; r < reps; ++r)
            if (rt[slow] < rt[r]) slow = r;
        keep[slow] = false;
        int fast = -1;
        for (int r = 0; r < reps; ++r)
            if (keep[r] && (fast < 0 || rt[r] < rt[fast])) fast = r;
        keep[fast] = false;
    }
    Truth t{0.0, 0.0, 0.0, 0.0, 0.0};
    int cnt = 0;
    for (int r = 0; r < reps; ++r) {
        if (!keep[r]) continue;
        t.perf = ocg::dadd(t.perf, pf[r]);
        t.power = ocg::dadd(t.power, pw[r]);
        t.eff = ocg::dadd(t.eff, ef[r]);
        t.energy = ocg::dadd(t.energy, en[r]);
        t.avg_power = ocg::dadd(t.avg_power, ap[r]);
        ++cnt;
    }
    const double nd = static_cast<double>(cnt);
    t.perf = ocg::ddiv(t.perf, nd);
    t.power = ocg::ddiv(t.power, nd);
    t.eff = ocg::ddiv(t.eff, nd);
    t.energy = ocg::ddiv(t.energy, nd);
    t.avg_power = ocg::ddiv(t.avg_power, nd);
    table[q] = t;
}

__device__ void fill_row(ocg_eval_row& row, int j, const Truth& e, const int32_t* cpu, const int32_t* gpu, int ngpu,
                         double e_base) {
    const int c = cpu[j / ngpu], g = gpu[j % ngpu];
    row.setting = j;
    row.cpu_cap_w = c;
    row.gpu_cap_w = g;
    row.true_perf = e.perf;
    row.true_loss = ocg::dsub(1.0, e.perf);
    row.energy_j = e.energy;
    row.avg_power_w = e.avg_power;
    row.efficiency = e.eff;
    // saving_at (policy.cpp:262-266)
    row.pred_saving = ocg::ddiv(ocg::dsub(e_base, ocg::ddiv(static_cast<double>(c + g), e.perf)), e_base);
}

__global__ void choose_kernel(int64_t napps, int ncpu, int ngpu, const int32_t* __restrict__ cpu,
                              const int32_t* __restrict__ gpu, const Truth* __restrict__ table, double gamma,
                              int npol, const int32_t* __restrict__ pols, const int32_t* __restrict__ open_idx,
                              const double* __restrict__ open_sav, ocg_eval_row* __restrict__ rows) {
    const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= napps * npol) return;
    const int64_t a = q / npol;
    const int kind = pols[q - a * npol];
    const int n = ncpu * ngpu, jb = n - 1;
    const Truth* tab = table + a * n;
    const double e_base = static_cast<double>(cpu[ncpu - 1] + gpu[ngpu - 1]);
    ocg_eval_row row{};
    if (kind == 0) {  // open: run_open_online's decision, its own pred_saving (policy.cpp:370-374)
        const int j = open_idx[a];
        fill_row(row, j, tab[j], cpu, gpu, ngpu, e_base);
        row.pred_saving = open_sav[a];
    } else {
        // candidate_set (policy.cpp:271-290) in the reference's order
        int cnt;
        if (kind == 1) cnt = 1;
        else if (kind == 2) cnt = ngpu;
        else if (kind == 3) cnt = ncpu;
        else cnt = n;
        int best = jb;
        for (int k = 0; k < cnt; ++k) {
            const int j = kind == 1 ? jb : (kind == 2 ? (ncpu - 1) * ngpu + k : (kind == 3 ? k * ngpu + (ngpu - 1) : k));
            const Truth& e = tab[j];
            if (ocg::dsub(1.0, e.perf) > gamma) continue;
            const Truth& b = tab[best];
            bool better;
            if (e.eff != b.eff) better = e.eff > b.eff;
            else if (e.perf != b.perf) better = e.perf > b.perf;
            else {
                const int sum = cpu[j / ngpu] + gpu[j % ngpu], bsum = cpu[best / ngpu] + gpu[best % ngpu];
                if (sum != bsum) better = sum < bsum;
                else better = j < best;  // lexicographic (cpu, gpu) == column order
            }
            if (better) best = j;
        }
        fill_row(row, best, tab[best], cpu, gpu, ngpu, e_base);
    }
    row.policy = kind;
    row.gamma = gamma;
    rows[q] = row;
}

// Aggregates by policy name as the reference does (policy.cpp:384-403): every row of
// that kind counts, in report order (app-major, then the policy list's order).
__global__ void aggregate_kernel(int64_t napps, int npol, const int32_t* __restrict__ pols,
                                 const ocg_eval_row* __restrict__ rows, ocg_eval_aggregate* __restrict__ aggs) {
    const int p = threadIdx.x;
    if (p >= npol) return;
    const int kind = pols[p];
    double eff = 0.0, loss = 0.0, perf = 0.0;
    int64_t cnt = 0;
    for (int64_t a = 0; a < napps; ++a)
        for (int k = 0; k < npol; ++k) {
            if (pols[k] != kind) continue;
            const ocg_eval_row& r = rows[a * npol + k];
            eff = ocg::dadd(eff, r.efficiency);
            loss = ocg::dadd(loss, r.true_loss);
            perf = ocg::dadd(perf, r.true_perf);
            ++cnt;
        }
    ocg_eval_aggregate g{};
    g.policy = kind;
    if (cnt > 0) {
        const double nd = static_cast<double>(cnt);
        g.mean_efficiency = ocg::ddiv(eff, nd);
        g.mean_true_loss = ocg::ddiv(loss, nd);
        g.mean_true_perf = ocg::ddiv(perf, nd);
        g.mean_gain_vs_no_cap = ocg::dsub(g.mean_efficiency, 1.0);
    }
    aggs[p] = g;
}

template <typename T>
struct DB {
    T* p = nullptr;
    ~DB() {
        if (p) cudaFree(p);
    }
    cudaError_t up(const T* h, size_t n, cudaStream_t s) {
        cudaError_t e = cudaMalloc(&p, sizeof(T) * (n ? n : 1));
        if (e == cudaSuccess && n) e = cudaMemcpyAsync(p, h, sizeof(T) * n, cudaMemcpyHostToDevice, s);
        return e;
    }
    cudaError_t alloc(size_t n) { return cudaMalloc(&p, sizeof(T) * (n ? n : 1)); }
};

}  // namespace

extern "C" {

int ocg_eval_suite(ocg_ctx* ctx, int64_t napps, const int32_t* cpu, int32_t ncpu, const int32_t* gpu, int32_t ngpu,
                   int32_t reps, const ocg_run_result* base_runs, const ocg_run_result* runs, double gamma,
                   int32_t npol, const int32_t* policies, const int32_t* open_idx, const double* open_pred_saving,
                   ocg_eval_row* rows, ocg_eval_aggregate* aggs) {
    if (reps < 1) return ocg_internal_fail(OCG_E_INVALID, "measure_truth: repetitions < 1");
    if (reps > 64) return ocg_internal_fail(OCG_E_UNSUPPORTED, "eval: more than 64 repetitions");
    if (!cpu || !gpu || ncpu <= 0 || ngpu <= 0) return ocg_internal_fail(OCG_E_INVALID, "cap list is empty");
    for (int k = 0; k < ncpu; ++k)
        if (cpu[k] <= 0 || (k > 0 && cpu[k] <= cpu[k - 1]))
            return ocg_internal_fail(OCG_E_INVALID, "cpu caps must be positive and strictly increasing");
    for (int k = 0; k < ngpu; ++k)
        if (gpu[k] <= 0 || (k > 0 && gpu[k] <= gpu[k - 1]))
            return ocg_internal_fail(OCG_E_INVALID, "gpu caps must be positive and strictly increasing");
    if (npol <= 0 || !policies) return ocg_internal_fail(OCG_E_INVALID, "eval: no policies");
    bool has_open = false;
    for (int p = 0; p < npol; ++p) {
        if (policies[p] < 0 || policies[p] > 4) return ocg_internal_fail(OCG_E_INVALID, "unknown policy");
        has_open = has_open || policies[p] == 0;
    }
    if (npol > 32) return ocg_internal_fail(OCG_E_UNSUPPORTED, "eval: more than 32 policies");
    if (napps < 0) return ocg_internal_fail(OCG_E_INVALID, "eval: negative app count");
    if (napps == 0) {  // the reference still reports one (zero) aggregate per policy
        if (aggs)
            for (int p = 0; p < npol; ++p) aggs[p] = ocg_eval_aggregate{policies[p], 0.0, 0.0, 0.0, 0.0};
        return OCG_OK;
    }
    if (!ctx || !base_runs || !runs || !rows || (has_open && (!open_idx || !open_pred_saving)))
        return ocg_internal_fail(OCG_E_INVALID, "eval: null argument");
    const int n = ncpu * ngpu;
    if (has_open)
        for (int64_t a = 0; a < napps; ++a)
            if (open_idx[a] < 0 || open_idx[a] >= n) return ocg_internal_fail(OCG_E_RANGE, "open decision out of range");
    cudaStream_t s = ocg_internal_stream(ctx);
    DB<ocg_run_result> db, dr;
    DB<int32_t> dc, dg, dp, doi;
    DB<double> dos;
    DB<Truth> dt;
    DB<ocg_eval_row> drow;
    DB<ocg_eval_aggregate> dagg;
    cudaError_t e = db.up(base_runs, static_cast<size_t>(napps * reps), s);
    if (e == cudaSuccess) e = dr.up(runs, static_cast<size_t>(napps * n * reps), s);
    if (e == cudaSuccess) e = dc.up(cpu, ncpu, s);
    if (e == cudaSuccess) e = dg.up(gpu, ngpu, s);
    if (e == cudaSuccess) e = dp.up(policies, npol, s);
    if (e == cudaSuccess && has_open) e = doi.up(open_idx, static_cast<size_t>(napps), s);
    if (e == cudaSuccess && has_open) e = dos.up(open_pred_saving, static_cast<size_t>(napps), s);
    if (e == cudaSuccess) e = dt.alloc(static_cast<size_t>(napps * n));
    if (e == cudaSuccess) e = drow.alloc(static_cast<size_t>(napps * npol));
    if (e == cudaSuccess) e = dagg.alloc(static_cast<size_t>(npol));
    if (e == cudaSuccess) {
        truth_kernel<<<static_cast<unsigned>((napps * n + 127) / 128), 128, 0, s>>>(napps, n, reps, db.p, dr.p, dt.p);
        choose_kernel<<<static_cast<unsigned>((napps * npol + 127) / 128), 128, 0, s>>>(
            napps, ncpu, ngpu, dc.p, dg.p, dt.p, gamma, npol, dp.p, doi.p, dos.p, drow.p);
        aggregate_kernel<<<1, 32, 0, s>>>(napps, npol, dp.p, drow.p, dagg.p);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(rows, drow.p, sizeof(ocg_eval_row) * napps * npol, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && aggs) e = cudaMemcpyAsync(aggs, dagg.p, sizeof(ocg_eval_aggregate) * npol, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return ocg_internal_fail(OCG_E_CUDA, std::string("eval: ") + cudaGetErrorString(e));
    return OCG_OK;
}

}  // extern "C"
