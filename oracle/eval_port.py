"""CPU restatement of policy::evaluate_suite's table/choice/aggregate logic
(TEST INFRASTRUCTURE ONLY: imported by tests/ as the checker, never by the product).

Follows /root/reference/proj/src/policy.cpp:
  measure_truth      :213-256  (paired repetitions, slowest then fastest dropped)
  saving_at          :262-266
  candidate_set      :268-290
  choose_exhaustive  :292-320
  row_from_truth     :322-337
  evaluate_suite     :373-405  (aggregates by policy name, report order)
Pure-Python float arithmetic is IEEE binary64 in the reference's operation order,
so it is bit-exact against the reference; pinned in tests/test_eval_harness.py
against the compiled reference (oracle/_ref ref_eval_default)."""
from __future__ import annotations


def measure_truth(base, capped):
    """base, capped: lists of (runtime_s, energy_j, avg_power_w) per repetition."""
    if len(base) < 1:
        raise ValueError("measure_truth: repetitions < 1")
    reps = []
    for b, c in zip(base, capped):
        perf = b[0] / c[0]
        power = c[2] / b[2]
        reps.append((c[0], perf, power, perf / power, c[1], c[2]))
    if len(reps) >= 3:
        slow = max(range(len(reps)), key=lambda i: (reps[i][0], -i))
        del reps[slow]
        fast = min(range(len(reps)), key=lambda i: (reps[i][0], i))
        del reps[fast]
    acc = [0.0] * 5
    for r in reps:
        for k in range(5):
            acc[k] += r[k + 1]
    n = float(len(reps))
    return tuple(a / n for a in acc)  # perf, power, eff, energy, avg_power


def candidates(kind, cpu, gpu):
    ncpu, ngpu = len(cpu), len(gpu)
    jb = ncpu * ngpu - 1
    if kind == 1:
        return [jb]
    if kind == 2:
        return [(ncpu - 1) * ngpu + g for g in range(ngpu)]
    if kind == 3:
        return [c * ngpu + ngpu - 1 for c in range(ncpu)]
    if kind == 4:
        return list(range(ncpu * ngpu))
    raise ValueError("candidate_set: open is not an exhaustive policy")


def choose(kind, table, cpu, gpu, gamma):
    ngpu = len(gpu)
    best = len(cpu) * ngpu - 1
    for j in candidates(kind, cpu, gpu):
        e, b = table[j], table[best]
        if 1.0 - e[0] > gamma:
            continue
        if e[2] != b[2]:
            better = e[2] > b[2]
        elif e[0] != b[0]:
            better = e[0] > b[0]
        else:
            s = cpu[j // ngpu] + gpu[j % ngpu]
            bs = cpu[best // ngpu] + gpu[best % ngpu]
            better = s < bs if s != bs else j < best
        if better:
            best = j
    return best


def row(j, e, cpu, gpu):
    """(setting, cpu, gpu, true_perf, true_loss, energy, avg_power, eff, pred_saving)."""
    ngpu = len(gpu)
    c, g = cpu[j // ngpu], gpu[j % ngpu]
    e_base = float(cpu[-1] + gpu[-1])
    sav = (e_base - float(c + g) / e[0]) / e_base
    return (j, c, g, e[0], 1.0 - e[0], e[3], e[4], e[2], sav)


def evaluate(base_runs, runs, cpu, gpu, kinds, gamma, open_idx=None, open_sav=None):
    """base_runs[a][r], runs[a][j][r] = (runtime_s, energy_j, avg_power_w).
    Returns (rows[a][p], aggs[p] = (mean_eff, mean_gain, mean_loss, mean_perf))."""
    n = len(cpu) * len(gpu)
    rows = []
    for a in range(len(base_runs)):
        table = [measure_truth(base_runs[a], runs[a][j]) for j in range(n)]
        out = []
        for k in kinds:
            if k == 0:
                r = list(row(open_idx[a], table[open_idx[a]], cpu, gpu))
                r[8] = open_sav[a]
                out.append(tuple(r))
            else:
                j = choose(k, table, cpu, gpu, gamma)
                out.append(row(j, table[j], cpu, gpu))
        rows.append(out)
    aggs = []
    for k in kinds:
        eff = loss = perf = 0.0
        cnt = 0
        for out in rows:
            for kk, r in zip(kinds, out):
                if kk != k:
                    continue
                eff += r[7]
                loss += r[4]
                perf += r[3]
                cnt += 1
        if cnt:
            eff, loss, perf = eff / cnt, loss / cnt, perf / cnt
            aggs.append((eff, eff - 1.0, loss, perf))
        else:
            aggs.append((0.0, 0.0, 0.0, 0.0))
    return rows, aggs
