"""Evaluation harness on the device: policy::evaluate_suite
(policy.cpp:373-405) for many apps at once.  The simulator (sim::run) is the
caller's: it hands in the repetition runs measure_truth (policy.cpp:213-256) would
draw, and the device builds the truth tables, the exhaustive policies' choices
(choose_exhaustive, policy.cpp:292-320), the rows (row_from_truth, :322-337) and the
per-policy aggregates, bit-exact in FP64."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check, lib, ptr
from .api import Context, PowerGrid, default_context

POLICY_NAMES = ("open", "no_cap", "gpu_cap_only", "cpu_cap_only", "oracle")


def policy_kind(name: str) -> int:
    """policy::policy_from_name (policy.cpp:203-211)."""
    if name not in POLICY_NAMES:
        raise _lib.InvalidArgument(_lib.OCG_E_INVALID, f"unknown policy: {name}")
    return POLICY_NAMES.index(name)


@dataclass
class EvalReport:
    rows: np.ndarray  # napps x npol structured (EvalRowC fields), report order
    aggregates: np.ndarray  # npol structured (EvalAggregateC fields)

    @property
    def policies(self) -> list[str]:
        return [POLICY_NAMES[k] for k in self.aggregates["policy"]]


_ROW_DTYPE = np.dtype([(n, np.int32 if t is _lib.c_i32 else np.float64) for n, t in _lib.EvalRowC._fields_],
                      align=True)
_AGG_DTYPE = np.dtype([(n, np.int32 if t is _lib.c_i32 else np.float64) for n, t in _lib.EvalAggregateC._fields_],
                      align=True)
assert _ROW_DTYPE.itemsize == _lib.ctypes.sizeof(_lib.EvalRowC)
assert _AGG_DTYPE.itemsize == _lib.ctypes.sizeof(_lib.EvalAggregateC)


def evaluate_suite(base_runs, runs, grid: PowerGrid, policies, gamma: float = 0.05, open_idx=None,
                   open_pred_saving=None, ctx: Context | None = None) -> EvalReport:
    """base_runs: napps x reps x 3 and runs: napps x n x reps x 3 of sim::RunResult
    (runtime_s, energy_j, avg_power_w); policies: names or kinds; open_idx /
    open_pred_saving: the open policy's run_open_online decisions per app."""
    ctx = ctx or default_context()
    b = np.ascontiguousarray(base_runs, np.float64)
    r = np.ascontiguousarray(runs, np.float64)
    napps, reps = b.shape[0], b.shape[1]
    n = grid.n
    if b.shape != (napps, reps, 3) or r.shape != (napps, n, reps, 3):
        raise _lib.InvalidArgument(_lib.OCG_E_INVALID, "run arrays do not match (napps, [n,] reps, 3)")
    kinds = np.asarray([policy_kind(p) if isinstance(p, str) else int(p) for p in policies], np.int32)
    oi = None if open_idx is None else np.ascontiguousarray(open_idx, np.int32)
    os_ = None if open_pred_saving is None else np.ascontiguousarray(open_pred_saving, np.float64)
    cpu, gpu = grid.arrays()
    rows = np.zeros((napps, len(kinds)), _ROW_DTYPE)
    aggs = np.zeros(len(kinds), _AGG_DTYPE)
    check(lib.ocg_eval_suite(ctx.handle, napps, ptr(cpu), len(cpu), ptr(gpu), len(gpu), reps, ptr(b), ptr(r),
                             gamma, len(kinds), ptr(kinds), ptr(oi), ptr(os_), ptr(rows), ptr(aggs)))
    return EvalReport(rows, aggs)
