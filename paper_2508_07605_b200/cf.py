"""The reference's cf:: operators over one whole matrix, every solver.

* ``cf_fit``      <- ``cf::fit``      (cfcomplete.hpp:59, cfcomplete.cpp:63-196)
* ``cf_complete`` <- ``cf::complete`` (cfcomplete.hpp:63, cfcomplete.cpp:198-213),
  optionally fused with ``policy::select_caps`` of every completed row.

Solvers: ``SOLVER_NCF_REF`` (the reference's NCF and schedule in FP64, operation
order of the chosen kernel lane: bit-identical parameters and meta),
``SOLVER_NCF_FAST`` (same NCF and schedule in FP32), ``SOLVER_ALS`` (rank-k ALS,
no reference counterpart).  Matrices are CSR (row_ptr int64, col int32
strictly ascending per row, val float64 in (0, 1.25]).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import LANE_AVX2, OCG_SOLVER_ALS, OCG_SOLVER_NCF_FAST, OCG_SOLVER_NCF_REF, check, lib, ptr
from .api import Context, NcfHyper, NcfMeta, NcfModel, PowerGrid, default_context, ncf_param_count

SOLVER_NCF_REF, SOLVER_NCF_FAST, SOLVER_ALS = OCG_SOLVER_NCF_REF, OCG_SOLVER_NCF_FAST, OCG_SOLVER_ALS


def _csr(row_ptr, col, val):
    return (np.ascontiguousarray(row_ptr, np.int64), np.ascontiguousarray(col, np.int32),
            np.ascontiguousarray(val, np.float64))


def cf_fit(row_ptr, col, val, n: int, hyper: NcfHyper | None = None, seed: int = 42,
           solver: int = SOLVER_NCF_REF, lane: int = LANE_AVX2, ctx: Context | None = None,
           stats: dict | None = None) -> NcfModel:
    """cf::fit of the m x n matrix given as CSR; returns the fitted NcfModel."""
    ctx = ctx or default_context()
    hyper = hyper or NcfHyper()
    rp, c, v = _csr(row_ptr, col, val)
    m = len(rp) - 1
    params = np.zeros(ncf_param_count(m, n, hyper))
    aseen, sseen = np.zeros(m, np.uint8), np.zeros(n, np.uint8)
    meta = _lib.NcfMetaC()
    h = hyper.to_c()
    steps, dms = ctypes.c_int64(), ctypes.c_double()
    check(lib.ocg_cf_fit_stats(ctx.handle, m, n, ptr(rp), ptr(c), ptr(v), ctypes.byref(h), seed, solver, lane,
                               ptr(params), ptr(aseen), ptr(sseen), ctypes.byref(meta), ctypes.byref(steps),
                               ctypes.byref(dms)))
    if stats is not None:
        stats.update(steps=steps.value, device_ms=dms.value)
    return NcfModel(hyper, m, n, params, aseen, sseen,
                    NcfMeta(meta.seed, meta.epochs_run, meta.initial_train_mse, meta.final_train_mse,
                            meta.best_val_mse))


@dataclass
class CompleteResult:
    completed: np.ndarray | None  # m x n, or None
    idx: np.ndarray | None        # selection per row (when a grid was given)
    saving: np.ndarray | None
    loss: np.ndarray | None
    ncand: np.ndarray | None


def cf_complete(row_ptr, col, val, n: int, hyper: NcfHyper | None = None, seed: int = 42,
                solver: int = SOLVER_NCF_REF, lane: int = LANE_AVX2, grid: PowerGrid | None = None,
                gamma: float = 0.05, als=None, want_completed: bool = True,
                ctx: Context | None = None) -> CompleteResult:
    """cf::complete (+ select_caps per row when ``grid`` is given)."""
    ctx = ctx or default_context()
    hyper = hyper or NcfHyper()
    rp, c, v = _csr(row_ptr, col, val)
    m = len(rp) - 1
    h = hyper.to_c()
    ah = None
    if solver == SOLVER_ALS:
        ah = als if isinstance(als, _lib.AlsHyperC) else _lib.AlsHyperC(*als)
    comp = np.zeros((m, n)) if want_completed else None
    idx = sav = loss = nc = None
    cpu = gpu = None
    ncpu = ngpu = 0
    if grid is not None:
        cpu, gpu = grid.arrays()
        ncpu, ngpu = len(cpu), len(gpu)
        idx, nc = np.zeros(m, np.int32), np.zeros(m, np.int32)
        sav, loss = np.zeros(m), np.zeros(m)
    check(lib.ocg_cf_complete(ctx.handle, m, n, ptr(rp), ptr(c), ptr(v), ctypes.byref(h),
                              ctypes.byref(ah) if ah is not None else None, seed, solver, lane, ptr(cpu), ncpu,
                              ptr(gpu), ngpu, gamma, ptr(comp), ptr(idx), ptr(sav), ptr(loss), ptr(nc)))
    return CompleteResult(comp, idx, sav, loss, nc)
