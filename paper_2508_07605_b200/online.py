"""Batched online-phase streams: the phase detector over many
GPU-power streams and run_open_online's probe ingest -> re-probe rule ->
per-app completion -> selection as one device pipeline."""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import LANE_AVX2, check, lib, ptr
from .api import META_DTYPE, Context, NcfHyper, OnlineBatchResult, PowerGrid, ProbePlan, default_context


def phase_detect_batch(power, lengths=None, delta_s: float = 0.2, window_s: float = 5.0, p_th_w: float = 60.0,
                       armed_start: bool = False, ctx: Context | None = None):
    """phase::Detector over every row of ``power`` (nstreams x nsamples).  Returns
    (fire_index, status): index of the firing sample or -1, and OCG_E_INVALID for a
    stream that feeds a negative sample.  armed_start: feeding begins at the first
    sample below the threshold (run_open_online's rule) instead of the first sample
    (detect_offline)."""
    ctx = ctx or default_context()
    p = np.ascontiguousarray(power, np.float64)
    if p.ndim == 1:
        p = p[None, :]
    ns, nt = p.shape
    ln = None if lengths is None else np.ascontiguousarray(lengths, np.int64)
    cfg = _lib.DetectorConfigC(delta_s, window_s, p_th_w)
    fire = np.zeros(ns, np.int64)
    st = np.zeros(ns, np.int32)
    check(lib.ocg_phase_detect_batch(ctx.handle, ctypes.byref(cfg), ns, nt, ptr(p), ptr(ln), int(armed_start),
                                     ptr(fire), ptr(st)))
    return fire, st


def online_ingest_complete_batch(block_vals, block_mask, counters, seeds, grid: PowerGrid, predictor,
                                 hyper: NcfHyper | None = None, gamma: float = 0.05, lane: int = LANE_AVX2,
                                 reprobe_counters=None, transition=None, plan: ProbePlan | None = None,
                                 want_completed: bool = True, ctx: Context | None = None):
    """run_open_online steps 2-4 for many apps on the device: predict_perf of each app's
    probe counters (napps x nplan x 7; the re-probe counters where ``transition`` is set),
    the estimates placed at the plan's columns, cf::complete against the dense block, and
    select_caps.  ``predictor`` is a device-resident predictor.Predictor.
    Returns (OnlineBatchResult, estimates napps x nplan)."""
    ctx = ctx or default_context()
    hyper = hyper or NcfHyper()
    plan = plan or ProbePlan.default_plan(grid)
    cols = np.asarray(plan.columns, np.int32)
    bv = np.ascontiguousarray(block_vals, np.float64)
    bm = np.ascontiguousarray(block_mask, np.uint8)
    c = np.ascontiguousarray(counters, np.float64).reshape(-1, len(cols), 7)
    napps = c.shape[0]
    rc_ = None if reprobe_counters is None else np.ascontiguousarray(reprobe_counters, np.float64)
    tr = None if transition is None else np.ascontiguousarray(transition, np.int32)
    sd = np.ascontiguousarray(seeds, np.uint64)
    cpu, gpu = grid.arrays()
    n = grid.n
    est = np.zeros((napps, len(cols)))
    comp = np.zeros((napps, n)) if want_completed else None
    idx, nc = np.zeros(napps, np.int32), np.zeros(napps, np.int32)
    sav, loss = np.zeros(napps), np.zeros(napps)
    meta = np.zeros(napps, META_DTYPE)
    status = np.zeros(napps, np.int32)
    h = hyper.to_c()
    check(lib.ocg_online_ingest_complete_batch(ctx.handle, bv.shape[0], ptr(bv), ptr(bm), napps, ptr(cols), len(cols),
                                               predictor.handle, ptr(c), ptr(rc_), ptr(tr), ptr(sd), ptr(cpu), len(cpu),
                                               ptr(gpu), len(gpu), ctypes.byref(h), gamma, lane, ptr(est), ptr(comp),
                                               ptr(idx), ptr(sav), ptr(loss), ptr(nc), ptr(meta), ptr(status)))
    return OnlineBatchResult(status, comp, idx, sav, loss, nc, meta), est
