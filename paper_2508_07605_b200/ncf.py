"""NCF completion + selection over a whole sparse matrix on the device.

cf::complete's imputation (cfcomplete.cpp:208-211, NcfModel::predict :47-58)
fused with policy::select_caps (policy.cpp:17-64) per row, through the C-ABI
(include/ocg.h: ocg_ncf_model_* / ocg_ncf_plan_*).  ``precision``:
EXACT (FP64, the reference lane's operation order: bit-identical) or FAST
(FP32 + tcgen05 tensor cores)."""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import OCG_NCF_EXACT, OCG_NCF_FAST, check, lib, ptr
from .api import LANE_AVX2, Context, NcfHyper, NcfModel, PowerGrid, default_context

EXACT, FAST = OCG_NCF_EXACT, OCG_NCF_FAST


class DeviceNcfModel:
    """A fitted cf::NcfModel resident in HBM (ocg_ncf_model)."""

    def __init__(self, model: NcfModel | None = None, *, json_text: str | None = None, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        self._h = ctypes.c_void_p()
        if json_text is not None:
            check(lib.ocg_ncf_model_from_json_text(self.ctx.handle, json_text.encode(), ctypes.byref(self._h)))
            self.model = None
            return
        h = model.hyper.to_c()
        self._keep = (np.ascontiguousarray(model.params, np.float64), np.ascontiguousarray(model.app_seen, np.uint8),
                      np.ascontiguousarray(model.setting_seen, np.uint8))
        check(lib.ocg_ncf_model_create(self.ctx.handle, ctypes.byref(h), model.m, model.n, *map(ptr, self._keep),
                                       ctypes.byref(self._h)))
        self.model = model

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            lib.ocg_ncf_model_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class NcfPlan:
    """A device model bound to a matrix (CSR of observed cells) and a grid."""

    def __init__(self, model: DeviceNcfModel, row_ptr, col, val, grid: PowerGrid, gamma: float = 0.05,
                 precision: int = FAST, lane: int = LANE_AVX2, on_device: bool = False):
        self.model = model
        self.m = int(len(row_ptr) - 1) if not on_device else None
        self.n = grid.n
        cpu, gpu = grid.arrays()
        self._h = ctypes.c_void_p()
        if on_device:
            args = (ctypes.c_void_p(row_ptr), ctypes.c_void_p(col), ctypes.c_void_p(val))
        else:
            self._keep = (np.ascontiguousarray(row_ptr, np.int64), np.ascontiguousarray(col, np.int32),
                          np.ascontiguousarray(val, np.float64))
            args = tuple(ptr(a) for a in self._keep)
        check(lib.ocg_ncf_plan_create(model.handle, *args, 1 if on_device else 0, ptr(cpu), len(cpu), ptr(gpu),
                                      len(gpu), gamma, precision, lane, ctypes.byref(self._h)))

    def upload(self, row_ptr, col, val):
        if isinstance(row_ptr, int):
            args = (ctypes.c_void_p(row_ptr), ctypes.c_void_p(col), ctypes.c_void_p(val))
        else:
            self._keep = (np.ascontiguousarray(row_ptr, np.int64), np.ascontiguousarray(col, np.int32),
                          np.ascontiguousarray(val, np.float64))
            args = tuple(ptr(a) for a in self._keep)
        check(lib.ocg_ncf_plan_upload(self._h, *args))

    def stage(self, row_ptr: int, col: int, val: int):
        """Queue the next step's CSR (host pointers, pinned memory) on the side copy stream."""
        check(lib.ocg_ncf_plan_stage(self._h, ctypes.c_void_p(row_ptr), ctypes.c_void_p(col), ctypes.c_void_p(val)))

    def results_async(self, out):
        """Queue the decisions' copies into host pointers out = (idx, saving, loss, ncand)."""
        check(lib.ocg_ncf_plan_results_async(self._h, *(ctypes.c_void_p(int(p)) for p in out)))

    def results_wait(self):
        check(lib.ocg_ncf_plan_results_wait(self._h))

    def run(self, timed: bool = True):
        """One completion + selection; returns (total_ms, [prep_ms, dense_ms]) when timed."""
        tot = ctypes.c_float(0.0)
        ph = (ctypes.c_float * 2)()
        check(lib.ocg_ncf_plan_run(self._h, ctypes.byref(tot) if timed else None, ph if timed else None))
        return float(tot.value), [float(x) for x in ph]

    def results(self, m: int):
        idx, ncand = np.zeros(m, np.int32), np.zeros(m, np.int32)
        saving, loss = np.zeros(m), np.zeros(m)
        check(lib.ocg_ncf_plan_results(self._h, ptr(idx), ptr(saving), ptr(loss), ptr(ncand)))
        return idx, saving, loss, ncand

    def completed_rows(self, rows) -> np.ndarray:
        r = np.ascontiguousarray(rows, np.int64)
        out = np.zeros((len(r), self.n))
        check(lib.ocg_ncf_plan_completed_rows(self._h, ptr(r), len(r), ptr(out)))
        return out

    def close(self):
        if self._h:
            lib.ocg_ncf_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def random_model(m: int, n: int, k: int = 32, seed: int = 0, emb_scale: float = 1.0) -> NcfModel:
    """Reference-format NCF model with synthetic weights (weights.random_ncf_params) for benches and
    tests at sizes the reference cannot fit (C2: 1M x 4096, k = 32)."""
    from .api import NcfMeta
    from .weights import random_ncf_params

    h = NcfHyper(app_dim=k, setting_dim=k)
    p = random_ncf_params(m, n, k, seed, emb_scale)
    return NcfModel(h, m, n, p, np.ones(m, np.uint8), np.ones(n, np.uint8), NcfMeta(seed, 0, 0.0, 0.0, 0.0))


def model_rows(model: NcfModel, r0: int, r1: int) -> NcfModel:
    """The model restricted to app rows [r0, r1) (a rank's shard): NcfModel::predict(i, j)
    reads only row i of the app table, so a row shard completes its rows identically."""
    k = model.hyper.app_dim
    p = np.concatenate([model.params[r0 * k: r1 * k], model.params[model.m * k:]])
    return NcfModel(model.hyper, r1 - r0, model.n, p, model.app_seen[r0:r1].copy(), model.setting_seen.copy(),
                    model.meta)
