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
    """Reference-format NCF weights for benches/tests at sizes the reference cannot fit
    (C2: 1M x 4096, k = 32): embedding rows uniform in +-emb_scale, the MLP with the
    reference's Glorot-uniform bound (nnkit.cpp:58-61), hidden {32, 16}; the output
    layer is scaled (x0.25, bias 0.7) so predictions spread over (0.01, 1.25] the way a
    fitted model's do (random Glorot output weights put ~55 % of cells on a clamp)."""
    from .api import NcfMeta, ncf_param_count
    h = NcfHyper(app_dim=k, setting_dim=k)
    rng = np.random.default_rng(seed)
    parts = [rng.uniform(-emb_scale, emb_scale, m * k), rng.uniform(-emb_scale, emb_scale, n * k)]
    dims = [2 * k, 32, 16, 1]
    for l in range(3):
        b = np.sqrt(6.0 / (dims[l] + dims[l + 1]))
        w = rng.uniform(-b, b, dims[l] * dims[l + 1])
        bias = rng.uniform(-0.1, 0.1, dims[l + 1])
        if l == 2:  # output layer: predictions centred in the normalized-performance range
            w *= 0.25
            bias[:] = 0.7
        parts += [w, bias]
    p = np.concatenate(parts)
    assert len(p) == ncf_param_count(m, n, h)
    return NcfModel(h, m, n, p, np.ones(m, np.uint8), np.ones(n, np.uint8), NcfMeta(seed, 0, 0.0, 0.0, 0.0))
