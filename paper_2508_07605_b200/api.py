"""Python mirror of the reference's operator surface for the online path.

Names, argument meaning and error behaviour follow the reference C++ API
(opencap::PowerGrid / cf::NcfHyper / cf::fit / cf::complete /
NcfModel::predict / policy::select_caps / ProbePlan::default_plan); every call
goes through the C-ABI in include/ocg.h into sm_100a kernels.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _lib
from ._lib import lib, check, ptr

__all__ = [
    "PowerGrid", "NcfHyper", "NcfMeta", "CapDecision", "ProbePlan", "Context", "derive_seed",
    "select_caps", "select_caps_batch", "online_complete_batch", "online_fit_batch_params", "ncf_predict",
    "ncf_param_count", "LANE_SCALAR", "LANE_AVX2", "OnlinePlan", "NcfModel",
]

LANE_SCALAR, LANE_AVX2 = _lib.LANE_SCALAR, _lib.LANE_AVX2


def derive_seed(root: int, tag: str, n: int = 0) -> int:
    """derive_seed (rng.hpp:53-60)."""
    return int(lib.ocg_derive_seed(root, tag.encode(), n))


@dataclass(frozen=True)
class PowerGrid:
    """opencap::PowerGrid (core.hpp:39-58): lexicographic (cpu, gpu) columns, baseline = last."""

    cpu_caps: tuple
    gpu_caps: tuple

    def __post_init__(self):
        for name, caps in (("cpu", self.cpu_caps), ("gpu", self.gpu_caps)):
            if len(caps) == 0:
                raise _lib.InvalidArgument(1, f"{name} cap list is empty")
            for i, c in enumerate(caps):
                if c <= 0:
                    raise _lib.InvalidArgument(1, f"{name} caps must be positive watts")
                if i and c <= caps[i - 1]:
                    raise _lib.InvalidArgument(1, f"{name} caps must be strictly increasing")
        object.__setattr__(self, "cpu_caps", tuple(int(c) for c in self.cpu_caps))
        object.__setattr__(self, "gpu_caps", tuple(int(c) for c in self.gpu_caps))

    @staticmethod
    def default_grid() -> "PowerGrid":  # core.cpp:55-57
        return PowerGrid((100, 125, 150, 175, 200), (100, 150, 200, 250))

    @staticmethod
    def spanning(ncpu: int, ngpu: int) -> "PowerGrid":
        """SURVEY §8d grids for C1-C3: cpu 60-250 W, gpu 100-400 W."""
        return PowerGrid(tuple(60 + (190 * i) // (ncpu - 1) for i in range(ncpu)),
                         tuple(100 + (300 * j) // (ngpu - 1) for j in range(ngpu)))

    def settings(self):
        return [(c, g) for c in self.cpu_caps for g in self.gpu_caps]

    def baseline(self):
        return (self.cpu_caps[-1], self.gpu_caps[-1])

    @property
    def n(self) -> int:
        return len(self.cpu_caps) * len(self.gpu_caps)

    def arrays(self):
        return np.asarray(self.cpu_caps, np.int32), np.asarray(self.gpu_caps, np.int32)


@dataclass
class NcfHyper:
    """cf::NcfHyper (cfcomplete.hpp:11-20) with the reference defaults."""

    app_dim: int = 8
    setting_dim: int = 8
    hidden: Sequence[int] = field(default_factory=lambda: [32, 16])
    lr: float = 1e-3
    max_epochs: int = 2000
    patience: int = 100
    val_fraction: float = 0.1
    batch_size: int = 32

    def to_c(self) -> _lib.NcfHyperC:
        h = _lib.NcfHyperC()
        h.app_dim, h.setting_dim = self.app_dim, self.setting_dim
        if len(self.hidden) > 8:
            raise _lib.InvalidArgument(1, "at most 8 hidden layers")
        for i, w in enumerate(self.hidden):
            h.hidden[i] = w
        h.n_hidden = len(self.hidden)
        h.lr, h.max_epochs, h.patience = self.lr, self.max_epochs, self.patience
        h.val_fraction, h.batch_size = self.val_fraction, self.batch_size
        return h


def ncf_param_count(m: int, n: int, h: NcfHyper) -> int:
    dims = [h.app_dim + h.setting_dim, *h.hidden, 1]
    return m * h.app_dim + n * h.setting_dim + sum(dims[i] * dims[i + 1] + dims[i + 1] for i in range(len(dims) - 1))


@dataclass
class NcfMeta:
    """NcfModel::Meta (cfcomplete.hpp:34-40)."""

    seed: int
    epochs_run: int
    initial_train_mse: float
    final_train_mse: float
    best_val_mse: float


@dataclass
class CapDecision:
    """policy::CapDecision (policy.hpp:22-27) + the column index of the setting."""

    setting: tuple
    index: int
    pred_saving: float
    pred_loss: float
    candidates_considered: int


class ProbePlan:
    """ProbePlan::default_plan (policy.cpp:66-82): the sampled-setting set."""

    def __init__(self, settings):
        self.settings = list(settings)

    @staticmethod
    def default_plan(grid: PowerGrid) -> "ProbePlan":
        cpu, gpu = grid.arrays()
        cols = np.zeros(6, np.int32)
        cnt = ctypes.c_int32()
        check(lib.ocg_default_plan(ptr(cpu), len(cpu), ptr(gpu), len(gpu), ptr(cols), ctypes.byref(cnt)))
        s = grid.settings()
        plan = ProbePlan(s[c] for c in cols[: cnt.value])
        plan.columns = [int(c) for c in cols[: cnt.value]]
        return plan


class Context:
    """One CUDA device + stream (ocg_ctx).  Owned by one thread at a time."""

    def __init__(self, device: int = 0):
        h = ctypes.c_void_p()
        check(lib.ocg_ctx_create(device, ctypes.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def info(self):
        sm, ma, mi = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        check(lib.ocg_ctx_device_info(self._h, ctypes.byref(sm), ctypes.byref(ma), ctypes.byref(mi)))
        return {"sm_count": sm.value, "cc": (ma.value, mi.value)}

    def close(self):
        if self._h:
            lib.ocg_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


_default_ctx = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def select_caps_batch(rows: np.ndarray, grid: PowerGrid, gamma: float = 0.05, ctx: Context | None = None):
    """policy::select_caps over every row of ``rows`` (nrows x grid.n, FP64).

    Returns (idx, saving, loss, ncand) arrays."""
    ctx = ctx or default_context()
    rows = np.ascontiguousarray(rows, dtype=np.float64)
    if rows.ndim != 2 or rows.shape[1] != grid.n:
        raise _lib.InvalidArgument(1, "select_caps: row length does not cover the grid")
    r = rows.shape[0]
    idx, ncand = np.zeros(r, np.int32), np.zeros(r, np.int32)
    sav, loss = np.zeros(r), np.zeros(r)
    cpu, gpu = grid.arrays()
    check(lib.ocg_select_caps(ctx.handle, ptr(rows), r, ptr(cpu), len(cpu), ptr(gpu), len(gpu), gamma,
                              ptr(idx), ptr(sav), ptr(loss), ptr(ncand)))
    return idx, sav, loss, ncand


def select_caps(row, grid: PowerGrid, gamma: float = 0.05, ctx: Context | None = None) -> CapDecision:
    """policy::select_caps (policy.cpp:17-64) for one row."""
    idx, sav, loss, ncand = select_caps_batch(np.asarray(row, np.float64)[None, :], grid, gamma, ctx)
    j = int(idx[0])
    return CapDecision(grid.settings()[j], j, float(sav[0]), float(loss[0]), int(ncand[0]))


@dataclass
class OnlineBatchResult:
    status: np.ndarray
    completed: np.ndarray
    idx: np.ndarray
    saving: np.ndarray
    loss: np.ndarray
    ncand: np.ndarray
    meta: np.ndarray  # structured: seed, epochs_run, initial/final train mse, best val mse


META_DTYPE = np.dtype([("seed", "<u8"), ("epochs_run", "<i4"), ("initial_train_mse", "<f8"),
                       ("final_train_mse", "<f8"), ("best_val_mse", "<f8")], align=True)
assert META_DTYPE.itemsize == ctypes.sizeof(_lib.NcfMetaC)


def online_complete_batch(block_vals, block_mask, probe_vals, probe_mask, seeds, grid: PowerGrid,
                          hyper: NcfHyper | None = None, gamma: float = 0.05, lane: int = LANE_AVX2,
                          ctx: Context | None = None) -> OnlineBatchResult:
    """run_open_online steps 3-4 (policy.cpp:178-189) for a batch of apps.

    block_*: offline dense block (D x n); probe_*: one probed row per app
    (napps x n); seeds: the cf::complete seed of each app.  Per-app failures are
    reported in ``status`` with the OCG code of the exception the reference
    would raise for that app."""
    ctx = ctx or default_context()
    hyper = hyper or NcfHyper()
    bv = np.ascontiguousarray(block_vals, np.float64)
    bm = np.ascontiguousarray(block_mask, np.uint8)
    pv = np.ascontiguousarray(probe_vals, np.float64)
    pm = np.ascontiguousarray(probe_mask, np.uint8)
    sd = np.ascontiguousarray(seeds, np.uint64)
    napps, n = pv.shape
    if n != grid.n or bv.shape[1] != n:
        raise _lib.InvalidArgument(1, "row length does not cover the grid")
    out = OnlineBatchResult(np.zeros(napps, np.int32), np.zeros((napps, n)), np.zeros(napps, np.int32),
                            np.zeros(napps), np.zeros(napps), np.zeros(napps, np.int32), np.zeros(napps, META_DTYPE))
    cpu, gpu = grid.arrays()
    h = hyper.to_c()
    check(lib.ocg_online_complete_batch(ctx.handle, bv.shape[0], ptr(bv), ptr(bm), napps, ptr(pv), ptr(pm),
                                        ptr(sd), ptr(cpu), len(cpu), ptr(gpu), len(gpu), ctypes.byref(h), gamma,
                                        lane, ptr(out.completed), ptr(out.idx), ptr(out.saving), ptr(out.loss),
                                        ptr(out.ncand), ptr(out.meta), ptr(out.status)))
    return out


def online_fit_batch_params(block_vals, block_mask, probe_vals, probe_mask, seeds, hyper: NcfHyper | None = None,
                            lane: int = LANE_AVX2, ctx: Context | None = None):
    """cf::fit of (block + app row) per app; returns (params[napps, T], meta, status)."""
    ctx = ctx or default_context()
    hyper = hyper or NcfHyper()
    bv = np.ascontiguousarray(block_vals, np.float64)
    bm = np.ascontiguousarray(block_mask, np.uint8)
    pv = np.ascontiguousarray(probe_vals, np.float64)
    pm = np.ascontiguousarray(probe_mask, np.uint8)
    sd = np.ascontiguousarray(seeds, np.uint64)
    napps, n = pv.shape
    T = ncf_param_count(bv.shape[0] + 1, n, hyper)
    params = np.zeros((napps, T))
    meta = np.zeros(napps, META_DTYPE)
    status = np.zeros(napps, np.int32)
    h = hyper.to_c()
    check(lib.ocg_online_fit_batch_params(ctx.handle, bv.shape[0], ptr(bv), ptr(bm), napps, ptr(pv), ptr(pm),
                                          ptr(sd), n, ctypes.byref(h), lane, ptr(params), T, ptr(meta),
                                          ptr(status)))
    return params, meta, status


def ncf_predict(m: int, n: int, hyper: NcfHyper, params, app_seen, setting_seen, rows, cols,
                lane: int = LANE_AVX2, ctx: Context | None = None) -> np.ndarray:
    """NcfModel::predict (cfcomplete.cpp:47-58) for (rows[k], cols[k]) pairs."""
    ctx = ctx or default_context()
    p = np.ascontiguousarray(params, np.float64)
    a = np.ascontiguousarray(app_seen, np.uint8)
    s = np.ascontiguousarray(setting_seen, np.uint8)
    r = np.ascontiguousarray(rows, np.int64)
    c = np.ascontiguousarray(cols, np.int64)
    out = np.zeros(len(r))
    h = hyper.to_c()
    check(lib.ocg_ncf_predict(ctx.handle, m, n, ctypes.byref(h), ptr(p), ptr(a), ptr(s), ptr(r), ptr(c), len(r),
                              lane, ptr(out)))
    return out


@dataclass
class NcfModel:
    """cf::NcfModel as data (cfcomplete.hpp:25-52): m apps, n settings, the flat
    parameter vector (Adam block order), seen masks and the training meta.
    ``to_json`` / ``from_json`` are the reference's model file (byte-identical
    text); ``predict`` runs NcfModel::predict on the device (FP64, lane-exact)."""

    hyper: NcfHyper
    m: int
    n: int
    params: np.ndarray
    app_seen: np.ndarray
    setting_seen: np.ndarray
    meta: NcfMeta

    def to_json(self) -> str:
        h = self.hyper.to_c()
        p = np.ascontiguousarray(self.params, np.float64)
        a = np.ascontiguousarray(self.app_seen, np.uint8)
        s = np.ascontiguousarray(self.setting_seen, np.uint8)
        mt = _lib.NcfMetaC()
        mt.seed, mt.epochs_run = self.meta.seed, self.meta.epochs_run
        mt.initial_train_mse, mt.final_train_mse, mt.best_val_mse = (self.meta.initial_train_mse,
                                                                    self.meta.final_train_mse,
                                                                    self.meta.best_val_mse)
        ln = ctypes.c_size_t()
        args = (ctypes.byref(h), self.m, self.n, ptr(p), ptr(a), ptr(s), ctypes.byref(mt))
        check(lib.ocg_ncf_model_to_json(*args, None, 0, ctypes.byref(ln)))
        buf = ctypes.create_string_buffer(ln.value)
        check(lib.ocg_ncf_model_to_json(*args, buf, ln.value, ctypes.byref(ln)))
        return buf.value.decode()

    @staticmethod
    def from_json(text: str) -> "NcfModel":
        raw = text.encode()
        h = _lib.NcfHyperC()
        m, n, npar = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        check(lib.ocg_ncf_model_from_json(raw, ctypes.byref(h), ctypes.byref(m), ctypes.byref(n), ctypes.byref(npar),
                                          None, None, None, None))
        p = np.zeros(npar.value)
        a, s = np.zeros(m.value, np.uint8), np.zeros(n.value, np.uint8)
        mt = _lib.NcfMetaC()
        check(lib.ocg_ncf_model_from_json(raw, ctypes.byref(h), ctypes.byref(m), ctypes.byref(n), ctypes.byref(npar),
                                          ptr(p), ptr(a), ptr(s), ctypes.byref(mt)))
        hyper = NcfHyper(app_dim=h.app_dim, setting_dim=h.setting_dim, hidden=[h.hidden[i] for i in range(h.n_hidden)])
        meta = NcfMeta(mt.seed, mt.epochs_run, mt.initial_train_mse, mt.final_train_mse, mt.best_val_mse)
        return NcfModel(hyper, m.value, n.value, p, a, s, meta)

    def predict(self, rows, cols, lane: int = LANE_AVX2, ctx: Context | None = None) -> np.ndarray:
        return ncf_predict(self.m, self.n, self.hyper, self.params, self.app_seen, self.setting_seen, rows, cols,
                           lane, ctx)


class OnlinePlan:
    """Device-resident per-app batch (ocg_online_plan): inputs uploaded once,
    the completion + selection kernel re-runnable on data already in HBM."""

    def __init__(self, block_vals, block_mask, probe_vals, probe_mask, seeds, grid: PowerGrid,
                 hyper: NcfHyper | None = None, gamma: float = 0.05, lane: int = LANE_AVX2,
                 want_completed: bool = True, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        hyper = hyper or NcfHyper()
        bv = np.ascontiguousarray(block_vals, np.float64)
        bm = np.ascontiguousarray(block_mask, np.uint8)
        pv = np.ascontiguousarray(probe_vals, np.float64)
        pm = np.ascontiguousarray(probe_mask, np.uint8)
        sd = np.ascontiguousarray(seeds, np.uint64)
        self.napps, self.n = pv.shape
        cpu, gpu = grid.arrays()
        h = hyper.to_c()
        self._h = ctypes.c_void_p()
        check(lib.ocg_online_plan_create(self.ctx.handle, bv.shape[0], ptr(bv), ptr(bm), self.napps, ptr(pv), ptr(pm),
                                         ptr(sd), ptr(cpu), len(cpu), ptr(gpu), len(gpu), ctypes.byref(h), gamma, lane,
                                         1 if want_completed else 0, ctypes.byref(self._h)))

    def run(self, timed: bool = True) -> float:
        """Re-run the kernel; returns its CUDA-event milliseconds when timed."""
        ms = ctypes.c_float(0.0)
        check(lib.ocg_online_plan_run(self._h, ctypes.byref(ms) if timed else None))
        return float(ms.value)

    def results(self) -> "OnlineBatchResult":
        n, napps = self.n, self.napps
        out = OnlineBatchResult(np.zeros(napps, np.int32), np.zeros((napps, n)), np.zeros(napps, np.int32),
                                np.zeros(napps), np.zeros(napps), np.zeros(napps, np.int32),
                                np.zeros(napps, META_DTYPE))
        check(lib.ocg_online_plan_results(self._h, ptr(out.completed), ptr(out.idx), ptr(out.saving), ptr(out.loss),
                                          ptr(out.ncand), ptr(out.meta), ptr(out.status)))
        return out

    def close(self):
        if self._h:
            lib.ocg_online_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
