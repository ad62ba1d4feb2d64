"""ALS completion + selection (joint mode) through the C-ABI (include/ocg.h).

No reference counterpart (the reference's CF is NCF only); semantics are the
CPU oracle's (oracle/ocg_oracle.c: ocgo_als_fit)."""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import lib, check, ptr
from .api import Context, PowerGrid, default_context


@dataclass
class AlsHyper:
    rank: int = 32
    lam: float = 0.003
    sweeps: int = 10
    seed: int = 42

    def to_c(self):
        h = _lib.AlsHyperC()
        h.rank, h.lambda_, h.sweeps, h.seed = self.rank, self.lam, self.sweeps, self.seed
        return h


class AlsPlan:
    """One joint completion problem resident on the device.

    csr: (m, row_ptr, col, val) host numpy arrays, or device addresses when
    ``on_device`` (ints; the caller keeps the buffers alive)."""

    def __init__(self, m, row_ptr, col, val, grid: PowerGrid, hyper: AlsHyper | None = None, gamma: float = 0.05,
                 on_device: bool = False, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        self.m, self.n = int(m), grid.n
        self.hyper = hyper or AlsHyper()
        cpu, gpu = grid.arrays()
        h = self.hyper.to_c()
        self._h = ctypes.c_void_p()
        if on_device:
            args = (ctypes.c_void_p(row_ptr), ctypes.c_void_p(col), ctypes.c_void_p(val))
        else:
            self._keep = (np.ascontiguousarray(row_ptr, np.int64), np.ascontiguousarray(col, np.int32),
                          np.ascontiguousarray(val, np.float32))
            args = tuple(ptr(a) for a in self._keep)
        check(lib.ocg_als_plan_create(self.ctx.handle, self.m, *args, 1 if on_device else 0, ptr(cpu), len(cpu),
                                      ptr(gpu), len(gpu), ctypes.byref(h), gamma, ctypes.byref(self._h)))

    def upload(self, row_ptr, col, val):
        """New observations (same m; nnz may change) from host memory: numpy arrays, or
        host addresses (ints, e.g. pinned buffers) the caller keeps alive until
        the next run completes."""
        if isinstance(row_ptr, int):
            args = (ctypes.c_void_p(row_ptr), ctypes.c_void_p(col), ctypes.c_void_p(val))
        else:
            self._keep = (np.ascontiguousarray(row_ptr, np.int64), np.ascontiguousarray(col, np.int32),
                          np.ascontiguousarray(val, np.float32))
            args = tuple(ptr(a) for a in self._keep)
        check(lib.ocg_als_plan_upload(self._h, *args))

    def upload_compact(self, row_ptr, col16, val):
        """upload() with uint16 column indices (n <= 65536); addresses or numpy arrays."""
        if isinstance(row_ptr, int):
            args = (ctypes.c_void_p(row_ptr), ctypes.c_void_p(col16), ctypes.c_void_p(val))
        else:
            self._keep = (np.ascontiguousarray(row_ptr, np.int64), np.ascontiguousarray(col16, np.uint16),
                          np.ascontiguousarray(val, np.float32))
            args = tuple(ptr(a) for a in self._keep)
        check(lib.ocg_als_plan_upload_compact(self._h, *args))

    def stage_compact(self, row_ptr, col16, val):
        """Double-buffered upload: the next step's CSR (16-bit columns) is copied on a side
        stream while the current step may still run; the next run() swaps it in.  Host
        addresses (pinned, unchanged until that run completes) or numpy arrays (kept alive
        by the plan)."""
        keep = None
        if isinstance(row_ptr, int):
            args = (ctypes.c_void_p(row_ptr), ctypes.c_void_p(col16), ctypes.c_void_p(val))
        else:
            keep = (np.ascontiguousarray(row_ptr, np.int64), np.ascontiguousarray(col16, np.uint16),
                    np.ascontiguousarray(val, np.float32))
            args = tuple(ptr(x) for x in keep)
        check(lib.ocg_als_plan_stage_compact(self._h, *args))
        if keep is not None:
            self._keep_staged = keep

    def results_async(self, out):
        """Enqueue the decisions' copy into 4 host addresses (pinned: int32[m], f64[m], f64[m],
        int32[m]) behind the current run; returns at once.  results_wait() blocks until done."""
        check(lib.ocg_als_plan_results_async(self._h, *(ctypes.c_void_p(a) for a in out)))

    def results_wait(self):
        check(lib.ocg_als_plan_results_wait(self._h))

    def add_observations(self, rows, cols, vals):
        """Merge new observed cells (sorted by (row, col), not observed yet) into the device
        CSR; only these cells cross PCIe.  Same matrix as upload() of the merged CSR."""
        r = np.ascontiguousarray(rows, np.int32)
        c = np.ascontiguousarray(cols, np.int32)
        v = np.ascontiguousarray(vals, np.float32)
        if not (len(r) == len(c) == len(v)):
            raise ValueError("rows/cols/vals lengths differ")
        check(lib.ocg_als_plan_add_observations(self._h, len(r), ptr(r), ptr(c), ptr(v)))

    def set_warm(self, sweeps: int):
        """Warm refits (deviation from from-scratch semantics): later runs start from the
        previous factors and run ``sweeps`` sweeps; 0 = from scratch."""
        check(lib.ocg_als_plan_set_warm(self._h, int(sweeps)))

    def run(self, timed: bool = True):
        """One step (CSC build + fit + fused imputation/selection).
        Returns (total_ms, [csc_ms, row_sweeps_ms, col_sweeps_ms, select_ms, row_gram_ms, col_gram_ms])."""
        tot = ctypes.c_float(0)
        ph = (ctypes.c_float * 6)()
        check(lib.ocg_als_plan_run(self._h, ctypes.byref(tot) if timed else None, ph if timed else None))
        return float(tot.value), [float(x) for x in ph]

    def results(self, out=None):
        """(idx, saving, loss, ncand) per row.  out: optional 4 host addresses (e.g.
        pinned buffers: int32[m], f64[m], f64[m], int32[m]) filled in place."""
        if out is not None:
            check(lib.ocg_als_plan_results(self._h, *(ctypes.c_void_p(a) for a in out), None, None))
            return None
        m = self.m
        idx, nc = np.zeros(m, np.int32), np.zeros(m, np.int32)
        sv, lo = np.zeros(m), np.zeros(m)
        check(lib.ocg_als_plan_results(self._h, ptr(idx), ptr(sv), ptr(lo), ptr(nc), None, None))
        return idx, sv, lo, nc

    def factors(self):
        U = np.zeros((self.m, self.hyper.rank), np.float32)
        V = np.zeros((self.n, self.hyper.rank), np.float32)
        check(lib.ocg_als_plan_results(self._h, None, None, None, None, ptr(U), ptr(V)))
        return U, V

    def completed_rows(self, row0: int, nrows: int) -> np.ndarray:
        out = np.zeros((nrows, self.n))
        check(lib.ocg_als_plan_completed_rows(self._h, row0, nrows, ptr(out)))
        return out

    def close(self):
        if getattr(self, "_h", None):
            lib.ocg_als_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
