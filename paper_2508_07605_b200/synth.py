"""Synthetic inputs (host side, via the C-ABI) for benches and tests.

See include/ocg.h "synthetic inputs": restatements of the reference's own
input generators (sim::make_suite / true_perf / profile_suite) and the
SURVEY §8d joint matrices C1-C3."""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import lib, check, ptr
from .api import PowerGrid

c_i32, c_i64, c_u64, c_dbl, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p


class WorkloadSpecC(ctypes.Structure):
    _fields_ = [("archetype", c_i32), ("kappa_c", c_dbl), ("alpha_c", c_dbl), ("kappa_g", c_dbl),
                ("alpha_g", c_dbl), ("base_runtime_s", c_dbl), ("cpu_phase_s", c_dbl), ("noise_sigma", c_dbl),
                ("ips_max", c_dbl), ("mem_tput_max", c_dbl), ("sm_clock_max", c_dbl)]


lib.ocg_synth_suite.argtypes = [c_vp, c_u64, ctypes.c_int, c_dbl, c_dbl, c_vp, c_i32, c_vp, c_i32, c_vp]
lib.ocg_synth_suite.restype = ctypes.c_int
lib.ocg_true_perf.argtypes = [c_vp, c_i32, c_i32]
lib.ocg_true_perf.restype = c_dbl
lib.ocg_synth_offline_block.argtypes = [c_u64, c_vp, c_i32, c_vp, c_i32, c_vp, c_vp]
lib.ocg_synth_offline_block.restype = ctypes.c_int
lib.ocg_synth_online_apps.argtypes = [c_i64, c_u64, c_vp, c_i32, c_vp, c_i32, c_vp, c_vp, c_vp]
lib.ocg_synth_online_apps.restype = ctypes.c_int
lib.ocg_synth_csr_count.argtypes = [c_i64, c_vp, c_i32, c_vp, c_i32, c_dbl, c_i64, c_u64, ctypes.c_int, c_vp]
lib.ocg_synth_csr_count.restype = ctypes.c_int
lib.ocg_synth_csr_fill.argtypes = [c_i64, c_vp, c_i32, c_vp, c_i32, c_dbl, c_i64, c_u64, ctypes.c_int, c_vp, c_vp,
                                   c_vp, c_vp]
lib.ocg_synth_csr_fill.restype = ctypes.c_int


lib.ocg_synth_rows_dense.argtypes = [c_i64, c_vp, c_i32, c_vp, c_i32, c_dbl, c_i64, c_u64, c_vp, c_i64, c_vp, c_vp]
lib.ocg_synth_rows_dense.restype = ctypes.c_int


def joint_rows_dense(m: int, grid: PowerGrid, density: float, dense_rows: int, rows, seed: int = 42):
    """Selected rows of joint_csr(...) as dense (values, mask)."""
    rows = np.ascontiguousarray(rows, np.int64)
    cpu, gpu = grid.arrays()
    vals = np.zeros((len(rows), grid.n))
    mask = np.zeros((len(rows), grid.n), np.uint8)
    check(lib.ocg_synth_rows_dense(m, ptr(cpu), len(cpu), ptr(gpu), len(gpu), density, dense_rows, seed, ptr(rows),
                                   len(rows), ptr(vals), ptr(mask)))
    return vals, mask


lib.ocg_synth_true_rows.argtypes = [c_i64, c_vp, c_i32, c_vp, c_i32, c_u64, c_vp, c_i64, c_vp]
lib.ocg_synth_true_rows.restype = ctypes.c_int


def true_rows(m: int, grid: PowerGrid, rows, seed: int = 42) -> np.ndarray:
    """sim::true_perf of every cell of the given rows of the joint matrix (len(rows) x n)."""
    rows = np.ascontiguousarray(rows, np.int64)
    cpu, gpu = grid.arrays()
    out = np.zeros((len(rows), grid.n))
    check(lib.ocg_synth_true_rows(m, ptr(cpu), len(cpu), ptr(gpu), len(gpu), seed, ptr(rows), len(rows), ptr(out)))
    return out


def make_suite(counts, seed: int, role: int, grid: PowerGrid, noise_sigma=0.01, cpu_phase_fraction=0.0):
    cnt = np.asarray(counts, np.int32)
    out = (WorkloadSpecC * int(cnt.sum()))()
    cpu, gpu = grid.arrays()
    check(lib.ocg_synth_suite(ptr(cnt), seed, role, noise_sigma, cpu_phase_fraction, ptr(cpu), len(cpu), ptr(gpu),
                              len(gpu), out))
    return out


lib.ocg_synth_counters.argtypes = [c_vp, c_i64, c_vp, c_i32, c_vp, c_i32, ctypes.c_int, ctypes.c_int, c_vp]
lib.ocg_synth_counters.restype = ctypes.c_int


def counters(specs, grid: PowerGrid, cpu_phase: bool = False, threads: int | None = None) -> np.ndarray:
    """sim::sample_counters of every spec at every setting: (len(specs) * grid.n, 7)."""
    threads = threads or max(1, min(64, os.cpu_count() or 1))
    arr = specs if isinstance(specs, ctypes.Array) else (WorkloadSpecC * len(specs))(*specs)
    cpu, gpu = grid.arrays()
    out = np.empty((len(arr) * grid.n, 7))
    check(lib.ocg_synth_counters(arr, len(arr), ptr(cpu), len(cpu), ptr(gpu), len(gpu), int(cpu_phase), threads,
                                 ptr(out)))
    return out


def true_perf(spec: WorkloadSpecC, cpu_cap: int, gpu_cap: int) -> float:
    return float(lib.ocg_true_perf(ctypes.byref(spec), cpu_cap, gpu_cap))


def offline_block(seed: int = 42, grid: PowerGrid | None = None) -> np.ndarray:
    grid = grid or PowerGrid.default_grid()
    cpu, gpu = grid.arrays()
    out = np.zeros((10, grid.n))
    rows = c_i64()
    check(lib.ocg_synth_offline_block(seed, ptr(cpu), len(cpu), ptr(gpu), len(gpu), ptr(out), ctypes.byref(rows)))
    return out[: rows.value]


def online_apps(napps: int, seed: int = 42, grid: PowerGrid | None = None):
    """(probe_vals, probe_mask, seeds) for napps eval-suite apps."""
    grid = grid or PowerGrid.default_grid()
    cpu, gpu = grid.arrays()
    pv = np.zeros((napps, grid.n))
    pm = np.zeros((napps, grid.n), np.uint8)
    sd = np.zeros(napps, np.uint64)
    check(lib.ocg_synth_online_apps(napps, seed, ptr(cpu), len(cpu), ptr(gpu), len(gpu), ptr(pv), ptr(pm), ptr(sd)))
    return pv, pm, sd


@dataclass
class CsrMatrix:
    m: int
    n: int
    row_ptr: np.ndarray  # int64 [m+1]
    col: np.ndarray      # int32 [nnz]
    val: np.ndarray      # float32 or float64 [nnz]

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])


lib.ocg_synth_csr_range_count.argtypes = [c_i64, c_i64, c_i64, c_vp, c_i32, c_vp, c_i32, c_dbl, c_i64, c_u64,
                                          ctypes.c_int, c_vp]
lib.ocg_synth_csr_range_count.restype = ctypes.c_int
lib.ocg_synth_csr_range_fill.argtypes = [c_i64, c_i64, c_i64, c_vp, c_i32, c_vp, c_i32, c_dbl, c_i64, c_u64,
                                         ctypes.c_int, c_vp, c_vp, c_vp, c_vp]
lib.ocg_synth_csr_range_fill.restype = ctypes.c_int


def joint_csr(m: int, grid: PowerGrid, density: float, dense_rows: int, seed: int = 42, dtype=np.float32,
              threads: int | None = None, rows: tuple | None = None) -> CsrMatrix:
    """SURVEY §8d synthetic joint matrix (C1: 10K x 256 @5%, C2: 1M x 4096 @2%, ...).
    rows=(r0, r1): only that row shard (local row_ptr), identical to the full matrix's rows."""
    threads = threads or max(1, min(64, os.cpu_count() or 1))
    r0, r1 = rows if rows is not None else (0, m)
    cpu, gpu = grid.arrays()
    rp = np.zeros(r1 - r0 + 1, np.int64)
    check(lib.ocg_synth_csr_range_count(m, r0, r1, ptr(cpu), len(cpu), ptr(gpu), len(gpu), density, dense_rows, seed,
                                        threads, ptr(rp)))
    nnz = int(rp[-1])
    col = np.empty(nnz, np.int32)
    v32 = np.empty(nnz, np.float32) if dtype == np.float32 else None
    v64 = np.empty(nnz, np.float64) if dtype == np.float64 else None
    check(lib.ocg_synth_csr_range_fill(m, r0, r1, ptr(cpu), len(cpu), ptr(gpu), len(gpu), density, dense_rows, seed,
                                       threads, ptr(rp), ptr(col), ptr(v32), ptr(v64)))
    return CsrMatrix(r1 - r0, grid.n, rp, col, v32 if v32 is not None else v64)
