"""File formats of the online phase's inputs (include/ocg.h "file formats").

* ``Matrix.read_csv`` / ``write_csv``: the reference's matrix CSV
  (read_matrix_csv_file / write_matrix_csv, core.cpp:191-254), byte-identical
  output, the reference's checks and exception kinds;
* ``Matrix.save_bin`` / ``load_bin``: the same matrix as a binary CSR;
* ``load_predictor``: pred::load_predictor (predictor.cpp:325-331) into a
  device-resident ``Predictor``.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from ._lib import check, lib, ptr


@dataclass
class Matrix:
    """PerformanceMatrix as CSR: app ids, per-column (cpu, gpu) settings, observed cells."""

    app_ids: list
    cpu: np.ndarray  # int32 [n]
    gpu: np.ndarray  # int32 [n]
    row_ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray

    @property
    def m(self) -> int:
        return len(self.app_ids)

    @property
    def n(self) -> int:
        return len(self.cpu)

    @staticmethod
    def _from_handle(h) -> "Matrix":
        m, n, nnz = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        try:
            check(lib.ocg_matrix_shape(h, ctypes.byref(m), ctypes.byref(n), ctypes.byref(nnz)))
            cpu, gpu = np.zeros(n.value, np.int32), np.zeros(n.value, np.int32)
            rp = np.zeros(m.value + 1, np.int64)
            col, val = np.zeros(nnz.value, np.int32), np.zeros(nnz.value)
            check(lib.ocg_matrix_get(h, ptr(cpu), ptr(gpu), ptr(rp), ptr(col), ptr(val)))
            ids = [lib.ocg_matrix_app_id(h, i).decode() for i in range(m.value)]
        finally:
            lib.ocg_matrix_destroy(h)
        return Matrix(ids, cpu, gpu, rp, col, val)

    def _handle(self):
        ids = (ctypes.c_char_p * self.m)(*[a.encode() for a in self.app_ids])
        cpu, gpu = np.ascontiguousarray(self.cpu, np.int32), np.ascontiguousarray(self.gpu, np.int32)
        rp = np.ascontiguousarray(self.row_ptr, np.int64)
        col, val = np.ascontiguousarray(self.col, np.int32), np.ascontiguousarray(self.val, np.float64)
        h = ctypes.c_void_p()
        check(lib.ocg_matrix_create(self.m, self.n, ctypes.cast(ids, ctypes.c_void_p), ptr(cpu), ptr(gpu), ptr(rp),
                                    ptr(col), ptr(val), ctypes.byref(h)))
        return h

    @staticmethod
    def read_csv(path) -> "Matrix":
        h = ctypes.c_void_p()
        check(lib.ocg_matrix_read_csv(str(path).encode(), ctypes.byref(h)))
        return Matrix._from_handle(h)

    @staticmethod
    def load_bin(path) -> "Matrix":
        h = ctypes.c_void_p()
        check(lib.ocg_matrix_load_bin(str(path).encode(), ctypes.byref(h)))
        return Matrix._from_handle(h)

    def write_csv(self, path) -> None:
        h = self._handle()
        try:
            check(lib.ocg_matrix_write_csv(h, str(path).encode()))
        finally:
            lib.ocg_matrix_destroy(h)

    def save_bin(self, path) -> None:
        h = self._handle()
        try:
            check(lib.ocg_matrix_save_bin(h, str(path).encode()))
        finally:
            lib.ocg_matrix_destroy(h)

    def dense(self):
        vals = np.zeros((self.m, self.n))
        mask = np.zeros((self.m, self.n), np.uint8)
        rows = np.repeat(np.arange(self.m), np.diff(self.row_ptr))
        vals[rows, self.col] = self.val
        mask[rows, self.col] = 1
        return vals, mask


def parse_predictor(text: str):
    """pred::predictor_from_json's checks, in C++: (dims, acts, params, mean, std, has_stats)."""
    raw = text.encode()
    nl, npar = ctypes.c_int32(), ctypes.c_int64()
    check(lib.ocg_predictor_parse(raw, ctypes.byref(nl), None, None, None, ctypes.byref(npar), None, None, None))
    dims, acts = np.zeros(nl.value + 1, np.int64), np.zeros(nl.value, np.int32)
    params, mean, std = np.zeros(npar.value), np.zeros(7), np.zeros(7)
    hs = ctypes.c_int()
    check(lib.ocg_predictor_parse(raw, ctypes.byref(nl), ptr(dims), ptr(acts), ptr(params), ctypes.byref(npar),
                                  ptr(mean), ptr(std), ctypes.byref(hs)))
    return dims, acts, params, mean, std, bool(hs.value)
