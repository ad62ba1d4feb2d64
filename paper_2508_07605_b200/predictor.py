"""Probe ingest: pred::predict_perf (predictor.cpp:151-157) batched on the GPU.

PredictorModel reads the reference's own predictor model file (nnkit model
JSON + feature_stats, predictor.cpp:292-316)."""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from ._lib import OCG_PRED_DEVICE_PTRS, OCG_PRED_GENERIC, check, lib, ptr
from .api import LANE_AVX2, Context, default_context

_ACT = {"selu": 0, "relu": 1, "identity": 2}


@dataclass
class PredictorModel:
    dims: list
    acts: list
    params: np.ndarray  # per layer W (out x in row-major) then b
    mean: np.ndarray
    std: np.ndarray
    has_stats: bool

    @staticmethod
    def from_json(text: str) -> "PredictorModel":
        """pred::predictor_from_json (predictor.cpp:302-316) / nn::model_from_json (nnkit.cpp:332-365),
        with the reference's shape / finiteness / activation checks (parsed in C++, formats.cpp)."""
        from .formats import parse_predictor

        dims, acts, params, mean, std, has_stats = parse_predictor(text)
        return PredictorModel([int(d) for d in dims], [int(a) for a in acts], params, mean, std, has_stats)

    @staticmethod
    def load(path) -> "PredictorModel":
        """pred::load_predictor (predictor.cpp:325-331): OCG_E_MISSING if the file is absent."""
        from pathlib import Path

        from ._lib import MissingArtifact, OCG_E_MISSING

        p = Path(path)
        if not p.is_file():
            raise MissingArtifact(OCG_E_MISSING, f"missing predictor model: {path}")
        return PredictorModel.from_json(p.read_text())


def predict_perf_batch(model: PredictorModel, counters, lane: int = LANE_AVX2,
                       ctx: Context | None = None) -> np.ndarray:
    """Normalized-performance estimates for counter samples (count x 7, CounterSample field order)."""
    ctx = ctx or default_context()
    c = np.ascontiguousarray(counters, np.float64).reshape(-1, 7)
    dims = np.asarray(model.dims, np.int64)
    acts = np.asarray(model.acts, np.int32)
    out = np.zeros(len(c))
    check(lib.ocg_predict_perf_batch(ctx.handle, len(acts), ptr(dims), ptr(acts), ptr(model.params), ptr(model.mean),
                                     ptr(model.std), 1 if model.has_stats else 0, ptr(c), len(c), lane, ptr(out)))
    return out


class Predictor:
    """A PredictorModel resident on the context's device (ocg_predictor_*)."""

    def __init__(self, model: PredictorModel, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        self.model = model
        dims = np.asarray(model.dims, np.int64)
        acts = np.asarray(model.acts, np.int32)
        h = ctypes.c_void_p()
        check(lib.ocg_predictor_create(self.ctx.handle, len(acts), ptr(dims), ptr(acts), ptr(model.params),
                                       ptr(model.mean), ptr(model.std), 1 if model.has_stats else 0,
                                       ctypes.byref(h)))
        self.handle = h

    def __call__(self, counters, lane: int = LANE_AVX2, generic: bool = False) -> np.ndarray:
        c = np.ascontiguousarray(counters, np.float64).reshape(-1, 7)
        out = np.zeros(len(c))
        check(lib.ocg_predictor_run(self.handle, ptr(c), len(c), lane, ptr(out), OCG_PRED_GENERIC if generic else 0))
        return out

    def run_device(self, counters_ptr: int, count: int, out_ptr: int, lane: int = LANE_AVX2,
                   generic: bool = False) -> None:
        """counters/out: device addresses (e.g. torch tensor data_ptr()) on the context's device."""
        flags = OCG_PRED_DEVICE_PTRS | (OCG_PRED_GENERIC if generic else 0)
        check(lib.ocg_predictor_run(self.handle, ctypes.c_void_p(counters_ptr), count, lane, ctypes.c_void_p(out_ptr),
                                    flags))

    def close(self):
        if self.handle:
            lib.ocg_predictor_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
