"""ctypes binding of the in-tree C-ABI library ``libocg.so`` (include/ocg.h).

The library is the only compute path: importing this module fails loudly if it
is missing, and every compute entry point returns ``OCG_E_CUDA`` when no sm_100
device is usable — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("OCG_LIB", _HERE / "libocg.so"))

if not LIB_PATH.exists():
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make -C paper_2508_07605_b200/csrc` "
        "or `python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)"
    )

lib = ctypes.CDLL(str(LIB_PATH))

OCG_OK, OCG_E_INVALID, OCG_E_MISSING, OCG_E_LOGIC = 0, 1, 2, 3
OCG_E_RANGE, OCG_E_COLD, OCG_E_DIVERGE, OCG_E_CUDA, OCG_E_UNSUPPORTED = 4, 5, 6, 7, 8
LANE_SCALAR, LANE_AVX2 = 0, 1

c_i32, c_i64, c_u64, c_dbl, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p


class NcfHyperC(ctypes.Structure):
    """ocg_ncf_hyper == cf::NcfHyper (cfcomplete.hpp:11-20)."""

    _fields_ = [
        ("app_dim", c_i64),
        ("setting_dim", c_i64),
        ("hidden", c_i64 * 8),
        ("n_hidden", c_i64),
        ("lr", c_dbl),
        ("max_epochs", c_i32),
        ("patience", c_i32),
        ("val_fraction", c_dbl),
        ("batch_size", c_i32),
    ]


class NcfMetaC(ctypes.Structure):
    """ocg_ncf_meta == NcfModel::Meta (cfcomplete.hpp:34-40)."""

    _fields_ = [
        ("seed", c_u64),
        ("epochs_run", c_i32),
        ("initial_train_mse", c_dbl),
        ("final_train_mse", c_dbl),
        ("best_val_mse", c_dbl),
    ]


def _sig(name, restype, *argtypes):
    fn = getattr(lib, name)
    fn.restype = restype
    fn.argtypes = list(argtypes)
    return fn


_sig("ocg_last_error", ctypes.c_char_p)
_sig("ocg_version", ctypes.c_int)
_sig("ocg_ncf_hyper_default", None, c_vp)
_sig("ocg_derive_seed", c_u64, c_u64, ctypes.c_char_p, c_u64)
_sig("ocg_ctx_create", ctypes.c_int, ctypes.c_int, ctypes.POINTER(c_vp))
_sig("ocg_ctx_destroy", None, c_vp)
_sig("ocg_ctx_device_info", ctypes.c_int, c_vp, c_vp, c_vp, c_vp)
_sig("ocg_select_caps", ctypes.c_int, c_vp, c_vp, c_i64, c_vp, c_i32, c_vp, c_i32, c_dbl, c_vp, c_vp, c_vp, c_vp)
_sig("ocg_select_caps_dev", ctypes.c_int, c_vp, c_vp, ctypes.c_int, c_i64, c_vp, c_i32, c_vp, c_i32, c_dbl,
     c_vp, c_vp, c_vp, c_vp)
_sig("ocg_default_plan", ctypes.c_int, c_vp, c_i32, c_vp, c_i32, c_vp, c_vp)
_sig("ocg_online_complete_batch", ctypes.c_int, c_vp, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_i32,
     c_vp, c_i32, c_vp, c_dbl, ctypes.c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp)
_sig("ocg_online_fit_batch_params", ctypes.c_int, c_vp, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_i32, c_vp,
     ctypes.c_int, c_vp, c_i64, c_vp, c_vp)
_sig("ocg_ncf_model_to_json", ctypes.c_int, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, ctypes.c_char_p,
     ctypes.c_size_t, c_vp)
_sig("ocg_ncf_model_from_json", ctypes.c_int, ctypes.c_char_p, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp)
_sig("ocg_ncf_predict", ctypes.c_int, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64,
     ctypes.c_int, c_vp)
_sig("ocg_debug_exp", ctypes.c_int, c_vp, c_vp, c_i64, c_vp)
_sig("ocg_debug_exp_host", c_dbl, c_dbl)
_sig("ocg_debug_rng", ctypes.c_int, c_vp, c_u64, c_i64, c_vp)


class OcgError(RuntimeError):
    """Raised for a non-zero ocg return code; ``code`` is the OCG_E_* value."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[ocg code {code}] {msg}")
        self.code = code


# reference exception types each return code stands for (ocg.h)
class InvalidArgument(OcgError, ValueError):
    pass


class OutOfRange(OcgError, IndexError):
    pass


class ColdError(OcgError):
    pass


class DivergenceError(OcgError):
    pass


class CudaError(OcgError):
    pass


class MissingArtifact(OcgError, FileNotFoundError):
    pass


_EXC = {OCG_E_INVALID: InvalidArgument, OCG_E_MISSING: MissingArtifact, OCG_E_RANGE: OutOfRange, OCG_E_COLD: ColdError,
        OCG_E_DIVERGE: DivergenceError, OCG_E_CUDA: CudaError}


def check(rc: int) -> None:
    if rc != OCG_OK:
        msg = (lib.ocg_last_error() or b"").decode(errors="replace")
        raise _EXC.get(rc, OcgError)(rc, msg)


def ptr(a):
    """Data pointer of a numpy array (or None)."""
    return None if a is None else ctypes.c_void_p(a.ctypes.data)

_sig("ocg_ctx_flush_l2", ctypes.c_int, c_vp)
_sig("ocg_ctx_synchronize", ctypes.c_int, c_vp)
_sig("ocg_online_plan_create", ctypes.c_int, c_vp, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_i32, c_vp,
     c_i32, c_vp, c_dbl, ctypes.c_int, ctypes.c_int, ctypes.POINTER(c_vp))
_sig("ocg_online_plan_run", ctypes.c_int, c_vp, ctypes.POINTER(ctypes.c_float))
_sig("ocg_online_plan_results", ctypes.c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp)
_sig("ocg_online_plan_destroy", None, c_vp)


class AlsHyperC(ctypes.Structure):
    """ocg_als_hyper."""

    _fields_ = [("rank", c_i32), ("lambda_", ctypes.c_float), ("sweeps", c_i32), ("seed", c_u64)]


_sig("ocg_als_plan_create", ctypes.c_int, c_vp, c_i64, c_vp, c_vp, c_vp, ctypes.c_int, c_vp, c_i32, c_vp, c_i32,
     c_vp, c_dbl, ctypes.POINTER(c_vp))
_sig("ocg_als_plan_run", ctypes.c_int, c_vp, c_vp, c_vp)
_sig("ocg_als_plan_upload", ctypes.c_int, c_vp, c_vp, c_vp, c_vp)
_sig("ocg_als_plan_upload_compact", ctypes.c_int, c_vp, c_vp, c_vp, c_vp)
_sig("ocg_als_plan_set_warm", ctypes.c_int, c_vp, ctypes.c_int32)
_sig("ocg_als_plan_add_observations", ctypes.c_int, c_vp, ctypes.c_int64, c_vp, c_vp, c_vp)
_sig("ocg_als_plan_stage_compact", ctypes.c_int, c_vp, c_vp, c_vp, c_vp)
_sig("ocg_als_plan_results_async", ctypes.c_int, c_vp, c_vp, c_vp, c_vp, c_vp)
_sig("ocg_als_plan_results_wait", ctypes.c_int, c_vp)
_sig("ocg_als_plan_results", ctypes.c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp)
_sig("ocg_als_plan_completed_rows", ctypes.c_int, c_vp, c_i64, c_i64, c_vp)
_sig("ocg_als_plan_destroy", None, c_vp)

_sig("ocg_ctx_set_stream", ctypes.c_int, c_vp, c_vp)
_sig("ocg_als_plan_begin", ctypes.c_int, c_vp)
_sig("ocg_als_plan_row_half", ctypes.c_int, c_vp)
_sig("ocg_als_plan_col_half", ctypes.c_int, c_vp)
_sig("ocg_als_plan_gram_floats", c_i64, c_vp)
_sig("ocg_als_plan_col_gram", ctypes.c_int, c_vp, c_vp)
_sig("ocg_als_plan_col_solve", ctypes.c_int, c_vp, c_vp)
_sig("ocg_als_plan_select", ctypes.c_int, c_vp)

_sig("ocg_predictor_create", ctypes.c_int, c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, ctypes.c_int,
     ctypes.POINTER(c_vp))
_sig("ocg_predictor_run", ctypes.c_int, c_vp, c_vp, c_i64, ctypes.c_int, c_vp, ctypes.c_uint32)
_sig("ocg_predictor_destroy", ctypes.c_int, c_vp)
OCG_PRED_DEVICE_PTRS, OCG_PRED_GENERIC = 1, 2
_sig("ocg_predict_perf_batch", ctypes.c_int, c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, ctypes.c_int, c_vp, c_i64,
     ctypes.c_int, c_vp)

# fused NCF completion + selection over a whole matrix (ocg_ncf_model_* / ocg_ncf_plan_*)
OCG_NCF_EXACT, OCG_NCF_FAST = 0, 1
_sig("ocg_ncf_model_create", ctypes.c_int, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, ctypes.POINTER(c_vp))
_sig("ocg_ncf_model_from_json_text", ctypes.c_int, c_vp, ctypes.c_char_p, ctypes.POINTER(c_vp))
_sig("ocg_ncf_model_destroy", None, c_vp)
_sig("ocg_ncf_plan_create", ctypes.c_int, c_vp, c_vp, c_vp, c_vp, ctypes.c_int, c_vp, c_i32, c_vp, c_i32, c_dbl,
     ctypes.c_int, ctypes.c_int, ctypes.POINTER(c_vp))
_sig("ocg_ncf_plan_upload", ctypes.c_int, c_vp, c_vp, c_vp, c_vp)
_sig("ocg_ncf_plan_run", ctypes.c_int, c_vp, c_vp, c_vp)
_sig("ocg_ncf_plan_results", ctypes.c_int, c_vp, c_vp, c_vp, c_vp, c_vp)
_sig("ocg_ncf_plan_completed_rows", ctypes.c_int, c_vp, c_vp, c_i64, c_vp)
_sig("ocg_ncf_plan_destroy", None, c_vp)

# cf:: over one whole matrix, every solver (ocg_cf_fit / ocg_cf_complete)
OCG_SOLVER_NCF_REF, OCG_SOLVER_NCF_FAST, OCG_SOLVER_ALS = 0, 1, 2
_sig("ocg_cf_fit", ctypes.c_int, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_u64, ctypes.c_int, ctypes.c_int, c_vp,
     c_vp, c_vp, c_vp)
_sig("ocg_cf_fit_stats", ctypes.c_int, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_u64, ctypes.c_int, ctypes.c_int,
     c_vp, c_vp, c_vp, c_vp, c_vp, c_vp)
_sig("ocg_cf_complete", ctypes.c_int, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_u64, ctypes.c_int,
     ctypes.c_int, c_vp, c_i32, c_vp, c_i32, c_dbl, c_vp, c_vp, c_vp, c_vp, c_vp)

# file formats (host only): matrix CSV / binary CSR, predictor model file
_sig("ocg_matrix_read_csv", ctypes.c_int, ctypes.c_char_p, ctypes.POINTER(c_vp))
_sig("ocg_matrix_write_csv", ctypes.c_int, c_vp, ctypes.c_char_p)
_sig("ocg_matrix_create", ctypes.c_int, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, ctypes.POINTER(c_vp))
_sig("ocg_matrix_shape", ctypes.c_int, c_vp, c_vp, c_vp, c_vp)
_sig("ocg_matrix_get", ctypes.c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp)
_sig("ocg_matrix_app_id", ctypes.c_char_p, c_vp, c_i64)
_sig("ocg_matrix_save_bin", ctypes.c_int, c_vp, ctypes.c_char_p)
_sig("ocg_matrix_load_bin", ctypes.c_int, ctypes.c_char_p, ctypes.POINTER(c_vp))
_sig("ocg_matrix_destroy", None, c_vp)
_sig("ocg_predictor_parse", ctypes.c_int, ctypes.c_char_p, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp)
_sig("ocg_predictor_from_json", ctypes.c_int, c_vp, ctypes.c_char_p, ctypes.POINTER(c_vp))
_sig("ocg_predictor_load", ctypes.c_int, c_vp, ctypes.c_char_p, ctypes.POINTER(c_vp))

# batched online-phase streams: phase detector, probe ingest wired into the per-app completion
class DetectorConfigC(ctypes.Structure):
    """ocg_detector_config == phase::DetectorConfig (phasedet.hpp:13-20)."""

    _fields_ = [("delta_s", c_dbl), ("window_s", c_dbl), ("p_th_w", c_dbl)]


_sig("ocg_phase_detect_batch", ctypes.c_int, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, ctypes.c_int, c_vp, c_vp)
_sig("ocg_online_ingest_complete_batch", ctypes.c_int, c_vp, c_i64, c_vp, c_vp, c_i64, c_vp, c_i32, c_vp, c_vp, c_vp,
     c_vp, c_vp, c_vp, c_i32, c_vp, c_i32, c_vp, c_dbl, ctypes.c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp)
_sig("ocg_ncf_plan_stage", ctypes.c_int, c_vp, c_vp, c_vp, c_vp)
_sig("ocg_ncf_plan_results_async", ctypes.c_int, c_vp, c_vp, c_vp, c_vp, c_vp)
_sig("ocg_ncf_plan_results_wait", ctypes.c_int, c_vp)

# evaluation harness: policy::evaluate_suite's truth tables, exhaustive choices and aggregates
class RunResultC(ctypes.Structure):
    _fields_ = [("runtime_s", c_dbl), ("energy_j", c_dbl), ("avg_power_w", c_dbl)]


class EvalRowC(ctypes.Structure):
    _fields_ = [("policy", c_i32), ("setting", c_i32), ("cpu_cap_w", c_i32), ("gpu_cap_w", c_i32), ("gamma", c_dbl),
                ("true_perf", c_dbl), ("true_loss", c_dbl), ("energy_j", c_dbl), ("avg_power_w", c_dbl),
                ("efficiency", c_dbl), ("pred_saving", c_dbl)]


class EvalAggregateC(ctypes.Structure):
    _fields_ = [("policy", c_i32), ("mean_efficiency", c_dbl), ("mean_gain_vs_no_cap", c_dbl),
                ("mean_true_loss", c_dbl), ("mean_true_perf", c_dbl)]


_sig("ocg_eval_suite", ctypes.c_int, c_vp, c_i64, c_vp, c_i32, c_vp, c_i32, c_i32, c_vp, c_vp, c_dbl, c_i32, c_vp,
     c_vp, c_vp, c_vp, c_vp)
