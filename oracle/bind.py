"""TEST INFRASTRUCTURE ONLY: ctypes bindings of the CPU oracle.

* ``Port``  — our plain-C restatement (oracle/_build/libocg_oracle.so)
* ``Ref``   — the reference library itself compiled from /root/reference
              (oracle/_ref/libopencap_ref.so, built by `make -C oracle ref`)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
leg may import this module, and only as the checker / CPU baseline.
"""
from __future__ import annotations

import ctypes
import json
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_LIB = HERE / "_build" / "libocg_oracle.so"
REF_LIB = HERE / "_ref" / "libopencap_ref.so"
REFERENCE_SRC = Path("/root/reference/proj/src")

c_i32, c_i64, c_u64, c_dbl, c_vp, c_sz = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double,
                                          ctypes.c_void_p, ctypes.c_size_t)


def P(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


class Hyper(ctypes.Structure):
    _fields_ = [("app_dim", c_i64), ("setting_dim", c_i64), ("hidden", c_i64 * 8), ("n_hidden", c_i64),
                ("lr", c_dbl), ("max_epochs", c_i32), ("patience", c_i32), ("val_fraction", c_dbl),
                ("batch_size", c_i32)]


class RefHyper(ctypes.Structure):
    _fields_ = [("app_dim", c_u64), ("setting_dim", c_u64), ("hidden", c_u64 * 8), ("n_hidden", c_u64),
                ("lr", c_dbl), ("max_epochs", c_i32), ("patience", c_i32), ("val_fraction", c_dbl),
                ("batch_size", c_i32)]


class Meta(ctypes.Structure):
    _fields_ = [("seed", c_u64), ("epochs_run", c_i32), ("initial_train_mse", c_dbl),
                ("final_train_mse", c_dbl), ("best_val_mse", c_dbl)]


class RefSpec(ctypes.Structure):
    _fields_ = [("archetype", c_i32), ("kappa_c", c_dbl), ("alpha_c", c_dbl), ("kappa_g", c_dbl),
                ("alpha_g", c_dbl), ("base_runtime_s", c_dbl), ("cpu_phase_s", c_dbl), ("noise_sigma", c_dbl),
                ("ips_max", c_dbl), ("mem_tput_max", c_dbl), ("sm_clock_max", c_dbl)]


class RefOnlineOut(ctypes.Structure):
    _fields_ = [("setting_idx", c_i32), ("pred_saving", c_dbl), ("pred_loss", c_dbl), ("candidates", c_i32),
                ("transition", c_i32), ("n_probes", c_i32), ("probe_idx", c_i32 * 64),
                ("probe_val", c_dbl * 64), ("completed_row", c_dbl * 4096)]


def _hyper(cls, app_dim=8, setting_dim=8, hidden=(32, 16), lr=1e-3, max_epochs=2000, patience=100,
           val_fraction=0.1, batch_size=32):
    h = cls()
    h.app_dim, h.setting_dim = app_dim, setting_dim
    for i, w in enumerate(hidden):
        h.hidden[i] = w
    h.n_hidden = len(hidden)
    h.lr, h.max_epochs, h.patience, h.val_fraction, h.batch_size = lr, max_epochs, patience, val_fraction, batch_size
    return h


def build(ref: bool = True) -> None:
    """Compile the port (always) and the reference library (when its sources exist)."""
    subprocess.run(["make", "-s", "-C", str(HERE), "port"], check=True)
    if ref and REFERENCE_SRC.exists():
        subprocess.run(["make", "-s", "-j8", "-C", str(HERE), "ref"], check=True)


def csr_of(values, mask):
    """Row-major CSR (row_ptr i64, col i32, val f64) of a dense masked matrix."""
    m, n = mask.shape
    rp = np.zeros(m + 1, np.int64)
    rp[1:] = np.cumsum(mask.sum(axis=1))
    ii, jj = np.nonzero(mask)
    return rp, jj.astype(np.int32), np.ascontiguousarray(values[ii, jj], np.float64)


class Port:
    """Our C restatement (scalar-lane FP order)."""

    def __init__(self, path=PORT_LIB):
        L = self.L = ctypes.CDLL(str(path))
        L.ocgo_last_error.restype = ctypes.c_char_p
        L.ocgo_derive_seed.restype = c_u64
        L.ocgo_derive_seed.argtypes = [c_u64, ctypes.c_char_p, c_u64]
        L.ocgo_rng_u64.argtypes = [c_u64, c_vp, c_sz]
        L.ocgo_rng_uniform.argtypes = [c_u64, c_dbl, c_dbl, c_vp, c_sz]
        L.ocgo_select_caps.argtypes = [c_vp, c_i64, c_vp, c_i32, c_vp, c_i32, c_dbl, c_vp, c_vp, c_vp, c_vp]
        L.ocgo_default_plan.argtypes = [c_vp, c_i32, c_vp, c_i32, c_vp, c_vp]
        L.ocgo_ncf_param_count.restype = c_i64
        L.ocgo_ncf_param_count.argtypes = [c_i64, c_i64, c_vp]
        L.ocgo_ncf_fit.argtypes = [c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_u64, c_vp, c_vp, c_vp, c_vp]
        L.ocgo_ncf_predict.argtypes = [c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp]
        L.ocgo_set_lane.argtypes = [ctypes.c_int]
        L.ocgo_als_fit.argtypes = [c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_dbl, c_i32, c_u64, c_vp,
                                   c_vp]
        L.ocgo_als_solve_rows.argtypes = [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_dbl]
        L.ocgo_als_col_gram.argtypes = [c_i64, c_vp, c_vp, c_vp, c_vp, c_i32, c_vp]
        L.ocgo_als_solve_from_gram.argtypes = [c_i64, c_vp, c_vp, c_i32, c_dbl]
        L.ocgo_als_init_value.restype = c_dbl
        L.ocgo_als_init_value.argtypes = [c_u64, c_i64, c_i32, c_i32]

    def set_lane(self, lane):
        """0: reference scalar lane FP order, 1: AVX2/FMA lane."""
        self.L.ocgo_set_lane(lane)

    def err(self):
        return self.L.ocgo_last_error().decode()

    def derive_seed(self, root, tag, n=0):
        return int(self.L.ocgo_derive_seed(root, tag.encode(), n))

    def rng_u64(self, seed, n):
        out = np.zeros(n, np.uint64)
        self.L.ocgo_rng_u64(seed, P(out), n)
        return out

    def select_caps(self, rows, cpu, gpu, gamma):
        rows = np.ascontiguousarray(rows, np.float64)
        r = rows.shape[0]
        cpu, gpu = np.asarray(cpu, np.int32), np.asarray(gpu, np.int32)
        idx, nc = np.zeros(r, np.int32), np.zeros(r, np.int32)
        sv, lo = np.zeros(r), np.zeros(r)
        rc = self.L.ocgo_select_caps(P(rows), r, P(cpu), len(cpu), P(gpu), len(gpu), gamma, P(idx), P(sv), P(lo),
                                     P(nc))
        return rc, idx, sv, lo, nc

    def default_plan(self, cpu, gpu):
        cpu, gpu = np.asarray(cpu, np.int32), np.asarray(gpu, np.int32)
        out = np.zeros(6, np.int32)
        cnt = c_i32()
        self.L.ocgo_default_plan(P(cpu), len(cpu), P(gpu), len(gpu), P(out), ctypes.byref(cnt))
        return out[: cnt.value].tolist()

    def ncf_fit(self, values, mask, seed, **hyper):
        m, n = mask.shape
        rp, col, val = csr_of(values, mask)
        h = _hyper(Hyper, **hyper)
        T = self.L.ocgo_ncf_param_count(m, n, ctypes.byref(h))
        p = np.zeros(T)
        meta = Meta()
        aseen, sseen = np.zeros(m, np.uint8), np.zeros(n, np.uint8)
        rc = self.L.ocgo_ncf_fit(m, n, P(rp), P(col), P(val), ctypes.byref(h), seed, P(p), ctypes.byref(meta),
                                 P(aseen), P(sseen))
        return rc, p, meta, aseen, sseen

    def ncf_predict(self, m, n, params, aseen, sseen, rows, cols, **hyper):
        h = _hyper(Hyper, **hyper)
        rows, cols = np.ascontiguousarray(rows, np.int64), np.ascontiguousarray(cols, np.int64)
        out = np.zeros(len(rows))
        rc = self.L.ocgo_ncf_predict(m, n, ctypes.byref(h), P(params), P(aseen), P(sseen), P(rows), P(cols),
                                     len(rows), P(out))
        return rc, out


def csc_of(m, n, row_ptr, col, val):
    """Stable CSC mirror (rows ascending inside a column) of a CSR matrix."""
    rows = np.repeat(np.arange(m, dtype=np.int32), np.diff(row_ptr))
    order = np.argsort(col, kind="stable")
    cp = np.zeros(n + 1, np.int64)
    cp[1:] = np.cumsum(np.bincount(col, minlength=n))
    return cp, rows[order].astype(np.int32), np.ascontiguousarray(val[order], np.float32)


def als_fit(port, m, n, row_ptr, col, val, k, lam, sweeps, seed):
    """FP64 ALS oracle (no reference counterpart)."""
    val = np.ascontiguousarray(val, np.float32)
    cp, crow, cval = csc_of(m, n, row_ptr, col, val)
    U, V = np.zeros((m, k)), np.zeros((n, k))
    rc = port.L.ocgo_als_fit(m, n, P(row_ptr), P(col), P(val), P(cp), P(crow), P(cval), k, lam, sweeps, seed,
                             P(U), P(V))
    assert rc == 0, port.err()
    return U, V


def als_completed_rows(U, V, row_ptr, col, val, rows):
    """oracle completed rows: observed verbatim (FP32 value widened), else clamp(u.v)."""
    out = np.clip(U[rows] @ V.T, 0.01, 1.25)
    for r, i in enumerate(rows):
        s, e = row_ptr[i], row_ptr[i + 1]
        out[r, col[s:e]] = val[s:e].astype(np.float64)
    return out


class Ref:
    """The reference library itself (compiled from /root/reference)."""

    def __init__(self, path=REF_LIB):
        L = self.L = ctypes.CDLL(str(path))
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_derive_seed.restype = c_u64
        L.ref_derive_seed.argtypes = [c_u64, ctypes.c_char_p, c_u64]
        L.ref_rng_u64.argtypes = [c_u64, c_vp, c_sz]
        L.ref_rng_uniform.argtypes = [c_u64, c_dbl, c_dbl, c_vp, c_sz]
        L.ref_select_caps.argtypes = [c_vp, c_sz, c_vp, c_sz, c_vp, c_sz, c_dbl, c_vp, c_vp, c_vp, c_vp]
        L.ref_default_plan.argtypes = [c_vp, c_sz, c_vp, c_sz, c_vp, c_vp]
        L.ref_ncf_fit.argtypes = [c_sz, c_vp, c_sz, c_vp, c_sz, c_vp, c_vp, c_vp, c_u64, ctypes.c_char_p, c_sz, c_vp,
                                  c_vp]
        L.ref_ncf_complete.argtypes = [c_sz, c_vp, c_sz, c_vp, c_sz, c_vp, c_vp, c_vp, c_u64, c_vp]
        L.ref_ncf_predict.argtypes = [ctypes.c_char_p, c_vp, c_vp, c_sz, c_vp]
        L.ref_predict_perf.argtypes = [ctypes.c_char_p, c_vp, c_sz, c_vp]
        L.ref_predict_perf_mt.argtypes = [ctypes.c_char_p, c_vp, c_sz, ctypes.c_int, c_vp]
        L.ref_predict_perf_mt.restype = c_dbl
        L.ref_make_suite.argtypes = [c_i32, c_i32, c_i32, c_i32, c_u64, c_dbl, c_i32, c_dbl, c_vp, c_sz, c_vp, c_sz,
                                     c_vp]
        L.ref_true_perf.restype = c_dbl
        L.ref_true_perf.argtypes = [c_vp, ctypes.c_int, ctypes.c_int]
        L.ref_sample_counters.argtypes = [c_vp, ctypes.c_int, ctypes.c_int, c_vp]
        L.ref_offline_default.argtypes = [c_u64, c_vp, c_vp, ctypes.c_char_p, c_sz, c_vp]
        L.ref_online_default.argtypes = [c_u64, ctypes.c_int, c_vp, c_sz, ctypes.c_char_p, c_vp]
        L.ref_online_batch.restype = c_dbl
        L.ref_online_batch.argtypes = [c_sz, c_vp, c_sz, c_vp, c_sz, c_vp, c_vp, c_vp, c_vp, c_sz, c_dbl, c_vp,
                                       ctypes.c_int, c_vp, c_vp]
        L.ref_force_lane.argtypes = [ctypes.c_int]
        L.ref_ncf_complete_select_rows.argtypes = [c_sz, c_sz, c_vp, c_sz, c_sz, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp,
                                                   c_sz, c_vp, c_vp, c_dbl, ctypes.c_int, c_vp, c_vp, c_vp, c_vp,
                                                   c_vp, c_vp]
        L.ref_joint_rows_dense.argtypes = [c_i64, c_vp, c_sz, c_vp, c_sz, c_dbl, c_i64, c_u64, c_vp, c_i64,
                                           ctypes.c_int, c_vp, c_vp]
        L.ref_matrix_csv_roundtrip.argtypes = [ctypes.c_char_p, ctypes.c_char_p, c_vp, c_vp, c_vp]
        L.ref_load_predictor.argtypes = [ctypes.c_char_p, c_vp]
        L.ref_run_trace.argtypes = [c_vp, ctypes.c_int, ctypes.c_int, c_u64, c_vp, c_sz, c_vp, c_vp]
        L.ref_detect.argtypes = [c_vp, c_sz, c_dbl, c_dbl, c_dbl, ctypes.c_int, c_vp]
        L.ref_eval_default.argtypes = [c_u64, ctypes.c_int, c_dbl, c_vp, c_sz, c_vp, c_vp, c_vp, c_vp, c_vp]
        L.ref_time_fit_step.argtypes = [c_sz, c_sz, c_sz, c_vp, c_sz, ctypes.c_int, c_vp]
        L.ref_time_fit_step.restype = c_dbl
        L.ref_complete_select_batch.restype = c_dbl
        L.ref_complete_select_batch.argtypes = [c_sz, c_sz, c_vp, c_sz, c_vp, c_sz, c_vp, c_vp, c_vp, c_vp, c_dbl,
                                                ctypes.c_int, c_vp]

    def err(self):
        return self.L.ref_last_error().decode()

    def force_lane(self, lane):
        assert self.L.ref_force_lane(lane) == 0

    def derive_seed(self, root, tag, n=0):
        return int(self.L.ref_derive_seed(root, tag.encode(), n))

    def rng_u64(self, seed, n):
        out = np.zeros(n, np.uint64)
        self.L.ref_rng_u64(seed, P(out), n)
        return out

    def select_caps(self, rows, cpu, gpu, gamma):
        rows = np.ascontiguousarray(rows, np.float64)
        r = rows.shape[0]
        cpu, gpu = np.asarray(cpu, np.int32), np.asarray(gpu, np.int32)
        idx, nc = np.zeros(r, np.int32), np.zeros(r, np.int32)
        sv, lo = np.zeros(r), np.zeros(r)
        rc = self.L.ref_select_caps(P(rows), r, P(cpu), len(cpu), P(gpu), len(gpu), gamma, P(idx), P(sv), P(lo),
                                    P(nc))
        return rc, idx, sv, lo, nc

    def default_plan(self, cpu, gpu):
        cpu, gpu = np.asarray(cpu, np.int32), np.asarray(gpu, np.int32)
        out = np.zeros(6, np.int32)
        cnt = c_sz()
        self.L.ref_default_plan(P(cpu), len(cpu), P(gpu), len(gpu), P(out), ctypes.byref(cnt))
        return out[: cnt.value].tolist()

    def ncf_fit(self, values, mask, cpu, gpu, seed, **hyper):
        m = mask.shape[0]
        cpu, gpu = np.asarray(cpu, np.int32), np.asarray(gpu, np.int32)
        values = np.ascontiguousarray(values, np.float64)
        mask = np.ascontiguousarray(mask, np.uint8)
        h = _hyper(RefHyper, **hyper)
        cap = 1 << 26
        buf = ctypes.create_string_buffer(cap)
        ln = c_sz()
        meta = Meta()
        rc = self.L.ref_ncf_fit(m, P(cpu), len(cpu), P(gpu), len(gpu), P(values), P(mask), ctypes.byref(h), seed, buf,
                                cap, ctypes.byref(ln), ctypes.byref(meta))
        return rc, (buf.value.decode() if rc == 0 else None), meta

    def ncf_complete(self, values, mask, cpu, gpu, seed, **hyper):
        m = mask.shape[0]
        cpu, gpu = np.asarray(cpu, np.int32), np.asarray(gpu, np.int32)
        values = np.ascontiguousarray(values, np.float64)
        mask = np.ascontiguousarray(mask, np.uint8)
        out = np.zeros_like(values)
        h = _hyper(RefHyper, **hyper)
        rc = self.L.ref_ncf_complete(m, P(cpu), len(cpu), P(gpu), len(gpu), P(values), P(mask), ctypes.byref(h),
                                     seed, P(out))
        return rc, out

    def ncf_predict(self, model_json, rows, cols):
        rows, cols = np.ascontiguousarray(rows, np.int64), np.ascontiguousarray(cols, np.int64)
        out = np.zeros(len(rows))
        rc = self.L.ref_ncf_predict(model_json.encode(), P(rows), P(cols), len(rows), P(out))
        return rc, out

    def ncf_complete_select_rows(self, ka, ks, hidden, params_sub, app_seen, setting_seen, cpu, gpu, values, mask,
                                 gamma=0.05, threads=1, want_completed=True):
        """NcfModel::predict of every unobserved cell of the given rows (a model whose app
        table holds exactly these rows) + policy::select_caps per row.  Returns
        (rc, completed | None, idx, saving, loss, ncand, seconds)."""
        values = np.ascontiguousarray(values, np.float64)
        mask = np.ascontiguousarray(mask, np.uint8)
        r = values.shape[0]
        cpu, gpu = np.asarray(cpu, np.int32), np.asarray(gpu, np.int32)
        hid = np.asarray(hidden, np.uint64)
        p = np.ascontiguousarray(params_sub, np.float64)
        aseen = np.ascontiguousarray(app_seen, np.uint8)
        sseen = np.ascontiguousarray(setting_seen, np.uint8)
        comp = np.zeros_like(values) if want_completed else None
        idx, nc = np.zeros(r, np.int32), np.zeros(r, np.int32)
        sv, lo = np.zeros(r), np.zeros(r)
        secs = c_dbl()
        rc = self.L.ref_ncf_complete_select_rows(ka, ks, P(hid), len(hid), r, P(p), P(aseen), P(sseen), P(cpu),
                                                 len(cpu), P(gpu), len(gpu), P(values), P(mask), gamma, threads,
                                                 P(comp), P(idx), P(sv), P(lo), P(nc), ctypes.byref(secs))
        return rc, comp, idx, sv, lo, nc, secs.value

    def joint_rows_dense(self, m, cpu, gpu, density, dense_rows, rows, seed=42, as_float=False):
        """SURVEY 8d joint-matrix rows generated by the reference's own sim/policy code."""
        cpu, gpu = np.asarray(cpu, np.int32), np.asarray(gpu, np.int32)
        rows = np.ascontiguousarray(rows, np.int64)
        n = len(cpu) * len(gpu)
        vals = np.zeros((len(rows), n))
        mask = np.zeros((len(rows), n), np.uint8)
        rc = self.L.ref_joint_rows_dense(m, P(cpu), len(cpu), P(gpu), len(gpu), density, dense_rows, seed, P(rows),
                                         len(rows), 1 if as_float else 0, P(vals), P(mask))
        assert rc == 0, self.err()
        return vals, mask

    def matrix_csv_roundtrip(self, in_path, out_path=None):
        """read_matrix_csv_file (+ write_matrix_csv): (rc, (m, n, nnz))."""
        m, n, nnz = c_sz(), c_sz(), c_sz()
        rc = self.L.ref_matrix_csv_roundtrip(str(in_path).encode(), None if out_path is None else str(out_path).encode(),
                                             ctypes.byref(m), ctypes.byref(n), ctypes.byref(nnz))
        return rc, (m.value, n.value, nnz.value)

    def time_fit_step(self, m, n, k, hidden=(32, 16), iters=3):
        """Seconds per cf::fit minibatch step composed from the reference's components."""
        hid = np.asarray(hidden, np.uint64)
        parts = np.zeros(3)
        secs = self.L.ref_time_fit_step(m, n, k, P(hid), len(hid), iters, P(parts))
        assert secs > 0, self.err()
        return secs, parts

    def run_trace(self, spec, cpu_cap, gpu_cap, seed, cap=1 << 16):
        """sim::run's GPU-power trace: (power samples, dt)."""
        out = np.zeros(cap)
        cnt, dt = c_sz(), c_dbl()
        rc = self.L.ref_run_trace(ctypes.byref(spec), cpu_cap, gpu_cap, seed, P(out), cap, ctypes.byref(cnt),
                                  ctypes.byref(dt))
        assert rc == 0, self.err()
        return out[: min(cnt.value, cap)].copy(), dt.value

    def detect(self, power, delta_s=0.2, window_s=5.0, p_th=60.0, armed=0):
        """(rc, fire index or -1) of the reference detector on one stream."""
        p = np.ascontiguousarray(power, np.float64)
        f = ctypes.c_int64()
        rc = self.L.ref_detect(P(p), len(p), delta_s, window_s, p_th, armed, ctypes.byref(f))
        return rc, f.value

    def eval_default(self, pols, seed=42, reps=5, gamma=0.05, napps=20, n=20):
        """policy::evaluate_suite of the default evaluation suite for baseline policies, and the
        sim::run results its truth tables come from: (rows, aggs, base, runs)."""
        pols = np.ascontiguousarray(pols, np.int32)
        rows = np.zeros((napps, len(pols), 8))
        aggs = np.zeros((len(pols), 4))
        base = np.zeros((napps, reps, 3))
        runs = np.zeros((napps, n, reps, 3))
        na = c_sz()
        rc = self.L.ref_eval_default(seed, reps, gamma, P(pols), len(pols), P(rows), P(aggs), P(base), P(runs),
                                     ctypes.byref(na))
        assert rc == 0 and na.value == napps, self.err()
        return rows, aggs, base, runs

    def load_predictor(self, path):
        hs = ctypes.c_int()
        rc = self.L.ref_load_predictor(str(path).encode(), ctypes.byref(hs))
        return rc, bool(hs.value)

    def offline_default(self, seed=42):
        dense = np.zeros(10 * 20)
        rows = c_sz()
        cap = 1 << 22
        buf = ctypes.create_string_buffer(cap)
        ln = c_sz()
        rc = self.L.ref_offline_default(seed, P(dense), ctypes.byref(rows), buf, cap, ctypes.byref(ln))
        assert rc == 0, self.err()
        return dense.reshape(rows.value, 20), buf.value.decode()

    def online_default(self, seed, eval_index, dense, predictor_json):
        out = RefOnlineOut()
        d = np.ascontiguousarray(dense, np.float64)
        rc = self.L.ref_online_default(seed, eval_index, P(d), d.shape[0], predictor_json.encode(),
                                       ctypes.byref(out))
        assert rc == 0, self.err()
        return out


def sub_model_params(params, m, n, ka, ks, rows):
    """Flat parameters of the model restricted to app rows `rows` (same setting table
    and MLP): NcfModel::predict(i, j) depends only on row i's embedding."""
    params = np.asarray(params, np.float64)
    app = params[: m * ka].reshape(m, ka)[np.asarray(rows, np.int64)].ravel()
    return np.concatenate([app, params[m * ka:]])


def model_params_from_json(text: str) -> np.ndarray:
    """Flat parameter vector (Adam block order) of a reference NcfModel JSON."""
    doc = json.loads(text)
    parts = [np.asarray(doc["embeddings"]["app"]["values"], np.float64).ravel(),
             np.asarray(doc["embeddings"]["setting"]["values"], np.float64).ravel()]
    for layer in doc["layers"]:
        parts.append(np.asarray(layer["weights"], np.float64).ravel())
        parts.append(np.asarray(layer["biases"], np.float64).ravel())
    return np.concatenate(parts)
