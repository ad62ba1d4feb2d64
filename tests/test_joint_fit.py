"""Joint-mode cf::fit (one model over a whole matrix): CPU side.

* the FP64 joint matrices the GPU tests fit are the reference's own
  (synth.joint_csr(dtype=float64) == ref_joint_rows_dense, bit for bit);
* the oracle restatement reproduces the reference's golden joint fits
  (tests/golden/joint_small.npz, made by tests/golden/make_joint_golden.py);
* ocg_cf_fit / ocg_cf_complete reject what the reference rejects, with the
  reference's exception type, before any device work (no GPU needed).
"""
import numpy as np
import pytest

import joint_cases as jc


@pytest.mark.parametrize("case", jc.small_cases()[:4], ids=lambda c: c["name"])
def test_joint_matrix_is_the_references(ref, case):
    grid, A = jc.matrix(case)
    cpu, gpu = grid.arrays()
    vals, mask = ref.joint_rows_dense(case["m"], cpu, gpu, case["density"], case["dense_rows"], np.arange(case["m"]))
    v, mk = jc.dense(A)
    np.testing.assert_array_equal(mk, mask)
    np.testing.assert_array_equal(v, vals)


@pytest.mark.parametrize("case", jc.small_cases(), ids=lambda c: c["name"])
def test_oracle_reproduces_reference_joint_fit(port, case):
    _, A = jc.matrix(case)
    vals, mask = jc.dense(A)
    port.set_lane(case["lane"])
    rc, params, meta, aseen, sseen = port.ncf_fit(vals, mask, case["seed"], **case["hyper"])
    assert rc == 0, port.err()
    assert meta.epochs_run == int(case["meta"][0])
    assert [meta.initial_train_mse, meta.final_train_mse, meta.best_val_mse] == list(case["meta"][1:])
    np.testing.assert_array_equal(params, case["params"])


def _csr():
    rp = np.array([0, 2, 3], np.int64)
    col = np.array([0, 2, 1], np.int32)
    val = np.array([0.5, 0.9, 1.0])
    return rp, col, val


def _fit(rp, col, val, n=3, **hyper):
    import ctypes

    from paper_2508_07605_b200 import NcfHyper
    from paper_2508_07605_b200._lib import check, lib, ptr

    h = NcfHyper(**hyper).to_c()
    check(lib.ocg_cf_fit(None, len(rp) - 1, n, ptr(rp), ptr(col), ptr(val), ctypes.byref(h), 1, 0, 1, None, None,
                         None, None))


@pytest.mark.parametrize("mut,exc", [
    (lambda rp, c, v: c.__setitem__(1, 3), "OutOfRange"),        # PerformanceMatrix::set index (core.cpp:143)
    (lambda rp, c, v: c.__setitem__(2, -1), "OutOfRange"),
    (lambda rp, c, v: v.__setitem__(0, 0.0), "InvalidArgument"),  # value outside (0, 1.25] (core.cpp:144-146)
    (lambda rp, c, v: v.__setitem__(2, 1.3), "InvalidArgument"),
    (lambda rp, c, v: v.__setitem__(1, np.nan), "InvalidArgument"),
    (lambda rp, c, v: c.__setitem__(1, 0), "InvalidArgument"),    # duplicate cell / unsorted columns
    (lambda rp, c, v: rp.__setitem__(1, 4), "InvalidArgument"),   # row_ptr not monotone
])
def test_cf_fit_rejects_bad_matrix(mut, exc):
    import paper_2508_07605_b200 as ocg

    rp, col, val = _csr()
    mut(rp, col, val)
    with pytest.raises(getattr(ocg, exc)):
        _fit(rp, col, val)


@pytest.mark.parametrize("hyper", [dict(app_dim=0), dict(lr=0.0), dict(max_epochs=0), dict(batch_size=0),
                                   dict(val_fraction=1.0), dict(val_fraction=-0.1), dict(hidden=[8, 0])])
def test_cf_fit_rejects_bad_hyper(hyper):
    import paper_2508_07605_b200 as ocg

    with pytest.raises(ocg.InvalidArgument, match="bad hyperparameters|zero layer width"):
        _fit(*_csr(), **hyper)


def test_cf_fit_rejects_empty_matrix():
    import paper_2508_07605_b200 as ocg

    with pytest.raises(ocg.InvalidArgument, match="no observed entries"):  # cfcomplete.cpp:72
        _fit(np.zeros(3, np.int64), np.zeros(0, np.int32), np.zeros(0))


def test_cf_complete_rejects_row_without_probes():
    import ctypes

    import paper_2508_07605_b200 as ocg
    from paper_2508_07605_b200._lib import check, lib, ptr

    rp = np.array([0, 2, 2], np.int64)  # row 1 has no observed entry (cfcomplete.cpp:199-205)
    col = np.array([0, 2], np.int32)
    val = np.array([0.5, 0.9])
    h = ocg.NcfHyper().to_c()
    with pytest.raises(ocg.InvalidArgument, match="no observed entries"):
        check(lib.ocg_cf_complete(None, 2, 3, ptr(rp), ptr(col), ptr(val), ctypes.byref(h), None, 1, 0, 1, None, 0,
                                  None, 0, 0.05, None, None, None, None, None))


def test_cf_fit_als_has_no_model():
    import ctypes

    import paper_2508_07605_b200 as ocg
    from paper_2508_07605_b200._lib import check, lib, ptr

    rp, col, val = _csr()
    h = ocg.NcfHyper().to_c()
    with pytest.raises(ocg.InvalidArgument, match="ALS"):
        check(lib.ocg_cf_fit(None, 2, 3, ptr(rp), ptr(col), ptr(val), ctypes.byref(h), 1, 2, 1, None, None, None,
                             None))
