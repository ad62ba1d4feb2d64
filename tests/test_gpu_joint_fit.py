"""Joint-mode cf::fit / cf::complete on the B200 through the C-ABI
(ocg_cf_fit, ocg_cf_complete) against the reference's own fits.

Bar: NCF_REF reproduces the reference's cf::fit bit for bit
— every parameter, epochs_run, the three MSEs — in both kernel lanes, on the
golden joint matrices and on the full C1 configuration (10K apps x 256
settings, k=8, 5 %, ~5 min per fit on the reference's host path); cf::complete
reproduces the reference's completed matrix bit for bit and select_caps'
decisions on it.  NCF_FAST (FP32, same schedule) is held to a stated quality
band against the FP64 fit.
"""
import time

import numpy as np
import pytest

import joint_cases as jc

pytestmark = pytest.mark.gpu


def _fit(case, ctx, solver=0, lane=None, stats=None):
    from paper_2508_07605_b200 import NcfHyper
    from paper_2508_07605_b200.cf import cf_fit

    _, A = jc.matrix(case)
    h = NcfHyper(**case["hyper"])
    return A, cf_fit(A.row_ptr, A.col, A.val, A.n, h, case["seed"], solver,
                     case["lane"] if lane is None else lane, ctx, stats)


def _assert_exact(model, case):
    meta = case["meta"]
    assert model.meta.epochs_run == int(meta[0])
    assert [model.meta.initial_train_mse, model.meta.final_train_mse, model.meta.best_val_mse] == list(meta[1:])
    mism = np.flatnonzero(model.params != case["params"])
    assert mism.size == 0, f"{mism.size} params differ, first at {mism[:5]}"


@pytest.mark.parametrize("case", jc.small_cases(), ids=lambda c: c["name"])
def test_joint_fit_bit_exact_small(ctx, case):
    _, model = _fit(case, ctx)
    _assert_exact(model, case)
    assert model.app_seen.all() and model.setting_seen.all()


@pytest.mark.parametrize("lane", [1, 0])
def test_joint_fit_bit_exact_c1(ctx, lane):
    case = jc.c1_case(lane)
    if case is None:
        pytest.skip("C1 golden not generated")
    stats = {}
    t0 = time.perf_counter()
    _, model = _fit(case, ctx, stats=stats)
    wall = time.perf_counter() - t0
    _assert_exact(model, case)
    print(f"\nC1 lane {lane}: {case['meta'][0]:.0f} epochs, {stats['steps']} steps, device {stats['device_ms'] / 1e3:.2f} s,"
          f" wall {wall:.2f} s (reference host path {case['host_seconds']:.0f} s)")


def test_joint_complete_select_matches_reference(ctx, ref):
    """cf::complete + select_caps over every row, NCF_REF, vs the reference's own."""
    from paper_2508_07605_b200 import NcfHyper
    from paper_2508_07605_b200.cf import cf_complete

    case = [c for c in jc.small_cases() if c["name"] == "d8_l1"][0]
    grid, A = jc.matrix(case)
    cpu, gpu = grid.arrays()
    vals, mask = jc.dense(A)
    ref.force_lane(1)
    rc, done = ref.ncf_complete(vals, mask, cpu, gpu, case["seed"], **case["hyper"])
    assert rc == 0, ref.err()
    r = cf_complete(A.row_ptr, A.col, A.val, A.n, NcfHyper(**case["hyper"]), case["seed"], 0, 1, grid, 0.05, ctx=ctx)
    np.testing.assert_array_equal(r.completed, done)
    rc, idx, sv, lo, nc = ref.select_caps(done, cpu, gpu, 0.05)
    assert rc == 0
    np.testing.assert_array_equal(r.idx, idx)
    np.testing.assert_array_equal(r.saving, sv)
    np.testing.assert_array_equal(r.loss, lo)
    np.testing.assert_array_equal(r.ncand, nc)


def test_joint_complete_fully_observed_is_identity(ctx):
    from paper_2508_07605_b200.cf import cf_complete

    rng = np.random.default_rng(3)
    m, n = 5, 6
    vals = rng.uniform(0.2, 1.2, (m, n))
    rp = np.arange(0, m * n + 1, n, dtype=np.int64)
    col = np.tile(np.arange(n, dtype=np.int32), m)
    r = cf_complete(rp, col, vals.ravel(), n, ctx=ctx)  # cfcomplete.cpp:206: no fit
    np.testing.assert_array_equal(r.completed, vals)


def test_joint_complete_cold_column(ctx):
    import paper_2508_07605_b200 as ocg
    from paper_2508_07605_b200.cf import cf_complete

    rp = np.array([0, 2, 4], np.int64)  # column 2 never observed -> predict() is cold (cfcomplete.cpp:53-55)
    col = np.array([0, 1, 0, 1], np.int32)
    val = np.array([0.5, 0.6, 0.7, 0.8])
    with pytest.raises(ocg.ColdError):
        cf_complete(rp, col, val, 3, ocg.NcfHyper(max_epochs=3), ctx=ctx)


def test_joint_fit_fast_fp32_quality(ctx, port, ref):
    """NCF_FAST (FP32, the reference schedule) vs the reference's FP64 fit on a
    golden case.  FP32 trajectories drift from FP64 ones (Adam over ~1K steps),
    so the bar is fit quality, not parameters: validation MSE within 5 % and
    train MSE within 10 % of the reference's, and the selection agreement of the two completed
    matrices reported."""
    case = [c for c in jc.small_cases() if c["name"] == "full_l1"][0]
    A, fast = _fit(case, ctx, solver=1)
    assert fast.meta.epochs_run == int(case["meta"][0])  # max_epochs-bound case
    exact = case["meta"]
    assert abs(fast.meta.best_val_mse - exact[3]) <= 0.05 * exact[3]
    assert abs(fast.meta.final_train_mse - exact[2]) <= 0.10 * exact[2]
    m, n = A.m, A.n
    kw = dict(case["hyper"])
    rows = np.repeat(np.arange(m), n)
    cols = np.tile(np.arange(n), m)
    port.set_lane(1)
    ones_m, ones_n = np.ones(m, np.uint8), np.ones(n, np.uint8)
    rc, pe = port.ncf_predict(m, n, case["params"], ones_m, ones_n, rows, cols, **kw)
    assert rc == 0
    rc, pf = port.ncf_predict(m, n, fast.params, ones_m, ones_n, rows, cols, **kw)
    assert rc == 0
    vals, mask = jc.dense(A)
    ce = np.where(mask == 1, vals, pe.reshape(m, n))
    cf = np.where(mask == 1, vals, pf.reshape(m, n))
    grid, _ = jc.matrix(case)
    cpu, gpu = grid.arrays()
    _, ie, *_ = ref.select_caps(ce, cpu, gpu, 0.05)
    _, i32, *_ = ref.select_caps(cf, cpu, gpu, 0.05)
    rel = np.abs(pf - pe) / pe
    agree = float((ie == i32).mean())
    print(f"\nFP32 vs FP64 fit: best_val {fast.meta.best_val_mse:.6g} vs {exact[3]:.6g}, final_train "
          f"{fast.meta.final_train_mse:.6g} vs {exact[2]:.6g}; prediction rel diff median {np.median(rel):.2e}; "
          f"selection agreement {agree:.3f}")
    assert agree > 0.5


def test_joint_fit_fast_code_path_in_fp64(ctx, monkeypatch):
    """The FP32 solver's formulas evaluated in FP64 (OCG_JOINT_FAST64, a
    diagnostic build of the same kernel) track the reference's FP64 fit to
    rounding: what separates NCF_FAST from NCF_REF is FP32 arithmetic only."""
    monkeypatch.setenv("OCG_JOINT_FAST64", "1")
    case = [c for c in jc.small_cases() if c["name"] == "full_l1"][0]
    _, m64 = _fit(case, ctx, solver=1)
    assert m64.meta.epochs_run == int(case["meta"][0])
    np.testing.assert_allclose(m64.params, case["params"], rtol=0, atol=1e-12)
    np.testing.assert_allclose([m64.meta.final_train_mse, m64.meta.best_val_mse], case["meta"][2:], rtol=1e-10)
