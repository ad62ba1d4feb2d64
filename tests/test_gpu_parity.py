"""GPU parity tests — through the C-ABI (libocg.so) against the reference's
golden vectors and the CPU oracle.  Bar: bit-exact (FP64, same operation
order as the selected reference kernel lane)."""
import numpy as np
import pytest

from conftest import DEFAULT_CPU, DEFAULT_GPU, fit_case

pytestmark = pytest.mark.gpu


def _grid(name):
    from paper_2508_07605_b200 import PowerGrid

    if name == "default":
        return PowerGrid.default_grid()
    return PowerGrid.spanning(*{"grid16": (16, 16), "grid64": (64, 64)}[name])


def test_device_is_b200(ctx):
    info = ctx.info()
    assert info["cc"][0] == 10 and info["sm_count"] >= 132


def test_device_exp_bit_exact(ctx, gold_npz):
    import ctypes

    from paper_2508_07605_b200 import _lib

    x, y = gold_npz["exp"]["x"], gold_npz["exp"]["y"]
    out = np.zeros_like(x)
    _lib.check(_lib.lib.ocg_debug_exp(ctx.handle, _lib.ptr(x), len(x), _lib.ptr(out)))
    np.testing.assert_array_equal(out.view(np.uint64), y.view(np.uint64))


def test_device_mt19937_64(ctx, golden):
    from paper_2508_07605_b200 import _lib

    for seed, stream in golden["rng"]["mt19937_64"].items():
        out = np.zeros(len(stream), np.uint64)
        _lib.check(_lib.lib.ocg_debug_rng(ctx.handle, int(seed), len(stream), _lib.ptr(out)))
        assert out.tolist() == [int(v) for v in stream]


def test_select_caps_bit_exact(ctx, golden, gold_npz):
    from paper_2508_07605_b200 import select_caps_batch

    s = gold_npz["select"]
    for k, case in enumerate(golden["select_cases"]):
        idx, sav, loss, nc = select_caps_batch(s[f"c{k}_rows"], _grid(case["name"]), case["gamma"], ctx)
        np.testing.assert_array_equal(idx, s[f"c{k}_idx"])
        np.testing.assert_array_equal(sav, s[f"c{k}_saving"])
        np.testing.assert_array_equal(loss, s[f"c{k}_loss"])
        np.testing.assert_array_equal(nc, s[f"c{k}_ncand"])


def test_select_caps_spec_example(ctx):
    from paper_2508_07605_b200 import PowerGrid, select_caps

    grid = PowerGrid.default_grid()
    row = np.full(20, 0.5)
    s = grid.settings()
    for st, p in {(200, 250): 1.0, (150, 200): 0.97, (125, 150): 0.90, (100, 100): 0.70}.items():
        row[s.index(st)] = p
    d = select_caps(row, grid, 0.05, ctx)
    assert d.setting == (150, 200) and d.candidates_considered == 2
    assert d.pred_saving == 0.19816723940435282 and d.pred_loss == 0.030000000000000027


def test_select_caps_errors(ctx):
    from paper_2508_07605_b200 import InvalidArgument, PowerGrid, select_caps_batch

    bad = np.full((3, 20), 0.9)
    bad[1, 4] = np.nan
    with pytest.raises(InvalidArgument):
        select_caps_batch(bad, PowerGrid.default_grid(), 0.05, ctx)
    with pytest.raises(InvalidArgument):
        select_caps_batch(np.full((1, 20), 0.9), PowerGrid.default_grid(), 1.5, ctx)


def test_select_caps_vs_oracle_random_large(ctx, port):
    from paper_2508_07605_b200 import PowerGrid, select_caps_batch

    rng = np.random.default_rng(9)
    grid = PowerGrid.spanning(64, 64)
    rows = rng.uniform(0.01, 1.25, (500, 4096))
    rows[:, -1] = rng.uniform(0.8, 1.25, 500)
    # force exact ties in saving and perf
    rows[::7, :] = np.maximum(np.round(rows[::7, :], 1), 0.1)
    idx, sav, loss, nc = select_caps_batch(rows, grid, 0.1, ctx)
    cpu, gpu = grid.arrays()
    rc, i2, s2, l2, n2 = port.select_caps(rows, cpu, gpu, 0.1)
    assert rc == 0
    np.testing.assert_array_equal(idx, i2)
    np.testing.assert_array_equal(sav, s2)
    np.testing.assert_array_equal(loss, l2)
    np.testing.assert_array_equal(nc, n2)


@pytest.mark.parametrize("lane", [0, 1])
@pytest.mark.parametrize("k", range(5))
def test_ncf_fit_params_bit_exact(ctx, golden, gold_npz, k, lane):
    """cf::fit on the device (one CTA per app) == reference, parameter for parameter."""
    from paper_2508_07605_b200 import NcfHyper, online_fit_batch_params

    name, values, mask, seed, hyper = fit_case(golden, gold_npz, k)
    h = NcfHyper(**hyper)
    params, meta, status = online_fit_batch_params(values[:-1], mask[:-1], values[-1:], mask[-1:], [seed], h, lane,
                                                   ctx)
    assert status[0] == 0
    np.testing.assert_array_equal(params[0], gold_npz["fit"][f"f{k}_lane{lane}_params"])
    g = golden["fit_cases"][k][f"lane{lane}"]
    assert meta[0]["epochs_run"] == g["epochs_run"]
    assert meta[0]["initial_train_mse"] == g["initial_train_mse"]
    assert meta[0]["final_train_mse"] == g["final_train_mse"]
    assert meta[0]["best_val_mse"] == g["best_val_mse"]
    assert meta[0]["seed"] == seed


@pytest.mark.parametrize("lane", [0, 1])
@pytest.mark.parametrize("k", range(5))
def test_ncf_predict_bit_exact(ctx, golden, gold_npz, k, lane):
    from paper_2508_07605_b200 import NcfHyper, ncf_predict

    name, values, mask, seed, hyper = fit_case(golden, gold_npz, k)
    m, n = mask.shape
    ii, jj = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
    params = gold_npz["fit"][f"f{k}_lane{lane}_params"]
    aseen = (mask.sum(1) > 0).astype(np.uint8)
    sseen = (mask.sum(0) > 0).astype(np.uint8)
    pred = ncf_predict(m, n, NcfHyper(**hyper), params, aseen, sseen, ii.ravel(), jj.ravel(), lane, ctx)
    np.testing.assert_array_equal(pred.reshape(m, n), gold_npz["fit"][f"f{k}_lane{lane}_pred"])


def _c0_batch(golden, gold_npz, lane, repeat=1):
    dense = gold_npz["c0"]["dense"]
    apps = [a for a in golden["c0_apps"] if a["lane"] == lane]
    napps = len(apps)
    pv = np.zeros((napps, 20))
    pm = np.zeros((napps, 20), np.uint8)
    for a, rec in enumerate(apps):
        for j, v in zip(rec["probe_idx"], rec["probe_val"]):
            pv[a, j], pm[a, j] = v, 1
    seeds = np.array([int(s) for s in golden["c0_complete_seeds"]], np.uint64)
    return dense, apps, np.tile(pv, (repeat, 1)), np.tile(pm, (repeat, 1)), np.tile(seeds, repeat)


@pytest.mark.parametrize("lane", [0, 1])
def test_online_c0_eval_suite_bit_exact(ctx, golden, gold_npz, lane):
    """The reference's online phase for the 20 paper-scale eval apps: completed
    rows and Algorithm-2 decisions bit-identical (policy.cpp:178-189)."""
    from paper_2508_07605_b200 import PowerGrid, online_complete_batch

    dense, apps, pv, pm, seeds = _c0_batch(golden, gold_npz, lane)
    r = online_complete_batch(dense, np.ones_like(dense, np.uint8), pv, pm, seeds, PowerGrid.default_grid(),
                              gamma=0.05, lane=lane, ctx=ctx)
    for a, rec in enumerate(apps):
        assert r.status[a] == 0
        np.testing.assert_array_equal(r.completed[a], gold_npz["c0"][f"lane{lane}_app{rec['eval_index']}_row"])
        assert r.idx[a] == rec["setting_idx"]
        assert r.saving[a] == rec["pred_saving"]
        assert r.loss[a] == rec["pred_loss"]
        assert r.ncand[a] == rec["candidates"]


def test_online_batch_many_apps_consistent(ctx, golden, gold_npz):
    """2000 apps (CTAs loop over several apps each): every copy of an app gives
    the same bits as the reference."""
    from paper_2508_07605_b200 import PowerGrid, online_complete_batch

    lane = 1
    dense, apps, pv, pm, seeds = _c0_batch(golden, gold_npz, lane, repeat=100)
    r = online_complete_batch(dense, np.ones_like(dense, np.uint8), pv, pm, seeds, PowerGrid.default_grid(),
                              lane=lane, ctx=ctx)
    assert (r.status == 0).all()
    want = np.array([rec["setting_idx"] for rec in apps] * 100)
    np.testing.assert_array_equal(r.idx, want)
    want_s = np.array([rec["pred_saving"] for rec in apps] * 100)
    np.testing.assert_array_equal(r.saving, want_s)


def test_online_batch_error_behaviour(ctx, golden, gold_npz):
    from paper_2508_07605_b200 import InvalidArgument, NcfHyper, PowerGrid, online_complete_batch

    dense, apps, pv, pm, seeds = _c0_batch(golden, gold_npz, 1)
    grid = PowerGrid.default_grid()
    pm2 = pm[:3].copy()
    pm2[1] = 0  # app without probes -> invalid_argument (cfcomplete.cpp:199-205)
    bm = np.ones_like(dense, np.uint8)
    bm[:, 7] = 0
    pm2[2, 7] = 0
    pm2[0, 7] = 1  # column 7 observed only by app 0
    pv2 = pv[:3].copy()
    pv2[0, 7] = 0.5
    r = online_complete_batch(dense, bm, pv2, pm2, seeds[:3], grid, NcfHyper(max_epochs=5), ctx=ctx)
    assert r.status[1] == 1  # invalid_argument
    assert r.status[2] == 5  # cold setting column (runtime_error)
    assert r.status[0] == 0
    with pytest.raises(InvalidArgument):
        online_complete_batch(dense, np.ones_like(dense, np.uint8), pv, pm, seeds, grid, NcfHyper(lr=0.0), ctx=ctx)
    with pytest.raises(InvalidArgument):
        online_complete_batch(dense, np.ones_like(dense, np.uint8), pv, pm, seeds, grid, gamma=0.0, ctx=ctx)


def test_online_fully_observed_row_not_refit(ctx, golden, gold_npz):
    from paper_2508_07605_b200 import PowerGrid, online_complete_batch

    dense = gold_npz["c0"]["dense"]
    row = dense[3:4].copy()
    r = online_complete_batch(dense, np.ones_like(dense, np.uint8), row, np.ones((1, 20), np.uint8), [1],
                              PowerGrid.default_grid(), ctx=ctx)
    assert r.status[0] == 0 and r.meta[0]["epochs_run"] == 0
    np.testing.assert_array_equal(r.completed[0], row[0])


@pytest.mark.parametrize("k", [0, 1])
def test_device_fit_model_file_identical_to_reference(ctx, ref, golden, gold_npz, k):
    """cf::fit on the device -> NcfModel::to_json text == the reference's own
    cf::fit + to_json on the same inputs (parameters, masks, meta, formatting)."""
    from paper_2508_07605_b200 import NcfHyper, NcfMeta, NcfModel, online_fit_batch_params

    name, values, mask, seed, hyper = fit_case(golden, gold_npz, k)
    hyper = dict(hyper, max_epochs=min(hyper.get("max_epochs", 2000), 40))
    h = NcfHyper(**hyper)
    params, meta, status = online_fit_batch_params(values[:-1], mask[:-1], values[-1:], mask[-1:], [seed], h, 1, ctx)
    assert status[0] == 0
    m, n = mask.shape
    mt = NcfMeta(int(meta[0]["seed"]), int(meta[0]["epochs_run"]), float(meta[0]["initial_train_mse"]),
                 float(meta[0]["final_train_mse"]), float(meta[0]["best_val_mse"]))
    model = NcfModel(h, m, n, params[0], (mask.sum(1) > 0).astype(np.uint8), (mask.sum(0) > 0).astype(np.uint8), mt)
    cpu, gpu = (list(DEFAULT_CPU), list(DEFAULT_GPU)) if n == 20 else ([1], list(range(1, n + 1)))
    ref.force_lane(1)
    rc, js, _ = ref.ncf_fit(values, mask, cpu, gpu, seed, **hyper)
    assert rc == 0
    assert model.to_json() == js
