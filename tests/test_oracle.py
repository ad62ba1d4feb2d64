"""Pin the CPU oracle (our plain-C restatement, oracle/ocg_oracle.c) against
golden vectors produced by the reference library itself, and — where the
reference is built on this host — directly against it.  No GPU needed."""
import numpy as np
import pytest

from conftest import DEFAULT_CPU, DEFAULT_GPU, fit_case


def test_derive_seed_and_mt19937_64(port, golden):
    for key, val in golden["rng"]["derive_seed"].items():
        root, tag, n = key.split("|")
        assert port.derive_seed(int(root), tag, int(n)) == int(val), key
    for seed, stream in golden["rng"]["mt19937_64"].items():
        assert port.rng_u64(int(seed), len(stream)).tolist() == [int(v) for v in stream]


def _grid(name):
    if name == "default":
        return DEFAULT_CPU, DEFAULT_GPU
    k = {"grid16": 16, "grid64": 64}[name]
    return ([60 + (190 * i) // (k - 1) for i in range(k)], [100 + (300 * j) // (k - 1) for j in range(k)])


def test_select_caps_golden(port, golden, gold_npz):
    s = gold_npz["select"]
    for k, case in enumerate(golden["select_cases"]):
        cpu, gpu = _grid(case["name"])
        rc, idx, sv, lo, nc = port.select_caps(s[f"c{k}_rows"], cpu, gpu, case["gamma"])
        assert rc == 0
        np.testing.assert_array_equal(idx, s[f"c{k}_idx"])
        np.testing.assert_array_equal(sv, s[f"c{k}_saving"])  # bit-exact
        np.testing.assert_array_equal(lo, s[f"c{k}_loss"])
        np.testing.assert_array_equal(nc, s[f"c{k}_ncand"])


def test_select_caps_spec_example(port):
    # SPEC.md:543 / :692 worked example
    row = np.full((1, 20), 0.5)
    s = [(c, g) for c in DEFAULT_CPU for g in DEFAULT_GPU]
    for st, p in {(200, 250): 1.0, (150, 200): 0.97, (125, 150): 0.90, (100, 100): 0.70}.items():
        row[0, s.index(st)] = p
    rc, idx, sv, lo, nc = port.select_caps(row, DEFAULT_CPU, DEFAULT_GPU, 0.05)
    assert rc == 0 and s[idx[0]] == (150, 200) and nc[0] == 2
    assert sv[0] == 0.19816723940435282 and lo[0] == 0.030000000000000027


def test_select_caps_errors(port, golden):
    bad = np.full((1, 20), 0.9)
    bad[0, 3] = -1.0
    assert port.select_caps(bad, DEFAULT_CPU, DEFAULT_GPU, 0.05)[0] == golden["select_rc_bad_entry"]
    assert port.select_caps(np.full((1, 20), 0.9), DEFAULT_CPU, DEFAULT_GPU, 1.0)[0] == golden["select_rc_bad_gamma"]


def test_default_plan(port, golden):
    for key, plan in golden["default_plans"].items():
        nc, ng = map(int, key.split("x"))
        cpu, gpu = (DEFAULT_CPU, DEFAULT_GPU) if (nc, ng) == (5, 4) else (
            [60 + (190 * i) // (nc - 1) for i in range(nc)], [100 + (300 * j) // (ng - 1) for j in range(ng)])
        assert port.default_plan(cpu, gpu) == plan


@pytest.mark.parametrize("lane", [0, 1])
@pytest.mark.parametrize("k", range(5))
def test_ncf_fit_bit_exact(port, golden, gold_npz, k, lane):
    name, values, mask, seed, hyper = fit_case(golden, gold_npz, k)
    port.set_lane(lane)
    try:
        rc, params, meta, aseen, sseen = port.ncf_fit(values, mask, seed, **hyper)
        m, n = mask.shape
        ii, jj = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
        rc2, pred = port.ncf_predict(m, n, params, aseen, sseen, ii.ravel(), jj.ravel(), **hyper)
    finally:
        port.set_lane(0)
    assert rc == 0 and rc2 == 0, port.err()
    np.testing.assert_array_equal(params, gold_npz["fit"][f"f{k}_lane{lane}_params"])
    np.testing.assert_array_equal(pred.reshape(m, n), gold_npz["fit"][f"f{k}_lane{lane}_pred"])
    g = golden["fit_cases"][k][f"lane{lane}"]
    assert meta.epochs_run == g["epochs_run"]
    assert meta.initial_train_mse == g["initial_train_mse"]
    assert meta.final_train_mse == g["final_train_mse"]
    assert meta.best_val_mse == g["best_val_mse"]


@pytest.mark.parametrize("lane", [0, 1])
def test_oracle_vs_reference_random_fits(port, ref, lane):
    """Fresh random matrices: port == reference in either lane, params and meta."""
    rng = np.random.default_rng(4242 + lane)
    ref.force_lane(lane)
    port.set_lane(lane)
    try:
        for trial in range(4):
            m, n = rng.integers(4, 14), rng.integers(3, 9)
            v = rng.uniform(0.05, 1.25, (m, n))
            mk = (rng.random((m, n)) < 0.5).astype(np.uint8)
            mk[np.arange(m), rng.integers(0, n, m)] = 1
            hyper = dict(app_dim=int(rng.integers(1, 6)), setting_dim=int(rng.integers(1, 6)),
                         hidden=(int(rng.integers(2, 12)),), max_epochs=40, patience=8,
                         batch_size=int(rng.integers(1, 20)))
            seed = int(rng.integers(0, 2**63))
            rc, js, meta_r = ref.ncf_fit(v, mk, [1], list(range(1, n + 1)), seed, **hyper)
            assert rc == 0
            from oracle.bind import model_params_from_json
            rc, p, meta_p, _, _ = port.ncf_fit(v, mk, seed, **hyper)
            assert rc == 0
            np.testing.assert_array_equal(p, model_params_from_json(js))
            assert meta_p.epochs_run == meta_r.epochs_run and meta_p.best_val_mse == meta_r.best_val_mse
    finally:
        ref.force_lane(1)
        port.set_lane(0)


def test_predictor_model_json_parse():
    """PredictorModel.from_json reads the reference's predictor file (predictor.cpp:302-316)."""
    from conftest import GOLD
    from paper_2508_07605_b200.predictor import PredictorModel

    m = PredictorModel.from_json((GOLD / "predictor.json").read_text())
    assert m.dims[0] == 7 and m.dims[-1] == 1 and m.has_stats
    assert len(m.params) == sum(a * b + b for a, b in zip(m.dims[:-1], m.dims[1:]))
    assert len(m.acts) == len(m.dims) - 1
