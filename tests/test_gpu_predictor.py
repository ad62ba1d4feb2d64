"""Probe ingest parity: batched pred::predict_perf (predictor.cpp:151-157) on
sm_100a vs the reference's own outputs (tests/golden/predictor.npz, produced
by oracle/_ref through ref_predict_perf in both kernel lanes)."""
import json

import numpy as np
import pytest

from conftest import GOLD

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def model():
    from paper_2508_07605_b200.predictor import PredictorModel

    return PredictorModel.from_json((GOLD / "predictor.json").read_text())


@pytest.mark.parametrize("lane", [0, 1])
def test_predict_perf_bit_exact(ctx, model, lane):
    from paper_2508_07605_b200.predictor import Predictor, predict_perf_batch

    g = np.load(GOLD / "predictor.npz")
    out = predict_perf_batch(model, g["counters"], lane, ctx)
    np.testing.assert_array_equal(out, g[f"lane{lane}"])
    p = Predictor(model, ctx)  # both kernels: thread-per-sample (reference arch) and warp-per-sample (any arch)
    np.testing.assert_array_equal(p(g["counters"], lane), g[f"lane{lane}"])
    np.testing.assert_array_equal(p(g["counters"], lane, generic=True), g[f"lane{lane}"])


def test_predict_perf_device_pointers(ctx, model):
    import torch

    from paper_2508_07605_b200.predictor import Predictor

    g = np.load(GOLD / "predictor.npz")
    dev = torch.device("cuda", 0)
    c = torch.from_numpy(g["counters"]).to(dev)
    out = torch.zeros(len(c), dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    Predictor(model, ctx).run_device(c.data_ptr(), len(c), out.data_ptr(), 1)
    np.testing.assert_array_equal(out.cpu().numpy(), g["lane1"])


def test_predict_perf_large_batch_consistent(ctx, model):
    """Every sample is independent: a 200K batch of tiled goldens gives the golden per row."""
    from paper_2508_07605_b200.predictor import predict_perf_batch

    g = np.load(GOLD / "predictor.npz")
    reps = 200_000 // len(g["counters"]) + 1
    out = predict_perf_batch(model, np.tile(g["counters"], (reps, 1)), 1, ctx)
    np.testing.assert_array_equal(out, np.tile(g["lane1"], reps))


def test_predict_perf_errors(ctx, model, golden):
    from paper_2508_07605_b200 import _lib
    from paper_2508_07605_b200.predictor import PredictorModel, predict_perf_batch

    g = np.load(GOLD / "predictor.npz")
    bad = g["counters"][:4].copy()
    bad[2, 2] = -1.0  # negative ips: validate_counters -> invalid_argument
    assert golden["predict_rc_negative_ips"] == _lib.OCG_E_INVALID
    with pytest.raises(_lib.InvalidArgument):
        predict_perf_batch(model, bad, 1, ctx)
    bad = g["counters"][:4].copy()
    bad[0, 5] = 1.5  # utilisation outside [0, 1]
    with pytest.raises(_lib.InvalidArgument):
        predict_perf_batch(model, bad, 1, ctx)
    doc = json.loads((GOLD / "predictor.json").read_text())
    doc.pop("feature_stats")
    nostats = PredictorModel.from_json(json.dumps(doc))
    with pytest.raises(_lib.OcgError) as e:
        predict_perf_batch(nostats, g["counters"][:4], 1, ctx)
    assert e.value.code == _lib.OCG_E_MISSING
    assert len(predict_perf_batch(model, np.zeros((0, 7)), 1, ctx)) == 0
