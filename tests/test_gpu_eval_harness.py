"""Evaluation harness on the B200: ocg_eval_suite against the
compiled reference's policy::evaluate_suite (truth tables from sim::run's
repetitions, exhaustive policies, aggregates) bit for bit, and against the pinned
restatement oracle/eval_port.py for the open policy's rows, ties and many apps."""
import numpy as np
import pytest

from conftest import DEFAULT_CPU, DEFAULT_GPU

pytestmark = pytest.mark.gpu

FIELDS = ["cpu_cap_w", "gpu_cap_w", "true_perf", "true_loss", "energy_j", "avg_power_w", "efficiency", "pred_saving"]


def _grid():
    from paper_2508_07605_b200 import PowerGrid

    return PowerGrid(list(DEFAULT_CPU), list(DEFAULT_GPU))


def _rows_array(rep):
    return np.stack([rep.rows[f].astype(np.float64) for f in FIELDS], axis=-1)


def _aggs_array(rep):
    a = rep.aggregates
    return np.stack([a["mean_efficiency"], a["mean_gain_vs_no_cap"], a["mean_true_loss"], a["mean_true_perf"]], -1)


@pytest.mark.parametrize("seed,reps,gamma,pols", [(42, 5, 0.05, [1, 2, 3, 4]), (7, 3, 0.10, [4, 3, 2, 1]),
                                                  (1234, 2, 0.0, [1, 2, 3, 4]), (99, 1, 0.2, [4]),
                                                  (5, 4, 0.05, [4, 1, 4])])
def test_eval_suite_matches_reference(ref, ctx, seed, reps, gamma, pols):
    from paper_2508_07605_b200.evaluate import evaluate_suite

    rows, aggs, base, runs = ref.eval_default(pols, seed=seed, reps=reps, gamma=gamma)
    rep = evaluate_suite(base[..., [0, 2, 1]], runs[..., [0, 2, 1]], _grid(), pols, gamma, ctx=ctx)
    assert np.array_equal(_rows_array(rep), rows)
    assert np.array_equal(_aggs_array(rep), aggs)
    assert rep.rows["policy"].tolist() == [pols] * rows.shape[0]
    assert np.all(rep.rows["gamma"] == gamma)


def _synthetic_runs(napps, reps, seed, quantize=None):
    rng = np.random.default_rng(seed)
    n = len(DEFAULT_CPU) * len(DEFAULT_GPU)
    base = np.empty((napps, reps, 3))
    base[..., 0] = rng.uniform(50, 150, (napps, reps))
    base[..., 2] = rng.uniform(200, 450, (napps, reps))
    base[..., 1] = base[..., 0] * base[..., 2]
    slow = rng.uniform(1.0, 1.3, (napps, n, reps))
    runs = np.empty((napps, n, reps, 3))
    runs[..., 0] = base[:, None, :, 0] * slow
    runs[..., 2] = base[:, None, :, 2] * rng.uniform(0.6, 1.0, (napps, n, reps))
    if quantize:  # coarse values: many equal efficiencies / performances, exercising the tie order
        runs[..., 0] = base[:, None, :, 0] * np.round(slow * quantize) / quantize
        runs[..., 2] = base[:, None, :, 2] * np.round(runs[..., 2] / base[:, None, :, 2] * quantize) / quantize
    runs[..., 1] = runs[..., 0] * runs[..., 2]
    runs[:, -1] = base  # the baseline setting measures the baseline run
    return base, runs


@pytest.mark.parametrize("napps,reps,quantize", [(600, 5, None), (600, 3, 4), (300, 4, 2), (200, 1, None)])
def test_eval_suite_open_ties_and_scale_match_port(ctx, napps, reps, quantize):
    from oracle import eval_port
    from paper_2508_07605_b200.evaluate import evaluate_suite

    base, runs = _synthetic_runs(napps, reps, seed=napps + reps, quantize=quantize)
    rng = np.random.default_rng(3)
    oi = rng.integers(0, runs.shape[1], napps).astype(np.int32)
    osv = rng.uniform(-0.2, 0.4, napps)
    pols = [0, 1, 2, 3, 4, 0]
    rep = evaluate_suite(base, runs, _grid(), pols, 0.08, open_idx=oi, open_pred_saving=osv, ctx=ctx)
    prow, pagg = eval_port.evaluate(base.tolist(), runs.tolist(), list(DEFAULT_CPU), list(DEFAULT_GPU), pols, 0.08,
                                    oi.tolist(), osv.tolist())
    want = np.array([[p[1:] for p in out] for out in prow])
    assert np.array_equal(_rows_array(rep), want)
    assert np.array_equal(rep.rows["setting"], np.array([[p[0] for p in out] for out in prow]))
    assert np.array_equal(_aggs_array(rep), np.array(pagg))
    assert np.array_equal(rep.rows["setting"][:, 0], oi)


def test_eval_suite_large_suite_invariants(ctx):
    """100k apps: every exhaustive choice is feasible and no candidate beats it."""
    from paper_2508_07605_b200.evaluate import evaluate_suite

    base, runs = _synthetic_runs(100_000, 3, seed=11)
    rep = evaluate_suite(base, runs, _grid(), ["oracle", "no_cap"], 0.05, ctx=ctx)
    r = rep.rows
    assert np.all(r["true_loss"][:, 0] <= 0.05)
    assert np.all(r["efficiency"][:, 0] >= r["efficiency"][:, 1])
    assert np.all(r["setting"][:, 1] == runs.shape[1] - 1)
    assert np.all(r["efficiency"][:, 1] == 1.0)
