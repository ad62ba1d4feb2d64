"""Evaluation harness, host side (no GPU): the CPU restatement oracle/eval_port.py
pinned against the compiled reference's policy::evaluate_suite (ref_eval_default on
sim::make_suite's default evaluation suite), and ocg_eval_suite's argument
rejections (measure_truth's repetitions < 1, PowerGrid's cap checks, unknown policy)."""
import ctypes

import numpy as np
import pytest

from conftest import DEFAULT_CPU, DEFAULT_GPU

POLS = [1, 2, 3, 4]


def _as_port(base, runs):
    # ref_eval_default dumps (runtime, avg_power, energy); RunResult order is (runtime, energy, avg_power)
    b = base[..., [0, 2, 1]]
    r = runs[..., [0, 2, 1]]
    return b.tolist(), r.tolist()


@pytest.mark.parametrize("seed,reps,gamma", [(42, 5, 0.05), (7, 3, 0.10), (1234, 2, 0.0), (99, 1, 0.2)])
def test_port_matches_reference_evaluate_suite(ref, seed, reps, gamma):
    from oracle import eval_port

    rows, aggs, base, runs = ref.eval_default(POLS, seed=seed, reps=reps, gamma=gamma)
    b, r = _as_port(base, runs)
    prow, pagg = eval_port.evaluate(b, r, list(DEFAULT_CPU), list(DEFAULT_GPU), POLS, gamma)
    got = np.array([[p[1:] for p in out] for out in prow])  # cpu, gpu, perf, loss, energy, avgp, eff, sav
    assert np.array_equal(got, rows)
    assert np.array_equal(np.array(pagg), aggs)


def test_port_duplicate_policies_aggregate_by_name(ref):
    from oracle import eval_port

    pols = [4, 1, 4]
    rows, aggs, base, runs = ref.eval_default(pols, seed=5, reps=3)
    b, r = _as_port(base, runs)
    prow, pagg = eval_port.evaluate(b, r, list(DEFAULT_CPU), list(DEFAULT_GPU), pols, 0.05)
    assert np.array_equal(np.array([[p[1:] for p in out] for out in prow]), rows)
    assert np.array_equal(np.array(pagg), aggs)


def _call(reps=3, cpu=DEFAULT_CPU, gpu=DEFAULT_GPU, pols=(1,), napps=1):
    from paper_2508_07605_b200 import _lib

    cpu, gpu = np.asarray(cpu, np.int32), np.asarray(gpu, np.int32)
    n = len(cpu) * len(gpu)
    na = max(napps, 1)
    base = np.ones((na, max(reps, 1), 3))
    runs = np.ones((na, n, max(reps, 1), 3))
    k = np.asarray(pols, np.int32)
    rows = np.zeros(max(napps, 1) * len(k) * ctypes.sizeof(_lib.EvalRowC), np.uint8)
    aggs = np.zeros(len(k) * ctypes.sizeof(_lib.EvalAggregateC), np.uint8)
    _lib.check(_lib.lib.ocg_eval_suite(None, napps, _lib.ptr(cpu), len(cpu), _lib.ptr(gpu), len(gpu), reps,
                                       _lib.ptr(base), _lib.ptr(runs), 0.05, len(k), _lib.ptr(k), None, None,
                                       _lib.ptr(rows), _lib.ptr(aggs)))
    return aggs


@pytest.mark.parametrize("kw", [dict(reps=0), dict(cpu=(100, 100)), dict(gpu=(150, 100)), dict(cpu=(0, 100)),
                                dict(pols=(5,)), dict(pols=(-1,)), dict(pols=(0,)), dict(napps=-1)])
def test_eval_suite_rejections(kw):
    import paper_2508_07605_b200 as ocg

    with pytest.raises(ocg.InvalidArgument):
        _call(**kw)


def test_eval_suite_no_apps_reports_zero_aggregates():
    from paper_2508_07605_b200.evaluate import _AGG_DTYPE

    a = np.frombuffer(_call(napps=0, pols=(4, 1)).tobytes(), dtype=_AGG_DTYPE)
    assert a["policy"].tolist() == [4, 1]
    assert np.all(a["mean_efficiency"] == 0.0)
