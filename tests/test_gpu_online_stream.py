"""Batched online streams on the B200 against the reference:
  * ocg_phase_detect_batch == phase::detect_offline / the reference Detector fed
    under run_open_online's arming rule, on the simulator's own power traces
    (sim::run, suites with CPU phases) and on adversarial synthetic streams;
  * ocg_online_ingest_complete_batch == pred::predict_perf of the same counters ->
    cf::complete of the dense block + the probed row -> select_caps, bit for bit,
    with the re-probe rule choosing which counters each app's estimates come from."""
import ctypes

import numpy as np
import pytest

from conftest import DEFAULT_CPU, DEFAULT_GPU, GOLD

pytestmark = pytest.mark.gpu


def _suite(ref, n_each, cpu_phase_fraction, seed=42):
    from oracle.bind import RefSpec

    cpu, gpu = np.asarray(DEFAULT_CPU, np.int32), np.asarray(DEFAULT_GPU, np.int32)
    out = (RefSpec * (4 * n_each))()
    rc = ref.L.ref_make_suite(n_each, n_each, n_each, n_each, seed, 0.01, 1, cpu_phase_fraction,
                              cpu.ctypes.data_as(ctypes.c_void_p), len(cpu), gpu.ctypes.data_as(ctypes.c_void_p),
                              len(gpu), out)
    assert rc == 0, ref.err()
    return out


@pytest.mark.parametrize("armed", [0, 1])
def test_detector_on_simulator_traces(ctx, ref, armed):
    from paper_2508_07605_b200.online import phase_detect_batch

    suite = _suite(ref, 6, 0.5)
    streams = []
    for k, spec in enumerate(suite):
        for (c, g) in [(100, 100), (150, 200), (200, 250)]:
            p, dt = ref.run_trace(spec, c, g, 1000 + k)
            assert abs(dt - 0.2) < 1e-12
            streams.append(p)
    T = max(len(p) for p in streams)
    P = np.zeros((len(streams), T))
    for i, p in enumerate(streams):
        P[i, :len(p)] = p
    lengths = np.array([len(p) for p in streams], np.int64)
    fire, st = phase_detect_batch(P, lengths, armed_start=bool(armed), ctx=ctx)
    want = np.array([ref.detect(p, armed=armed)[1] for p in streams])
    np.testing.assert_array_equal(fire, want)
    assert (st == 0).all()
    assert (want >= 0).sum() > 5 and (want < 0).sum() >= 0


@pytest.mark.parametrize("armed", [0, 1])
def test_detector_adversarial_streams(ctx, ref, armed):
    from paper_2508_07605_b200.online import phase_detect_batch

    rng = np.random.default_rng(4)
    S, T = 300, 160
    P = np.where(rng.random((S, T)) < 0.08, rng.uniform(0, 59.99, (S, T)), rng.uniform(60.0, 200.0, (S, T)))
    P[::7, :] = np.where(P[::7, :] < 60, 60.0, P[::7, :])       # exactly at the threshold counts as high
    P[3::11, 40:] = 150.0                                         # a clean high run
    P[5::13, rng.integers(0, T)] = -3.0                           # negative samples (invalid when fed)
    P[9::17, 20] = np.nan                                         # NaN: never below the threshold
    lengths = rng.integers(0, T + 1, S).astype(np.int64)
    fire, st = phase_detect_batch(P, lengths, armed_start=bool(armed), ctx=ctx)
    for s in range(S):
        rc, f = ref.detect(P[s, :lengths[s]], armed=armed)
        if rc:
            assert st[s] == rc, s
        else:
            assert st[s] == 0 and fire[s] == f, (s, fire[s], f)


def test_ingest_complete_matches_reference(ctx, ref, port):
    """counters -> predict_perf -> estimates at the plan columns -> cf::complete (per app,
    the paper-scale offline block) -> select_caps, against the reference's pieces."""
    import paper_2508_07605_b200 as ocg
    from oracle import bind
    from paper_2508_07605_b200 import synth
    from paper_2508_07605_b200.online import online_ingest_complete_batch
    from paper_2508_07605_b200.predictor import Predictor, PredictorModel

    grid = ocg.PowerGrid.default_grid()
    block = synth.offline_block(42, grid)
    plan = ocg.ProbePlan.default_plan(grid)
    pj = (GOLD / "predictor.json").read_text()
    pred = Predictor(PredictorModel.from_json(pj), ctx=ctx)
    suite = _suite(ref, 3, 0.0, seed=7)
    napps = len(suite)
    settings = grid.settings()
    counters = np.zeros((napps, len(plan.columns), 7))
    reprobe = np.zeros_like(counters)
    for a, spec in enumerate(suite):
        for p, j in enumerate(plan.columns):
            c, g = settings[j]
            ref.L.ref_sample_counters(ctypes.byref(spec), c, g, bind.P(counters[a, p]))
    reprobe[:] = counters
    reprobe[:, :, 2] *= 0.9  # the post-transition samples differ
    transition = (np.arange(napps) % 3 == 0).astype(np.int32)
    seeds = np.arange(napps, dtype=np.uint64) * 977 + 5
    hyper = ocg.NcfHyper(max_epochs=40, patience=10)
    res, est = online_ingest_complete_batch(block, np.ones_like(block, np.uint8), counters, seeds, grid, pred, hyper,
                                            reprobe_counters=reprobe, transition=transition, ctx=ctx)
    assert (res.status == 0).all(), res.status
    cpu, gpu = grid.arrays()
    ref.force_lane(1)
    for a in range(napps):
        use = reprobe[a] if transition[a] else counters[a]
        out = np.zeros(len(plan.columns))
        assert ref.L.ref_predict_perf(pj.encode(), bind.P(np.ascontiguousarray(use)), len(use), bind.P(out)) == 0
        np.testing.assert_array_equal(est[a], out)
        vals = np.vstack([block, np.zeros(grid.n)])
        mask = np.vstack([np.ones_like(block, np.uint8), np.zeros(grid.n, np.uint8)])
        vals[-1, plan.columns] = out
        mask[-1, plan.columns] = 1
        rc, done = ref.ncf_complete(vals, mask, cpu, gpu, int(seeds[a]), max_epochs=40, patience=10)
        assert rc == 0, ref.err()
        np.testing.assert_array_equal(res.completed[a], done[-1])
        rc, i2, s2, l2, n2 = ref.select_caps(done[-1:], cpu, gpu, 0.05)
        assert (res.idx[a], res.saving[a], res.loss[a], res.ncand[a]) == (i2[0], s2[0], l2[0], n2[0])


def test_ingest_invalid_counters_flag_the_app(ctx):
    import paper_2508_07605_b200 as ocg
    from paper_2508_07605_b200 import synth
    from paper_2508_07605_b200.online import online_ingest_complete_batch
    from paper_2508_07605_b200.predictor import Predictor, PredictorModel

    grid = ocg.PowerGrid.default_grid()
    block = synth.offline_block(42, grid)
    pred = Predictor(PredictorModel.from_json((GOLD / "predictor.json").read_text()), ctx=ctx)
    c = np.tile(np.array([150.0, 200.0, 1e9, 1e9, 1.5e9, 0.5, 0.4]), (3, 6, 1))
    c[1, 2, 5] = 1.5   # activity outside [0, 1] (validate_counters, core.cpp:80-82)
    res, _ = online_ingest_complete_batch(block, np.ones_like(block, np.uint8), c, np.arange(3, dtype=np.uint64),
                                          grid, pred, ocg.NcfHyper(max_epochs=5), ctx=ctx)
    assert list(res.status) == [0, ocg._lib.OCG_E_INVALID, 0]
