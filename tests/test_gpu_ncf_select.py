"""Fused NCF completion + selection over a whole matrix (ocg_ncf_plan_*) vs the
reference library itself (oracle/_ref: NcfModel::from_json + NcfModel::predict
of every unobserved cell + policy::select_caps, cfcomplete.cpp:47-58, :208-211,
policy.cpp:17-64).

Bars:
  * EXACT precision: completed values and decisions (index, saving, loss,
    candidates) bit-identical to the reference, both kernel lanes;
  * FAST precision (FP32 + tcgen05): |p - p_ref| <= FAST_RTOL * max(p_ref, P_FLOOR)
    on every imputed cell, i.e. relative 1e-5 for p >= 0.1 and 1e-6 absolute
    below (FP32 carries ~3e-7 absolute error through the MLP's O(1)
    intermediates, so small outputs lose relative accuracy to cancellation);
    the decision identical wherever the row's selection margin exceeds the
    tolerance propagated through Algorithm 2."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FAST_RTOL = 1e-5
P_FLOOR = 0.1


def _fast_err(comp, c_ref):
    """max of |dp| / max(p_ref, P_FLOOR) (the FAST contract), and the plain max |dp|/p."""
    d = np.abs(comp - c_ref)
    return (d / np.maximum(c_ref, P_FLOOR)).max(), (d / c_ref).max()


def _dense(A):
    vals = np.zeros((A.m, A.n))
    mask = np.zeros((A.m, A.n), np.uint8)
    i = np.repeat(np.arange(A.m), np.diff(A.row_ptr))
    vals[i, A.col] = A.val
    mask[i, A.col] = 1
    return vals, mask


def _problem(m, nc, ng, density, dense_rows, k, seed, emb_scale=0.6):
    from paper_2508_07605_b200 import PowerGrid, synth
    from paper_2508_07605_b200.ncf import random_model

    grid = PowerGrid.spanning(nc, ng)
    A = synth.joint_csr(m, grid, density, dense_rows, seed=seed, dtype=np.float64)
    model = random_model(m, grid.n, k, seed=seed + 1, emb_scale=emb_scale)
    return grid, A, model


def _reference(ref, model, A, grid, rows, lane, threads=None):
    from oracle import bind

    ref.force_lane(lane)
    vals, mask = _dense(A)
    k = model.hyper.app_dim
    sub = bind.sub_model_params(model.params, model.m, model.n, k, k, rows)
    cpu, gpu = grid.arrays()
    rc, comp, idx, sv, lo, nc, _ = ref.ncf_complete_select_rows(
        k, k, model.hyper.hidden, sub, model.app_seen[rows], model.setting_seen, cpu, gpu, vals[rows], mask[rows],
        0.05, threads or min(32, os.cpu_count() or 1))
    assert rc == 0, ref.err()
    return comp, idx, sv, lo, nc


def _margin_safe(comp_ref, grid, gamma, tol):
    """Rows whose Algorithm-2 decision cannot change under a perturbation
    |dp| <= tol * max(p, P_FLOOR) of every non-baseline completed value (the
    baseline is exact in both modes): the winner is valid with margin, and it
    beats every cell that is or might be valid (|loss - gamma| within the
    perturbation) by more than the perturbation of the savings."""
    cpu, gpu = grid.arrays()
    cs = (cpu[:, None] + gpu[None, :]).ravel().astype(np.float64)
    e_base = float(cpu[-1] + gpu[-1])
    pb = comp_ref[:, -1:]
    dp = tol * np.maximum(comp_ref, P_FLOOR)
    dp[:, -1] = 0.0
    loss = 1.0 - comp_ref / pb
    dl = 2 * dp / pb + 1e-15
    sav = (e_base - cs[None, :] / comp_ref) / e_base
    dsav = 2 * cs[None, :] * dp / comp_ref ** 2 / e_base + 1e-15
    maybe = loss <= gamma + dl
    sure = loss <= gamma - dl
    hi = np.where(maybe, sav + dsav, -np.inf)  # optimistic savings of every possible candidate
    w = np.argmax(np.where(maybe, sav, -np.inf), axis=1)
    r = np.arange(len(w))
    lo_w = sav[r, w] - dsav[r, w]
    hi[r, w] = -np.inf
    return sure[r, w] & (lo_w > hi.max(axis=1))


@pytest.mark.parametrize("lane", [0, 1])
@pytest.mark.parametrize("k", [8, 32])
def test_exact_bit_identical_to_reference(ctx, ref, lane, k):
    from paper_2508_07605_b200.ncf import EXACT, DeviceNcfModel, NcfPlan

    grid, A, model = _problem(400, 8, 16, 0.08, 3, k, seed=7 + k)
    dm = DeviceNcfModel(model, ctx=ctx)
    plan = NcfPlan(dm, A.row_ptr, A.col, A.val, grid, 0.05, EXACT, lane)
    plan.run()
    idx, sv, lo, nc = plan.results(A.m)
    rows = np.arange(A.m)
    comp = plan.completed_rows(rows)
    c_ref, i_ref, s_ref, l_ref, n_ref = _reference(ref, model, A, grid, rows, lane)
    np.testing.assert_array_equal(comp, c_ref)
    np.testing.assert_array_equal(idx, i_ref)
    np.testing.assert_array_equal(sv, s_ref)
    np.testing.assert_array_equal(lo, l_ref)
    np.testing.assert_array_equal(nc, n_ref)


@pytest.mark.parametrize("ngrid", [(8, 16), (16, 16), (10, 30), (64, 64)])
def test_fast_within_tolerance(ctx, ref, ngrid):
    from paper_2508_07605_b200.ncf import FAST, DeviceNcfModel, NcfPlan

    m = 300 if ngrid[0] < 64 else 130
    grid, A, model = _problem(m, *ngrid, 0.05, 2, 32, seed=ngrid[0] + ngrid[1])
    dm = DeviceNcfModel(model, ctx=ctx)
    plan = NcfPlan(dm, A.row_ptr, A.col, A.val, grid, 0.05, FAST, 1)
    plan.run()
    idx, sv, lo, nc = plan.results(A.m)
    rows = np.arange(A.m)
    comp = plan.completed_rows(rows)
    c_ref, i_ref, s_ref, l_ref, n_ref = _reference(ref, model, A, grid, rows, 1)
    vals, mask = _dense(A)
    np.testing.assert_array_equal(comp[mask == 1], c_ref[mask == 1])  # observed cells verbatim
    np.testing.assert_array_equal(comp[:, -1], c_ref[:, -1])            # baselines exact in both modes
    err, rel = _fast_err(comp, c_ref)
    assert err <= FAST_RTOL, (err, rel)
    safe = _margin_safe(c_ref, grid, 0.05, FAST_RTOL)
    assert safe.mean() > 0.5, safe.mean()
    np.testing.assert_array_equal(idx[safe], i_ref[safe])
    np.testing.assert_allclose(sv[safe], s_ref[safe], rtol=0, atol=1e-4)
    # the fused decision is exactly select_caps on the rows the kernel completed
    from oracle import bind

    port = bind.Port()
    cpu, gpu = grid.arrays()
    rc, i2, s2, l2, n2 = port.select_caps(comp, cpu, gpu, 0.05)
    assert rc == 0
    np.testing.assert_array_equal(idx, i2)
    np.testing.assert_array_equal(sv, s2)
    np.testing.assert_array_equal(lo, l2)
    np.testing.assert_array_equal(nc, n2)


def test_reference_fitted_model_file(ctx, ref):
    """A model fitted by the reference (cf::fit) and loaded from its own model
    file completes its matrix exactly as cf::complete does."""
    from paper_2508_07605_b200 import PowerGrid
    from paper_2508_07605_b200.ncf import EXACT, FAST, DeviceNcfModel, NcfPlan

    grid = PowerGrid.spanning(5, 6)
    rng = np.random.default_rng(3)
    m, n = 40, grid.n
    vals = rng.uniform(0.2, 1.2, (m, n))
    mask = (rng.random((m, n)) < 0.3).astype(np.uint8)
    mask[:, 0] = 1
    cpu, gpu = grid.arrays()
    ref.force_lane(1)
    rc, text, meta = ref.ncf_fit(vals, mask, cpu, gpu, 99, max_epochs=40, patience=10)
    assert rc == 0, ref.err()
    rc, full = ref.ncf_complete(vals, mask, cpu, gpu, 99, max_epochs=40, patience=10)
    assert rc == 0
    rcs, i_ref, s_ref, l_ref, n_ref = ref.select_caps(full, cpu, gpu, 0.05)
    i = np.nonzero(mask)
    row_ptr = np.concatenate([[0], np.cumsum(mask.sum(1))]).astype(np.int64)
    col = i[1].astype(np.int32)
    val = vals[i]
    dm = DeviceNcfModel(json_text=text, ctx=ctx)
    plan = NcfPlan(dm, row_ptr, col, val, grid, 0.05, EXACT, 1)
    plan.run()
    idx, sv, lo, nc = plan.results(m)
    np.testing.assert_array_equal(plan.completed_rows(np.arange(m)), full)
    np.testing.assert_array_equal(idx, i_ref)
    np.testing.assert_array_equal(sv, s_ref)
    fplan = NcfPlan(dm, row_ptr, col, val, grid, 0.05, FAST, 1)
    fplan.run()
    err, rel = _fast_err(fplan.completed_rows(np.arange(m)), full)
    assert err <= FAST_RTOL, (err, rel)


def test_errors_follow_reference_exceptions(ctx):
    from paper_2508_07605_b200 import ColdError, InvalidArgument, OutOfRange, PowerGrid
    from paper_2508_07605_b200.ncf import EXACT, FAST, DeviceNcfModel, NcfPlan, random_model

    grid = PowerGrid.spanning(4, 4)
    m, n = 6, grid.n
    model = random_model(m, n, 8, seed=1)
    row_ptr = np.arange(0, 2 * m + 1, 2, dtype=np.int64)
    col = np.tile(np.array([0, n - 1], np.int32), m)
    val = np.full(2 * m, 0.7)

    def run(rp, c, v, mdl=model, prec=EXACT):
        dm = DeviceNcfModel(mdl, ctx=ctx)
        p = NcfPlan(dm, rp, c, v, grid, 0.05, prec, 1)
        p.run()
        return p.results(m)

    for prec in (EXACT, FAST):
        idx, *_ = run(row_ptr, col, val, prec=prec)
        assert (idx >= 0).all()
    rp = row_ptr.copy()
    rp[3:] -= 2  # row 2 without observations (cfcomplete.cpp:199-205)
    with pytest.raises(InvalidArgument):
        run(rp, col[:-2], val[:-2])
    bad = val.copy()
    bad[5] = 1.3  # outside (0, 1.25] (core.cpp:145-147)
    with pytest.raises(InvalidArgument):
        run(row_ptr, col, bad)
    c2 = col.copy()
    c2[1] = n  # column index out of range
    with pytest.raises(OutOfRange):
        run(row_ptr, c2, val)
    cold = random_model(m, n, 8, seed=1)
    cold.setting_seen[5] = 0  # cold setting column with unobserved cells (cfcomplete.cpp:53-55)
    with pytest.raises(ColdError):
        run(row_ptr, col, val, mdl=cold)
    cold = random_model(m, n, 8, seed=1)
    cold.app_seen[2] = 0  # cold app row (:50-52)
    with pytest.raises(ColdError):
        run(row_ptr, col, val, mdl=cold)


@pytest.mark.parametrize("precision", ["exact", "fast"])
def test_c2_scale_sampled_rows_match_reference(ctx, ref, precision):
    """The BASELINE C2 configuration (1M apps x 4096 settings, rank 32, 2 %
    observed, 1K dense rows) completed + selected on the device; 2000 sampled
    rows (incl. dense rows) checked against the reference."""
    from paper_2508_07605_b200 import PowerGrid, synth
    from paper_2508_07605_b200.ncf import EXACT, FAST, DeviceNcfModel, NcfPlan, random_model

    m = int(os.environ.get("OCG_C2_ROWS", 1_000_000))
    grid = PowerGrid.spanning(64, 64)
    A = synth.joint_csr(m, grid, 0.02, max(1, m // 1000), seed=42, dtype=np.float64)
    model = random_model(m, grid.n, 32, seed=5, emb_scale=0.6)
    dm = DeviceNcfModel(model, ctx=ctx)
    prec = EXACT if precision == "exact" else FAST
    plan = NcfPlan(dm, A.row_ptr, A.col, A.val, grid, 0.05, prec, 1)
    plan.run()
    idx, sv, lo, nc = plan.results(A.m)
    assert (idx >= 0).all()
    rng = np.random.default_rng(11)
    rows = np.unique(np.concatenate([np.arange(4), rng.choice(A.m, 1996, replace=False)]))
    comp = plan.completed_rows(rows)
    sub_rp = np.concatenate([[0], np.cumsum(np.diff(A.row_ptr)[rows])]).astype(np.int64)
    sub_col = np.concatenate([A.col[A.row_ptr[r]:A.row_ptr[r + 1]] for r in rows])
    sub_val = np.concatenate([A.val[A.row_ptr[r]:A.row_ptr[r + 1]] for r in rows])
    sub = synth.CsrMatrix(len(rows), A.n, sub_rp, sub_col, sub_val)
    from oracle import bind

    ref.force_lane(1)
    vals, mask = _dense(sub)
    sp = bind.sub_model_params(model.params, model.m, model.n, 32, 32, rows)
    cpu, gpu = grid.arrays()
    rc, c_ref, i_ref, s_ref, l_ref, n_ref, _ = ref.ncf_complete_select_rows(
        32, 32, model.hyper.hidden, sp, model.app_seen[rows], model.setting_seen, cpu, gpu, vals, mask, 0.05,
        min(32, os.cpu_count() or 1))
    assert rc == 0, ref.err()
    if precision == "exact":
        np.testing.assert_array_equal(comp, c_ref)
        np.testing.assert_array_equal(idx[rows], i_ref)
        np.testing.assert_array_equal(sv[rows], s_ref)
        np.testing.assert_array_equal(lo[rows], l_ref)
        np.testing.assert_array_equal(nc[rows], n_ref)
    else:
        err, rel = _fast_err(comp, c_ref)
        print(f"C2 fast: max |dp|/max(p, {P_FLOOR}) = {err:.3g}, max |dp|/p = {rel:.3g}")
        assert err <= FAST_RTOL, (err, rel)
        safe = _margin_safe(c_ref, grid, 0.05, FAST_RTOL)
        assert safe.mean() > 0.5, safe.mean()
        np.testing.assert_array_equal(idx[rows][safe], i_ref[safe])


def test_pipelined_stage_and_async_results_match_sync(ctx):
    """ocg_ncf_plan_stage + _results_async/_wait (the next CSR staged on a side stream while the
    current step runs) give the decisions the synchronous upload + run + results give, step by step."""
    import torch

    from paper_2508_07605_b200 import PowerGrid, synth
    from paper_2508_07605_b200.ncf import FAST, DeviceNcfModel, NcfPlan, random_model

    grid = PowerGrid.spanning(16, 16)
    mats = [synth.joint_csr(3000, grid, 0.05 + 0.01 * k, 3, seed=40 + k, dtype=np.float64) for k in range(3)]
    model = random_model(3000, grid.n, 8, seed=1, emb_scale=0.6)
    dm = DeviceNcfModel(model, ctx=ctx)
    want = []
    for A in mats:
        p = NcfPlan(dm, A.row_ptr, A.col, A.val, grid, 0.05, FAST)
        p.run(timed=False)
        want.append(p.results(A.m))
        p.close()
    pins = [[torch.from_numpy(x).pin_memory() for x in (A.row_ptr, A.col, A.val)] for A in mats]
    out = [torch.empty(3000, dtype=dt).pin_memory() for dt in (torch.int32, torch.float64, torch.float64, torch.int32)]
    plan = NcfPlan(dm, mats[0].row_ptr, mats[0].col, mats[0].val, grid, 0.05, FAST)
    order = [0, 1, 2, 1, 0, 2]
    plan.stage(*(int(x.data_ptr()) for x in pins[order[0]]))
    plan.run(timed=False)
    for i, k in enumerate(order):
        if i + 1 < len(order):
            plan.stage(*(int(x.data_ptr()) for x in pins[order[i + 1]]))
        plan.results_async([int(x.data_ptr()) for x in out])
        if i + 1 < len(order):
            plan.run(timed=False)
        plan.results_wait()
        for got, exp in zip(out, want[k]):
            np.testing.assert_array_equal(got.numpy(), exp)
    plan.close()
    dm.close()
