"""ALS completion + fused selection on the GPU vs the FP64 CPU oracle.

ALS has no reference counterpart (parity vs the reference: unpinned); the
oracle (oracle/ocg_oracle.c) defines it.  Bars:
  * factors / predictions: FP32 GPU vs FP64 oracle within PRED_RTOL;
  * selection: bit-exact w.r.t. the completed rows the kernel used
    (oracle select_caps on the GPU's completed rows);
  * end-to-end decisions: identical to the oracle's wherever the row's
    selection margin exceeds the prediction tolerance."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

PRED_RTOL = 2e-3  # FP32 ALS vs FP64 oracle, relative, on imputed cells


def _problem(m, nc, ng, density, dense_rows, seed):
    from paper_2508_07605_b200 import PowerGrid, synth

    grid = PowerGrid.spanning(nc, ng)
    return grid, synth.joint_csr(m, grid, density, dense_rows, seed=seed)


@pytest.mark.parametrize("k", [8, 16, 32, 64])
def test_als_factors_and_predictions_match_oracle(ctx, port, k):
    from oracle import bind
    from paper_2508_07605_b200.als import AlsHyper, AlsPlan

    grid, A = _problem(1500, 8, 16, 0.15, 4, seed=3)
    hyp = AlsHyper(rank=k, lam=0.003, sweeps=6, seed=11)
    plan = AlsPlan(A.m, A.row_ptr, A.col, A.val, grid, hyp, 0.05, ctx=ctx)
    plan.run()
    Ug, Vg = plan.factors()
    Uo, Vo = bind.als_fit(port, A.m, A.n, A.row_ptr, A.col, A.val, k, 0.003, 6, 11)
    Pg = np.clip(Ug.astype(np.float64) @ Vg.T.astype(np.float64), 0.01, 1.25)
    Po = np.clip(Uo @ Vo.T, 0.01, 1.25)
    rel = np.abs(Pg - Po) / Po
    assert np.quantile(rel, 0.999) < PRED_RTOL, (rel.max(), np.quantile(rel, 0.999))


@pytest.mark.parametrize("rank", [16, 32, 64])  # 32/64: tensor-core imputation + selection
@pytest.mark.parametrize("n_grid", [(8, 16), (16, 16), (64, 64), (10, 30)])
def test_als_fused_selection_exact_on_completed_rows(ctx, port, n_grid, rank):
    """The fused kernel's decision == policy::select_caps on the very rows it
    completed (bit-exact: index, saving, loss, candidates)."""
    from paper_2508_07605_b200.als import AlsHyper, AlsPlan

    m = 700 if n_grid[0] < 64 else 200
    grid, A = _problem(m, *n_grid, 0.05, 2, seed=5)
    plan = AlsPlan(A.m, A.row_ptr, A.col, A.val, grid, AlsHyper(rank=rank, sweeps=4), 0.05, ctx=ctx)
    plan.run()
    idx, sav, loss, nc = plan.results()
    rows = plan.completed_rows(0, A.m)
    # observed cells verbatim
    i = np.repeat(np.arange(A.m), np.diff(A.row_ptr))
    np.testing.assert_array_equal(rows[i, A.col], A.val.astype(np.float64))
    assert ((rows >= 0.01) & (rows <= 1.25)).all()
    cpu, gpu = grid.arrays()
    rc, i2, s2, l2, n2 = port.select_caps(rows, cpu, gpu, 0.05)
    assert rc == 0
    np.testing.assert_array_equal(idx, i2)
    np.testing.assert_array_equal(sav, s2)
    np.testing.assert_array_equal(loss, l2)
    np.testing.assert_array_equal(nc, n2)


@pytest.mark.parametrize("rank", [8, 32, 64])
def test_als_selection_ties_and_clamps(ctx, port, rank):
    """Rows engineered to hit the clamp floor/ceiling and exact saving ties."""
    from paper_2508_07605_b200.als import AlsHyper, AlsPlan
    from paper_2508_07605_b200 import PowerGrid

    grid = PowerGrid.spanning(4, 8)
    n = grid.n
    rng = np.random.default_rng(0)
    m = 400
    dense = rng.choice([0.01, 0.5, 0.9, 1.0, 1.25], size=(m, n))
    mask = rng.random((m, n)) < 0.7
    mask[:, -1] = True
    rp = np.zeros(m + 1, np.int64)
    rp[1:] = np.cumsum(mask.sum(1))
    ii, jj = np.nonzero(mask)
    col, val = jj.astype(np.int32), dense[ii, jj].astype(np.float32)
    plan = AlsPlan(m, rp, col, val, grid, AlsHyper(rank=rank, sweeps=3), 0.1, ctx=ctx)
    plan.run()
    idx, sav, loss, nc = plan.results()
    rows = plan.completed_rows(0, m)
    cpu, gpu = grid.arrays()
    rc, i2, s2, l2, n2 = port.select_caps(rows, cpu, gpu, 0.1)
    np.testing.assert_array_equal(idx, i2)
    np.testing.assert_array_equal(sav, s2)
    np.testing.assert_array_equal(loss, l2)
    np.testing.assert_array_equal(nc, n2)


@pytest.mark.parametrize("rank", [16, 32, 64])
def test_als_end_to_end_decisions_match_oracle_where_margin_allows(ctx, port, rank):
    from oracle import bind
    from paper_2508_07605_b200.als import AlsHyper, AlsPlan

    grid, A = _problem(2000, 16, 16, 0.05, 2, seed=9)
    hyp = AlsHyper(rank=rank, lam=0.003, sweeps=8, seed=2)
    plan = AlsPlan(A.m, A.row_ptr, A.col, A.val, grid, hyp, 0.05, ctx=ctx)
    plan.run()
    idx, sav, loss, nc = plan.results()
    Uo, Vo = bind.als_fit(port, A.m, A.n, A.row_ptr, A.col, A.val, rank, 0.003, 8, 2)
    rows_o = bind.als_completed_rows(Uo, Vo, A.row_ptr, A.col, A.val, np.arange(A.m))
    cpu, gpu = grid.arrays()
    rc, io_, so, lo, no = port.select_caps(rows_o, cpu, gpu, 0.05)
    # a row's decision is "safe" when no perturbation of its predictions within
    # the tolerance can change it: every other setting is either clearly worse
    # (saving below best - tol) or clearly invalid (loss above gamma + tol), and
    # the winner is clearly valid
    E = cpu[-1] + gpu[-1]
    caps = np.add.outer(cpu, gpu).ravel().astype(np.float64)
    sav_all = (E - caps[None, :] / rows_o) / E
    loss_all = 1.0 - rows_o / rows_o[:, -1:]
    tol = 4 * PRED_RTOL
    r = np.arange(A.m)
    best_s = sav_all[r, io_]
    other_ok = (sav_all < best_s[:, None] - tol) | (loss_all > 0.05 + tol)
    other_ok[r, io_] = True
    safe = other_ok.all(axis=1) & (loss_all[r, io_] < 0.05 - tol)
    assert safe.mean() > 0.5
    np.testing.assert_array_equal(idx[safe], io_[safe])
    agree = (idx == io_).mean()
    assert agree > 0.9, agree


def test_als_upload_refit_matches_fresh_plan(ctx):
    """ocg_als_plan_upload + run == a plan created on the new data (streaming refit)."""
    from paper_2508_07605_b200.als import AlsHyper, AlsPlan

    grid, A = _problem(900, 8, 16, 0.08, 2, seed=13)
    hyp = AlsHyper(rank=32, sweeps=3)
    plan = AlsPlan(A.m, A.row_ptr, A.col, A.val, grid, hyp, 0.05, ctx=ctx)
    plan.run()
    rng = np.random.default_rng(1)
    val2 = np.clip(A.val * rng.uniform(0.9, 1.1, A.val.shape), 0.01, 1.25).astype(np.float32)
    plan.upload(A.row_ptr, A.col, val2)
    plan.run()
    got = plan.results()
    plan.upload_compact(A.row_ptr, A.col.astype(np.uint16), val2)  # 16-bit column indices
    plan.run()
    for g_, c_ in zip(got, plan.results()):
        np.testing.assert_array_equal(g_, c_)
    fresh = AlsPlan(A.m, A.row_ptr, A.col, val2, grid, hyp, 0.05, ctx=ctx)
    fresh.run()
    want = fresh.results()
    for g_, w_ in zip(got, want):
        np.testing.assert_array_equal(g_, w_)
    # streaming arrival (nnz grows): one new observation in 1% of the rows
    from paper_2508_07605_b200 import stream

    B = stream.add_observations(A, grid, frac=0.01, seed=5)
    assert B.nnz > A.nnz
    plan.upload(B.row_ptr, B.col, B.val)
    plan.run()
    got = plan.results()
    fresh = AlsPlan(B.m, B.row_ptr, B.col, B.val, grid, hyp, 0.05, ctx=ctx)
    fresh.run()
    for g_, w_ in zip(got, fresh.results()):
        np.testing.assert_array_equal(g_, w_)
    # warm refit (flagged deviation): starts from the previous factors, still a valid fit
    plan.set_warm(2)
    plan.upload(A.row_ptr, A.col, A.val)
    plan.run()
    idx, sav, loss, nc = plan.results()
    assert (idx >= 0).all() and (nc >= 1).all()


def test_als_rank32_multisegment_rows_and_empty_items(ctx, port):
    """Rank 32 (tensor-core path) with rows longer than one segment (dense rows over
    2048 settings -> 2 segments, reduced in segment order), a column nobody observed
    (zero factor, like ocgo_als_fit) and an app row with no observations.  Such a
    matrix is rejected for decisions (test_gpu_als_validation.py); the factors stay
    inspectable and match the oracle."""
    from oracle import bind
    from paper_2508_07605_b200 import PowerGrid
    from paper_2508_07605_b200.als import AlsHyper, AlsPlan

    grid = PowerGrid.spanning(64, 32)
    n = grid.n
    rng = np.random.default_rng(7)
    m = 300
    mask = rng.random((m, n)) < 0.03
    mask[:3, :] = True        # dense rows: 2048 observations = 2 segments
    mask[:, 5] = False        # cold column
    mask[10, :] = False       # app without observations
    mask[3:, -1] = True       # baseline observed elsewhere
    mask[10, :] = False
    vals = rng.uniform(0.2, 1.2, (m, n))
    rp = np.zeros(m + 1, np.int64)
    rp[1:] = np.cumsum(mask.sum(1))
    ii, jj = np.nonzero(mask)
    col, val = jj.astype(np.int32), vals[ii, jj].astype(np.float32)
    hyp = AlsHyper(rank=32, lam=0.003, sweeps=4, seed=5)
    plan = AlsPlan(m, rp, col, val, grid, hyp, 0.05, ctx=ctx)
    plan.run()
    Ug, Vg = plan.factors()
    Uo, Vo = bind.als_fit(port, m, n, rp, col, val, 32, 0.003, 4, 5)
    assert np.all(Vg[5] == 0) and np.all(Ug[10] == 0)
    assert np.all(Vo[5] == 0) and np.all(Uo[10] == 0)
    Pg = np.clip(Ug.astype(np.float64) @ Vg.T.astype(np.float64), 0.01, 1.25)
    Po = np.clip(Uo @ Vo.T, 0.01, 1.25)
    rel = np.abs(Pg - Po) / Po
    assert np.quantile(rel, 0.999) < PRED_RTOL, (rel.max(), np.quantile(rel, 0.999))


@pytest.mark.parametrize("rank", [16, 32])
def test_als_add_observations_matches_merged_upload(ctx, rank):
    """ocg_als_plan_add_observations (device-side merge of new cells) == a plan on the
    merged CSR: same factors and decisions, bit for bit; bad arrivals are rejected
    and leave the plan usable."""
    from paper_2508_07605_b200 import stream
    from paper_2508_07605_b200.als import AlsHyper, AlsPlan

    grid, A = _problem(1200, 8, 16, 0.1, 3, seed=17)
    hyp = AlsHyper(rank=rank, sweeps=3)
    plan = AlsPlan(A.m, A.row_ptr, A.col, A.val, grid, hyp, 0.05, ctx=ctx)
    plan.run()
    B, (r, c, v) = stream.add_observations(A, grid, frac=0.05, seed=9, return_delta=True)
    plan.add_observations(r, c, v)
    plan.run()
    fresh = AlsPlan(B.m, B.row_ptr, B.col, B.val, grid, hyp, 0.05, ctx=ctx)
    fresh.run()
    for g_, w_ in zip(plan.factors(), fresh.factors()):
        np.testing.assert_array_equal(g_, w_)
    for g_, w_ in zip(plan.results(), fresh.results()):
        np.testing.assert_array_equal(g_, w_)
    # a second arrival on top of the first
    C, (r2, c2, v2) = stream.add_observations(B, grid, frac=0.02, seed=10, return_delta=True)
    plan.add_observations(r2, c2, v2)
    plan.run()
    fresh = AlsPlan(C.m, C.row_ptr, C.col, C.val, grid, hyp, 0.05, ctx=ctx)
    fresh.run()
    for g_, w_ in zip(plan.results(), fresh.results()):
        np.testing.assert_array_equal(g_, w_)
    # rejected: an observed cell, unsorted cells, out-of-range column
    row0 = int(np.nonzero(np.diff(C.row_ptr) > 0)[0][0])
    for bad in ((np.array([row0]), np.array([C.col[C.row_ptr[row0]]]), np.array([0.5])),
                (np.array([5, 4]), np.array([0, 0]), np.array([0.5, 0.5])),
                (np.array([0]), np.array([grid.n]), np.array([0.5]))):
        with pytest.raises(Exception):
            plan.add_observations(*bad)
    plan.run()
    for g_, w_ in zip(plan.results(), fresh.results()):
        np.testing.assert_array_equal(g_, w_)


def test_als_stage_compact_pipelined_matches_upload(ctx):
    """ocg_als_plan_stage_compact (side-stream copy, swapped in by the next run) gives the
    same decisions as a synchronous upload, also when the next CSR is staged while the
    current run is still in flight, and when its nnz differs."""
    from paper_2508_07605_b200 import stream
    from paper_2508_07605_b200.als import AlsHyper, AlsPlan

    grid, A = _problem(1500, 8, 16, 0.1, 3, seed=23)
    B = stream.add_observations(A, grid, frac=0.2, seed=4)
    hyp = AlsHyper(rank=32, sweeps=3)
    want = {}
    for name, M in (("A", A), ("B", B)):
        p = AlsPlan(M.m, M.row_ptr, M.col, M.val, grid, hyp, 0.05, ctx=ctx)
        p.run()
        want[name] = p.results()
        p.close()
    plan = AlsPlan(A.m, A.row_ptr, A.col, A.val, grid, hyp, 0.05, ctx=ctx)
    seq = ["B", "A", "B", "B", "A"]
    mats = {"A": A, "B": B}
    plan.stage_compact(B.row_ptr, B.col.astype(np.uint16), B.val)
    with pytest.raises(Exception):  # one staged CSR at a time
        plan.stage_compact(A.row_ptr, A.col.astype(np.uint16), A.val)
    keep = []
    for i, name in enumerate(seq):
        plan.run(timed=False)
        if i + 1 < len(seq):  # stage the next input while this run is in flight
            M = mats[seq[i + 1]]
            arrs = (M.row_ptr.copy(), M.col.astype(np.uint16), M.val.copy())
            keep.append(arrs)
            plan.stage_compact(*(int(x.ctypes.data) for x in arrs))
        for g_, w_ in zip(plan.results(), want[name]):
            np.testing.assert_array_equal(g_, w_)


@pytest.mark.parametrize("k", [16, 32])
def test_als_csc_packed_keys_identical_to_pair_sort(ctx, k, monkeypatch):
    """The packed 32-bit-key CSC build (col << rb | row, default when m and n fit) and the
    64-bit-payload radix sort (OCG_CSC_PAIRS=1) give the same CSC, so the fits are
    bit-identical; includes fully observed rows and an empty row (which makes the
    matrix invalid for decisions, as cf::complete refuses it; the factors compare)."""
    import paper_2508_07605_b200 as ocg
    from paper_2508_07605_b200.als import AlsHyper, AlsPlan
    from paper_2508_07605_b200.synth import CsrMatrix

    grid, A = _problem(2500, 8, 16, 0.2, 5, seed=29)
    keep = np.ones(A.nnz, bool)
    keep[A.row_ptr[11]:A.row_ptr[12]] = False
    cnt = np.diff(A.row_ptr).copy()
    cnt[11] = 0
    A = CsrMatrix(A.m, A.n, np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64), A.col[keep], A.val[keep])
    hyp = AlsHyper(rank=k, lam=0.003, sweeps=3, seed=5)
    out = []
    for forced in ("0", "1"):
        monkeypatch.setenv("OCG_CSC_PAIRS", forced)
        plan = AlsPlan(A.m, A.row_ptr, A.col, A.val, grid, hyp, 0.05, ctx=ctx)
        plan.run()
        out.append(plan.factors())
        with pytest.raises(ocg.InvalidArgument):
            plan.results()
        plan.close()
    for a, b in zip(out[0], out[1]):
        np.testing.assert_array_equal(a, b)


def test_als_results_async_matches_results(ctx):
    """ocg_als_plan_results_async + _results_wait (copies queued behind the run, the next run
    queued right after) return what the synchronous ocg_als_plan_results returns."""
    import torch

    from paper_2508_07605_b200.als import AlsHyper, AlsPlan

    grid, A = _problem(1000, 8, 16, 0.1, 2, seed=31)
    plan = AlsPlan(A.m, A.row_ptr, A.col, A.val, grid, AlsHyper(rank=32, sweeps=3), 0.05, ctx=ctx)
    plan.run(timed=False)
    want = plan.results()
    outs = [torch.empty(A.m, dtype=dt).pin_memory() for dt in (torch.int32, torch.float64, torch.float64,
                                                                torch.int32)]
    plan.results_async([int(x.data_ptr()) for x in outs])
    plan.run(timed=False)  # queued behind the copy: must not disturb it
    plan.results_wait()
    for g_, w_ in zip(outs, want):
        np.testing.assert_array_equal(g_.numpy(), w_)
    plan.results_wait()  # the second run (same inputs) gives the same decisions
    for g_, w_ in zip(plan.results(), want):
        np.testing.assert_array_equal(g_, w_)
