"""ALS plan input validation on the device (the checks the reference applies to
the same matrix: PerformanceMatrix::set core.cpp:142-148, cf::complete
cfcomplete.cpp:199-205, the cold-column rule :53-55), reported as the reference's
exception kind by results(); bad entries never reach the fit out of bounds."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _csr():
    from paper_2508_07605_b200 import PowerGrid, synth

    grid = PowerGrid.spanning(8, 8)
    A = synth.joint_csr(300, grid, 0.1, 2, seed=7)
    return grid, A


def _run(ctx, grid, rp, col, val, upload=False):
    from paper_2508_07605_b200.als import AlsHyper, AlsPlan

    if upload:
        _, A = _csr()
        plan = AlsPlan(len(rp) - 1, A.row_ptr, A.col, A.val, grid, AlsHyper(rank=32, sweeps=2), 0.05, ctx=ctx)
        plan.run()
        plan.results()
        plan.upload(rp, col, val)
    else:
        plan = AlsPlan(len(rp) - 1, rp, col, val, grid, AlsHyper(rank=32, sweeps=2), 0.05, ctx=ctx)
    plan.run()
    return plan


@pytest.mark.parametrize("upload", [False, True])
@pytest.mark.parametrize("kind", ["range", "neg", "zero", "big", "nan", "unsorted", "empty_row", "cold"])
def test_als_rejects_like_the_reference(ctx, kind, upload):
    import paper_2508_07605_b200 as ocg

    grid, A = _csr()
    rp, col, val = A.row_ptr.copy(), A.col.copy(), A.val.copy()
    exc = ocg.InvalidArgument
    if kind == "range":
        col[rp[5] + 1] = grid.n + 3
        exc = ocg.OutOfRange
    elif kind == "neg":
        col[rp[9]] = -1
        exc = ocg.OutOfRange
    elif kind == "zero":
        val[17] = 0.0
    elif kind == "big":
        val[40] = 1.3
    elif kind == "nan":
        val[3] = np.nan
    elif kind == "unsorted":
        q = rp[20]
        col[q], col[q + 1] = col[q + 1], col[q]
    elif kind == "empty_row":  # drop every observation of row 30
        keep = np.ones(len(col), bool)
        keep[rp[30]:rp[31]] = False
        col, val = col[keep], val[keep]
        cnt = np.diff(rp)
        cnt[30] = 0
        rp = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
    elif kind == "cold":  # setting column 3 never observed
        keep = col != 3
        rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))[keep]
        col, val = col[keep], val[keep]
        rp = np.concatenate([[0], np.cumsum(np.bincount(rows, minlength=len(rp) - 1))]).astype(np.int64)
        exc = ocg.ColdError
    plan = _run(ctx, grid, rp, col, val, upload)
    with pytest.raises(exc):
        plan.results()
    with pytest.raises(exc):
        plan.completed_rows(0, 4)


def test_als_rejects_bad_row_ptr_and_grid(ctx):
    import paper_2508_07605_b200 as ocg
    from paper_2508_07605_b200 import PowerGrid
    from paper_2508_07605_b200.als import AlsHyper, AlsPlan

    grid, A = _csr()
    rp = A.row_ptr.copy()
    rp[10], rp[11] = rp[11], rp[10]
    with pytest.raises(ocg.InvalidArgument):
        AlsPlan(A.m, rp, A.col, A.val, grid, AlsHyper(rank=16), 0.05, ctx=ctx)
    bad = PowerGrid.__new__(PowerGrid)  # bypass the Python-side check: the C side must refuse too
    object.__setattr__(bad, "cpu_caps", (100, 90, 120, 130, 140, 150, 160, 170))
    object.__setattr__(bad, "gpu_caps", grid.gpu_caps)
    with pytest.raises(ocg.InvalidArgument):
        AlsPlan(A.m, A.row_ptr, A.col, A.val, bad, AlsHyper(rank=16), 0.05, ctx=ctx)


def test_als_valid_input_still_runs_after_a_rejected_one(ctx):
    grid, A = _csr()
    val = A.val.copy()
    val[0] = 2.0
    plan = _run(ctx, grid, A.row_ptr, A.col, val)
    import paper_2508_07605_b200 as ocg

    with pytest.raises(ocg.InvalidArgument):
        plan.results()
    plan.upload(A.row_ptr, A.col, A.val)
    plan.run()
    idx, *_ = plan.results()
    assert (idx >= 0).all()
