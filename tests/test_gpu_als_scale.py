"""ALS at C2 scale (VERDICT r1 "C2-scale code paths are untested"): a 200K x 4096
matrix at 2 % with 200 dense rows and the always-observed default-plan columns
(~200K observations each: hundreds of segments, the level-2 group reduce, the
band-strided segment order) — every half-sweep's output is checked against the
FP64 oracle solving the SAME inputs (the GPU's own previous factors) on sampled
rows (dense ones included) and columns (the baseline and plan columns included),
with a MAX bound on the relative difference of the predictions they imply."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
K, LAM = 32, 0.003
MAX_REL = 2e-3


def _csc_cols(A, cols):
    """CSC of the selected columns (rows ascending), as the oracle's column solve takes it."""
    rows = np.repeat(np.arange(A.m, dtype=np.int32), np.diff(A.row_ptr))
    cp, crow, cval = [0], [], []
    for j in cols:
        sel = A.col == j
        crow.append(rows[sel])
        cval.append(A.val[sel].astype(np.float32))
        cp.append(cp[-1] + int(sel.sum()))
    return np.asarray(cp, np.int64), np.concatenate(crow).astype(np.int32), np.concatenate(cval)


def _check_rows(port, A, rows, V, U_gpu):
    from oracle.bind import P

    rp = np.concatenate([[0], np.cumsum(np.diff(A.row_ptr)[rows])]).astype(np.int64)
    col = np.concatenate([A.col[A.row_ptr[i]:A.row_ptr[i + 1]] for i in rows]).astype(np.int32)
    val = np.concatenate([A.val[A.row_ptr[i]:A.row_ptr[i + 1]] for i in rows]).astype(np.float32)
    Vd = np.ascontiguousarray(V, np.float64)
    Uo = np.zeros((len(rows), K))
    port.L.ocgo_als_solve_rows(len(rows), P(rp), P(col), P(val), P(Vd), P(Uo), K, LAM)
    po = np.clip(Uo @ Vd.T, 0.01, 1.25)
    pg = np.clip(U_gpu[rows].astype(np.float64) @ Vd.T, 0.01, 1.25)
    return float(np.max(np.abs(pg - po) / po))


def _check_cols(port, A, cols, U, V_gpu, prow):
    from oracle.bind import P

    cp, crow, cval = _csc_cols(A, cols)
    Ud = np.ascontiguousarray(U, np.float64)
    G = np.zeros(len(cols) * (K * K + K + 1))
    port.L.ocgo_als_col_gram(len(cols), P(cp), P(crow), P(cval), P(Ud), K, P(G))
    Vo = np.zeros((len(cols), K))
    port.L.ocgo_als_solve_from_gram(len(cols), P(G), P(Vo), K, LAM)
    po = np.clip(Ud[prow] @ Vo.T, 0.01, 1.25)
    pg = np.clip(Ud[prow] @ V_gpu[cols].astype(np.float64).T, 0.01, 1.25)
    return float(np.max(np.abs(pg - po) / po)), np.diff(cp)


def test_als_c2_scale_half_sweeps_match_oracle(ctx, port):
    import paper_2508_07605_b200._lib as L
    from paper_2508_07605_b200 import PowerGrid, ProbePlan, synth
    from paper_2508_07605_b200.als import AlsHyper, AlsPlan

    grid = PowerGrid.spanning(64, 64)
    m = 200_000
    A = synth.joint_csr(m, grid, 0.02, 200, seed=42)
    plan = AlsPlan(m, A.row_ptr, A.col, A.val, grid, AlsHyper(rank=K, lam=LAM, sweeps=1, seed=42), 0.05, ctx=ctx)
    rng = np.random.default_rng(1)
    rows = np.concatenate([np.arange(0, 200, 10), rng.choice(np.arange(200, m), 300, replace=False)])
    plan_cols = ProbePlan.default_plan(grid).columns
    cols = np.unique(np.concatenate([plan_cols, [grid.n - 1], rng.choice(grid.n, 40, replace=False)]))
    prow = rng.choice(m, 400, replace=False)
    L.check(L.lib.ocg_als_plan_begin(plan._h))
    worst = []
    for sweep in range(3):
        _, V_prev = plan.factors()
        L.check(L.lib.ocg_als_plan_row_half(plan._h))
        U, _ = plan.factors()
        worst.append(("rows", sweep, _check_rows(port, A, rows, V_prev, U)))
        L.check(L.lib.ocg_als_plan_col_half(plan._h))
        U2, V = plan.factors()
        np.testing.assert_array_equal(U2, U)
        err, counts = _check_cols(port, A, cols, U, V, prow)
        worst.append(("cols", sweep, err))
    assert counts.max() > 150_000  # the baseline / plan columns: ~m observations each
    print("\nmax rel prediction diff per half-sweep:", [(s, i, f"{e:.2e}") for s, i, e in worst])
    assert max(e for *_, e in worst) < MAX_REL, worst
    plan.close()
