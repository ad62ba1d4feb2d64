"""Model-agnostic ALS checks (parity contract item 5): ALS has no
reference counterpart, so besides the FP64 oracle (test_gpu_als.py) the device
fit is pinned against matrices whose completion is known exactly:
  * rank-1 noiseless data p_ij = u_i v_j is recovered on the unobserved cells;
  * a constant matrix completes to the constant;
  * column-mean dominance: p_ij = c_j (every app the same profile) completes each
    unobserved cell to its column's value.
Every row and column is observed well beyond the rank (a rank-k fit of fewer
observations is not identifiable), and the fit runs 100 sweeps (the FP64 oracle needs
as many on these matrices).  The tolerance covers FP32 arithmetic and the
lambda * n_i ridge bias at lambda = 1e-5."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

# relative error over the unobserved cells (measured on B200 at 100 sweeps: max <= 2.4e-4,
# median <= 3.5e-5 across these cases)
MAX = 1e-3
MEDIAN = 1e-4


def _check(rel):
    med = np.median(rel)
    print(f"rel err: median {med:.2e}  max {rel.max():.2e}")
    assert rel.max() < MAX and med < MEDIAN, (med, rel.max())


def _csr_from_dense(P, mask):
    from paper_2508_07605_b200.synth import CsrMatrix

    m, n = P.shape
    rows, cols = np.nonzero(mask)
    rp = np.zeros(m + 1, np.int64)
    np.add.at(rp, rows + 1, 1)
    rp = np.cumsum(rp)
    return CsrMatrix(m, n, rp, cols.astype(np.int32), P[rows, cols].astype(np.float32))


def _mask(m, n, density, rng):
    mask = rng.random((m, n)) < density
    mask[np.arange(m), rng.integers(0, n, m)] = True  # every row observed somewhere
    mask[rng.integers(0, m, n), np.arange(n)] = True  # and every column
    return mask


def _fit_predict(ctx, A, grid, rank, sweeps=100):  # ALS needs ~100 sweeps to converge here (FP64 oracle: same)
    from paper_2508_07605_b200.als import AlsHyper, AlsPlan

    plan = AlsPlan(A.m, A.row_ptr, A.col, A.val, grid, AlsHyper(rank=rank, lam=1e-5, sweeps=sweeps, seed=3),
                   0.05, ctx=ctx)
    plan.run()
    U, V = plan.factors()
    plan.close()
    return np.clip(U.astype(np.float64) @ V.T.astype(np.float64), 0.01, 1.25)


@pytest.mark.parametrize("rank,nc,ng,density", [(8, 8, 8, 0.6), (16, 8, 8, 0.6), (32, 16, 16, 0.5),
                                                (64, 16, 16, 0.7)])
def test_als_recovers_rank1_noiseless(ctx, rank, nc, ng, density):
    from paper_2508_07605_b200 import PowerGrid

    rng = np.random.default_rng(rank)
    grid = PowerGrid.spanning(nc, ng)
    m, n = 3000, grid.n
    u = rng.uniform(0.5, 1.0, m)
    v = rng.uniform(0.3, 1.2, n)
    P = np.outer(u, v)
    mask = _mask(m, n, density, rng)
    got = _fit_predict(ctx, _csr_from_dense(P, mask), grid, rank)
    rel = np.abs(got - P)[~mask] / P[~mask]
    _check(rel)


@pytest.mark.parametrize("rank", [8, 32])
def test_als_constant_matrix_completes_to_the_constant(ctx, rank):
    from paper_2508_07605_b200 import PowerGrid

    rng = np.random.default_rng(7)
    grid = PowerGrid.spanning(6, 10)
    m, n = 2000, grid.n
    P = np.full((m, n), 0.8)
    mask = _mask(m, n, 0.2, rng)
    got = _fit_predict(ctx, _csr_from_dense(P, mask), grid, rank)
    rel = np.abs(got - P)[~mask] / P[~mask]
    _check(rel)


@pytest.mark.parametrize("rank,nc,ng,density", [(16, 8, 16, 0.6), (64, 16, 16, 0.7)])
def test_als_column_profile_dominance(ctx, rank, nc, ng, density):
    from paper_2508_07605_b200 import PowerGrid

    rng = np.random.default_rng(11)
    grid = PowerGrid.spanning(nc, ng)
    m, n = 2500, grid.n
    c = rng.uniform(0.2, 1.2, n)
    P = np.tile(c, (m, 1))
    mask = _mask(m, n, density, rng)
    got = _fit_predict(ctx, _csr_from_dense(P, mask), grid, rank)
    rel = np.abs(got - P)[~mask] / P[~mask]
    _check(rel)
