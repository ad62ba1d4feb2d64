"""The multi-GPU ALS schedule on real sm_100a kernels, emulated on one GPU:
two row shards = two plans; the column Gram records of both are summed (what
NCCL allreduce does across ranks) and both shards solve the same records."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("k", [16, 32, 64])  # 32/64: tensor-core Gram records (MODE 1)
def test_two_shard_schedule_matches_oracle(ctx, port, k):
    import torch

    from oracle import bind
    from paper_2508_07605_b200 import PowerGrid, synth
    from paper_2508_07605_b200.als import AlsHyper, AlsPlan
    from paper_2508_07605_b200.dist import GpuAlsBackend, shard_rows

    grid = PowerGrid.spanning(8, 16)
    m, sweeps = 2000, 5
    hyp = AlsHyper(rank=k, lam=0.003, sweeps=sweeps, seed=3)
    A = synth.joint_csr(m, grid, 0.1, 4, seed=21)
    dev = torch.device("cuda", 0)
    backs, shards = [], []
    for r in range(2):
        r0, r1 = shard_rows(m, 2, r)
        S = synth.joint_csr(m, grid, 0.1, 4, seed=21, rows=(r0, r1))
        plan = AlsPlan(S.m, S.row_ptr, S.col, S.val, grid, hyp, 0.05)
        backs.append(GpuAlsBackend(plan, dev))
        shards.append((r0, r1, plan))
    for b in backs:
        b.begin()
    for _ in range(sweeps):
        for b in backs:
            b.row_half()
        G = backs[0].col_gram().clone() + backs[1].col_gram()
        for b in backs:
            b.col_solve(G)
    for b in backs:
        b.select()
    torch.cuda.synchronize()
    U = np.zeros((m, k), np.float32)
    Vs = []
    for r0, r1, plan in shards:
        Ur, Vr = plan.factors()
        U[r0:r1] = Ur
        Vs.append(Vr)
    np.testing.assert_array_equal(Vs[0], Vs[1])  # replicated V is bit-identical
    Uo, Vo = bind.als_fit(port, A.m, A.n, A.row_ptr, A.col, A.val, k, 0.003, sweeps, 3)
    Pg = np.clip(U.astype(np.float64) @ Vs[0].T.astype(np.float64), 0.01, 1.25)
    Po = np.clip(Uo @ Vo.T, 0.01, 1.25)
    rel = np.abs(Pg - Po) / Po
    assert np.quantile(rel, 0.999) < 2e-3, rel.max()
    # per-shard selection == select_caps on the shard's completed rows
    cpu, gpu = grid.arrays()
    for r0, r1, plan in shards:
        idx, sav, loss, nc = plan.results()
        rows = plan.completed_rows(0, r1 - r0)
        rc, i2, s2, l2, n2 = port.select_caps(rows, cpu, gpu, 0.05)
        np.testing.assert_array_equal(idx, i2)
        np.testing.assert_array_equal(sav, s2)
