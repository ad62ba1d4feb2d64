"""World-size-2 check of the row-sharded ALS schedule (paper_2508_07605_b200.dist)
on CPU: gloo allreduce + the FP64 oracle as the backend.  The sharded result
must equal the single-process oracle ALS (same algorithm, reassociated sums)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT

K, LAM, SWEEPS, SEED = 8, 0.003, 4, 5
M, NC, NG = 300, 4, 8


def _problem():
    from paper_2508_07605_b200 import PowerGrid, synth

    grid = PowerGrid.spanning(NC, NG)
    return grid, synth.joint_csr(M, grid, 0.2, 2, seed=13)


class OracleBackend:
    def __init__(self, port, A, r0, r1, n):
        from oracle import bind

        self.port, self.n = port, n
        rp = A.row_ptr[r0:r1 + 1] - A.row_ptr[r0]
        s, e = A.row_ptr[r0], A.row_ptr[r1]
        self.rp, self.col, self.val = rp, A.col[s:e].copy(), A.val[s:e].copy()
        self.m = r1 - r0
        self.cp, self.crow, self.cval = bind.csc_of(self.m, n, self.rp, self.col, self.val)
        self.U = np.zeros((self.m, K))
        self.V = np.zeros((n, K))

    def begin(self):
        for j in range(self.n):
            for f in range(K):
                self.V[j, f] = self.port.L.ocgo_als_init_value(SEED, j, f, K)

    def row_half(self):
        from oracle.bind import P

        self.port.L.ocgo_als_solve_rows(self.m, P(self.rp), P(self.col), P(self.val), P(self.V), P(self.U), K, LAM)

    def col_half(self):
        g = self.col_gram()
        self.col_solve(g)

    def col_gram(self):
        import torch

        from oracle.bind import P

        G = np.zeros(self.n * (K * K + K + 1))
        self.port.L.ocgo_als_col_gram(self.n, P(self.cp), P(self.crow), P(self.cval), P(self.U), K, P(G))
        return torch.from_numpy(G)

    def col_solve(self, g):
        from oracle.bind import P

        G = np.ascontiguousarray(g.numpy())
        self.port.L.ocgo_als_solve_from_gram(self.n, P(G), P(self.V), K, LAM)

    def select(self):
        pass


def _worker(rank, world, port_no, out):
    import sys

    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import bind
    from paper_2508_07605_b200.dist import ShardedAlsDriver, shard_rows

    grid, A = _problem()
    r0, r1 = shard_rows(M, world, rank)
    be = OracleBackend(bind.Port(), A, r0, r1, grid.n)
    ShardedAlsDriver(be, world, lambda g: dist.all_reduce(g)).run(SWEEPS)
    out[rank] = (r0, r1, be.U.copy(), be.V.copy())
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_rows_partition():
    from paper_2508_07605_b200.dist import shard_rows

    for m in (1, 7, 1000, 1_000_000):
        for w in (1, 2, 3, 8):
            parts = [shard_rows(m, w, r) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == m
            assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))
            assert max(b - a for a, b in parts) - min(b - a for a, b in parts) <= 1


def test_row_sharded_als_matches_single_process(port):
    from oracle import bind

    grid, A = _problem()
    U1, V1 = bind.als_fit(port, A.m, A.n, A.row_ptr, A.col, A.val, K, LAM, SWEEPS, SEED)
    mgr = mp.Manager()
    out = mgr.dict()
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    Us = np.zeros_like(U1)
    for r in range(world):
        r0, r1, U, V = out[r]
        Us[r0:r1] = U
        np.testing.assert_allclose(V, V1, rtol=1e-9, atol=1e-12)
    np.testing.assert_array_equal(out[0][3], out[1][3])  # V replicated bit-identically
    np.testing.assert_allclose(Us, U1, rtol=1e-9, atol=1e-12)
