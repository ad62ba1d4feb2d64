"""Streaming arrivals: the merged CSR is valid and adds exactly
one previously unobserved cell to the chosen rows (host-side, no GPU)."""
import numpy as np


def test_add_observations_merges_one_new_cell_per_row():
    from paper_2508_07605_b200 import PowerGrid, synth
    from paper_2508_07605_b200.stream import add_observations

    grid = PowerGrid.spanning(8, 16)
    A = synth.joint_csr(3000, grid, 0.05, 3, seed=4)
    B = add_observations(A, grid, frac=0.01, seed=9)
    added = np.diff(B.row_ptr) - np.diff(A.row_ptr)
    assert set(np.unique(added)) <= {0, 1} and added.sum() == 30 and B.nnz == A.nnz + 30
    for i in range(A.m):
        a = A.col[A.row_ptr[i]:A.row_ptr[i + 1]]
        b = B.col[B.row_ptr[i]:B.row_ptr[i + 1]]
        assert np.all(np.diff(b) > 0)  # ascending, unique
        assert np.isin(a, b).all()
        va = A.val[A.row_ptr[i]:A.row_ptr[i + 1]]
        vb = B.val[B.row_ptr[i]:B.row_ptr[i + 1]]
        np.testing.assert_array_equal(vb[np.isin(b, a)], va)  # old observations verbatim
    assert ((B.val > 0.0) & (B.val <= 1.25)).all()
    # dense rows (all columns observed) are never chosen
    assert (added[:3] == 0).all()
