"""Streaming arrivals for online refits.

Each arrival batch adds ONE new observation to each of ``frac`` of the rows
(seeded): a column the row has not observed yet, valued like the row's nearest
observed setting with the profiling noise form of the reference
(``exp(0.01 N(0,1))``, simnode.cpp:127) and clamped to the matrix domain
(0.01, 1.25] (core.cpp:142-148).  The result is a new CSR (columns ascending
per row) that ``AlsPlan.upload`` takes as is; refits then complete it from
scratch (reference semantics) or warm (``AlsPlan.set_warm``, a flagged
deviation).  Host-side input generation only — nothing here is on the device
path."""
from __future__ import annotations

import numpy as np

from .api import PowerGrid
from .synth import CsrMatrix


def add_observations(A: CsrMatrix, grid: PowerGrid, frac: float = 0.01, seed: int = 0, return_delta: bool = False):
    """The merged CSR; with return_delta also the new cells (rows, cols, vals), sorted by
    (row, col) -- the arguments of ``AlsPlan.add_observations``."""
    m, n = A.m, grid.n
    rng = np.random.default_rng(seed)
    rp = A.row_ptr
    cnt = np.diff(rp)
    cand = np.nonzero(cnt < n)[0]  # rows with an unobserved column left
    k = min(len(cand), max(1, int(round(frac * m))))
    rows = np.sort(rng.choice(cand, size=k, replace=False)).astype(np.int64)
    keys = np.repeat(np.arange(m, dtype=np.int64), cnt) * n + A.col.astype(np.int64)
    cols = rng.integers(0, n, size=k)
    todo = np.ones(k, bool)
    for _ in range(64):  # rejection: a column the row has not observed (rows are < 100% full)
        q = rows[todo] * n + cols[todo]
        pos = np.searchsorted(keys, q)
        hit = (pos < len(keys)) & (keys[np.minimum(pos, len(keys) - 1)] == q)
        idx = np.nonzero(todo)[0]
        todo[idx[~hit]] = False
        if not todo.any():
            break
        cols[idx[hit]] = rng.integers(0, n, size=int(hit.sum()))
    ok = ~todo
    rows, cols = rows[ok], cols[ok].astype(np.int64)
    ins = rows * n + cols
    # value: the row's nearest observed setting, with profiling noise
    pos = np.searchsorted(keys, ins)
    lo = np.clip(pos - 1, rp[rows], rp[rows + 1] - 1)
    hi = np.clip(pos, rp[rows], rp[rows + 1] - 1)
    near = np.where(np.abs(A.col[lo] - cols) <= np.abs(A.col[hi] - cols), lo, hi)
    vals = np.clip(A.val[near].astype(np.float64) * np.exp(0.01 * rng.standard_normal(len(rows))), 0.01, 1.25)
    # merge: old entry q moves by the number of insertions before it; insertion t lands
    # after the old entries before it plus the t insertions before it
    nnz2 = A.nnz + len(rows)
    col2 = np.empty(nnz2, np.int32)
    val2 = np.empty(nnz2, A.val.dtype)
    old_dst = np.arange(A.nnz, dtype=np.int64) + np.searchsorted(ins, keys)
    new_dst = pos + np.arange(len(rows), dtype=np.int64)
    col2[old_dst] = A.col
    val2[old_dst] = A.val
    col2[new_dst] = cols
    val2[new_dst] = vals.astype(A.val.dtype)
    add = np.zeros(m, np.int64)
    add[rows] = 1
    rp2 = rp.copy()
    rp2[1:] += np.cumsum(add)
    B = CsrMatrix(m, n, rp2, col2, val2)
    if return_delta:
        return B, (rows.astype(np.int32), cols.astype(np.int32), vals.astype(A.val.dtype))
    return B
