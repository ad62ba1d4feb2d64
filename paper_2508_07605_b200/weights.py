"""Pure-numpy synthetic inputs shared by the product's benches and the reference
arm (no library import: bench.py's reference leg loads this file standalone so
the reference run never maps libocg.so)."""
from __future__ import annotations

import numpy as np


def spanning_caps(ncpu: int, ngpu: int):
    """SURVEY §8d grids for C1-C3 (cpu 60-250 W, gpu 100-400 W), as PowerGrid.spanning."""
    return (np.array([60 + (190 * i) // (ncpu - 1) for i in range(ncpu)], np.int32),
            np.array([100 + (300 * j) // (ngpu - 1) for j in range(ngpu)], np.int32))


def random_ncf_params(m: int, n: int, k: int = 32, seed: int = 0, emb_scale: float = 1.0) -> np.ndarray:
    """Flat parameters [app m x k | setting n x k | W0 b0 W1 b1 W2 b2] of a reference-layout NCF
    model with hidden {32, 16}: embeddings uniform in +-emb_scale, the MLP with the reference's
    Glorot-uniform bound (nnkit.cpp:58-61); the output layer is scaled (x0.25, bias 0.7) so the
    predictions spread over (0.01, 1.25] the way a fitted model's do."""
    rng = np.random.default_rng(seed)
    parts = [rng.uniform(-emb_scale, emb_scale, m * k), rng.uniform(-emb_scale, emb_scale, n * k)]
    dims = [2 * k, 32, 16, 1]
    for l in range(3):
        b = np.sqrt(6.0 / (dims[l] + dims[l + 1]))
        w = rng.uniform(-b, b, dims[l] * dims[l + 1])
        bias = rng.uniform(-0.1, 0.1, dims[l + 1])
        if l == 2:
            w *= 0.25
            bias[:] = 0.7
        parts += [w, bias]
    return np.concatenate(parts)
