"""Golden joint-mode NCF fits (tests/golden/make_joint_golden.py, produced by the
reference's own cf::fit) and the matrices they were fitted on."""
from __future__ import annotations

from pathlib import Path

import numpy as np

GOLD = Path(__file__).resolve().parent / "golden"


def spanning(nc, ng):
    return [60 + (190 * i) // (nc - 1) for i in range(nc)], [100 + (300 * j) // (ng - 1) for j in range(ng)]


def small_cases():
    z = np.load(GOLD / "joint_small.npz")
    names = sorted({k.split("/")[0] for k in z.files})
    out = []
    for name in names:
        cfg = z[f"{name}/cfg"]
        hi = z[f"{name}/hyper_i"]
        hf = z[f"{name}/hyper_f"]
        hyper = dict(app_dim=int(hi[0]), setting_dim=int(hi[1]), hidden=tuple(int(x) for x in z[f"{name}/hidden"][: hi[2]]),
                     max_epochs=int(hi[3]), patience=int(hi[4]), batch_size=int(hi[5]), lr=float(hf[0]),
                     val_fraction=float(hf[1]))
        out.append(dict(name=name, m=int(cfg[0]), grid=(int(cfg[1]), int(cfg[2])), dense_rows=int(cfg[3]),
                        seed=int(cfg[4]), lane=int(cfg[5]), density=float(z[f"{name}/density"][0]), hyper=hyper,
                        params=z[f"{name}/params"], meta=z[f"{name}/meta"]))
    return out


def c1_case(lane):
    p = GOLD / f"joint_c1_lane{lane}.npz"
    if not p.exists():
        return None
    z = np.load(p)
    cfg = z["cfg"]
    return dict(name=f"c1_l{lane}", m=int(cfg[0]), grid=(int(cfg[1]), int(cfg[2])), dense_rows=int(cfg[3]),
                seed=int(cfg[4]), lane=int(cfg[5]), density=float(z["density"][0]), hyper={}, params=z["params"],
                meta=z["meta"], host_seconds=float(z["host_seconds"][0]))


def matrix(case):
    """CSR (FP64 values) of the case's SURVEY §8d joint matrix (matrix seed 42)."""
    from paper_2508_07605_b200 import PowerGrid, synth

    grid = PowerGrid(tuple(spanning(*case["grid"])[0]), tuple(spanning(*case["grid"])[1]))
    A = synth.joint_csr(case["m"], grid, case["density"], case["dense_rows"], seed=42, dtype=np.float64, threads=4)
    return grid, A


def dense(A):
    vals = np.zeros((A.m, A.n))
    mask = np.zeros((A.m, A.n), np.uint8)
    rows = np.repeat(np.arange(A.m), np.diff(A.row_ptr))
    vals[rows, A.col] = A.val
    mask[rows, A.col] = 1
    return vals, mask
