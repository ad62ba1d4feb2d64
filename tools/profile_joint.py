"""Time the joint-mode NCF fit (ocg_cf_fit) on the C1 matrix for a few epochs.

    OCG_JOINT_PROFILE=1 python tools/profile_joint.py [epochs] [solver] [lane] [k]
"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2508_07605_b200 import Context, NcfHyper, PowerGrid, synth  # noqa: E402
from paper_2508_07605_b200.cf import cf_fit  # noqa: E402

epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 20
solver = int(sys.argv[2]) if len(sys.argv) > 2 else 0
lane = int(sys.argv[3]) if len(sys.argv) > 3 else 1
k = int(sys.argv[4]) if len(sys.argv) > 4 else 8
m = int(sys.argv[5]) if len(sys.argv) > 5 else 10_000
grid = PowerGrid.spanning(16, 16) if m <= 100_000 else PowerGrid.spanning(64, 64)
dens = 0.05 if m <= 100_000 else 0.02
A = synth.joint_csr(m, grid, dens, max(1, m // 1000), seed=42, dtype=np.float64)
with Context(0) as ctx:
    h = NcfHyper(app_dim=k, setting_dim=k, max_epochs=epochs, patience=10_000)
    st = {}
    t0 = time.perf_counter()
    model = cf_fit(A.row_ptr, A.col, A.val, A.n, h, 42, solver, lane, ctx, st)
    wall = time.perf_counter() - t0
print(f"m={m} n={A.n} nnz={A.nnz} k={k} solver={solver} lane={lane}: {model.meta.epochs_run} epochs, "
      f"{st['steps']} steps, device {st['device_ms']:.1f} ms = {st['device_ms'] * 1e3 / max(st['steps'], 1):.2f} us/step, "
      f"wall {wall:.2f} s, best_val {model.meta.best_val_mse:.6g}")
