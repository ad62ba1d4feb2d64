"""One fused NCF completion + selection pass on a C2-shaped matrix with fewer rows
(default 200K), for ncu:  ncu --set full -k regex:ncf_fast_kernel python tools/profile_ncf.py"""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2508_07605_b200 as ocg  # noqa: E402
from paper_2508_07605_b200 import synth  # noqa: E402
from paper_2508_07605_b200.ncf import EXACT, FAST, DeviceNcfModel, NcfPlan, random_model  # noqa: E402

m = int(os.environ.get("OCG_ROWS", 200_000))
prec = EXACT if os.environ.get("OCG_PREC", "fast") == "exact" else FAST
grid = ocg.PowerGrid.spanning(64, 64)
A = synth.joint_csr(m, grid, 0.02, max(1, m // 1000), seed=42, dtype=np.float64)
model = random_model(m, grid.n, 32, seed=5, emb_scale=0.6)
ctx = ocg.Context(0)
dm = DeviceNcfModel(model, ctx=ctx)
plan = NcfPlan(dm, A.row_ptr, A.col, A.val, grid, 0.05, prec, 1)
for _ in range(int(os.environ.get("OCG_REPS", 2))):
    ms, ph = plan.run(timed=True)
    print(f"total {ms:.3f} ms, phases {ph}")
