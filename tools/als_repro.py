"""Small ALS run for compute-sanitizer / debugging on the GPU box."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

from paper_2508_07605_b200 import PowerGrid, synth
from paper_2508_07605_b200.als import AlsHyper, AlsPlan

k = int(sys.argv[1]) if len(sys.argv) > 1 else 8
grid = PowerGrid.spanning(8, 16)
A = synth.joint_csr(1500, grid, 0.15, 4, seed=3)
plan = AlsPlan(A.m, A.row_ptr, A.col, A.val, grid, AlsHyper(rank=k, lam=0.003, sweeps=2, seed=11), 0.05)
print(plan.run())
print(plan.results()[0][:10])
