import time, numpy as np, torch, sys
sys.path.insert(0, '.')
import bench
import paper_2508_07605_b200 as ocg
from paper_2508_07605_b200.als import AlsHyper, AlsPlan
cfg, grid, A = bench._joint_matrix("c2", 0, 1)
ctx = ocg.Context(0)
hyp = AlsHyper(rank=32, lam=0.003, sweeps=10, seed=42)
pin = [torch.from_numpy(x).pin_memory() for x in (A.row_ptr, A.col.astype(np.uint16), A.val)]
ptrs = [int(x.data_ptr()) for x in pin]
res = [torch.empty(A.m, dtype=dt).pin_memory() for dt in (torch.int32, torch.float64, torch.float64, torch.int32)]
rp = [int(x.data_ptr()) for x in res]
p = AlsPlan(A.m, A.row_ptr, A.col, A.val, grid, hyp, 0.05, ctx=ctx)
p.run(timed=False); p.results(out=rp)
def t(f, n=5):
    torch.cuda.synchronize(); t0 = time.perf_counter(); f(n); torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e3
def runs(n):
    for _ in range(n): p.run(timed=False)
def runs_res(n):
    for _ in range(n): p.run(timed=False); p.results(out=rp)
def serial(n):
    for _ in range(n): p.upload_compact(*ptrs); p.run(timed=False); p.results(out=rp)
def upl(n):
    for _ in range(n): p.upload_compact(*ptrs)
def piped(n):
    p.stage_compact(*ptrs)
    for i in range(n):
        p.run(timed=False)
        if i + 1 < n: p.stage_compact(*ptrs)
        p.results(out=rp)
for name, f in [("runs", runs), ("runs+results", runs_res), ("upload only", upl), ("serial", serial), ("piped", piped), ("runs", runs), ("piped", piped)]:
    print(f"{name:14s} {t(f):8.2f} ms/step", flush=True)
