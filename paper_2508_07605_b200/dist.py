"""Row-sharded multi-GPU ALS completion + selection.

Each rank owns a contiguous shard of application rows (its CSR rows, its U
rows); V (n x k) is replicated.  Per sweep:
  row half-sweep      local (needs only V)
  column half-sweep   every rank forms its shard's column Gram records
                      [k*k Gram | k rhs | count] per column, one allreduce(sum)
                      combines them (NCCL over NVLink; 17.3 MB at C2), and every
                      rank solves the same records -> identical V everywhere
  selection           local rows, no exchange
The driver is backend-agnostic: GpuAlsBackend drives the sm_100a plan on
torch's current stream (so torch's NCCL allreduce is stream-ordered with our
kernels); the tests drive the same schedule with the FP64 CPU oracle over gloo.
"""
from __future__ import annotations

import ctypes
from typing import Callable


def shard_rows(m: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced row shard [r0, r1) of rank."""
    base, extra = divmod(m, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


class ShardedAlsDriver:
    """One ALS completion step over row shards.  allreduce(buf) sums buf in
    place across ranks (a no-op when world == 1)."""

    def __init__(self, backend, world: int, allreduce: Callable | None = None):
        self.b, self.world, self.allreduce = backend, world, allreduce

    def run(self, sweeps: int) -> None:
        b = self.b
        b.begin()
        for _ in range(sweeps):
            b.row_half()
            if self.world == 1:
                b.col_half()
            else:
                g = b.col_gram()
                self.allreduce(g)
                b.col_solve(g)
        b.select()


class GpuAlsBackend:
    """AlsPlan phases on torch's current CUDA stream + a torch Gram buffer."""

    def __init__(self, plan, device):
        import torch

        from . import _lib

        self._lib = _lib
        self.plan = plan
        stream = torch.cuda.current_stream(device)
        _lib.check(_lib.lib.ocg_ctx_set_stream(plan.ctx.handle, ctypes.c_void_p(stream.cuda_stream)))
        n = int(_lib.lib.ocg_als_plan_gram_floats(plan._h))
        self.G = torch.empty(n, dtype=torch.float32, device=device)

    def _c(self, fn, *args):
        self._lib.check(fn(self.plan._h, *args))

    def begin(self):
        self._c(self._lib.lib.ocg_als_plan_begin)

    def row_half(self):
        self._c(self._lib.lib.ocg_als_plan_row_half)

    def col_half(self):
        self._c(self._lib.lib.ocg_als_plan_col_half)

    def col_gram(self):
        self._c(self._lib.lib.ocg_als_plan_col_gram, ctypes.c_void_p(self.G.data_ptr()))
        return self.G

    def col_solve(self, g):
        self._c(self._lib.lib.ocg_als_plan_col_solve, ctypes.c_void_p(g.data_ptr()))

    def select(self):
        self._c(self._lib.lib.ocg_als_plan_select)
