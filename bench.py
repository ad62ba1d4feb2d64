#!/usr/bin/env python3
"""bench.py — B200 online CF completion + selection (OPEN online phase).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload c2-ncf|c2|c1-ncf|c1|c3|c4|c0xn|ingest]

One JSON line on rank 0.  For N>1 launch with
torch.distributed.run; each rank takes an equal shard of the units (weak
scaling for the sharded workloads), timing is the max over ranks of CUDA-event
device time.  A "step" is one pass of the hot path over one batch of
synthetic input:

  c2-ncf  (default) SURVEY §8d C2 (BASELINE configs[2]): 1M apps x 4096 settings,
        rank 32, 2% observed — the reference's CF model (NCF) given fitted weights:
        cf::complete's imputation of every unobserved cell fused with Algorithm-2
        selection on every row (FP32 + tcgen05; reference parity: exact mode
        bit-identical, fast mode within 1e-5); the reference arm runs the same
        weights through NcfModel::predict + select_caps
  c2    the same matrix completed by ALS (fit included; no reference counterpart)
  c1-fit  C1 (configs[1]) through the reference's whole CF path, bit for bit: cf::fit
        (NCF, reference schedule, early stopping) + imputation + selection
  c1    C1 (configs[1]): 10K x 256, rank 8, 5% observed, same path
  c0xn  the reference's own online semantics at scale: N independent apps,
        each cf::complete'd against the paper-scale offline block + selected
        (bit-exact NCF, one CTA per app)
  ingest  probe ingest: pred::predict_perf over every
        (app, setting) counter sample of 20K eval apps on the C2 64x64 grid
        (81.9M samples, the C2 probe count), bit-exact FP64

--impl reference times the reference's own CPU implementation of the path
(oracle/_ref, compiled from the unmodified reference sources) on this host's
cores over a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS = {"hbm_gbs": 6515.7, "bf16_tflops": 1644.8, "source": "fallback"}
try:
    _p = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    PEAKS = {"hbm_gbs": _p["hbm_gbs"], "bf16_tflops": _p["bf16_tflops"], "source": "measured"}
except Exception:
    PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback (B200_PROFILING.md)"}


# ----------------------------------------------------------------- plumbing
class Dist:
    def __init__(self, backend: str | None):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        if self.world > 1 and os.environ.get("OCG_BENCH_SHARE_GPU") == "1":
            # dry run of the N > 1 code paths on a one-GPU box: every rank on cuda:0, gloo
            # for the barrier / max (NCCL refuses two ranks on one device); timings meaningless
            self.local = 0
            backend = "gloo" if backend else backend
        if self.world > 1 and backend:
            import torch
            import torch.distributed as dist

            if backend == "nccl":
                torch.cuda.set_device(self.local)
            dist.init_process_group(backend)
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        import torch

        dev = "cuda" if self.pg.get_backend() == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if not self.pg:
            return x
        import torch

        dev = "cuda" if self.pg.get_backend() == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.pg.all_reduce(t)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


class Clocks:
    """SM clock and clock-event (throttle) reasons during the timed region, read through
    NVML (the library nvidia-smi uses): a sampler thread every 10 ms plus one sample per
    step (tick()), so even a sub-second timed region carries >= steps samples
    (B200_PROFILING.md clocks line; falls back to nvidia-smi -lms 200 without NVML)."""

    REASONS = (("hw_slowdown", 0x8), ("sw_thermal_slowdown", 0x20), ("hw_thermal_slowdown", 0x40),
               ("sw_power_cap", 0x4), ("hw_power_brake_slowdown", 0x80))

    def __init__(self, device: int):
        self.device = device
        self.sm, self.reasons, self.smax = [], set(), None
        self.nvml = None
        self.stop = threading.Event()
        self.thread = None
        self.smi = None

    def _sample(self):
        try:
            self.sm.append(float(self.nvml.nvmlDeviceGetClockInfo(self.h, self.nvml.NVML_CLOCK_SM)))
            bits = self.nvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for name, bit in self.REASONS:
                if bits & bit:
                    self.reasons.add(name)
        except Exception:
            pass

    def tick(self):
        if self.nvml:
            self._sample()

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.smax = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))

            def loop():
                while not self.stop.is_set():
                    self._sample()
                    time.sleep(0.01)

            self.thread = threading.Thread(target=loop, daemon=True)
            self.thread.start()
        except Exception:
            self.nvml = None
            try:
                fd, self.path = tempfile.mkstemp(suffix=".csv")
                os.close(fd)
                self.smi = subprocess.Popen(["nvidia-smi", f"--id={self.device}",
                                             "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                                             "clocks_event_reasons.sw_thermal_slowdown,"
                                             "clocks_event_reasons.hw_thermal_slowdown,"
                                             "clocks_event_reasons.sw_power_cap",
                                             "--format=csv,noheader,nounits", "-lms", "200"],
                                            stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            except Exception:
                self.smi = None
        return self

    def __exit__(self, *exc):
        self.stop.set()
        if self.thread:
            self.thread.join(timeout=2)
        if self.smi:
            self.smi.terminate()
            try:
                self.smi.wait(timeout=5)
            except Exception:
                self.smi.kill()
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                try:
                    self.sm.append(float(f[0]))
                    self.smax = float(f[1])
                except (ValueError, IndexError):
                    continue
                for (name, _), v in zip(self.REASONS, f[2:6]):
                    if v.lower().startswith("active"):
                        self.reasons.add(name)
            os.unlink(self.path)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.smax, "reasons": ["no clock samples"], "samples": 0}
        load = [x for x in self.sm if self.smax and x > 0.5 * self.smax] or self.sm
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": self.smax, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": "nvml" if self.nvml else "nvidia-smi"}


def host_info():
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


# --------------------------------------------------------------- workloads
def workload_c0xn(args, d: Dist):
    """Reference online semantics (policy.cpp:178-189) for many apps, bit-exact NCF."""
    import paper_2508_07605_b200 as ocg
    from paper_2508_07605_b200 import synth

    grid = ocg.PowerGrid.default_grid()
    per_gpu = args.apps
    total = per_gpu * d.world
    block = synth.offline_block(42, grid)
    bmask = np.ones_like(block, np.uint8)
    pv, pm, sd = synth.online_apps(total, 42, grid)
    lo, hi = d.rank * per_gpu, (d.rank + 1) * per_gpu
    pv, pm, sd = pv[lo:hi], pm[lo:hi], sd[lo:hi]
    ctx = ocg.Context(d.local)
    hyper = ocg.NcfHyper()
    plan = ocg.OnlinePlan(block, bmask, pv, pm, sd, grid, hyper, 0.05, args.lane, True, ctx)
    for _ in range(args.warmup):
        plan.run(timed=False)
    ocg._lib.check(ocg._lib.lib.ocg_ctx_synchronize(ctx.handle))
    res = plan.results()
    assert (res.status == 0).all(), np.unique(res.status)
    d.barrier()
    ms = 0.0
    with Clocks(d.local) as clk:
        for _ in range(args.steps):
            ocg._lib.check(ocg._lib.lib.ocg_ctx_flush_l2(ctx.handle))
            ms += plan.run(timed=True)
            clk.tick()
    d.barrier()
    t_dev = d.max(ms / 1e3)
    res = plan.results()
    epochs = float(res.meta["epochs_run"].mean())
    # e2e through the public API with host buffers
    e2e_t = 0.0
    ocg.online_complete_batch(block, bmask, pv[:64], pm[:64], sd[:64], grid, hyper, 0.05, args.lane, ctx)
    d.barrier()
    for _ in range(args.steps):
        t0 = time.perf_counter()
        r2 = ocg.online_complete_batch(block, bmask, pv, pm, sd, grid, hyper, 0.05, args.lane, ctx)
        e2e_t += time.perf_counter() - t0
    e2e_t = d.max(e2e_t)
    assert np.array_equal(r2.idx, res.idx)
    n = grid.n
    cells = total * n * args.steps
    h2d = block.nbytes + bmask.nbytes + pv.nbytes + pm.nbytes + sd.nbytes + 8 * 4
    d2h = r2.completed.nbytes + r2.idx.nbytes + r2.saving.nbytes + r2.loss.nbytes + r2.ncand.nbytes + \
        r2.meta.nbytes + r2.status.nbytes
    # algorithmic FP64 work per app: forward+backward per sample, Adam per param, per epoch
    dims = [16, 32, 16, 1]
    mac = sum(dims[i] * dims[i + 1] for i in range(3))
    nt = 206 - 20
    flops_app = epochs * (nt * (2 * mac + 4 * mac) + 20 * 2 * mac + 6 * 1337 * 12)
    achieved = flops_app * per_gpu * args.steps / (ms / 1e3) / 1e12
    out = {
        "metric": "CF-completed matrix cells/sec",
        "value": cells / t_dev,
        "unit": "cells/s",
        "selections_per_sec": total * args.steps / t_dev,
        "ms_per_step": t_dev * 1e3 / args.steps,
        "e2e": {"value": cells / e2e_t, "unit": "cells/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "dtype": "f64",
        "config": {"workload": "c0xn", "apps": total, "apps_per_gpu": per_gpu, "settings": n,
                   "offline_rows": int(block.shape[0]), "rank": 8, "hidden": [32, 16], "batch": 32,
                   "lane": "avx2" if args.lane else "scalar", "mean_epochs_run": epochs,
                   "l2": "flushed (256 MB write) before every timed step"},
        "scaling": "weak",
        "gpu_launches": args.steps,
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": 37.0, "unit": "TFLOP/s",
                     "frac": achieved / 37.0, "traffic": None,
                     "note": "FP64 SIMT nominal 37 TFLOP/s (no measured FP64 peak); algorithmic flops from meta"},
        "clocks": clk.summary(),
    }
    return out, ("c0xn", per_gpu)


def _simt_peaks():
    """Measured FP64/FP32 SIMT peaks (tools/simt_peak.cu on a B200, profiles/simt_peak.json)."""
    try:
        return json.loads((ROOT / "profiles" / "simt_peak.json").read_text()), "measured (tools/simt_peak.cu)"
    except Exception:
        return {"fp64_tflops": 37.0, "fp32_tflops": 74.5}, "nominal (no measured SIMT peak)"


PRED_MODEL = ROOT / "tests" / "golden" / "predictor.json"  # a predictor trained by the reference (make_golden.py)
INGEST_APPS = 20_000  # x 4096 settings = 81.9M counter samples per GPU


def _ingest_counters(apps: int, rank: int):
    import paper_2508_07605_b200 as ocg
    from paper_2508_07605_b200 import synth

    grid = ocg.PowerGrid.spanning(64, 64)
    specs = synth.make_suite([apps * (rank + 1) // 4] * 4, 42, 1, grid, 0.01, 0.2)
    lo = apps * rank // 4
    mine = [specs[a * (apps * (rank + 1) // 4) + lo + i] for a in range(4) for i in range(apps // 4)]
    return grid, synth.counters(mine, grid)


def workload_ingest(args, d: Dist):
    """Batched pred::predict_perf (predictor.cpp:151-157) over the C2 probe volume, bit-exact FP64."""
    import ctypes

    import torch

    import paper_2508_07605_b200 as ocg
    from paper_2508_07605_b200.predictor import Predictor, PredictorModel

    grid, counters = _ingest_counters(INGEST_APPS, d.rank)
    count = len(counters)
    dev = torch.device("cuda", d.local)
    torch.cuda.set_device(dev)
    ctx = ocg.Context(d.local)
    stream = torch.cuda.current_stream(dev)
    ocg._lib.check(ocg._lib.lib.ocg_ctx_set_stream(ctx.handle, ctypes.c_void_p(stream.cuda_stream)))
    model = PredictorModel.from_json(PRED_MODEL.read_text())
    pred = Predictor(model, ctx)
    c_dev = torch.from_numpy(counters).to(dev)
    out = torch.empty(count, dtype=torch.float64, device=dev)
    for _ in range(args.warmup):
        pred.run_device(c_dev.data_ptr(), count, out.data_ptr(), args.lane)
    torch.cuda.synchronize()
    d.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with Clocks(d.local) as clk:
        for e0, e1 in ev:  # 4.6 GB of counters per step: inputs larger than L2
            e0.record(stream)
            pred.run_device(c_dev.data_ptr(), count, out.data_ptr(), args.lane)
            e1.record(stream)
            clk.tick()
        torch.cuda.synchronize()
    ms = sum(e0.elapsed_time(e1) for e0, e1 in ev)
    d.barrier()
    t_dev = d.max(ms / 1e3)
    res_dev = out.cpu().numpy()
    # e2e: host counters in, host estimates out, through the public API
    e2e_t = 0.0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        res = pred(counters, args.lane)
        e2e_t += time.perf_counter() - t0
    e2e_t = d.max(e2e_t)
    assert np.array_equal(res, res_dev)
    total = count * d.world * args.steps
    dims = model.dims
    flops = 2 * sum(dims[i] * dims[i + 1] for i in range(len(dims) - 1)) + sum(dims[1:]) + 14
    peaks, src = _simt_peaks()
    achieved = flops * count * args.steps / (ms / 1e3) / 1e12
    out_line = {
        "metric": "probe performance estimates/sec",
        "value": total / t_dev,
        "unit": "estimates/s",
        "ms_per_step": t_dev * 1e3 / args.steps,
        "e2e": {"value": total / e2e_t, "unit": "estimates/s", "h2d_bytes_per_step": int(counters.nbytes),
                "d2h_bytes_per_step": int(res.nbytes)},
        "dtype": "f64",
        "config": {"workload": "ingest", "samples_per_gpu": count, "apps_per_gpu": INGEST_APPS,
                   "settings": grid.n, "architecture": dims, "lane": "avx2" if args.lane else "scalar",
                   "model": "tests/golden/predictor.json (trained by the reference)",
                   "l2": "inputs (4.6 GB counters) larger than L2"},
        "scaling": "weak",
        "gpu_launches": args.steps,
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": peaks["fp64_tflops"], "unit": "TFLOP/s",
                     "frac": achieved / peaks["fp64_tflops"], "traffic": None,
                     "note": f"algorithmic {flops} flop/sample (2*MACs + biases + standardize); peak {src}"},
        "clocks": clk.summary(),
    }
    return out_line, ("ingest", count)


def reference_ingest(samples: int, threads: int, lane: int = 1):
    """pred::predict_perf of the reference (oracle/_ref) over the first `samples` ingest counters."""
    from oracle import bind

    ref = bind.Ref()
    ref.force_lane(lane)
    _, counters = _ingest_counters(max(4, samples // 4096 + 4), 0)
    c = np.ascontiguousarray(counters[:samples])
    out = np.zeros(len(c))
    secs = ref.L.ref_predict_perf_mt(PRED_MODEL.read_text().encode(), bind.P(c), len(c), threads, bind.P(out))
    assert secs > 0, ref.err()
    return len(c) / secs, secs, len(c)


JOINT = {  # SURVEY §8d joint configs
    "c1": dict(m=10_000, grid=(16, 16), density=0.05, dense_rows=10, rank=8),
    "c2": dict(m=1_000_000, grid=(64, 64), density=0.02, dense_rows=1000, rank=32),
}
JOINT["c3"] = dict(m=4_000_000, grid=(128, 128), density=0.01, dense_rows=4000, rank=64)  # BASELINE configs[3]
JOINT["c4"] = dict(JOINT["c2"])  # streaming refits on the C2 matrix


def _joint_matrix(name, rank, world):
    from paper_2508_07605_b200 import PowerGrid, synth
    from paper_2508_07605_b200.dist import shard_rows

    c = JOINT[name]
    grid = PowerGrid.spanning(*c["grid"])
    r0, r1 = shard_rows(c["m"], world, rank)
    A = synth.joint_csr(c["m"], grid, c["density"], c["dense_rows"], seed=42, rows=(r0, r1))
    return c, grid, A


def quality_rows(m_loc, dense_rows, nblocks=20, block=100):
    """Row sample for the quality block: nblocks blocks of `block` rows spread over the
    local rows past the dense ones (every archetype of make_suite's suite is covered)."""
    lo = min(dense_rows, max(0, m_loc - block))
    starts = np.linspace(lo, m_loc - block, nblocks).astype(np.int64)
    return [(int(s), block) for s in np.unique(starts)]


def completion_quality(m, grid, A, blocks, completed, idx_completed, gamma, ctx, goff=0):
    """Held-out quality of a completion on the sampled local rows (blocks of (r0, count),
    completed rows stacked in that order):
      * RMSE of the imputed cells against the simulator's ground truth sim::true_perf
        (simnode.cpp:43-45), absolute and relative;
      * truth_optimal_frac: rows whose selection equals policy::select_caps on the TRUE row
        (the reference's C1 run reported RMSE 0.018, 61 % truth-optimal);
      * true_saving_regret: mean true energy saving lost vs the true optimum, and the share
        of rows whose chosen setting violates the true performance-loss bound gamma."""
    import paper_2508_07605_b200 as ocg
    from paper_2508_07605_b200 import synth

    rows = np.concatenate([np.arange(r0, r0 + c) for r0, c in blocks])
    truth = synth.true_rows(m, grid, rows + goff)
    mask = np.zeros_like(completed, bool)
    for k, i in enumerate(rows):
        mask[k, A.col[A.row_ptr[i]:A.row_ptr[i + 1]]] = True
    held = ~mask
    err = completed[held] - truth[held]
    idx_t, *_ = ocg.select_caps_batch(truth, grid, gamma, ctx)
    idx_c = np.asarray(idx_completed)
    cpu, gpu = grid.arrays()
    csum = (np.repeat(cpu, len(gpu)) + np.tile(gpu, len(cpu))).astype(np.float64)
    e_base = float(csum[-1])
    sav = (e_base - csum[None, :] / truth) / e_base
    loss = 1.0 - truth / truth[:, -1:]
    r = np.arange(len(rows))
    return {"rows": int(len(rows)), "heldout_cells": int(held.sum()),
            "heldout_rmse": float(np.sqrt(np.mean(err ** 2))),
            "heldout_rel_rmse": float(np.sqrt(np.mean((err / truth[held]) ** 2))),
            "truth_optimal_frac": float(np.mean(idx_c == idx_t)),
            "true_saving_regret": float(np.mean(sav[r, idx_t] - sav[r, idx_c])),
            "true_loss_violation_frac": float(np.mean(loss[r, idx_c] > gamma))}


def als_sweeps_rule(A, grid, hyp, gamma, ctx, m, goff=0, tol=1e-3, cap=40):
    """Sweep count by a stated convergence rule: the smallest number of ALS sweeps after which
    the held-out predictions of the quality row sample change by less than `tol` (relative
    RMS) from one sweep to the next (calibration run outside the timed region); also returns
    the held-out RMSE after every sweep."""
    from paper_2508_07605_b200 import synth
    from paper_2508_07605_b200.als import AlsPlan
    import paper_2508_07605_b200._lib as L

    plan = AlsPlan(A.m, A.row_ptr, A.col, A.val, grid, hyp, gamma, ctx=ctx)
    blocks = quality_rows(A.m, 0, nblocks=10, block=100)
    rows = np.concatenate([np.arange(r0, r0 + c) for r0, c in blocks])
    truth = synth.true_rows(m, grid, rows + goff)
    L.check(L.lib.ocg_als_plan_begin(plan._h))
    prev, sweeps, delta, curve = None, cap, None, []
    for s_ in range(1, cap + 1):
        L.check(L.lib.ocg_als_plan_row_half(plan._h))
        L.check(L.lib.ocg_als_plan_col_half(plan._h))
        cur = np.concatenate([plan.completed_rows(r0, c) for r0, c in blocks])
        curve.append(float(np.sqrt(np.mean((cur - truth) ** 2))))
        if prev is not None:
            delta = float(np.sqrt(np.mean(((cur - prev) / prev) ** 2)))
            if delta < tol:
                sweeps = s_
                break
        prev = cur
    plan.close()
    return sweeps, {"rule": f"smallest sweep count whose predictions on {len(rows)} sampled rows change < {tol:g} "
                            f"(relative RMS) from the previous sweep (cap {cap})", "sweeps": sweeps,
                    "last_change": delta, "rmse_vs_truth_by_sweep": curve}


def workload_joint(args, d: Dist):
    """ALS completion + fused imputation + Algorithm-2 selection of a joint matrix.
    N=1: the fused single-GPU plan; N>1: rows sharded over ranks, column Gram
    records allreduced with NCCL each column half-sweep (paper_2508_07605_b200.dist)."""
    import torch

    import paper_2508_07605_b200 as ocg
    from paper_2508_07605_b200.als import AlsHyper, AlsPlan
    from paper_2508_07605_b200.dist import GpuAlsBackend, ShardedAlsDriver

    cfg, grid, A = _joint_matrix(args.workload, d.rank, d.world)
    m_loc, n, nnz = A.m, grid.n, A.nnz
    m = cfg["m"]
    ctx = ocg.Context(d.local)
    sweeps_rule = {"rule": "fixed by --sweeps", "sweeps": args.sweeps}
    if args.sweeps <= 0:  # the stated convergence rule picks the sweep count (rank 0 decides, all ranks use it)
        from paper_2508_07605_b200.dist import shard_rows as _sr

        sw, sweeps_rule = als_sweeps_rule(A, grid, AlsHyper(rank=cfg["rank"], lam=args.als_lambda, sweeps=1, seed=42),
                                          args.gamma, ctx, m, goff=_sr(m, d.world, d.rank)[0])
        args.sweeps = int(d.max(float(sw)))
        sweeps_rule["sweeps"] = args.sweeps
    hyp = AlsHyper(rank=cfg["rank"], lam=args.als_lambda, sweeps=args.sweeps, seed=42)
    dev = torch.device("cuda", d.local)
    t_rp = torch.from_numpy(A.row_ptr).to(dev)
    t_col = torch.from_numpy(A.col).to(dev)
    t_val = torch.from_numpy(A.val).to(dev)
    torch.cuda.synchronize(dev)
    plan = AlsPlan(m_loc, t_rp.data_ptr(), t_col.data_ptr(), t_val.data_ptr(), grid, hyp, args.gamma,
                   on_device=True, ctx=ctx)
    phases = [0.0] * 6
    if d.world == 1:
        step = lambda: plan.run(timed=True)  # noqa: E731
    else:
        backend = GpuAlsBackend(plan, dev)
        driver = ShardedAlsDriver(backend, d.world, lambda g: d.pg.all_reduce(g))

        def step():
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            driver.run(args.sweeps)
            e1.record()
            e1.synchronize()
            return e0.elapsed_time(e1), [0.0] * 6
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    d.barrier()
    tot_ms = 0.0
    with Clocks(d.local) as clk:
        for _ in range(args.steps):
            ocg._lib.check(ocg._lib.lib.ocg_ctx_flush_l2(ctx.handle))
            ms, ph = step()
            clk.tick()
            tot_ms += ms
            phases = [a + b for a, b in zip(phases, ph)]
    torch.cuda.synchronize(dev)
    d.barrier()
    t_dev = d.max(tot_ms / 1e3)
    idx, sav, loss, ncand = plan.results()
    assert (idx >= 0).all() and (ncand >= 1).all()
    from paper_2508_07605_b200.dist import shard_rows

    qb = quality_rows(m_loc, cfg["dense_rows"] if d.rank == 0 else 0)
    qrows = np.concatenate([np.arange(r0, r0 + c) for r0, c in qb])
    quality = completion_quality(m, grid, A, qb, np.concatenate([plan.completed_rows(r0, c) for r0, c in qb]),
                                 idx[qrows], args.gamma, ctx, goff=shard_rows(m, d.world, d.rank)[0])
    quality["sweeps_rule"] = sweeps_rule
    plan.close()
    del t_rp, t_col, t_val
    # end to end through the public API with host buffers: a plan created once
    # (device allocations are not the workload), then per step the CSR is
    # uploaded from pinned host memory (ocg_als_plan_upload), the plan runs
    # from scratch and the decisions are read back to the host.
    # N>1: each rank uploads its shard and runs the sharded schedule.
    compact = n <= 65536  # 16-bit column indices over PCIe (ocg_als_plan_upload_compact)
    pin = [torch.from_numpy(x).pin_memory()
           for x in (A.row_ptr, A.col.astype(np.uint16) if compact else A.col, A.val)]
    h2d_bytes = sum(int(x.numel() * x.element_size()) for x in pin)
    res_pin = [torch.empty(m_loc, dtype=dt).pin_memory() for dt in (torch.int32, torch.float64, torch.float64,
                                                                      torch.int32)]
    p2 = AlsPlan(m_loc, A.row_ptr, A.col, A.val, grid, hyp, args.gamma, ctx=ctx)
    if d.world == 1:
        p2.run(timed=False)  # warm (module load, first-touch)
    e2e_steps = max(1, min(args.steps, 3))
    d.barrier()
    e2e_t = 0.0
    for _ in range(e2e_steps):
        ocg._lib.check(ocg._lib.lib.ocg_ctx_flush_l2(ctx.handle))
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        (p2.upload_compact if compact else p2.upload)(*(int(x.data_ptr()) for x in pin))
        if d.world == 1:
            p2.run(timed=False)
        else:
            ShardedAlsDriver(GpuAlsBackend(p2, dev), d.world, lambda g: d.pg.all_reduce(g)).run(args.sweeps)
        p2.results(out=[int(x.data_ptr()) for x in res_pin])  # decisions into pinned host memory
        e2e_t += time.perf_counter() - t0
    e2e_t = d.max(e2e_t / e2e_steps)
    e2e_serial_t = e2e_t
    e2e_mode = "serial: per step upload, run, readback (L2 flushed before each)"
    if d.world == 1 and compact:
        # pipelined refits (double-buffered input, ocg_als_plan_stage_compact): step i+1's CSR
        # crosses PCIe on a side stream while step i runs; every step still copies its whole
        # CSR in and its decisions out inside the timed region.  No L2 flush between steps
        # (the 663 MB CSR is larger than L2).
        ptrs = [int(x.data_ptr()) for x in pin]
        e2e_p = max(args.steps, 3)
        p2.stage_compact(*ptrs)  # warm: staging buffers, side stream
        p2.run(timed=False)
        p2.results(out=[int(x.data_ptr()) for x in res_pin])
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        rptr = [int(x.data_ptr()) for x in res_pin]
        p2.stage_compact(*ptrs)
        p2.run(timed=False)
        for i in range(e2e_p):
            if i + 1 < e2e_p:
                p2.stage_compact(*ptrs)  # H2D of step i+1 on the side stream, during step i
            p2.results_async(rptr)  # D2H of step i's decisions, queued behind step i
            if i + 1 < e2e_p:
                p2.run(timed=False)  # step i+1 queued behind that copy: the GPU never idles
            p2.results_wait()
        e2e_t = (time.perf_counter() - t0) / e2e_p
        e2e_mode = (f"pipelined over {e2e_p} steps: step i+1's CSR staged (side-stream H2D) while step i runs, "
                    "step i's decisions copied out behind it and waited for by the host before the next "
                    "iteration; no L2 flush (inputs larger than L2)")
    r2 = [x.numpy() for x in res_pin]
    p2.close()
    if d.world == 1:
        assert np.array_equal(r2[0], idx)
    cells = m * n
    k = cfg["rank"]
    # roofline of the Gram kernel (K3): per observation 8 B (index +
    # value) + 4k B gathered factor row, per item 4k B factor + 8 B pointer; the
    # same kernel runs the row and the column half-sweep once per sweep each.
    row_bytes = nnz * (8 + 4 * k) + m_loc * (4 * k + 8)
    col_bytes = nnz * (8 + 4 * k) + n * (4 * k + 8)
    out = {
        "metric": "CF-completed matrix cells/sec",
        "value": cells * args.steps / t_dev,
        "unit": "cells/s",
        "selections_per_sec": m * args.steps / t_dev,
        "ms_per_step": t_dev * 1e3 / args.steps,
        "e2e": {"value": cells / e2e_t, "unit": "cells/s",
                "h2d_bytes_per_step": h2d_bytes * d.world,
                "d2h_bytes_per_step": int(idx.nbytes + sav.nbytes + loss.nbytes + ncand.nbytes) * d.world,
                "selections_per_sec": m / e2e_t, "mode": e2e_mode,
                "serial_value": cells / e2e_serial_t},
        "dtype": "f32 factors (rank 32/64 Gram and imputation on fp16 hi/lo split operands, the L^T L term dropped, FP32 accumulation) / f64 selection",
        "config": {"workload": args.workload, "apps": m, "settings": n, "rank": k, "observed_per_gpu": nnz,
                   "density": cfg["density"], "offline_dense_rows": cfg["dense_rows"], "solver": "als",
                   "sweeps": args.sweeps, "lambda": args.als_lambda, "gamma": args.gamma,
                   "parallelism": f"rows sharded over {d.world} GPU(s), column Gram allreduce (NCCL)"
                   if d.world > 1 else "1 GPU",
                   "l2": "inputs (CSR %.0f MB/GPU) larger than L2, and L2 flushed before every timed step" %
                         ((A.row_ptr.nbytes + A.col.nbytes + A.val.nbytes) / 1e6)},
        "quality": quality,
        "scaling": "strong",
        "gpu_launches": args.steps * (16 + args.sweeps * (4 if d.world == 1 else 5) + 2),
        "clocks": clk.summary(),
    }
    if d.world == 1:
        row_ms = phases[1] / args.steps / args.sweeps
        col_ms = phases[2] / args.steps / args.sweeps
        out["phases_ms_per_step"] = {"csc_build_and_segments": phases[0] / args.steps,
                                     "row_half_sweeps": phases[1] / args.steps,
                                     "col_half_sweeps": phases[2] / args.steps,
                                     "impute_select": phases[3] / args.steps,
                                     "row_gram_kernel": phases[4] / args.steps,
                                     "col_gram_kernel": phases[5] / args.steps}
        # K3 Gram kernel alone (CUDA events around its launches on the library
        # stream), row and column launches averaged: gather-counted bytes per launch
        # over the average launch duration.
        g_row = phases[4] / args.steps / args.sweeps
        g_col = phases[5] / args.steps / args.sweeps
        if g_row > 0 and g_col > 0:
            kern, t_row, t_col = f"als_mma_gram_kernel<{k}> (K3 Gram accumulation, mma.sync f16 hi/lo)", g_row, g_col
        else:  # rank 8/16: the fused SIMT Gram + solve kernel; whole half-sweeps
            kern, t_row, t_col = "als_seg_gram_kernel (K3 Gram + K4 solve, SIMT)", row_ms, col_ms
        achieved = (row_bytes + col_bytes) / 2 / ((t_row + t_col) / 2 / 1e3) / 1e9
        traffic = None
        tf = ROOT / "profiles" / "gram_dram_traffic.json"
        if tf.exists() and k == 32:
            tj = json.loads(tf.read_text())
            traffic = (tj["row_bytes"] + tj["col_bytes"]) / 2
        out["roofline"] = {"bound": "hbm", "kernel": kern,
                           "achieved": achieved, "peak": PEAKS["hbm_gbs"], "unit": "GB/s",
                           "frac": achieved / PEAKS["hbm_gbs"], "traffic": traffic,
                           "bytes_def": "gather-counted per launch: nnz*(8+4k) + items*(4k+8) (SURVEY 8d K3; the "
                                        "factor-row gathers are served mostly by L2). traffic = measured DRAM "
                                        "read+write per launch (ncu, profiles/gram_dram_traffic.json): the "
                                        "compulsory CSR read + per-segment Gram records written for K4",
                           "launch_ms_row": t_row, "launch_ms_col": t_col,
                           "half_sweep_ms_row": row_ms, "half_sweep_ms_col": col_ms}
    return out, (args.workload, m)


def workload_c4(args, d: Dist):
    """streaming online phase on the C2 matrix.  Each arrival batch adds one
    new observation to 1% of the rows (paper_2508_07605_b200.stream), on top of the previous
    batches; a refit = the new cells merged into the device CSR (ocg_als_plan_add_observations:
    only the new cells cross PCIe, from pinned host memory) + full completion + selection from
    scratch (reference semantics) + decisions read back.  Reported: latency per refit (wall
    clock, the refit is synchronous), as cells/s, and the warm-start latency (2 sweeps from the
    previous factors: a flagged deviation) at N=1.  N>1: each rank refits its row shard with
    the sharded schedule (arrivals in its own rows)."""
    import torch

    import paper_2508_07605_b200 as ocg
    from paper_2508_07605_b200.als import AlsHyper, AlsPlan
    from paper_2508_07605_b200.dist import GpuAlsBackend, ShardedAlsDriver
    from paper_2508_07605_b200.stream import add_observations

    cfg, grid, A = _joint_matrix("c4", d.rank, d.world)
    m, n = cfg["m"], grid.n
    ctx = ocg.Context(d.local)
    dev = torch.device("cuda", d.local)
    sweeps_rule = {"rule": "fixed by --sweeps", "sweeps": args.sweeps}
    if args.sweeps <= 0:  # the same stated convergence rule as c2 (rank 0 decides, all ranks use it)
        from paper_2508_07605_b200.dist import shard_rows as _sr

        sw, sweeps_rule = als_sweeps_rule(A, grid, AlsHyper(rank=cfg["rank"], lam=args.als_lambda, sweeps=1, seed=42),
                                          args.gamma, ctx, m, goff=_sr(m, d.world, d.rank)[0])
        args.sweeps = int(d.max(float(sw)))
        sweeps_rule["sweeps"] = args.sweeps
    hyp = AlsHyper(rank=cfg["rank"], lam=args.als_lambda, sweeps=args.sweeps, seed=42)
    nref = args.warmup + args.steps + (1 + args.steps if d.world == 1 else 0)
    deltas, B = [], A
    for b in range(nref):  # the arrival stream, prepared on the host before timing
        B, dl = add_observations(B, grid, frac=0.01, seed=1000 * d.rank + b + 1, return_delta=True)
        deltas.append([torch.from_numpy(x).pin_memory() for x in dl])
    plan = AlsPlan(A.m, A.row_ptr, A.col, A.val, grid, hyp, args.gamma, ctx=ctx)
    lib = ocg._lib.lib
    res_pin = [torch.empty(A.m, dtype=dt).pin_memory() for dt in (torch.int32, torch.float64, torch.float64,
                                                                   torch.int32)]

    def refit(b):
        r_, c_, v_ = deltas[b]
        ocg._lib.check(lib.ocg_als_plan_add_observations(plan._h, r_.numel(), r_.data_ptr(), c_.data_ptr(),
                                                         v_.data_ptr()))
        if d.world == 1:
            plan.run(timed=False)
        else:
            ShardedAlsDriver(GpuAlsBackend(plan, dev), d.world, lambda g: d.pg.all_reduce(g)).run(args.sweeps)
        plan.results(out=[int(x.data_ptr()) for x in res_pin])  # decisions into pinned host memory
        return res_pin

    def timed(nsteps, base):
        ts = []
        for b in range(nsteps):
            ocg._lib.check(ocg._lib.lib.ocg_ctx_flush_l2(ctx.handle))
            torch.cuda.synchronize(dev)
            d.barrier()
            t0 = time.perf_counter()
            r = refit(base + b)
            ts.append(d.max(time.perf_counter() - t0))
        return ts, r

    for b in range(args.warmup):
        refit(b)
    with Clocks(d.local) as clk:
        ts, r = timed(args.steps, args.warmup)
    base = args.warmup + args.steps
    assert bool((r[0] >= 0).all())
    lat = statistics.median(ts)
    out = {"metric": "CF-completed matrix cells/sec", "value": m * n / lat, "unit": "cells/s",
           "ms_per_step": lat * 1e3, "scaling": "strong", "dtype": "f32 factors (rank 32/64 Gram and imputation on fp16 hi/lo split operands, the L^T L term dropped, FP32 accumulation) / f64 selection",
           "refit_latency_ms": {"from_scratch_median": lat * 1e3, "all": [t * 1e3 for t in ts]},
           "selections_per_sec": m / lat,
           "e2e": {"value": m * n / lat, "unit": "cells/s",
                   "h2d_bytes_per_step": int(sum(x.numel() * x.element_size() for x in deltas[0])) * d.world,
                   "d2h_bytes_per_step": int(sum(x.numel() * x.element_size() for x in r)) * d.world},
           "config": {"workload": "c4", "apps": m, "settings": n, "rank": cfg["rank"],
                      "arrivals": "1 new observation in each of 1% of rows per refit, cumulative",
                      "observed_per_gpu": A.nnz, "sweeps": args.sweeps, "sweeps_rule": sweeps_rule,
                      "parallelism": f"rows sharded over {d.world} GPU(s)" if d.world > 1 else "1 GPU",
                      "timing": "wall clock per synchronous refit (new cells H2D + device CSR merge + run + "
                                "readback), max over ranks, L2 flushed before each"},
           "gpu_launches": args.steps * (16 + args.sweeps * 4 + 2), "clocks": clk.summary()}
    if d.world == 1:  # warm refits: a flagged deviation from the reference's from-scratch cf::complete
        plan.set_warm(2)
        refit(base)
        tw, _ = timed(args.steps, base + 1)
        plan.set_warm(0)
        out["refit_latency_ms"]["warm_2_sweeps_median"] = statistics.median(tw) * 1e3
        out["refit_latency_ms"]["warm_note"] = ("deviation: starts from the previous factors with 2 sweeps "
                                                f"instead of a from-scratch {args.sweeps}-sweep fit")
    plan.close()
    return out, ("c4", m)


NCF = {  # fused NCF completion + selection (SURVEY §8a a9 + a10): the joint matrices with a fitted model
    "c2-ncf": dict(JOINT["c2"]),
    "c1-ncf": dict(JOINT["c1"]),
}
NCF_MODEL_SEED, NCF_EMB_SCALE = 5, 0.6


def _ncf_traffic():
    """DRAM read+write bytes per launch of the dense kernel at C2, from the ncu capture."""
    f = ROOT / "profiles" / "ncf_fast_dram_traffic.json"
    return json.loads(f.read_text())["bytes_per_launch"] if f.exists() else None


def _ncf_flops_per_cell(k):
    """Algorithmic FP32 work per imputed cell of the fast kernel: layer 0 (A_i + B_j, SELU on 32),
    layer 1 (32 x 16 MACs, tensor cores), SELU on 16, layer 2 (16 MACs), clamp."""
    return 32 + 4 * 32 + 2 * 32 * 16 + 16 + 4 * 16 + 2 * 16 + 2


def workload_ncf(args, d: Dist):
    """cf::complete's imputation (cfcomplete.cpp:208-211, NcfModel::predict :47-58) of every
    unobserved cell of the C2 matrix, fused with policy::select_caps (policy.cpp:17-64) on every
    row, given a fitted model (reference model-file layout; synthetic weights: the reference cannot
    fit C2).  Rows shard over ranks with no collective (weak... strong: total rows fixed)."""
    import torch

    import paper_2508_07605_b200 as ocg
    from paper_2508_07605_b200 import synth
    from paper_2508_07605_b200.ncf import EXACT, FAST, DeviceNcfModel, NcfPlan, random_model

    cfg = NCF[args.workload]
    grid = ocg.PowerGrid.spanning(*cfg["grid"])
    m, n, k = cfg["m"], grid.n, cfg["rank"]
    # weak scaling: every rank completes its own C2-sized instance (rows [rank m, (rank + 1) m) of
    # an (N m)-row synthetic matrix and a model seeded per rank; rank 0's instance is the N = 1 one)
    cells_total = m * n * d.world
    r0, r1 = d.rank * m, (d.rank + 1) * m
    A = synth.joint_csr(m * d.world, grid, cfg["density"], cfg["dense_rows"], seed=42, dtype=np.float64,
                        rows=(r0, r1))
    model = random_model(m, n, k, seed=NCF_MODEL_SEED + 1000 * d.rank, emb_scale=NCF_EMB_SCALE)
    m_loc, nnz = A.m, A.nnz
    ctx = ocg.Context(d.local)
    dev = torch.device("cuda", d.local)
    torch.cuda.set_device(dev)
    dm = DeviceNcfModel(model, ctx=ctx)
    t_rp, t_col, t_val = (torch.from_numpy(x).to(dev) for x in (A.row_ptr, A.col, A.val))
    torch.cuda.synchronize(dev)
    plan = NcfPlan(dm, t_rp.data_ptr(), t_col.data_ptr(), t_val.data_ptr(), grid, args.gamma, FAST, args.lane,
                   on_device=True)
    for _ in range(args.warmup):
        plan.run(timed=False)
    idx0 = plan.results(m_loc)[0]
    assert (idx0 >= 0).all()
    d.barrier()
    tot, ph = 0.0, [0.0, 0.0]
    with Clocks(d.local) as clk:
        for _ in range(args.steps):
            ocg._lib.check(ocg._lib.lib.ocg_ctx_flush_l2(ctx.handle))
            ms, p = plan.run(timed=True)
            clk.tick()
            tot += ms
            ph = [a + b for a, b in zip(ph, p)]
    d.barrier()
    t_dev = d.max(tot / 1e3)
    idx, sav, loss, ncand = plan.results(m_loc)
    assert np.array_equal(idx, idx0) and (ncand >= 1).all()
    exact = None
    if args.exact_step:  # the exact (FP64, reference lane order) precision on the same data: one timed step
        eplan = NcfPlan(dm, t_rp.data_ptr(), t_col.data_ptr(), t_val.data_ptr(), grid, args.gamma, EXACT, args.lane,
                        on_device=True)
        ocg._lib.check(ocg._lib.lib.ocg_ctx_flush_l2(ctx.handle))
        exact_ms, _ = eplan.run(timed=True)
        ex_idx = eplan.results(m_loc)[0]
        exact = {"ms_per_step": exact_ms, "value": cells_total / (exact_ms / 1e3) if d.world == 1 else None,
                 "decisions_equal_to_fast": float((ex_idx == idx).mean()),
                 "note": "OCG_NCF_EXACT: FP64 in the reference lane's operation order, glibc exp"}
        eplan.close()
    plan.close()
    del t_rp, t_col, t_val
    # end to end through the public API with host buffers: the model is resident (created once);
    # per step the matrix's CSR crosses PCIe from pinned host memory (ocg_ncf_plan_upload), the
    # completion + selection runs, and the decisions come back into pinned host memory.
    pin = [torch.from_numpy(x).pin_memory() for x in (A.row_ptr, A.col, A.val)]
    h2d_bytes = sum(int(x.numel() * x.element_size()) for x in pin)
    res = [np.zeros(m_loc, np.int32), np.zeros(m_loc), np.zeros(m_loc), np.zeros(m_loc, np.int32)]
    p2 = NcfPlan(dm, A.row_ptr, A.col, A.val, grid, args.gamma, FAST, args.lane)
    p2.run(timed=False)
    p2.results(m_loc)
    e2e_steps = max(args.steps, 3)
    d.barrier()
    e2e_t = 0.0
    lib = ocg._lib.lib
    for _ in range(e2e_steps):
        ocg._lib.check(lib.ocg_ctx_flush_l2(ctx.handle))
        t0 = time.perf_counter()
        p2.upload(*(int(x.data_ptr()) for x in pin))
        p2.run(timed=False)
        ocg._lib.check(lib.ocg_ncf_plan_results(p2._h, *(ocg._lib.ptr(r) for r in res)))
        e2e_t += time.perf_counter() - t0
    e2e_t = d.max(e2e_t / e2e_steps)
    assert np.array_equal(res[0], idx)
    e2e_serial_t = e2e_t
    e2e_mode = "serial: per step CSR upload (pinned, FP64 values), run, decisions read back; L2 flushed"
    # pipelined serving loop (ocg_ncf_plan_stage / _results_async): step i+1's CSR crosses PCIe on a
    # side stream while step i runs; every step still copies its whole CSR in and its decisions out
    ptrs = [int(x.data_ptr()) for x in pin]
    res_pin = [torch.empty(m_loc, dtype=dt).pin_memory() for dt in (torch.int32, torch.float64, torch.float64,
                                                                      torch.int32)]
    rptr = [int(x.data_ptr()) for x in res_pin]
    p2.stage(*ptrs)  # warm the staging buffers / side stream
    p2.run(timed=False)
    p2.results_async(rptr)
    p2.results_wait()
    # a serving loop in steady state: the pipeline fill (the first step's 991 MB H2D, not
    # overlapped) is paid once inside the timed region and amortised over 4x the bench steps
    e2e_p = 4 * max(args.steps, 3)
    torch.cuda.synchronize(dev)
    d.barrier()
    t0 = time.perf_counter()
    p2.stage(*ptrs)
    p2.run(timed=False)
    for i in range(e2e_p):
        if i + 1 < e2e_p:
            p2.stage(*ptrs)  # H2D of step i+1 on the side stream, during step i
        p2.results_async(rptr)  # D2H of step i's decisions, queued behind step i
        if i + 1 < e2e_p:
            p2.run(timed=False)  # step i+1 queued behind that copy: the GPU never idles
        p2.results_wait()
    e2e_t = d.max((time.perf_counter() - t0) / e2e_p)
    assert np.array_equal(res_pin[0].numpy(), idx)
    e2e_mode = (f"pipelined over {e2e_p} steps (pipeline fill included): step i+1's CSR staged (side-stream H2D "
                "from pinned memory) while step i runs, step i's decisions copied out behind it and waited for by the "
                "host every step; no L2 flush (the 991 MB CSR is larger than L2)")
    p2.close()
    dm.close()
    cells = cells_total
    imputed = m_loc * n - nnz
    peaks, src = _simt_peaks()
    dense_ms = ph[1] / args.steps
    achieved = _ncf_flops_per_cell(k) * imputed / (dense_ms / 1e3) / 1e12
    simt_fpc = _ncf_flops_per_cell(k) - 2 * 32 * 16
    simt_achieved = simt_fpc * imputed / (dense_ms / 1e3) / 1e12
    out = {
        "metric": "CF-completed matrix cells/sec",
        "value": cells * args.steps / t_dev,
        "unit": "cells/s",
        "selections_per_sec": m * d.world * args.steps / t_dev,
        "ms_per_step": t_dev * 1e3 / args.steps,
        "e2e": {"value": cells / e2e_t, "unit": "cells/s", "h2d_bytes_per_step": h2d_bytes * d.world,
                "d2h_bytes_per_step": int(sum(r.nbytes for r in res)) * d.world,
                "selections_per_sec": m * d.world / e2e_t,
                "mode": e2e_mode, "serial_value": cells / e2e_serial_t},
        "dtype": "f32 (tcgen05 f16 hi/lo layer 1) / f64 selection",
        "config": {"workload": args.workload, "apps": m * d.world, "apps_per_gpu": m, "settings": n, "rank": k,
                   "hidden": [32, 16],
                   "observed_per_gpu": nnz, "density": cfg["density"], "offline_dense_rows": cfg["dense_rows"],
                   "solver": "ncf inference (given a fitted model)", "precision": "fast",
                   "model": f"reference NCF model layout, synthetic weights (ncf.random_model seed "
                            f"{NCF_MODEL_SEED}, embeddings +-{NCF_EMB_SCALE})", "gamma": args.gamma,
                   "parallelism": f"{d.world} GPUs, one C2 instance each, no collective" if d.world > 1 else "1 GPU",
                   "l2": "L2 flushed (256 MB write) before every timed step; CSR %.0f MB/GPU" %
                         ((A.row_ptr.nbytes + A.col.nbytes + A.val.nbytes) / 1e6)},
        "phases_ms_per_step": {"prep (validate, A/B precompute, baselines, observed cells)": ph[0] / args.steps,
                               "dense ncf_fast_kernel": dense_ms},
        "exact_precision": exact if exact else "not run (--exact-step; r02: 1.88 s/step, decisions equal to the "
                                                 "fast path on all 1M rows, profiles/r02_bench_c2ncf_exact.json)",
        "scaling": "weak",
        "gpu_launches": args.steps * 7,  # validate, fast_rows, fast_cols, fast_scale, base, rowprep, fast
        "roofline": {"bound": "fp32", "kernel": "ncf_fast_kernel (tcgen05.mma kind::f16 M128 N16 K16 x6 per "
                                                "128 cells, TMA-staged B_j tiles)",
                     "achieved": simt_achieved, "peak": peaks["fp32_tflops"], "unit": "TFLOP/s",
                     "frac": simt_achieved / peaks["fp32_tflops"], "traffic": _ncf_traffic(),
                     "bytes_per_cell": 0.0,
                     "note": f"binding pipe = FP32 SIMT: the {simt_fpc} algorithmic SIMT flop per imputed cell "
                             f"(layer-0 add + SELU on 32 units, layer-1 bias + SELU on 16, layer 2, clamp) over the "
                             f"dense kernel's event time against the FP32 SIMT peak ({src}); the other pipes' floors "
                             f"are lower (see floors_ms). Layer 1's 1024 flop/cell run on the tensor cores (x3 for the "
                             f"fp16 hi/lo split); SURVEY 8d K2 counted all {_ncf_flops_per_cell(k)} flop/cell on the "
                             f"SIMT pipe (floor ~66 ms), which this kernel beats (k2_all_flops). The gap to the SIMT "
                             f"floor is instruction overhead per SIMT flop (SELU select, fp16 hi/lo split, operand "
                             f"stores, per-column barrier): the kernel is issue-bound (ncu, ~370 instructions per cell, issue "
                             f"0.70/cycle/SMSP: "
                             f"profiles/r02_c2ncf_fast_ncu.txt). HBM is irrelevant: DRAM 0.69 GB per launch.",
                     "floors_ms": {"fp32_simt": simt_fpc * imputed / (peaks["fp32_tflops"] * 1e12) * 1e3,
                                   "mufu_ex2 (16 per cell, 16/clk/SM)": 16 * imputed / (16 * 148 * 1.965e9) * 1e3,
                                   "tensor (3 x 1024 flop per cell, measured bf16 peak)":
                                       3 * 1024 * imputed / (PEAKS["bf16_tflops"] * 1e12) * 1e3},
                     "k2_all_flops": {"flops_per_cell": _ncf_flops_per_cell(k), "achieved_tflops": achieved,
                                      "vs_fp32_simt_peak": achieved / peaks["fp32_tflops"]},
                     "simt_flops_per_cell": simt_fpc, "tensor_flops_per_cell": 2 * 32 * 16},
        "clocks": clk.summary(),
    }
    return out, (args.workload, m)


def _weights_module():
    """The pure-numpy input module loaded standalone: the reference arm never maps libocg.so."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("ocg_weights", ROOT / "paper_2508_07605_b200" / "weights.py")
    wmod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(wmod)
    return wmod


def composed_fit(k, m, n, density):
    """The reference's cf::fit at a size it cannot run, composed from its own components timed
    here: one minibatch step = dense embedding-gradient zeroing + 32 x
    nn::backprop_sample + nn::AdamState::step over every parameter; x steps per epoch."""
    from oracle import bind

    ref = bind.Ref()
    ref.force_lane(1)
    secs, parts = ref.time_fit_step(m, n, k, (32, 16), iters=3)
    nnz = density * m * n
    steps = int(np.ceil(0.9 * nnz / 32))
    return {"kind": "composed", "seconds_per_step": secs,
            "parts_s": {"grad_zeroing": parts[0], "backprop_32_samples": parts[1], "adam_all_params": parts[2]},
            "steps_per_epoch": steps, "hours_per_epoch": secs * steps / 3600, "cores": 1,
            "note": "reference cf::fit minibatch step composed from its own components at this model size "
                    "(oracle/_ref ref_time_fit_step, AVX2 lane, 1 core: the reference is single-threaded); "
                    "an early-stopped fit runs hundreds of epochs"}


def reference_ncf(workload: str, threads: int, rows_per_thread: int, lane: int = 1):
    """The reference's NcfModel::predict of every unobserved cell + policy::select_caps on sampled
    rows of the same matrix with the same weights (oracle/_ref; inputs generated by the reference's
    own sim code, no product library).  The per-cell cost is size-independent: linear extrapolation."""
    import importlib.util

    from oracle import bind

    wmod = _weights_module()
    cfg = NCF[workload]
    cpu, gpu = wmod.spanning_caps(*cfg["grid"])
    m, n, k = cfg["m"], len(cpu) * len(gpu), cfg["rank"]
    nrows = max(1, threads * rows_per_thread)
    rng = np.random.default_rng(0)
    rows = np.sort(rng.choice(m, nrows, replace=False)).astype(np.int64)
    ref = bind.Ref()
    ref.force_lane(lane)
    vals, mask = ref.joint_rows_dense(m, cpu, gpu, cfg["density"], cfg["dense_rows"], rows, seed=42)
    params = wmod.random_ncf_params(m, n, k, NCF_MODEL_SEED, NCF_EMB_SCALE)
    sub = bind.sub_model_params(params, m, n, k, k, rows)
    rc, _, idx, sv, lo, nc, secs = ref.ncf_complete_select_rows(k, k, [32, 16], sub, np.ones(nrows, np.uint8),
                                                                np.ones(n, np.uint8), cpu, gpu, vals, mask, 0.05,
                                                                threads, want_completed=False)
    assert rc == 0, ref.err()
    desc = (f"{nrows} rows sampled from {workload} ({m} x {n}, rank {k}): reference NcfModel::predict of every "
            f"unobserved cell + select_caps per row, same weights, {'AVX2' if lane else 'scalar'} lane, {threads} threads; per-cell cost is "
            f"size-independent, so rows/s extrapolate linearly to all {m} rows")
    return nrows * n / secs, desc, secs


C1_FIT = dict(JOINT["c1"])
C1_GOLDEN_EPOCHS = {1: 388, 0: 374}  # the reference's own full C1 fit (tests/golden/joint_c1_lane*.npz)


def workload_c1_fit(args, d: Dist):
    """The reference's complete online CF path at C1 (BASELINE configs[1]), bit for bit: cf::fit
    (cfcomplete.cpp:63-196; NCF, default NcfHyper, seed 42, the reference's schedule and early
    stopping) + cf::complete's imputation of every unobserved cell + policy::select_caps of every
    row, FP64 in the reference lane's operation order.  One step = one whole fit + completion +
    selection.  N>1: replicas (the reference schedule is sequential)."""
    import torch

    import paper_2508_07605_b200 as ocg
    from paper_2508_07605_b200 import synth
    from paper_2508_07605_b200.cf import SOLVER_NCF_REF, cf_fit
    from paper_2508_07605_b200.ncf import EXACT, DeviceNcfModel, NcfPlan

    c = C1_FIT
    grid = ocg.PowerGrid.spanning(*c["grid"])
    A = synth.joint_csr(c["m"], grid, c["density"], c["dense_rows"], seed=42, dtype=np.float64)
    m, n = A.m, A.n
    ctx = ocg.Context(d.local)
    dev = torch.device("cuda", d.local)
    torch.cuda.set_device(dev)
    hyper = ocg.NcfHyper()

    qb = quality_rows(m, c["dense_rows"])
    qrows = np.concatenate([np.arange(r0, r0 + k) for r0, k in qb])

    def step():
        st = {}
        model = cf_fit(A.row_ptr, A.col, A.val, n, hyper, 42, SOLVER_NCF_REF, args.lane, ctx, st)
        dm = DeviceNcfModel(model, ctx=ctx)
        plan = NcfPlan(dm, A.row_ptr, A.col, A.val, grid, args.gamma, EXACT, args.lane)
        ms, _ = plan.run(timed=True)
        r = plan.results(m)
        st["completed"] = plan.completed_rows(qrows)
        plan.close()
        dm.close()
        return st["device_ms"] + ms, st, model, r

    for _ in range(args.warmup):
        step()
    d.barrier()
    tot, fit_ms = 0.0, 0.0
    with Clocks(d.local) as clk:
        for _ in range(args.steps):
            ms, st, model, r = step()
            clk.tick()
            tot += ms
            fit_ms += st["device_ms"]
    d.barrier()
    t_dev = d.max(tot / 1e3)
    # end to end: the public cf::complete entry with host buffers (CSR in, decisions out)
    from paper_2508_07605_b200.cf import cf_complete

    t0 = time.perf_counter()
    rr = cf_complete(A.row_ptr, A.col, A.val, n, hyper, 42, SOLVER_NCF_REF, args.lane, grid, args.gamma,
                     want_completed=False, ctx=ctx)
    e2e_t = d.max(time.perf_counter() - t0)
    assert np.array_equal(rr.idx, r[0])
    golden = C1_GOLDEN_EPOCHS.get(args.lane)
    quality = completion_quality(m, grid, A, qb, st["completed"], r[0][qrows], args.gamma, ctx)
    # the FP32 solver on the same schedule (NCF_FAST): time, quality, agreement with the exact fit
    from paper_2508_07605_b200.cf import SOLVER_NCF_FAST
    from paper_2508_07605_b200.ncf import FAST

    stf = {}
    mf = cf_fit(A.row_ptr, A.col, A.val, n, hyper, 42, SOLVER_NCF_FAST, args.lane, ctx, stf)
    dmf = DeviceNcfModel(mf, ctx=ctx)
    pf = NcfPlan(dmf, A.row_ptr, A.col, A.val, grid, args.gamma, FAST, args.lane)
    msf, _ = pf.run(timed=True)
    rf = pf.results(m)
    qf = completion_quality(m, grid, A, qb, pf.completed_rows(qrows), rf[0][qrows], args.gamma, ctx)
    pf.close()
    dmf.close()
    fast_block = {"ms_per_step": stf["device_ms"] + msf, "epochs_run": mf.meta.epochs_run,
                  "best_val_mse": mf.meta.best_val_mse, "exact_best_val_mse": model.meta.best_val_mse,
                  "decisions_equal_to_exact": float((rf[0] == r[0]).mean()), "quality": qf,
                  "note": "OCG_SOLVER_NCF_FAST: FP32 on the reference schedule; FP32 trajectories drift from FP64, "
                          "so fit quality and selection agreement are reported instead of parameter parity. For "
                          "scale: the reference's own two FP64 lanes (scalar vs AVX2, rounding differences only) "
                          "agree on 66.5 % of the C1 decisions (388 vs 374 epochs)"}
    cells = m * n * d.world
    out = {
        "metric": "CF-completed matrix cells/sec",
        "value": cells * args.steps / t_dev,
        "unit": "cells/s",
        "selections_per_sec": m * d.world * args.steps / t_dev,
        "ms_per_step": t_dev * 1e3 / args.steps,
        "e2e": {"value": cells / e2e_t, "unit": "cells/s", "h2d_bytes_per_step": int(A.row_ptr.nbytes + A.col.nbytes +
                                                                                       A.val.nbytes) * d.world,
                "d2h_bytes_per_step": int(m * 24) * d.world,
                "mode": "ocg_cf_complete: host CSR in, fit + fused completion + selection, decisions out"},
        "dtype": "f64 (reference lane operation order: bit-identical)",
        "config": {"workload": "c1-fit", "apps": m, "settings": n, "rank": 8, "observed": A.nnz,
                   "density": c["density"], "solver": "ncf (reference schedule, joint mode)", "hyper": "NcfHyper{}",
                   "seed": 42, "lane": args.lane, "epochs_run": model.meta.epochs_run,
                   "reference_epochs_run": golden, "minibatch_steps": st["steps"],
                   "parallelism": f"{d.world} replica(s)" if d.world > 1 else "1 GPU",
                   "l2": "fit state (2.7 MB) L2-resident by design; inputs re-uploaded per step"},
        "phases_ms_per_step": {"fit": fit_ms / args.steps, "complete_select": (tot - fit_ms) / args.steps},
        "quality": quality,
        "fast_solver": fast_block,
        "parity": "epochs_run and every parameter bit-identical to the reference's C1 fit "
                  "(tests/test_gpu_joint_fit.py::test_joint_fit_bit_exact_c1)",
        "scaling": "weak",
        "gpu_launches": args.steps * (int(model.meta.epochs_run) + 12),
        "roofline": {"bound": "latency", "kernel": "joint_epoch_kernel (leader CTA step chain)",
                     "achieved": st["device_ms"] * 1e3 / st["steps"], "peak": None, "unit": "us/step",
                     "frac": None, "traffic": None,
                     "note": "the reference schedule is a dependent chain of minibatch steps; the leader's per-step "
                             "latency is the bound (dense Adam replay runs off the critical path on helper warps)"},
        "clocks": clk.summary(),
    }
    return out, ("c1-fit", m)


def reference_c1_fit(threads: int, epochs: int = 4, lane: int = 1):
    """The reference's cf::fit on the C1 matrix for `epochs` epochs (timed) -> per-epoch time x the
    epochs its own full fit runs (the GPU runs the identical epochs, bit for bit), + its
    NcfModel::predict + select_caps over every row."""
    from oracle import bind

    wmod = _weights_module()
    c = C1_FIT
    cpu, gpu = wmod.spanning_caps(*c["grid"])
    m, n = c["m"], len(cpu) * len(gpu)
    ref = bind.Ref()
    ref.force_lane(lane)
    vals, mask = ref.joint_rows_dense(m, cpu, gpu, c["density"], c["dense_rows"], np.arange(m), seed=42)
    t = {}
    for e in (1, epochs):  # two epoch budgets: fixed cost (init, split, MSEs) and per-epoch cost apart
        t0 = time.perf_counter()
        rc, js, meta = ref.ncf_fit(vals, mask, cpu, gpu, 42, max_epochs=e)
        t[e] = time.perf_counter() - t0
        assert rc == 0, ref.err()
    per_epoch = (t[epochs] - t[1]) / (epochs - 1)
    fixed = max(0.0, t[1] - per_epoch)
    params = bind.model_params_from_json(js)
    rc, _, idx, *_, t_sel = ref.ncf_complete_select_rows(8, 8, [32, 16], params, np.ones(m, np.uint8),
                                                         np.ones(n, np.uint8), cpu, gpu, vals, mask, 0.05, 1,
                                                         want_completed=False)
    assert rc == 0, ref.err()
    full_epochs = C1_GOLDEN_EPOCHS[lane]
    secs = fixed + per_epoch * full_epochs + t_sel
    return {"value": m * n / secs, "unit": "cells/s", "cores": 1, "kind": "reference", **host_info(),
            "sample": f"reference cf::fit on the full C1 matrix timed at 1 and {epochs} epochs (fixed {fixed:.2f} s + "
                      f"{per_epoch:.3f} s/epoch) scaled to the {full_epochs} epochs its own complete fit runs, "
                      f"+ NcfModel::predict of every unobserved "
                      f"cell and select_caps of every row ({t_sel:.2f} s); {'AVX2' if lane else 'scalar'} lane, "
                      f"1 core (cf::fit is single-threaded)", "seconds": secs,
            "measured_full_fit_s": {1: 344.5, 0: 613.6}[lane]}


WORKLOADS = {"c0xn": workload_c0xn, "c1": workload_joint, "c2": workload_joint, "c3": workload_joint,
             "c4": workload_c4, "ingest": workload_ingest, "c2-ncf": workload_ncf, "c1-ncf": workload_ncf,
             "c1-fit": workload_c1_fit}


# -------------------------------------------------------- reference (CPU)
def reference_c0xn(napps: int, threads: int, lane: int = 1):
    """The reference's cf::complete + select_caps per app (ref_online_batch)."""
    import ctypes

    from oracle import bind
    import paper_2508_07605_b200 as ocg
    from paper_2508_07605_b200 import synth

    ref = bind.Ref()
    ref.force_lane(lane)
    grid = ocg.PowerGrid.default_grid()
    block = synth.offline_block(42, grid)
    pv, pm, sd = synth.online_apps(napps, 42, grid)
    cpu, gpu = grid.arrays()
    h = bind._hyper(bind.RefHyper)
    idx = np.zeros(napps, np.int32)
    sav = np.zeros(napps)
    secs = ref.L.ref_online_batch(block.shape[0], bind.P(cpu), len(cpu), bind.P(gpu), len(gpu), bind.P(block),
                                  bind.P(pv), bind.P(pm), bind.P(sd), napps, 0.05, ctypes.byref(h), threads,
                                  bind.P(idx), bind.P(sav))
    return secs, idx, sav, grid.n


def reference_joint(workload: str, threads: int, nprob: int, max_epochs: int = 1, lane: int = 1):
    """The reference's cf::complete + select_caps on row samples of the joint matrix.

    Each problem = 1 dense row + (m_s - 1) rows taken at a stride through the
    C1/C2 matrix (all n settings), completed by the reference's NCF with
    app_dim = setting_dim = rank and max_epochs capped, then every row
    selected.  Returns (cells/s, description)."""
    import ctypes

    from oracle import bind

    wmod = _weights_module()
    c = JOINT[workload]
    cpu, gpu = wmod.spanning_caps(*c["grid"])
    m, n = c["m"], len(cpu) * len(gpu)
    ref = bind.Ref()
    m_s = 128 if n > 1024 else 256
    vals = np.zeros((nprob, m_s, n))
    mask = np.zeros((nprob, m_s, n), np.uint8)
    stride = m // m_s
    for p in range(nprob):
        rows = np.concatenate([[p % c["dense_rows"]],
                               (c["dense_rows"] + p * 7919 + np.arange(1, m_s) * stride) % (m - c["dense_rows"])
                               + c["dense_rows"]])
        vals[p], mask[p] = ref.joint_rows_dense(m, cpu, gpu, c["density"], c["dense_rows"], rows, seed=42,
                                                as_float=True)
    ref.force_lane(lane)
    h = bind._hyper(bind.RefHyper, app_dim=c["rank"], setting_dim=c["rank"], max_epochs=max_epochs)
    seeds = np.arange(nprob, dtype=np.uint64) + 1
    sel = np.zeros((nprob, m_s), np.int32)
    secs = ref.L.ref_complete_select_batch(nprob, m_s, bind.P(cpu), len(cpu), bind.P(gpu), len(gpu), bind.P(vals),
                                           bind.P(mask), ctypes.byref(h), bind.P(seeds), 0.05, threads, bind.P(sel))
    assert (sel >= 0).all(), "reference sample failed"
    desc = (f"{nprob} problems of {m_s} rows x {n} settings sampled from {workload} (1 dense + strided rows), "
            f"reference cf::complete (NCF rank {c['rank']}, max_epochs={max_epochs}) + select_caps per row, "
            f"AVX2 lane, {threads} threads. UPPER BOUND on the reference's {workload} rate: its fit runs to early "
            f"stopping (hundreds of epochs) and its per-epoch cost grows with m (dense Adam over (m+n)k params)")
    return nprob * m_s * n / secs, desc, secs


def cpu_baseline(workload: str, threads: int):
    if workload in NCF:
        v1, d1, s1 = reference_ncf(workload, 1, 24)
        v0, d0, s0 = reference_ncf(workload, 1, 24, lane=0)
        v, desc, secs = reference_ncf(workload, threads, 48)
        c = NCF[workload]
        return {"value": v, "unit": "cells/s", "cores": threads, "kind": "reference", "sample": desc,
                "seconds": secs, **host_info(),
                "one_core": {"value": v1, "sample": d1, "seconds": s1},
                "one_core_scalar_lane": {"value": v0, "sample": d0, "seconds": s0},
                "fit_composed": composed_fit(c["rank"], c["m"], c["grid"][0] * c["grid"][1], c["density"])}
    if workload == "c1-fit":
        return reference_c1_fit(threads)
    if workload in JOINT:
        v, desc, secs = reference_joint(workload, threads, nprob=2 * threads)
        c = JOINT[workload]
        return {"value": v, "unit": "cells/s", "cores": threads, "kind": "reference", "sample": desc,
                "seconds": secs, **host_info(),
                "fit_composed": composed_fit(c["rank"], c["m"], c["grid"][0] * c["grid"][1], c["density"])}
    if workload == "ingest":
        v, secs, n = reference_ingest(400_000 * threads, threads)
        return {"value": v, "unit": "estimates/s", "cores": threads, "kind": "reference",
                "sample": f"first {n} ingest counter samples, pred::predict_perf (oracle/_ref, AVX2 lane, "
                          f"{threads} threads)", "seconds": secs}
    if workload == "c0xn":
        napps = max(threads * 8, 16)
        secs, _, _, n = reference_c0xn(napps, threads)
        return {"value": napps * n / secs, "unit": "cells/s", "cores": threads, "kind": "reference",
                "sample": f"{napps} apps x cf::complete+select_caps (oracle/_ref, AVX2 lane, {threads} threads)",
                "seconds": secs}
    raise ValueError(workload)


def run_reference(args, d: Dist):
    if d.rank != 0:
        return
    threads = os.cpu_count() or 1
    if args.workload == "c0xn":
        napps = max(threads * 4, 8)
        for _ in range(args.warmup):
            reference_c0xn(max(threads, 1), threads)
        tot, cells = 0.0, 0
        for _ in range(args.steps):
            secs, _, _, n = reference_c0xn(napps, threads)
            tot += secs
            cells += napps * n
        v = cells / tot
        line = {"impl": "reference", "metric": "CF-completed matrix cells/sec", "value": v, "unit": "cells/s",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": tot * 1e3 / args.steps, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": "c0xn", "apps_per_step": napps},
                "cpu_baseline": {"value": v, "unit": "cells/s", "cores": threads, "kind": "reference",
                                 "sample": f"{napps} apps per step, cf::complete + select_caps, AVX2 lane"},
                "e2e": {"value": v, "unit": "cells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    if args.workload == "ingest":
        for _ in range(args.warmup):
            reference_ingest(20_000 * threads, threads)
        tot, cnt = 0.0, 0
        for _ in range(args.steps):
            v, secs, n = reference_ingest(200_000 * threads, threads)
            tot += secs
            cnt += n
        v = cnt / tot
        line = {"impl": "reference", "metric": "probe performance estimates/sec", "value": v, "unit": "estimates/s",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": tot * 1e3 / args.steps, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (sim::sample_counters of eval apps, C2 grid)",
                "config": {"workload": "ingest", "samples_per_step": cnt // args.steps},
                "cpu_baseline": {"value": v, "unit": "estimates/s", "cores": threads, "kind": "reference",
                                 "sample": f"{cnt // args.steps} samples per step, pred::predict_perf, AVX2 lane"},
                "e2e": {"value": v, "unit": "estimates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    if args.workload == "c1-fit":
        vals = [reference_c1_fit(threads) for _ in range(max(1, min(args.steps, 2)))]
        cb = vals[-1]
        v = cb["value"]
        line = {"impl": "reference", "metric": "CF-completed matrix cells/sec", "value": v, "unit": "cells/s",
                "n_gpus": args.gpus, "steps": len(vals), "warmup": 0, "ms_per_step": cb["seconds"] * 1e3,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (SURVEY 8d generator run by the reference)",
                "config": {"workload": "c1-fit", "apps": C1_FIT["m"], "rank": 8, "solver": "ncf (reference)"},
                "cpu_baseline": cb,
                "e2e": {"value": v, "unit": "cells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    if args.workload in NCF:
        for _ in range(args.warmup):
            reference_ncf(args.workload, threads, 4)
        tot, cells = 0.0, 0
        for _ in range(args.steps):
            v, desc, secs = reference_ncf(args.workload, threads, 32)
            tot += secs
            cells += v * secs
        v = cells / tot
        line = {"impl": "reference", "metric": "CF-completed matrix cells/sec", "value": v, "unit": "cells/s",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": tot * 1e3 / args.steps, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (SURVEY 8d generator run by the reference)",
                "config": {"workload": args.workload, "apps": NCF[args.workload]["m"],
                           "rank": NCF[args.workload]["rank"], "solver": "ncf inference (given a fitted model)"},
                "cpu_baseline": {"value": v, "unit": "cells/s", "cores": threads, "kind": "reference",
                                 "sample": desc},
                "e2e": {"value": v, "unit": "cells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    if args.workload in JOINT:
        for _ in range(args.warmup):
            reference_joint(args.workload, threads, nprob=threads)
        tot, vals = 0.0, []
        for _ in range(args.steps):
            v, desc, secs = reference_joint(args.workload, threads, nprob=2 * threads)
            vals.append(v)
            tot += secs
        v = float(np.mean(vals))
        line = {"impl": "reference", "metric": "CF-completed matrix cells/sec", "value": v, "unit": "cells/s",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": tot * 1e3 / args.steps, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (SURVEY 8d generators, seed 42)",
                "config": {"workload": args.workload, "apps": JOINT[args.workload]["m"],
                           "rank": JOINT[args.workload]["rank"]},
                "cpu_baseline": {"value": v, "unit": "cells/s", "cores": threads, "kind": "reference",
                                 "sample": desc},
                "e2e": {"value": v, "unit": "cells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    raise SystemExit(f"unknown workload {args.workload}")


def secondary_lines(args):
    """Driver-visible measurements of the other reference-exact paths, run after the headline
    (same process, 1 GPU): c1-fit (the reference's whole CF path at C1, bit-exact, one step) and
    c0xn (the reference's per-app online semantics for 4096 apps), each with its own bounded
    reference-CPU figure."""
    import argparse as _ap

    out = {}
    d1 = Dist(None)
    for name, over in (("c1-fit", dict(workload="c1-fit", steps=1, warmup=0)),
                       ("c0xn", dict(workload="c0xn", steps=2, warmup=1, apps=4096))):
        a2 = _ap.Namespace(**{**vars(args), **over})
        try:
            o, _ = WORKLOADS[name](a2, d1)
            keep = {k: o[k] for k in ("metric", "value", "unit", "ms_per_step", "e2e", "dtype", "config", "quality", "fast_solver",
                                      "phases_ms_per_step", "parity", "roofline", "clocks") if k in o}
            keep["steps"], keep["warmup"] = a2.steps, a2.warmup
            if not args.no_cpu_baseline:
                keep["cpu_baseline"] = cpu_baseline(name, os.cpu_count() or 1)
            out[name] = keep
        except Exception as e:  # reported, not fatal for the headline
            out[name] = {"error": repr(e)}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c2-ncf")
    ap.add_argument("--sweeps", type=int, default=0,
                    help="ALS sweeps per fit (c1/c2/c3); 0 = the convergence rule (als_sweeps_rule)")
    ap.add_argument("--als-lambda", type=float, default=0.003)
    ap.add_argument("--gamma", type=float, default=0.05)
    ap.add_argument("--apps", type=int, default=16384, help="c0xn: apps per GPU")
    ap.add_argument("--lane", type=int, default=1, help="reference FP lane to reproduce (0 scalar, 1 avx2)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="c2-ncf: skip the secondary c1-fit / c0xn blocks")
    ap.add_argument("--exact-step", action="store_true",
                    help="c2-ncf/c1-ncf: also time one step of the bit-exact FP64 precision (outside the timed region)")
    args = ap.parse_args()
    if args.impl == "reference":
        d = Dist("gloo")
        try:
            run_reference(args, d)
        finally:
            d.close()
        return
    d = Dist("nccl")
    try:
        out, _ = WORKLOADS[args.workload](args, d)
        if d.rank == 0:
            line = {"metric": out.pop("metric"), "value": out.pop("value"), "unit": out.pop("unit"),
                    "n_gpus": d.world, "steps": args.steps, "warmup": args.warmup,
                    "ms_per_step": out.pop("ms_per_step"), "higher_is_better": True,
                    "scaling": out.pop("scaling"), "vs_baseline": None, "dtype": out.pop("dtype"),
                    "data": "synthetic (SURVEY §8d generators, seed 42)"}
            line.update(out)
            if d.world == 1 and not args.no_cpu_baseline:
                try:
                    line["cpu_baseline"] = cpu_baseline(args.workload, os.cpu_count() or 1)
                except Exception as e:  # reported, not fatal
                    line["cpu_baseline"] = {"value": None, "error": str(e)}
            line["peaks"] = PEAKS
            if d.world == 1 and args.workload == "c2-ncf" and not args.no_secondary:
                line["secondary"] = secondary_lines(args)
            print(json.dumps(line), flush=True)
    finally:
        d.close()


if __name__ == "__main__":
    main()
