#!/usr/bin/env python3
"""Generate the golden vectors in tests/golden/ from the REFERENCE itself.

Runs only in the build container (needs /root/reference): it builds
oracle/_ref/libopencap_ref.so from the unmodified reference sources and drives
the reference's public API through the ctypes shim (oracle/ref_capi.cpp).
The outputs are committed; tests never need /root/reference at run time.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import bind  # noqa: E402

OUT = Path(__file__).resolve().parent
DEFAULT_CPU = [100, 125, 150, 175, 200]
DEFAULT_GPU = [100, 150, 200, 250]


def spanning(nc, ng):
    return [60 + (190 * i) // (nc - 1) for i in range(nc)], [100 + (300 * j) // (ng - 1) for j in range(ng)]


def golden_select(ref: bind.Ref):
    rng = np.random.default_rng(20250807)
    out = {}
    cases = []
    # SPEC.md:543 worked example
    n = 20
    row = np.full(n, 0.5)
    s = [(c, g) for c in DEFAULT_CPU for g in DEFAULT_GPU]
    row[s.index((200, 250))] = 1.0
    row[s.index((150, 200))] = 0.97
    row[s.index((125, 150))] = 0.90
    row[s.index((100, 100))] = 0.70
    rows = [row]
    # random rows (>= 1000 rows)
    r = rng.uniform(0.3, 1.2, size=(1200, n))
    r[:, -1] = rng.uniform(0.6, 1.25, size=1200)
    rows.extend(r)
    # ties: repeated values, identical savings via equal cap sums
    t = rng.choice([0.5, 0.8, 0.9, 0.95, 1.0], size=(300, n))
    rows.extend(t)
    rows = np.array(rows)
    for gamma in (0.05, 0.15):
        rc, idx, sv, lo, nc = ref.select_caps(rows, DEFAULT_CPU, DEFAULT_GPU, gamma)
        assert rc == 0, ref.err()
        cases.append(("default", gamma, rows, idx, sv, lo, nc))
    c16, g16 = spanning(16, 16)
    rows16 = rng.uniform(0.2, 1.25, size=(300, 256))
    rc, idx, sv, lo, nc = ref.select_caps(rows16, c16, g16, 0.05)
    assert rc == 0
    cases.append(("grid16", 0.05, rows16, idx, sv, lo, nc))
    c64, g64 = spanning(64, 64)
    rows64 = rng.uniform(0.2, 1.25, size=(12, 4096))
    rows64[:, -1] = 1.0
    rc, idx, sv, lo, nc = ref.select_caps(rows64, c64, g64, 0.05)
    assert rc == 0
    cases.append(("grid64", 0.05, rows64, idx, sv, lo, nc))
    for k, (name, gamma, rows_, idx, sv, lo, nc) in enumerate(cases):
        out[f"c{k}_rows"] = rows_
        out[f"c{k}_idx"], out[f"c{k}_saving"], out[f"c{k}_loss"], out[f"c{k}_ncand"] = idx, sv, lo, nc
    meta = [{"name": c[0], "gamma": c[1]} for c in cases]
    np.savez_compressed(OUT / "select.npz", **out)
    # error behaviour (policy.cpp:19-25)
    bad = np.full((1, 20), 0.9)
    bad[0, 3] = -1.0
    rc_bad = ref.select_caps(bad, DEFAULT_CPU, DEFAULT_GPU, 0.05)[0]
    rc_gamma = ref.select_caps(rows[:1], DEFAULT_CPU, DEFAULT_GPU, 1.0)[0]
    # default plans
    plans = {f"{nc}x{ng}": ref.default_plan(*((DEFAULT_CPU, DEFAULT_GPU) if nc == 5 and ng == 4 else spanning(nc, ng)))
             for nc, ng in [(5, 4), (16, 16), (64, 64), (128, 128), (2, 2), (3, 7)]}
    return {"select_cases": meta, "select_rc_bad_entry": rc_bad, "select_rc_bad_gamma": rc_gamma,
            "default_plans": plans}


def golden_rng(ref: bind.Ref):
    seeds = {}
    for root, tag, n in [(42, "ncf.fit", 0), (42, "online.ncf.ev_gpu_sensitive_0", 0), (7, "synth.mask", 12345),
                         (2**64 - 1, "x", 2**63), (0, "", 0)]:
        seeds[f"{root}|{tag}|{n}"] = str(ref.derive_seed(root, tag, n))
    streams = {str(s): [str(v) for v in ref.rng_u64(s, 700)] for s in (0, 42, 2**63 + 12345)}
    return {"derive_seed": seeds, "mt19937_64": streams}


def golden_exp():
    rng = np.random.default_rng(7)
    xs = np.concatenate([rng.uniform(-20, 0, 60000), rng.uniform(-745, 709.7, 10000), rng.uniform(-1e-9, 0, 2000),
                         -np.logspace(-300, 2.8, 2000), np.array([0.0, -0.0, -1e-320, -708.5, -745.2, 1e-300])])
    ys = np.array([math.exp(float(x)) for x in xs])
    np.savez_compressed(OUT / "exp.npz", x=xs, y=ys)


def ncf_cases(ref: bind.Ref, dense):
    """(name, values, mask, seed, hyper) fit cases; last row is the 'app row'."""
    cases = []
    rng = np.random.default_rng(11)
    # C0: offline dense block + an app probed on the default plan
    plan = ref.default_plan(DEFAULT_CPU, DEFAULT_GPU)
    vals = np.zeros((11, 20))
    mask = np.zeros((11, 20), np.uint8)
    vals[:10], mask[:10] = dense, 1
    for j in plan:
        vals[10, j], mask[10, j] = rng.uniform(0.3, 1.0), 1
    cases.append(("c0", vals, mask, 1234, {}))
    # random sparse 24x12, small model with odd widths (AVX2 tails everywhere)
    m, n = 24, 12
    v = rng.uniform(0.05, 1.2, (m, n))
    mk = (rng.random((m, n)) < 0.45).astype(np.uint8)
    mk[np.arange(m), rng.integers(0, n, m)] = 1
    mk[rng.integers(0, m, n), np.arange(n)] = 1
    cases.append(("odd", v, mk, 99, dict(app_dim=3, setting_dim=5, hidden=(6, 5), batch_size=7, max_epochs=60,
                                         patience=10)))
    # one hidden layer, val_fraction 0.25, lr 3e-3
    cases.append(("h1", v, mk, 5, dict(app_dim=4, setting_dim=4, hidden=(9,), val_fraction=0.25, lr=3e-3,
                                       max_epochs=80, patience=15)))
    # tiny matrix: 5 observed cells -> val_count 0 (monitor = train)
    v2 = rng.uniform(0.2, 1.0, (3, 4))
    mk2 = np.zeros((3, 4), np.uint8)
    mk2[0, 0] = mk2[0, 1] = mk2[1, 2] = mk2[2, 3] = mk2[2, 1] = 1
    cases.append(("tiny", v2, mk2, 3, dict(max_epochs=50, patience=5)))
    # three hidden layers, no early stop inside max_epochs
    cases.append(("deep", v, mk, 17, dict(app_dim=8, setting_dim=8, hidden=(16, 12, 8), max_epochs=25,
                                          patience=1000)))
    return cases


def golden_fit(ref: bind.Ref, dense):
    out = {}
    meta = []
    for k, (name, vals, mask, seed, hyper) in enumerate(ncf_cases(ref, dense)):
        out[f"f{k}_values"], out[f"f{k}_mask"] = vals, mask
        entry = {"name": name, "seed": seed, "hyper": {kk: list(vv) if isinstance(vv, tuple) else vv
                                                       for kk, vv in hyper.items()}}
        m, n = mask.shape
        ii, jj = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
        for lane in (0, 1):
            ref.force_lane(lane)
            # the grid only labels columns; fit does not depend on it -> use a synthetic 1 x n grid
            rc, js, mt = ref.ncf_fit(vals, mask, [1], list(range(1, n + 1)), seed, **hyper)
            assert rc == 0, ref.err()
            out[f"f{k}_lane{lane}_params"] = bind.model_params_from_json(js)
            entry[f"lane{lane}"] = {"epochs_run": mt.epochs_run, "initial_train_mse": mt.initial_train_mse,
                                    "final_train_mse": mt.final_train_mse, "best_val_mse": mt.best_val_mse}
            rc, pred = ref.ncf_predict(js, ii.ravel(), jj.ravel())
            if rc == 0:
                out[f"f{k}_lane{lane}_pred"] = pred.reshape(m, n)
            entry[f"lane{lane}_predict_rc"] = rc
            rc, comp = ref.ncf_complete(vals, mask, [1], list(range(1, n + 1)), seed, **hyper)
            entry[f"lane{lane}_complete_rc"] = rc
            if rc == 0:
                out[f"f{k}_lane{lane}_completed"] = comp
        meta.append(entry)
    ref.force_lane(1)
    np.savez_compressed(OUT / "fit.npz", **out)
    return meta


def golden_c0(ref: bind.Ref):
    """The reference CLI flow at paper scale: offline (seed 42) + online for the 20 eval apps."""
    dense, pred_json = ref.offline_default(42)
    out = {"dense": dense}
    apps = []
    for lane in (0, 1):
        ref.force_lane(lane)
        for e in range(20):
            o = ref.online_default(42, e, dense, pred_json)
            rec = {"eval_index": e, "lane": lane, "setting_idx": o.setting_idx, "pred_saving": o.pred_saving,
                   "pred_loss": o.pred_loss, "candidates": o.candidates, "transition": o.transition,
                   "probe_idx": list(o.probe_idx[: o.n_probes]), "probe_val": list(o.probe_val[: o.n_probes])}
            out[f"lane{lane}_app{e}_row"] = np.array(o.completed_row[:20])
            apps.append(rec)
    ref.force_lane(1)
    np.savez_compressed(OUT / "c0.npz", **out)
    (OUT / "predictor.json").write_text(pred_json)
    return apps


def golden_predictor(ref: bind.Ref, pred_json: str):
    """pred::predict_perf on counters of the eval suite at every default-grid setting (+ CPU-phase counters)."""
    import ctypes

    specs = (bind.RefSpec * 20)()
    cpu, gpu = np.asarray(DEFAULT_CPU, np.int32), np.asarray(DEFAULT_GPU, np.int32)
    assert ref.L.ref_make_suite(5, 5, 5, 5, 42, 0.01, 1, 0.2, bind.P(cpu), 5, bind.P(gpu), 4, specs) == 0
    rows = []
    for sp in specs:
        for c in DEFAULT_CPU:
            for g in DEFAULT_GPU:
                v = np.zeros(7)
                ref.L.ref_sample_counters(ctypes.byref(sp), c, g, bind.P(v))
                rows.append(v)
    counters = np.array(rows)
    # extremes: zero activity, saturated activity, huge throughput
    extra = counters[:8].copy()
    extra[0, 5] = extra[0, 6] = 0.0
    extra[1, 5] = extra[1, 6] = 1.0
    extra[2, 2] *= 50.0
    extra[3, 4] = 0.0
    counters = np.vstack([counters, extra])
    out = {"counters": counters}
    for lane in (0, 1):
        ref.force_lane(lane)
        o = np.zeros(len(counters))
        rc = ref.L.ref_predict_perf(pred_json.encode(), bind.P(counters), len(counters), bind.P(o))
        assert rc == 0, ref.err()
        out[f"lane{lane}"] = o
    ref.force_lane(1)
    bad = counters[:1].copy()
    bad[0, 2] = -1.0
    rc_bad = ref.L.ref_predict_perf(pred_json.encode(), bind.P(bad), 1, bind.P(np.zeros(1)))
    np.savez_compressed(OUT / "predictor.npz", **out)
    return {"predict_rc_negative_ips": rc_bad}


def main():
    bind.build(ref=True)
    ref = bind.Ref()
    golden = {"generated_by": "tests/golden/make_golden.py from oracle/_ref (the reference library)"}
    golden.update(golden_select(ref))
    golden["rng"] = golden_rng(ref)
    golden_exp()
    c0 = golden_c0(ref)
    golden["c0_apps"] = c0
    dense = np.load(OUT / "c0.npz")["dense"]
    golden["fit_cases"] = golden_fit(ref, dense)
    golden.update(golden_predictor(ref, (OUT / "predictor.json").read_text()))
    # cf::complete seeds used by run_open_online for the 20 eval apps
    specs = ["ev_gpu_sensitive_%d", "ev_cpu_sensitive_%d", "ev_both_sensitive_%d", "ev_insensitive_%d"]
    ids = [s % k for s in specs for k in range(5)]
    golden["c0_app_ids"] = ids
    golden["c0_complete_seeds"] = [str(ref.derive_seed(ref.derive_seed(42, "open." + a), "online.ncf." + a))
                                   for a in ids]
    (OUT / "golden.json").write_text(json.dumps(golden, indent=1))
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
