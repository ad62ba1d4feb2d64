"""Drop-in check: the reference's OWN run_open_online (policy.cpp:114-191),
compiled from the reference sources, with cf::complete replaced by the B200
adapter (integration/opencap_cfcomplete_b200.cpp -> include/ocg.h) gives the
reference's decisions bit for bit in both kernel lanes."""
import os
import subprocess

import pytest

from conftest import GOLD, ROOT

pytestmark = pytest.mark.gpu
DEMO = ROOT / "integration" / "_build" / "online_demo"


@pytest.mark.parametrize("lane", ["scalar", "avx2"])
def test_reference_pipeline_with_b200_cf_complete(golden, lane):
    if not DEMO.exists():
        pytest.skip("integration demo not built (needs the reference sources at build time)")
    env = dict(os.environ, OPENCAP_KERNEL=lane)
    out = subprocess.run([str(DEMO), str(GOLD / "predictor.json")], capture_output=True, text=True, env=env,
                         timeout=600, check=True).stdout.split("\n")
    lane_id = 0 if lane == "scalar" else 1
    want = {a["eval_index"]: a for a in golden["c0_apps"] if a["lane"] == lane_id}
    got = [line.split() for line in out if line.strip()]
    assert len(got) == 20
    for e, idx, sav, cand in got:
        w = want[int(e)]
        assert int(idx) == w["setting_idx"]
        assert float.fromhex(sav) == w["pred_saving"]
        assert int(cand) == w["candidates"]


JDEMO = ROOT / "integration" / "_build" / "joint_demo"


def _write_matrix_csv(path, grid, A):
    """The reference's matrix CSV (core.cpp:192-205): header app,c<CPU>_g<GPU>,...;
    empty cells unobserved; values in shortest round-trip decimal."""
    lines = ["app," + ",".join(f"c{c}_g{g}" for c, g in grid.settings())]
    for i in range(A.m):
        row = [""] * A.n
        for q in range(A.row_ptr[i], A.row_ptr[i + 1]):
            row[A.col[q]] = repr(float(A.val[q]))
        lines.append(f"a{i}," + ",".join(row))
    path.write_text("\n".join(lines) + "\n")


def test_reference_api_joint_complete_above_paper_scale(tmp_path, ref):
    """read_matrix_csv_file -> cf::complete -> select_caps, the reference's own
    code with the adapter: a 400 x 64 matrix (4.8K parameters, beyond the per-app
    kernel) completes on the joint path with the reference's decisions, bit for bit."""
    import joint_cases as jc
    import numpy as np

    if not JDEMO.exists():
        pytest.skip("integration demo not built (needs the reference sources at build time)")
    case = [c for c in jc.small_cases() if c["name"] == "d8_l1"][0]
    grid, A = jc.matrix(case)
    csv = tmp_path / "m.csv"
    _write_matrix_csv(csv, grid, A)
    env = dict(os.environ, OPENCAP_KERNEL="avx2")
    out = subprocess.run([str(JDEMO), "complete", str(csv)], capture_output=True, text=True, env=env, timeout=600,
                         check=True).stdout.split("\n")
    got = [line.split() for line in out if line.strip()]
    assert len(got) == A.m
    vals, mask = jc.dense(A)
    cpu, gpu = grid.arrays()
    ref.force_lane(1)
    rc, done = ref.ncf_complete(vals, mask, cpu, gpu, 42)
    assert rc == 0, ref.err()
    rc, idx, sv, lo, nc = ref.select_caps(done, cpu, gpu, 0.05)
    for i, (r, k, s, l, c) in enumerate(got):
        assert int(r) == i
        assert (int(k), float.fromhex(s), float.fromhex(l), int(c)) == (idx[i], sv[i], lo[i], nc[i]), i


def test_reference_api_joint_fit_c1(tmp_path):
    """cf::fit of the full C1 matrix through the reference's own loader and
    cf::fit signature: the model file's parameters equal the reference's fit."""
    import joint_cases as jc
    import numpy as np

    from oracle.bind import model_params_from_json

    if not JDEMO.exists():
        pytest.skip("integration demo not built (needs the reference sources at build time)")
    case = jc.c1_case(1)
    if case is None:
        pytest.skip("C1 golden not generated")
    grid, A = jc.matrix(case)
    csv = tmp_path / "c1.csv"
    _write_matrix_csv(csv, grid, A)
    model = tmp_path / "model.json"
    env = dict(os.environ, OPENCAP_KERNEL="avx2")
    out = subprocess.run([str(JDEMO), "fit", str(csv), str(model)], capture_output=True, text=True, env=env,
                         timeout=900, check=True).stdout
    assert out.split()[1] == str(int(case["meta"][0]))
    np.testing.assert_array_equal(model_params_from_json(model.read_text()), case["params"])
