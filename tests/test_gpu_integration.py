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
