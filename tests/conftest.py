import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLD = ROOT / "tests" / "golden"

DEFAULT_CPU = (100, 125, 150, 175, 200)
DEFAULT_GPU = (100, 150, 200, 250)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; parity tests through the C-ABI")


@pytest.fixture(scope="session")
def golden():
    return json.loads((GOLD / "golden.json").read_text())


@pytest.fixture(scope="session")
def gold_npz():
    return {k: np.load(GOLD / f"{k}.npz") for k in ("select", "fit", "c0", "exp")}


@pytest.fixture(scope="session")
def port():
    from oracle import bind

    if not bind.PORT_LIB.exists():
        bind.build(ref=False)
    return bind.Port()


@pytest.fixture(scope="session")
def ref():
    from oracle import bind

    if not bind.REF_LIB.exists():
        pytest.skip("oracle/_ref not built (reference sources absent on this host)")
    return bind.Ref()


@pytest.fixture(scope="session")
def ctx():
    from paper_2508_07605_b200 import Context

    return Context(0)


def fit_case(golden, gold_npz, k):
    """(name, values, mask, seed, hyper kwargs) of golden fit case k."""
    f = gold_npz["fit"]
    case = golden["fit_cases"][k]
    hyper = dict(case["hyper"])
    if "hidden" in hyper:
        hyper["hidden"] = tuple(hyper["hidden"])
    return case["name"], f[f"f{k}_values"], f[f"f{k}_mask"].astype(np.uint8), case["seed"], hyper
