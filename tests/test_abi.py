"""C-ABI library checks that need no GPU: it loads, exports every symbol
include/ocg.h declares, its host-only helpers match the reference goldens, and
compute entry points fail loudly (no CPU fallback) when no device is usable."""
import math
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import DEFAULT_CPU, DEFAULT_GPU, ROOT

HEADER = ROOT / "include" / "ocg.h"


def _declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(ocg_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2508_07605_b200 import _lib

    names = _declared()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(_lib.lib, n)]
    assert not missing, missing


def test_library_is_sm100a():
    so = ROOT / "paper_2508_07605_b200" / "libocg.so"
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(so)], capture_output=True, text=True)
    assert "sm_100a" in out.stdout, out.stdout + out.stderr


def test_derive_seed_matches_reference(golden):
    from paper_2508_07605_b200 import derive_seed

    for key, val in golden["rng"]["derive_seed"].items():
        root, tag, n = key.split("|")
        assert derive_seed(int(root), tag, int(n)) == int(val)


def test_default_plan_matches_reference(golden):
    from paper_2508_07605_b200 import PowerGrid, ProbePlan

    for key, plan in golden["default_plans"].items():
        nc, ng = map(int, key.split("x"))
        grid = PowerGrid.default_grid() if (nc, ng) == (5, 4) else PowerGrid.spanning(nc, ng)
        assert ProbePlan.default_plan(grid).columns == plan


def test_hyper_defaults_match_reference():
    import ctypes

    from paper_2508_07605_b200 import NcfHyper, _lib

    h = _lib.NcfHyperC()
    _lib.lib.ocg_ncf_hyper_default(ctypes.byref(h))
    d = NcfHyper()
    assert (h.app_dim, h.setting_dim, h.n_hidden, list(h.hidden)[:2]) == (d.app_dim, d.setting_dim, 2, [32, 16])
    assert (h.lr, h.max_epochs, h.patience, h.val_fraction, h.batch_size) == (1e-3, 2000, 100, 0.1, 32)


def test_grid_validation():
    from paper_2508_07605_b200 import InvalidArgument, PowerGrid

    with pytest.raises(InvalidArgument):
        PowerGrid((100, 100), (100,))
    with pytest.raises(InvalidArgument):
        PowerGrid((), (100,))
    assert PowerGrid.spanning(64, 64).n == 4096


def test_host_exp_replica_matches_libm(gold_npz):
    """The same glibc-exp restatement the kernels use, host build, vs libm."""
    from paper_2508_07605_b200 import _lib

    e = gold_npz["exp"]
    f = _lib.lib.ocg_debug_exp_host
    xs, ys = e["x"], e["y"]
    got = np.array([f(float(x)) for x in xs])
    assert np.array_equal(got.view(np.uint64), ys.view(np.uint64))
    rng = np.random.default_rng(123)
    fresh = rng.uniform(-40.0, 0.0, 100000)
    assert all(f(float(x)) == math.exp(float(x)) for x in fresh)


def test_compute_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2508_07605_b200 import Context, CudaError

    with pytest.raises(CudaError):
        Context(0)
