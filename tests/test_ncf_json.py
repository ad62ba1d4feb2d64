"""NCF model file (SURVEY §8b ocg_model_to_json / from_json; §8f-2): the
reference's own model files (tests/golden/ncf_model_*.json, written by
cf::fit + NcfModel::to_json through oracle/_ref) load into the flat parameter
layout and are written back BYTE-IDENTICAL.  Host-only: no GPU."""
import json

import numpy as np
import pytest

from conftest import GOLD


@pytest.mark.parametrize("name", ["c0", "odd"])
def test_reference_model_file_round_trips_byte_identical(name):
    from oracle import bind
    from paper_2508_07605_b200 import NcfModel

    text = (GOLD / f"ncf_model_{name}.json").read_text()
    model = NcfModel.from_json(text)
    doc = json.loads(text)
    np.testing.assert_array_equal(model.params, bind.model_params_from_json(text))
    assert model.m == doc["embeddings"]["app"]["rows"] and model.n == doc["embeddings"]["setting"]["rows"]
    assert model.meta.epochs_run == doc["training"]["epochs_run"]
    assert list(model.app_seen) == doc["observed"]["app_seen"]
    assert model.to_json() == text


def test_model_file_errors():
    from paper_2508_07605_b200 import NcfModel, OcgError

    text = (GOLD / "ncf_model_odd.json").read_text()
    doc = json.loads(text)
    doc["format_version"] = 2
    with pytest.raises(OcgError):
        NcfModel.from_json(json.dumps(doc))
    doc = json.loads(text)
    doc["embeddings"]["app"]["values"][0] = doc["embeddings"]["app"]["values"][0][:-1]
    with pytest.raises(OcgError):
        NcfModel.from_json(json.dumps(doc))
    with pytest.raises(OcgError):
        NcfModel.from_json("{not json")


def test_fresh_reference_fits_round_trip(ref):
    """Fresh random fits of the reference library (when it is built here)."""
    from paper_2508_07605_b200 import NcfModel

    rng = np.random.default_rng(2)
    for seed in (1, 2):
        m, n = 9, 6
        v = rng.uniform(0.1, 1.2, (m, n))
        mk = (rng.random((m, n)) < 0.6).astype(np.uint8)
        mk[:, 0] = 1
        rc, js, _ = ref.ncf_fit(v, mk, [1], list(range(1, n + 1)), seed, app_dim=3, setting_dim=2, hidden=(5,),
                                max_epochs=20, patience=5)
        assert rc == 0
        assert NcfModel.from_json(js).to_json() == js
