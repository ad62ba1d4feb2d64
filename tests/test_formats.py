"""File formats against the reference's own loaders / writers (no GPU):
matrix CSV (read_matrix_csv_file / write_matrix_csv, core.cpp:191-254),
binary CSR, and the predictor model file (pred::load_predictor,
predictor.cpp:301-331)."""
import json

import numpy as np
import pytest

import joint_cases as jc


def _matrix():
    from paper_2508_07605_b200.formats import Matrix

    case = [c for c in jc.small_cases() if c["name"] == "odd_l1"][0]
    grid, A = jc.matrix(case)
    cpu = np.repeat(np.asarray(grid.cpu_caps, np.int32), len(grid.gpu_caps))
    gpu = np.tile(np.asarray(grid.gpu_caps, np.int32), len(grid.cpu_caps))
    val = A.val.copy()
    val[::7] = np.nextafter(val[::7], 2.0)  # values needing all 17 significant digits
    val[1] = 1.25
    val[2] = 5e-324
    return Matrix([f"app_{i}" for i in range(A.m)], cpu, gpu, A.row_ptr, A.col, val)


def test_csv_write_is_byte_identical_to_reference(tmp_path, ref):
    M = _matrix()
    mine = tmp_path / "mine.csv"
    M.write_csv(mine)
    theirs = tmp_path / "theirs.csv"
    rc, shape = ref.matrix_csv_roundtrip(mine, theirs)  # the reference reads ours and writes its own
    assert rc == 0, ref.err()
    assert shape == (M.m, M.n, len(M.val))
    assert mine.read_bytes() == theirs.read_bytes()


def test_csv_read_matches_reference_written_file(tmp_path, ref):
    from paper_2508_07605_b200.formats import Matrix

    M = _matrix()
    src = tmp_path / "src.csv"
    M.write_csv(src)
    theirs = tmp_path / "theirs.csv"
    assert ref.matrix_csv_roundtrip(src, theirs)[0] == 0
    R = Matrix.read_csv(theirs)
    assert R.app_ids == M.app_ids
    for a, b in ((R.cpu, M.cpu), (R.gpu, M.gpu), (R.row_ptr, M.row_ptr), (R.col, M.col), (R.val, M.val)):
        np.testing.assert_array_equal(a, b)


def test_binary_round_trip(tmp_path):
    from paper_2508_07605_b200.formats import Matrix

    M = _matrix()
    M.save_bin(tmp_path / "m.bin")
    R = Matrix.load_bin(tmp_path / "m.bin")
    assert R.app_ids == M.app_ids
    np.testing.assert_array_equal(R.val, M.val)
    np.testing.assert_array_equal(R.col, M.col)
    np.testing.assert_array_equal(R.row_ptr, M.row_ptr)


BAD_CSV = {
    "empty": "",
    "header": "name,c1_g1\na,0.5\n",
    "no_settings": "app\na\n",
    "label": "app,c1g1\na,0.5\n",
    "label_zero": "app,c0_g1\na,0.5\n",
    "ragged": "app,c1_g1,c1_g2\na,0.5\n",
    "dup_app": "app,c1_g1\na,0.5\na,0.6\n",
    "dup_setting": "app,c1_g1,c1_g1\na,0.5,0.6\n",
    "no_rows": "app,c1_g1\n",
    "non_numeric": "app,c1_g1\na,x\n",
    "spaces": "app,c1_g1\na, 0.5\n",
    "too_big": "app,c1_g1\na,1.3\n",
    "zero": "app,c1_g1\na,0\n",
    "nan": "app,c1_g1\na,nan\n",
    "empty_id": "app,c1_g1\n,0.5\n",
}


@pytest.mark.parametrize("name", sorted(BAD_CSV))
def test_csv_rejections_match_reference(tmp_path, ref, name):
    import paper_2508_07605_b200 as ocg
    from paper_2508_07605_b200.formats import Matrix

    p = tmp_path / f"{name}.csv"
    p.write_text(BAD_CSV[name])
    rc_ref, _ = ref.matrix_csv_roundtrip(p)
    assert rc_ref != 0
    with pytest.raises(ocg.OcgError) as e:
        Matrix.read_csv(p)
    assert e.value.code == rc_ref, (e.value, ref.err())


def test_csv_missing_file(tmp_path, ref):
    import paper_2508_07605_b200 as ocg
    from paper_2508_07605_b200.formats import Matrix

    assert ref.matrix_csv_roundtrip(tmp_path / "nope.csv")[0] == 2
    with pytest.raises(ocg.MissingArtifact):
        Matrix.read_csv(tmp_path / "nope.csv")


def _mutations():
    base = json.loads((jc.GOLD / "predictor.json").read_text())

    def mod(f):
        d = json.loads(json.dumps(base))
        f(d)
        return d

    return {
        "ok": base,
        "version": mod(lambda d: d.__setitem__("format_version", 2)),
        "arch": mod(lambda d: d["architecture"]["activations"].pop()),
        "layers": mod(lambda d: d["layers"].pop()),
        "wrows": mod(lambda d: d["layers"][0]["weights"].pop()),
        "wcols": mod(lambda d: d["layers"][1]["weights"][3].pop()),
        "bias": mod(lambda d: d["layers"][2]["biases"].append(0.0)),
        "act": mod(lambda d: d["architecture"]["activations"].__setitem__(0, "tanh")),
        "stats": mod(lambda d: d["feature_stats"]["mean"].pop()),
        "no_stats": mod(lambda d: d.pop("feature_stats")),
        "type": mod(lambda d: d["layers"][0].__setitem__("biases", "zero")),
    }


@pytest.mark.parametrize("name", sorted(_mutations()))
def test_predictor_file_checks_match_reference(tmp_path, ref, name):
    import paper_2508_07605_b200 as ocg
    from paper_2508_07605_b200.predictor import PredictorModel

    p = tmp_path / "pred.json"
    p.write_text(json.dumps(_mutations()[name]))
    rc_ref, has_stats = ref.load_predictor(p)
    if rc_ref == 0:
        m = PredictorModel.load(p)
        assert m.has_stats == has_stats
        assert m.dims[0] == 7 and m.dims[-1] == 1
    else:
        with pytest.raises(ocg.OcgError) as e:
            PredictorModel.load(p)
        assert e.value.code == rc_ref, (e.value, ref.err())


def test_predictor_missing_file(tmp_path, ref):
    import paper_2508_07605_b200 as ocg
    from paper_2508_07605_b200.predictor import PredictorModel

    assert ref.load_predictor(tmp_path / "nope.json")[0] == 2
    with pytest.raises(ocg.MissingArtifact):
        PredictorModel.load(tmp_path / "nope.json")
