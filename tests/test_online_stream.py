"""Batched online streams, host side (no GPU): phase::DetectorConfig::validate's
rejections (phasedet.cpp:12-25) and the reference detector shims themselves."""
import ctypes

import numpy as np
import pytest


@pytest.mark.parametrize("cfg", [(0.0, 5.0, 60.0), (0.2, 0.0, 60.0), (0.2, 5.0, -1.0), (0.3, 5.0, 60.0),
                                 (0.2, 5.1, 60.0), (0.4, 5.0, 60.0), (0.2, 4.6, 60.0)])
def test_detector_config_rejections(ref, cfg):
    import paper_2508_07605_b200 as ocg
    from paper_2508_07605_b200 import _lib

    p = np.full(40, 100.0)
    rc_ref, _ = ref.detect(p, *cfg)
    assert rc_ref == 1
    c = _lib.DetectorConfigC(*cfg)
    fire = np.zeros(1, np.int64)
    with pytest.raises(ocg.InvalidArgument):
        _lib.check(_lib.lib.ocg_phase_detect_batch(None, ctypes.byref(c), 1, 40, _lib.ptr(p), None, 0,
                                                   _lib.ptr(fire), None))


def test_reference_detector_modes(ref):
    # 30 W for 10 samples, then 100 W: offline fires at the 25th high sample either way;
    # a stream that starts high fires offline at sample 24 but never arms online
    low_then_high = np.concatenate([np.full(10, 30.0), np.full(40, 100.0)])
    assert ref.detect(low_then_high, armed=0) == (0, 34)
    assert ref.detect(low_then_high, armed=1) == (0, 34)
    high = np.full(60, 100.0)
    assert ref.detect(high, armed=0) == (0, 24)
    assert ref.detect(high, armed=1) == (0, -1)
